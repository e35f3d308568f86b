"""Accepted-token statistics of draft-then-verify decoding.

Same contract as the reference (pkg/src/specpipe/acceptance.py): per round the
verifier commits the longest correct draft prefix plus one bonus token, so the
committed count lives on {1, …, n_cand+1}; under i.i.d. Bernoulli(p)
acceptance its pmf is P[k] = p^(k−1)(1−p) (k ≤ n_cand), P[n_cand+1] = p^n_cand.
The engine uses :func:`sample_accepted` for the forced-acceptance benchmark
mode (synthetic weights accept nothing) — same inverse-CDF draw
on a caller-owned ``np.random.Generator`` as acceptance.py:55-72, so a given
seed yields the reference's exact counts (tests/golden/ref_specpipe.json).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class AcceptanceModel:
    p: float
    n_cand: int

    def __post_init__(self):
        if not 0.0 <= self.p <= 1.0:
            raise ValidationError("p must be in [0, 1]")
        if self.n_cand < 1:
            raise ValidationError("n_cand must be >= 1")


def pmf(model: AcceptanceModel) -> np.ndarray:
    n = model.n_cand
    accepted = np.arange(n + 1, dtype=np.float64)  # draft tokens accepted before the first rejection
    probs = model.p ** accepted * (1.0 - model.p)
    probs[n] = model.p ** n  # every draft token accepted (no rejection term)
    return probs


def expected_accepted(model: AcceptanceModel) -> float:
    """E[k] = Σ k·P[k] = (1 − p^(n+1)) / (1 − p), and n+1 at p = 1."""
    if model.p == 1.0:
        return float(model.n_cand + 1)
    return float((1.0 - model.p ** (model.n_cand + 1)) / (1.0 - model.p))


def committed_per_verify(model: AcceptanceModel, max_new: int) -> float:
    """Expected tokens committed per verification when every sequence generates
    exactly ``max_new`` tokens and the last verification is clamped to what is
    left (simulator.py:213-214): max_new / E[verifications to finish], with
    V(r) = 1 + Σ_k P[k] · V(r − k) for r > 0 (V ≤ 0 = 0) — the steady-state
    rate of a pool whose finished sequences are immediately replaced."""
    if max_new <= 0:
        return expected_accepted(model)
    probs = pmf(model)
    V = np.zeros(max_new + 1)
    for r in range(1, max_new + 1):
        V[r] = 1.0 + sum(probs[k - 1] * V[max(r - k, 0)] for k in range(1, model.n_cand + 2))
    return float(max_new / V[max_new])


def sample_accepted(model: AcceptanceModel, rng: np.random.Generator, size: int | None = None):
    cdf = np.cumsum(pmf(model))
    cdf[-1] = 1.0
    draws = rng.random(1 if size is None else size)
    k = np.searchsorted(cdf, draws, side="right") + 1
    k = np.minimum(k, model.n_cand + 1).astype(np.int64)
    return int(k[0]) if size is None else k


def input_uniforms(seed: int, rnd: int, batch: int, kind: int, shape) -> np.ndarray:
    """Uniform inputs of round ``rnd`` (−2 = prefill, −1 = first draft) for one batch.

    kind 0 = draft sampling, 1 = accept tests, 2 = resample, 3 = first token.
    The randomness is an *input* of the bit-exact accept/reject contract, so
    the engine and the CPU oracle derive it the same way.
    """
    return np.random.default_rng([seed, rnd + 2, batch, kind]).random(shape, dtype=np.float32)


def forced_counts(seed: int, rnd: int, batch: int, p: float, n_cand: int, size: int) -> np.ndarray:
    rng = np.random.default_rng([seed, rnd + 2, batch, 7])
    return sample_accepted(AcceptanceModel(p, n_cand), rng, size).astype(np.int32)
