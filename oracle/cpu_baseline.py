"""ORACLE — test infrastructure only.  Times the CPU port (oracle/model_ref.py)
on a bounded sample of the benchmark workload, for bench.py's
``cpu_baseline`` object and its ``--impl reference`` arm.

The reference ships no executable inference path, so the CPU
baseline is this port of the path, run on the box's host cores: one verify
layer of the target and one decode layer of the draft at full 8x22B /
Mistral-7B shapes, on ``sample_seqs`` sequences at the benchmark's context
length; a full round is extrapolated as
    n_layer_t·t_target_layer + t_lm_head + (n_cand+1)·(n_layer_d·t_draft_layer + t_lm_head_d)
and committed tokens as sample_seqs·E[k] (forced acceptance at p).
"""
from __future__ import annotations

import dataclasses
import os
import time

import numpy as np

from . import accept_ref
from .model_ref import KV, Arch, forward


def _arch(a, n_layer=1) -> Arch:
    return Arch(vocab=a.vocab, hidden=a.hidden, inter=a.inter, n_layer=n_layer, n_head=a.n_head,
                n_kv_head=a.n_kv_head, head_dim=a.head_dim, n_expert=a.n_expert, rope_theta=a.rope_theta, eps=a.eps)


def _weights(a: Arch, seed: int) -> dict:
    """Random weights of the benchmark's distribution (N(0, 0.02²))."""
    rng = np.random.default_rng(seed)
    H, I, E, dh = a.hidden, a.inter, a.n_expert, a.head_dim

    def filled(*shape):
        return rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)

    L = {"attn_norm": np.ones(H, np.float32), "ffn_norm": np.ones(H, np.float32),
         "wq": filled(a.n_head * dh, H), "wk": filled(a.n_kv_head * dh, H), "wv": filled(a.n_kv_head * dh, H),
         "wo": filled(H, a.n_head * dh)}
    if E:
        L["router"] = rng.normal(0, 0.1, size=(E, H)).astype(np.float32)
        L["w_gate"], L["w_up"], L["w_down"] = filled(E, I, H), filled(E, I, H), filled(E, H, I)
    else:
        L["w_gate"], L["w_up"], L["w_down"] = filled(I, H), filled(I, H), filled(H, I)
    return {"embed": rng.normal(0, 1, size=(a.vocab, H)).astype(np.float32), "final_norm": np.ones(H, np.float32),
            "lm_head": filled(a.vocab, H), "layers": [L]}


@dataclasses.dataclass
class CpuSample:
    tokens_per_s: float     # extrapolated: sample_seqs·E[k] per extrapolated round
    t_target_layer: float
    t_draft_layer: float
    t_round: float          # extrapolated round time (not executed)
    sample: str
    cores: int
    t_sample: float = 0.0   # wall time of the work actually executed (one step of the reference arm)


def measure(target, draft, n_cand: int, p: float, ctx: int, sample_seqs: int = 4, seed: int = 0,
            cache: dict | None = None, commits_per_verify: float | None = None) -> CpuSample:
    """target/draft: objects with the ModelArch fields (vocab, hidden, ...).
    ``cache`` (a dict kept by the caller) holds the weights between repeated
    measurements, so each repetition times only the forward passes."""
    at, ad = _arch(target), _arch(draft)
    rng = np.random.default_rng(seed)
    cache = {} if cache is None else cache
    wt = cache.get("t") or cache.setdefault("t", _weights(at, 0))
    kv = KV(at, sample_seqs, ctx + n_cand + 2)
    kv.k[...] = rng.standard_normal(kv.k.shape, dtype=np.float32)
    kv.v[...] = rng.standard_normal(kv.v.shape, dtype=np.float32)
    toks = [rng.integers(0, at.vocab, n_cand + 1) for _ in range(sample_seqs)]
    t0 = time.perf_counter()
    forward(at, wt, kv, list(range(sample_seqs)), toks, [ctx] * sample_seqs, True, "all")
    t_t = time.perf_counter() - t0
    del kv
    wd = cache.get("d") or cache.setdefault("d", _weights(ad, 1))
    kvd = KV(ad, sample_seqs, ctx + n_cand + 2)
    t0 = time.perf_counter()
    forward(ad, wd, kvd, list(range(sample_seqs)), [[int(t[0])] for t in toks], [ctx] * sample_seqs, True, "last")
    t_d = time.perf_counter() - t0
    # the one-layer timings include one LM head each; count it once per pass
    t_round = target.n_layer * t_t + (n_cand + 1) * draft.n_layer * t_d
    # committed tokens per verified sequence: E[k], or the caller's clamped steady-state figure
    # (16-token requests, the GPU arm's workload)
    e = commits_per_verify or accept_ref.expected_accepted(p, n_cand)
    cores = len(os.sched_getaffinity(0))
    sample = (f"1 target layer ({target.name if hasattr(target, 'name') else 'target'}) verify of {sample_seqs} seqs × "
              f"{n_cand + 1} tokens at ctx {ctx} + 1 draft layer decode step, NumPy fp32 on {cores} cores, "
              f"extrapolated to {target.n_layer}+{n_cand + 1}×{draft.n_layer} layers per round, {e:.4f} commits per verify")
    return CpuSample(sample_seqs * e / t_round, t_t, t_d, t_round, sample, cores, t_t + t_d)
