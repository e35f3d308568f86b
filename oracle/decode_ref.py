"""ORACLE — test infrastructure only.  CPU restatement of the offloaded
speculative decoding loop (prefill → dual-batch rotation → accept/reject),
token for token, against which the B200 engine's ``generate`` is checked.

Round structure (reference: simulator.py:155-215):
  round r verifies batch b = r % 2 with the drafts made for it in round r-1
  and drafts batch 1-b from that batch's state after its last verification;
  a barrier closes the round.  One verification per round (the
  reference's simulator decrements both batches per round; a physical
  executor verifies one).
Per sequence: ctx = tokens already in both KV caches; t_last = the newest
committed token (not yet in KV).  A draft round feeds t_last, d_1..d_n at
positions ctx..ctx+n (n+1 draft steps, the last one only fills KV), a verify
pass feeds the same n+1 tokens to the target; committing c tokens advances
ctx by c for both models (their KV rows ctx..ctx+c-1 hold exactly the
committed inputs), so no cache ever needs a rollback copy.
"""
from __future__ import annotations

import numpy as np

from . import accept_ref, canon_ref
from .model_ref import KV, Arch
from .model_ref import forward as _forward_np


def uniforms(seed: int, rnd: int, batch: int, kind: int, shape) -> np.ndarray:
    """Input randomness shared by the engine and the oracle (not an algorithm)."""
    return np.random.default_rng([seed, rnd + 2, batch, kind]).random(shape, dtype=np.float32)


def forced_counts(seed: int, rnd: int, batch: int, p: float, n_cand: int, size: int) -> np.ndarray:
    rng = np.random.default_rng([seed, rnd + 2, batch, 7])
    return accept_ref.sample_accepted(p, n_cand, rng, size).astype(np.int32)


def generate(tarch: Arch, tW: dict, darch: Arch, dW: dict, prompts: list, max_new: int, n_cand: int,
             bs_decoding: int, mode: str = "greedy", seed: int = 0, forced_p: float | None = None,
             temperature: float = 1.0, mirror: bool = True, record: list | None = None,
             margins: list | None = None, arith: str = "numpy"):
    """Returns (committed token lists, rounds).  ``margins`` (optional, filled
    per sequence) receives the top-1 − top-2 logit gap of the target row that
    produced each committed token.  ``arith="canonical"`` evaluates both models
    in the canonical float order (canon_ref) — the order the B200 parity mode
    reproduces bit for bit, so its tokens must equal these exactly;
    ``"numpy"`` is the NumPy restatement (``mirror`` = bf16 rounding points)."""
    if arith == "canonical":
        def forward(arch, W, kv, seqs, toks, starts, _mirror, rows):
            return canon_ref.forward(arch, W, kv, seqs, toks, starts, rows)

        new_kv = canon_ref.KV16
    elif arith == "numpy":
        forward, new_kv = _forward_np, KV
    else:
        raise ValueError(f"arith must be 'numpy' or 'canonical', got {arith!r}")
    S = len(prompts)
    gap = [[] for _ in range(S)]

    def top2_gap(row):
        part = np.partition(row, -2)
        return float(part[-1] - part[-2])

    assert 1 <= S <= 2 * bs_decoding
    batches = [list(range(0, min(bs_decoding, S))), list(range(bs_decoding, S))]
    max_len = max(len(p) for p in prompts) + max_new + n_cand + 2
    tkv, dkv = new_kv(tarch, S, max_len), new_kv(darch, S, max_len)
    all_seq = list(range(S))
    starts0 = [0] * S
    tl = forward(tarch, tW, tkv, all_seq, [np.asarray(p) for p in prompts], starts0, mirror, "last")
    forward(darch, dW, dkv, all_seq, [np.asarray(p) for p in prompts], starts0, mirror, "last")
    out = [[] for _ in range(S)]
    remaining = np.full(S, max_new, np.int32)
    t_last = np.zeros(S, np.int32)
    ctx = np.array([len(p) for p in prompts], np.int64)
    for b, members in enumerate(batches):
        if not members:
            continue
        lg = np.concatenate([tl[i] for i in members])
        if mode == "greedy":
            first = accept_ref.sample_tokens(lg)
        else:
            first = accept_ref.sample_tokens(lg, uniforms(seed, -2, b, 3, len(members)), temperature)
        for j, i in enumerate(members):
            out[i].append(int(first[j]))
            gap[i].append(top2_gap(lg[j]))
            remaining[i] -= 1
            t_last[i] = first[j]

    def draft(b: int, rnd: int):
        members = batches[b]
        toks = t_last[members].copy()
        d = np.zeros((len(members), n_cand), np.int32)
        q = np.zeros((len(members), n_cand, darch.vocab), np.float32) if mode == "sample" else None
        u = uniforms(seed, rnd, b, 0, (len(members), n_cand)) if mode == "sample" else None
        for j in range(n_cand + 1):
            lg = forward(darch, dW, dkv, members, [[int(t)] for t in toks], list(ctx[members] + j), mirror, "last")
            if j == n_cand:
                break  # KV fill for d_n only
            lg = np.concatenate(lg)
            if mode == "sample":
                tok, probs = accept_ref.sample_tokens(lg, u[:, j], temperature, want_probs=True)
                q[:, j, :] = probs
            else:
                tok = accept_ref.sample_tokens(lg)
            d[:, j] = tok
            toks = tok
        return d, q

    drafts = {}
    if batches[0]:
        drafts[0] = draft(0, -1)
    rnd = 0
    while (remaining > 0).any():
        b = rnd % 2
        members = batches[b]
        if members and (remaining[members] > 0).any():
            d, q = drafts[b]
            vt = [[int(t_last[i])] + [int(x) for x in d[j]] for j, i in enumerate(members)]
            lg = np.stack(forward(tarch, tW, tkv, members, vt, list(ctx[members]), mirror, "all"))
            if mode == "sample":
                tok, cnt = accept_ref.accept_sample(d, lg, q, uniforms(seed, rnd, b, 1, (len(members), n_cand)),
                                                    uniforms(seed, rnd, b, 2, len(members)), remaining[members],
                                                    temperature)
            else:
                forced = None
                if forced_p is not None:
                    forced = forced_counts(seed, rnd, b, forced_p, n_cand, len(members))
                tok, cnt = accept_ref.accept_greedy(d, lg, remaining[members], forced)
            if record is not None:
                record.append({"round": rnd, "batch": b, "counts": cnt.copy(), "logits": lg})
            for j, i in enumerate(members):
                c = int(cnt[j])
                if c > 0:
                    out[i].extend(int(x) for x in tok[j, :c])
                    gap[i].extend(top2_gap(lg[j, m]) for m in range(c))
                    remaining[i] -= c
                    t_last[i] = tok[j, c - 1]
                    ctx[i] += c
        o = 1 - b
        if batches[o] and (remaining[batches[o]] > 0).any():
            drafts[o] = draft(o, rnd)
        rnd += 1
    if margins is not None:
        margins.extend(gap)
    return out, rnd
