"""ORACLE — test infrastructure only (tests/, smoke(), bench cpu_baseline).

NumPy restatement of the target/draft forward passes the B200 path runs, and
of the dual-batch speculative decoding loop around them.  Not importable by
the product package; it is the checker.

What it restates, and from where:
  * the per-layer dataflow attention → FFN load → FFN compute of the target,
    PAPER.md:157 and simulator.py:168-192 (the reference only models it);
  * Mixtral / Mistral block arithmetic (RMSNorm, GQA attention with
    rotate-half RoPE, top-2-of-E routing with pair renormalisation, SwiGLU
    experts) — third-party, transformers `modeling_mixtral.py` /
    `modeling_mistral.py`; pinned against those modules by
    tests/golden/make_hf_golden.py → tests/golden/hf_tiny.npz;
  * dual-batch rotation: round r verifies batch r % 2 and drafts batch
    1 - r % 2 (simulator.py:156-157), barrier per round
    (simulator.py:209-211), committed = accepted prefix + 1 bonus clamped to
    the remaining budget (acceptance.py:1-6, simulator.py:213-214).

``mirror_bf16=True`` rounds activations to bf16 at exactly the points the
CUDA path stores bf16 (GEMM outputs, norms, residual sums); ``False`` keeps
fp32 throughout (used to compare with the HF fp32 reference).
Token-level parity of a full decode is unpinned by the reference itself
(SURVEY.md §0.3): the golden vectors here are HF-pinned, not specpipe-pinned.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


def bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 → bf16 (round-to-nearest-even), returned as fp32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)).astype(np.uint32)
    return r.view(np.float32)


@dataclasses.dataclass(frozen=True)
class Arch:
    """Architecture constants (presets.py:6-11 for the full-size shapes)."""

    vocab: int
    hidden: int
    inter: int
    n_layer: int
    n_head: int
    n_kv_head: int
    head_dim: int
    n_expert: int  # 0 = dense MLP (draft)
    top_k: int = 2
    rope_theta: float = 1e6
    eps: float = 1e-5


def init_weights(arch: Arch, seed: int, std: float = 0.02, embed_std: float = 1.0) -> dict:
    """Deterministic fp32 weights whose values are bf16-representable."""
    rng = np.random.default_rng(seed)
    H, I, E, dh = arch.hidden, arch.inter, arch.n_expert, arch.head_dim

    def w(*shape, s=std):
        return bf16(rng.normal(0.0, s, size=shape).astype(np.float32))

    W = {
        "embed": w(arch.vocab, H, s=embed_std),
        "final_norm": bf16(1.0 + 0.1 * rng.standard_normal(H).astype(np.float32)),
        "lm_head": w(arch.vocab, H, s=embed_std / math.sqrt(H) * 4.0),
        "layers": [],
    }
    for _ in range(arch.n_layer):
        L = {
            "attn_norm": bf16(1.0 + 0.1 * rng.standard_normal(H).astype(np.float32)),
            "wq": w(arch.n_head * dh, H),
            "wk": w(arch.n_kv_head * dh, H),
            "wv": w(arch.n_kv_head * dh, H),
            "wo": w(H, arch.n_head * dh),
            "ffn_norm": bf16(1.0 + 0.1 * rng.standard_normal(H).astype(np.float32)),
        }
        if E:
            L["router"] = w(E, H, s=0.1)
            L["w_gate"] = w(E, I, H)
            L["w_up"] = w(E, I, H)
            L["w_down"] = w(E, H, I)
        else:
            L["w_gate"] = w(I, H)
            L["w_up"] = w(I, H)
            L["w_down"] = w(H, I)
        W["layers"].append(L)
    return W


def rmsnorm(x, w, eps, mirror):
    x = np.asarray(x, np.float32)
    var = np.mean(x.astype(np.float64) ** 2, axis=-1, keepdims=True).astype(np.float32)
    y = x * (1.0 / np.sqrt(var + np.float32(eps))).astype(np.float32)
    if mirror:
        return bf16(bf16(y) * w)
    return y * w


def rope(x, pos, theta):
    """x [T, heads, dh] fp32, pos [T] → rotate-half RoPE in fp32."""
    dh = x.shape[-1]
    half = dh // 2
    inv = (1.0 / np.power(np.float32(theta), np.arange(0, dh, 2, dtype=np.float32) / np.float32(dh))).astype(np.float32)
    ang = pos.astype(np.float32)[:, None] * inv[None, :]
    c = np.cos(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    s = np.sin(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    x0, x1 = x[..., :half], x[..., half:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


class KV:
    """Dense per-sequence KV store of the oracle: k[layer][seq] -> [pos, hkv, dh]."""

    def __init__(self, arch: Arch, n_seq: int, max_len: int):
        self.k = np.zeros((arch.n_layer, n_seq, max_len, arch.n_kv_head, arch.head_dim), np.float32)
        self.v = np.zeros_like(self.k)


def forward(arch: Arch, W: dict, kv: KV, seqs: list[int], tokens: list[np.ndarray], starts: list[int],
            mirror: bool = True, logits_rows: str = "all") -> list[np.ndarray]:
    """Run new tokens of several sequences through the model.

    seqs[i] is the KV slot, tokens[i] its new token ids, placed at positions
    starts[i] .. starts[i]+len-1 and attending causally to everything before.
    Returns per-sequence fp32 logits ([len, V], or [1, V] for "last").
    """
    H, dh, hq, hkv = arch.hidden, arch.head_dim, arch.n_head, arch.n_kv_head
    G = hq // hkv
    rnd = bf16 if mirror else (lambda a: np.asarray(a, np.float32))
    lens = [len(t) for t in tokens]
    tok = np.concatenate([np.asarray(t, np.int64) for t in tokens])
    pos = np.concatenate([np.arange(s, s + n) for s, n in zip(starts, lens)])
    x = W["embed"][tok].astype(np.float32)
    bounds = np.cumsum([0] + lens)
    for li, L in enumerate(W["layers"]):
        xn = rmsnorm(x, L["attn_norm"], arch.eps, mirror)
        q = rnd(xn @ L["wq"].T).reshape(-1, hq, dh)
        k = rnd(xn @ L["wk"].T).reshape(-1, hkv, dh)
        v = rnd(xn @ L["wv"].T).reshape(-1, hkv, dh)
        q = rnd(rope(q, pos, arch.rope_theta))
        k = rnd(rope(k, pos, arch.rope_theta))
        attn = np.zeros((x.shape[0], hq, dh), np.float32)
        for i, s in enumerate(seqs):
            a, b = bounds[i], bounds[i + 1]
            p0 = starts[i]
            kv.k[li, s, p0:p0 + lens[i]] = k[a:b]
            kv.v[li, s, p0:p0 + lens[i]] = v[a:b]
            K = kv.k[li, s, :p0 + lens[i]]  # [n_keys, hkv, dh]
            Vv = kv.v[li, s, :p0 + lens[i]]
            for h in range(hq):
                g = h // G
                S = (q[a:b, h, :].astype(np.float64) @ K[:, g, :].T.astype(np.float64)) / math.sqrt(dh)
                n_keys = K.shape[0]
                qpos = np.arange(p0, p0 + lens[i])[:, None]
                S = np.where(np.arange(n_keys)[None, :] <= qpos, S, -np.inf)
                S = S - S.max(axis=1, keepdims=True)
                P = np.exp(S)
                P /= P.sum(axis=1, keepdims=True)
                attn[a:b, h, :] = (P @ Vv[:, g, :].astype(np.float64)).astype(np.float32)
        attn = rnd(attn).reshape(-1, hq * dh)
        h = rnd(rnd(attn @ L["wo"].T) + x)
        hn = rmsnorm(h, L["ffn_norm"], arch.eps, mirror)
        if arch.n_expert:
            logits_r = (hn.astype(np.float64) @ L["router"].T.astype(np.float64)).astype(np.float32)
            # top-2, ties → lower expert index (stable sort of −logit)
            top = np.argsort(-logits_r, axis=1, kind="stable")[:, :2]
            rows = np.arange(h.shape[0])
            l0, l1 = logits_r[rows, top[:, 0]], logits_r[rows, top[:, 1]]
            w1 = (np.float32(1.0) / (np.float32(1.0) + np.exp(l0 - l1))).astype(np.float32)
            wts = np.stack([np.float32(1.0) - w1, w1], axis=1)
            ys = np.zeros((h.shape[0], 2, h.shape[1]), np.float32)
            for e in range(arch.n_expert):  # experts process their routed rows as one batch
                tok, slot = np.nonzero(top == e)
                if tok.size == 0:
                    continue
                xe = hn[tok]
                act = rnd(silu(xe @ L["w_gate"][e].T) * (xe @ L["w_up"][e].T))
                ys[tok, slot] = rnd((act @ L["w_down"][e].T) * wts[tok, slot][:, None])
            x = rnd(h + rnd(ys[:, 0] + ys[:, 1]))
        else:
            g = hn @ L["w_gate"].T
            u = hn @ L["w_up"].T
            act = rnd(silu(g) * u)
            x = rnd(rnd(act @ L["w_down"].T) + h)
    if logits_rows == "last":
        idx = bounds[1:] - 1
        x = x[idx]
    xn = rmsnorm(x, W["final_norm"], arch.eps, mirror)
    logits = (xn.astype(np.float64) @ W["lm_head"].T.astype(np.float64)).astype(np.float32)
    if logits_rows == "last":
        return [logits[i:i + 1] for i in range(len(seqs))]
    return [logits[bounds[i]:bounds[i + 1]] for i in range(len(seqs))]
