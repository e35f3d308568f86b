"""ORACLE — test infrastructure only.  The canonical-order forward pass: the
same block dataflow as ``model_ref.forward`` (simulator.py:168-192;
Mixtral / Mistral arithmetic of transformers, pinned by tests/golden/hf_tiny.npz
in fp32) evaluated with the single-definition float order of
oracle/csrc/canon_oracle.c.  The B200 path's parity mode (``arith="canonical"``,
paper_2505_10259_b200/csrc/canon.cu) must reproduce these logits bit for bit,
and therefore every greedy and sampled token (north star: bit-exact accepted
tokens on the tiny config).

Rounding points are those of the product path (models.py):
  xn = rmsnorm(x); qkv = bf16(xn·Wqkvᵀ); q, k = rope; att = attention;
  h = bf16(bf16(att·Woᵀ) + x); hn = rmsnorm(h);
  MoE: route(hn) → act = swiglu → y = bf16(act·W_downᵀ · w) →
       x = bf16(h + bf16(y₀ + y₁));   dense: x = bf16(bf16(act·W_downᵀ) + h);
  logits = rmsnorm(x)·lm_headᵀ in fp32.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_canon.so")
_lib = None
_P = ctypes.c_void_p
EPI_BF16, EPI_F32, EPI_BF16_RESID, EPI_BF16_ROWSCALE = 0, 1, 2, 4


def _l():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        _lib = ctypes.CDLL(_SO)
        i, f = ctypes.c_int, ctypes.c_float
        _lib.canon_gemm.argtypes = [_P, _P, i, i, i, _P, i, i, _P]
        _lib.canon_swiglu.argtypes = [_P, _P, _P, i, i, i, _P]
        _lib.canon_rmsnorm.argtypes = [_P, _P, i, i, f, _P]
        _lib.canon_rope.argtypes = [_P, i, i, i, _P, _P, _P]
        _lib.canon_attn.argtypes = [_P, _P, _P, i, i, i, i, i, f, _P]
        _lib.canon_route.argtypes = [_P, _P, i, i, i, _P, _P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_P)


def to_u16(a: np.ndarray) -> np.ndarray:
    """bf16-valued fp32 array → its bf16 bit patterns."""
    a = np.ascontiguousarray(a, np.float32)
    return (a.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def to_f32(u: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


_W16: dict = {}


def _w(a: np.ndarray) -> np.ndarray:
    """Cached bf16 bits of a weight array (weights are built once per test)."""
    key = (id(a), a.shape)
    hit = _W16.get(key)
    if hit is None or hit[0] is not a:
        hit = (a, to_u16(a))
        _W16[key] = hit
    return hit[1]


def gemm(a16, b16, epi=EPI_BF16, aux=None):
    a16 = np.ascontiguousarray(a16, np.uint16)
    M, K = a16.shape
    N = b16.shape[0]
    out = np.zeros((M, N), np.float32 if epi == EPI_F32 else np.uint16)
    if aux is not None:
        aux = np.ascontiguousarray(aux, np.float32 if epi == EPI_BF16_ROWSCALE else np.uint16)
    _l().canon_gemm(_p(a16), _p(b16), M, N, K, _p(out), N, epi, _p(aux))
    return out


def swiglu(a16, g16, u16):
    a16 = np.ascontiguousarray(a16, np.uint16)
    M, K = a16.shape
    N = g16.shape[0]
    out = np.zeros((M, N), np.uint16)
    _l().canon_swiglu(_p(a16), _p(g16), _p(u16), M, N, K, _p(out))
    return out


def rmsnorm(x16, w16, eps):
    x16 = np.ascontiguousarray(x16, np.uint16)
    T, H = x16.shape
    out = np.zeros_like(x16)
    _l().canon_rmsnorm(_p(x16), _p(w16), T, H, np.float32(eps), _p(out))
    return out


def rope_table(dh: int, theta: float, rows: int) -> np.ndarray:
    """[rows, dh] fp32: cos(p·f_i) | sin(p·f_i), f_i = θ^(−2i/dh), float64 then rounded."""
    inv = 1.0 / theta ** (np.arange(0, dh, 2, dtype=np.float64) / dh)
    ang = np.arange(rows, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def rope(x16, pos, table):
    x16 = np.ascontiguousarray(x16, np.uint16)
    T, heads, dh = x16.shape
    pos = np.ascontiguousarray(pos, np.int32)
    out = np.zeros_like(x16)
    _l().canon_rope(_p(x16), T, heads, dh, _p(pos), _p(np.ascontiguousarray(table, np.float32)), _p(out))
    return out


def attn(q16, k16, v16, p0, scale):
    q16 = np.ascontiguousarray(q16, np.uint16)
    n_q, hq, dh = q16.shape
    hkv = k16.shape[1]
    out = np.zeros_like(q16)
    _l().canon_attn(_p(q16), _p(np.ascontiguousarray(k16, np.uint16)), _p(np.ascontiguousarray(v16, np.uint16)),
                    n_q, p0, hq, hkv, dh, np.float32(scale), _p(out))
    return out


def route(x16, wg16):
    x16 = np.ascontiguousarray(x16, np.uint16)
    T, H = x16.shape
    E = wg16.shape[0]
    idx = np.zeros((T, 2), np.int32)
    w = np.zeros((T, 2), np.float32)
    _l().canon_route(_p(x16), _p(wg16), T, H, E, _p(idx), _p(w))
    return idx, w


class KV16:
    """Per-sequence KV store of bf16 bit patterns: k[layer, seq, pos, hkv, dh]."""

    def __init__(self, arch, n_seq: int, max_len: int):
        self.k = np.zeros((arch.n_layer, n_seq, max_len, arch.n_kv_head, arch.head_dim), np.uint16)
        self.v = np.zeros_like(self.k)
        self.table = rope_table(arch.head_dim, arch.rope_theta, max_len)


def forward(arch, W: dict, kv: KV16, seqs, tokens, starts, logits_rows: str = "all"):
    """model_ref.forward's contract (per-sequence fp32 logits) in canonical order."""
    H, dh, hq, hkv = arch.hidden, arch.head_dim, arch.n_head, arch.n_kv_head
    lens = [len(t) for t in tokens]
    tok = np.concatenate([np.asarray(t, np.int64) for t in tokens])
    pos = np.concatenate([np.arange(s, s + n) for s, n in zip(starts, lens)]).astype(np.int32)
    bounds = np.cumsum([0] + lens)
    x = _w(W["embed"])[tok]
    scale = np.float32(1.0 / math.sqrt(dh))
    for li, L in enumerate(W["layers"]):
        xn = rmsnorm(x, _w(L["attn_norm"]), arch.eps)
        q = rope(gemm(xn, _w(L["wq"])).reshape(-1, hq, dh), pos, kv.table)
        k = rope(gemm(xn, _w(L["wk"])).reshape(-1, hkv, dh), pos, kv.table)
        v = gemm(xn, _w(L["wv"])).reshape(-1, hkv, dh)
        att = np.zeros((x.shape[0], hq, dh), np.uint16)
        for i, s in enumerate(seqs):
            a, b = bounds[i], bounds[i + 1]
            p0 = starts[i]
            kv.k[li, s, p0:p0 + lens[i]] = k[a:b]
            kv.v[li, s, p0:p0 + lens[i]] = v[a:b]
            att[a:b] = attn(q[a:b], kv.k[li, s, :p0 + lens[i]], kv.v[li, s, :p0 + lens[i]], p0, scale)
        h = gemm(att.reshape(-1, hq * dh), _w(L["wo"]), EPI_BF16_RESID, x)
        hn = rmsnorm(h, _w(L["ffn_norm"]), arch.eps)
        if arch.n_expert:
            idx, wts = route(hn, _w(L["router"]))
            ys = np.zeros((h.shape[0], 2, H), np.float32)
            for e in range(arch.n_expert):
                t_e, slot = np.nonzero(idx == e)
                if t_e.size == 0:
                    continue
                act = swiglu(hn[t_e], _w(L["w_gate"])[e], _w(L["w_up"])[e])
                ys[t_e, slot] = to_f32(gemm(act, _w(L["w_down"])[e], EPI_BF16_ROWSCALE, wts[t_e, slot]))
            moe = to_u16(_bf16(ys[:, 0] + ys[:, 1]))
            x = to_u16(_bf16(to_f32(h) + to_f32(moe)))
        else:
            act = swiglu(hn, _w(L["w_gate"]), _w(L["w_up"]))
            x = gemm(act, _w(L["w_down"]), EPI_BF16_RESID, h)
    if logits_rows == "last":
        x = x[bounds[1:] - 1]
    xf = rmsnorm(x, _w(W["final_norm"]), arch.eps)
    logits = gemm(xf, _w(W["lm_head"]), EPI_F32)
    if logits_rows == "last":
        return [logits[i:i + 1] for i in range(len(seqs))]
    return [logits[bounds[i]:bounds[i + 1]] for i in range(len(seqs))]


def _bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.astype(np.uint32).view(np.float32)
