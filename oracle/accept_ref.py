"""ORACLE — test infrastructure only.  ctypes wrapper of oracle/csrc/accept_oracle.c
(the CPU restatement of the K7 accept/reject step; see that file's header for
the reference lines it follows) plus the statistical acceptance model.

The statistical part restates pkg/src/specpipe/acceptance.py:
  pmf                acceptance.py:29-38   P[k] = p^(k-1)(1-p), P[n+1] = p^n
  expected_accepted  acceptance.py:41-52   (1 - p^(n+1)) / (1 - p); n+1 at p = 1
  sample_accepted    acceptance.py:55-72   inverse CDF on np.random.Generator
and is pinned against the reference by tests/golden/ref_specpipe.json.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_accept.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def _l():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i, f = ctypes.c_int, ctypes.c_float
        _lib.oracle_accept_greedy.argtypes = [P, P, P, P, i, i, i, P, P]
        _lib.oracle_accept_sample.argtypes = [P, P, P, P, P, P, f, i, i, i, P, P]
        _lib.oracle_sample_tokens.argtypes = [P, P, f, i, i, P, P]
        _lib.oracle_det_exp.argtypes = [f]
        _lib.oracle_det_exp.restype = f
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def det_exp(x: float) -> float:
    return float(_l().oracle_det_exp(float(x)))


def accept_greedy(draft, logits, remaining, forced=None):
    draft = np.ascontiguousarray(draft, np.int32)
    logits = np.ascontiguousarray(logits, np.float32)
    remaining = np.ascontiguousarray(remaining, np.int32)
    bs, n = draft.shape
    V = logits.shape[-1]
    f = None if forced is None else np.ascontiguousarray(forced, np.int32)
    tok = np.zeros((bs, n + 1), np.int32)
    cnt = np.zeros(bs, np.int32)
    _l().oracle_accept_greedy(_p(draft), _p(logits), _p(remaining), _p(f), bs, n, V, _p(tok), _p(cnt))
    return tok, cnt


def accept_sample(draft, logits, qprobs, u_acc, u_res, remaining, temperature=1.0):
    draft = np.ascontiguousarray(draft, np.int32)
    logits = np.ascontiguousarray(logits, np.float32)
    qprobs = np.ascontiguousarray(qprobs, np.float32)
    u_acc = np.ascontiguousarray(u_acc, np.float32)
    u_res = np.ascontiguousarray(u_res, np.float32)
    remaining = np.ascontiguousarray(remaining, np.int32)
    bs, n = draft.shape
    V = logits.shape[-1]
    tok = np.zeros((bs, n + 1), np.int32)
    cnt = np.zeros(bs, np.int32)
    _l().oracle_accept_sample(_p(draft), _p(logits), _p(qprobs), _p(u_acc), _p(u_res), _p(remaining),
                              np.float32(1.0 / temperature), bs, n, V, _p(tok), _p(cnt))
    return tok, cnt


def sample_tokens(logits, uniforms=None, temperature=1.0, want_probs=False):
    logits = np.ascontiguousarray(logits, np.float32)
    rows, V = logits.shape
    u = None if uniforms is None else np.ascontiguousarray(uniforms, np.float32)
    tok = np.zeros(rows, np.int32)
    probs = np.zeros((rows, V), np.float32) if want_probs else None
    _l().oracle_sample_tokens(_p(logits), _p(u), np.float32(1.0 / temperature), rows, V, _p(tok), _p(probs))
    return (tok, probs) if want_probs else tok


# ---- statistical acceptance model (acceptance.py restatement) ----

def pmf(p: float, n_cand: int) -> np.ndarray:
    k = np.arange(1, n_cand + 2, dtype=np.float64)
    out = p ** (k - 1) * (1.0 - p)
    out[-1] = p ** n_cand
    return out


def expected_accepted(p: float, n_cand: int) -> float:
    if p == 1.0:
        return float(n_cand + 1)
    return float((1.0 - p ** (n_cand + 1)) / (1.0 - p))


def sample_accepted(p: float, n_cand: int, rng: np.random.Generator, size: int) -> np.ndarray:
    cdf = np.cumsum(pmf(p, n_cand))
    cdf[-1] = 1.0
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right") + 1, n_cand + 1).astype(np.int64)
