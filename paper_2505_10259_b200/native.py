"""ctypes binding of the C ABI in ``include/specoffload_b200.h``.

This is the one place the Python host layer touches native code.  Every
wrapper takes torch tensors (device memory owned by PyTorch, SURVEY.md §8b
"Ownership"), checks shapes/dtypes, and enqueues on the current (or given)
CUDA stream.  A non-zero status raises :class:`NativeError`.  There is no CPU
fallback: if the shared library is missing, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from ctypes import c_float, c_int, c_int64, c_size_t, c_void_p

import torch

from .errors import NativeError, NativeLibraryMissing

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_native", "libspecoffload_b200.so")
_lib = None

EPI_BF16 = 0
EPI_F32 = 1
EPI_BF16_RESID = 2
EPI_SWIGLU = 3
EPI_BF16_ROWSCALE = 4

# name -> (restype, argtypes); mirrors include/specoffload_b200.h
_P = c_void_p
_SIGNATURES = {
    "so_abi_version": (c_int, []),
    "so_status_string": (ctypes.c_char_p, [c_int]),
    "so_device_sm_count": (c_int, []),
    "so_set_device": (c_int, [c_int]),
    "so_accept_greedy": (c_int, [_P, _P, _P, _P, c_int, c_int, c_int, _P, _P, _P]),
    "so_accept_sample": (c_int, [_P, _P, _P, _P, _P, _P, c_float, c_int, c_int, c_int, _P, _P, _P]),
    "so_sample_tokens": (c_int, [_P, c_int64, _P, c_float, c_int, c_int, _P, c_int64, _P, c_int64, _P]),
    "so_router_workspace_bytes": (c_size_t, [c_int, c_int]),
    "so_router_top2": (c_int, [_P, _P, c_int, c_int, c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "so_moe_combine": (c_int, [_P, _P, _P, c_int, c_int, _P, _P]),
    "so_gemm_bf16": (c_int, [_P, _P, c_int, c_int, c_int, _P, c_int, c_int, _P, _P]),
    "so_gemm_workspace_bytes": (c_size_t, [c_int, c_int, c_int]),
    "so_gemm_bf16_ex": (c_int, [_P, _P, c_int, c_int, c_int, _P, c_int, c_int, _P, _P, c_size_t, _P]),
    "so_gemm_grouped_bf16": (c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, _P, c_int, c_int, _P, _P]),
    "so_gemm_bf16_v": (c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, _P, c_int, c_int, _P, _P, c_size_t, c_int, _P]),
    "so_gemv_workspace_bytes": (c_size_t, [c_int, c_int, c_int]),
    "so_gemv_bf16": (c_int, [_P, _P, c_int, c_int, c_int, _P, c_int, c_int, _P, _P, c_size_t, _P]),
    "so_embed": (c_int, [_P, _P, c_int, c_int, _P, _P]),
    "so_rmsnorm": (c_int, [_P, _P, c_int, c_int, c_float, _P, _P]),
    "so_rope_kv_append": (c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, c_float, c_int, _P, _P, _P, _P]),
    "so_attn_paged": (c_int, [_P, _P, _P, _P, c_int, _P, _P, c_int, c_int, c_int, c_int, c_int, c_int,
                              c_float, _P, _P]),
    "so_attn_paged_tc": (c_int, [_P, _P, _P, _P, c_int, _P, _P, c_int, c_int, c_int, c_int, c_int, c_int,
                                 c_float, _P, _P]),
    "so_attn_paged_v": (c_int, [_P, _P, _P, _P, c_int, _P, _P, c_int, c_int, c_int, c_int, c_int, c_int,
                                c_float, _P, c_int, _P]),
    "so_canon_gemm": (c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, _P, c_int, c_int, _P, _P]),
    "so_canon_rmsnorm": (c_int, [_P, _P, c_int, c_int, c_float, _P, _P]),
    "so_canon_rope_kv_append": (c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, _P, c_int, c_int, _P, _P, _P, _P]),
    "so_canon_attn_paged": (c_int, [_P, _P, _P, _P, c_int, _P, _P, c_int, c_int, c_int, c_int, c_int, c_int,
                                    c_float, _P, _P]),
    "so_canon_router_top2": (c_int, [_P, _P, c_int, c_int, c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "so_stream_layer": (c_int, [_P, _P, c_size_t, c_size_t, _P, _P]),
    "so_event_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "so_event_destroy": (c_int, [_P]),
    "so_event_record": (c_int, [_P, _P]),
    "so_stream_wait_event": (c_int, [_P, _P]),
    "so_event_synchronize": (c_int, [_P]),
    "so_event_elapsed_ms": (c_int, [_P, _P, ctypes.POINTER(c_float)]),
    "so_memcpy_async": (c_int, [_P, _P, c_size_t, _P]),
    "so_stream_synchronize": (c_int, [_P]),
    "so_stream_query": (c_int, [_P]),
    "so_event_query": (c_int, [_P]),
    "so_copy_sm": (c_int, [_P, _P, c_size_t, _P]),
    "so_build_verify_tokens": (c_int, [_P, _P, c_int, c_int, c_int, _P, _P, _P]),
    "so_gather_i32": (c_int, [_P, _P, c_int, _P, _P]),
    "so_scatter_i32": (c_int, [_P, _P, _P, c_int, _P]),
    "so_xc4_scratch_bytes": (c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "so_xc4_bound": (c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "so_xc4_encode": (c_int, [_P, ctypes.c_uint64, ctypes.c_uint32, c_int, _P, c_size_t, _P,
                              ctypes.POINTER(ctypes.c_uint64), _P, _P]),
    "so_xc4_decode": (c_int, [_P, _P, ctypes.c_uint32, ctypes.c_uint32, _P, _P]),
    "so_xc4_stream": (c_int, [_P, _P, ctypes.c_uint32, ctypes.c_uint32, _P, c_size_t, c_int, _P,
                              ctypes.POINTER(ctypes.c_uint64), _P, _P, _P, _P]),
}

_PLUMBING = {"so_event_create", "so_event_destroy", "so_event_record", "so_stream_wait_event", "so_event_synchronize",
             "so_event_elapsed_ms", "so_memcpy_async", "so_stream_synchronize", "so_set_device",
             "so_stream_query", "so_event_query"}


def library_path() -> str:
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raise if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise NativeLibraryMissing(
                f"{_LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)"
            )
        handle = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


# kernels (or copy-engine DMA batches) each entry point enqueues; summed into
# ``launches`` so bench.py can report how many of our kernels ran
_KERNELS_PER_CALL = {"so_router_top2": 1, "so_canon_router_top2": 3, "so_stream_layer": 0, "so_xc4_encode": 5}
launches = {"kernels": 0, "copies": 0}
_count_lock = threading.Lock()  # the verify and draft streams are enqueued from two threads


def reset_launch_counter() -> None:
    with _count_lock:
        launches["kernels"] = 0
        launches["copies"] = 0


def set_device(index: int) -> None:
    """Make ``index`` current for this thread in the library's runtime as well."""
    _check(lib().so_set_device(index), "so_set_device")


def _check(rc: int, what: str) -> None:
    if what not in _PLUMBING:
        with _count_lock:
            if what == "so_stream_layer":
                launches["copies"] += 1
            elif what in ("so_xc4_stream", "so_xc4_decode"):
                pass  # counted per frame by the caller
            else:
                launches["kernels"] += _KERNELS_PER_CALL.get(what, 1)
    if rc != 0:
        msg = lib().so_status_string(rc).decode()
        raise NativeError(f"{what} failed with status {rc}: {msg}", rc)


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


# ---------------------------------------------------------------- K7 accept ---

def accept_greedy(draft, logits, remaining, out_tokens, out_counts, forced=None, stream=None):
    bs, n_cand = draft.shape
    V = logits.shape[-1]
    _need(draft, torch.int32, "draft"); _need(logits, torch.float32, "logits")
    _need(remaining, torch.int32, "remaining")
    assert logits.numel() == bs * (n_cand + 1) * V
    if forced is not None:
        _need(forced, torch.int32, "forced")
    _check(lib().so_accept_greedy(_ptr(draft), _ptr(logits), _ptr(remaining), _ptr(forced), bs, n_cand, V,
                                  _ptr(out_tokens), _ptr(out_counts), _stream(stream)), "so_accept_greedy")


def accept_sample(draft, logits, draft_probs, u_accept, u_resample, remaining, out_tokens, out_counts,
                  temperature=1.0, stream=None):
    bs, n_cand = draft.shape
    V = logits.shape[-1]
    for t, n in ((logits, "logits"), (draft_probs, "draft_probs"), (u_accept, "u_accept"),
                 (u_resample, "u_resample")):
        _need(t, torch.float32, n)
    _check(lib().so_accept_sample(_ptr(draft), _ptr(logits), _ptr(draft_probs), _ptr(u_accept),
                                  _ptr(u_resample), _ptr(remaining), 1.0 / temperature, bs, n_cand, V,
                                  _ptr(out_tokens), _ptr(out_counts), _stream(stream)), "so_accept_sample")


def sample_tokens(logits, out_tokens, uniforms=None, out_probs=None, temperature=1.0, stream=None):
    """Rows of ``logits`` [rows, V] (row stride may exceed V) → one token each."""
    rows, V = logits.shape
    assert logits.dtype == torch.float32 and logits.stride(1) == 1
    tok_stride = out_tokens.stride(0) if out_tokens.dim() else 1
    probs_stride = out_probs.stride(0) if out_probs is not None else 0
    _check(lib().so_sample_tokens(_ptr(logits), logits.stride(0), _ptr(uniforms), 1.0 / temperature, rows, V,
                                  _ptr(out_tokens), tok_stride, _ptr(out_probs), probs_stride,
                                  _stream(stream)), "so_sample_tokens")


# ---------------------------------------------------------------- K2 router ---

def router_workspace_bytes(T: int, E: int) -> int:
    return int(lib().so_router_workspace_bytes(T, E))


def router_top2(x, w_gate, expert_offsets, perm_token, row_weight, token_rows, x_perm, workspace,
                topk_idx=None, topk_w=None, stream=None):
    T, H = x.shape
    E = w_gate.shape[0]
    _need(x, torch.bfloat16, "x"); _need(w_gate, torch.bfloat16, "w_gate")
    _check(lib().so_router_top2(_ptr(x), _ptr(w_gate), T, H, E, _ptr(topk_idx), _ptr(topk_w),
                                _ptr(expert_offsets), _ptr(perm_token), _ptr(row_weight), _ptr(token_rows),
                                _ptr(x_perm), _ptr(workspace), _stream(stream)), "so_router_top2")


def moe_combine(y_perm, token_rows, resid, out, stream=None):
    T, H = resid.shape
    _check(lib().so_moe_combine(_ptr(y_perm), _ptr(token_rows), _ptr(resid), T, H, _ptr(out),
                                _stream(stream)), "so_moe_combine")


# ---------------------------------------------------------------- GEMMs ---

_splitk_ws: dict[int, torch.Tensor] = {}  # stream handle → grow-only split-K scratch (one per enqueuing stream)
_splitk_lock = threading.Lock()


def _stream_ws(pool: dict, need: int, stream: int, device) -> tuple[int, int]:
    if need == 0:
        return 0, 0
    with _splitk_lock:
        ws = pool.get(stream)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 16 << 20), dtype=torch.uint8, device=device)
            pool[stream] = ws
    return ws.data_ptr(), ws.numel()


def gemm(a, b, out, epilogue=EPI_BF16, aux=None, stream=None, variant: int = 0):
    """out = epilogue(a[M,K] · b[N,K]ᵀ) on tcgen05 (decode steps: the K5c cluster
    split-K kernel; other skinny shapes: split-K over the SMs).
    ``variant``: tile choice (0 = auto; see so_gemm_bf16_v) — tests and benchmarks only."""
    M, K = a.shape
    N = b.shape[-2]
    assert b.shape[-1] == K
    _need(a, torch.bfloat16, "a")
    assert b.dtype == torch.bfloat16
    st = _stream(stream)
    # decode steps go to K5c, which reduces in distributed shared memory (no scratch)
    gemv = variant in (0, 4) and epilogue != EPI_BF16_ROWSCALE and lib().so_gemv_workspace_bytes(M, N, K) > 0
    if gemv:
        ws, ws_bytes = 0, 0
    elif variant != 3:
        ws, ws_bytes = _stream_ws(_splitk_ws, int(lib().so_gemm_workspace_bytes(M, N, K)), st, a.device)
    else:
        ws, ws_bytes = 0, 0
    _check(lib().so_gemm_bf16_v(_ptr(a), _ptr(b), None, 1, M, N, K, _ptr(out), out.stride(0), epilogue, _ptr(aux), ws,
                                ws_bytes, variant, st), "so_gemm_bf16")
    if ws and not gemv:
        with _count_lock:
            launches["kernels"] += 1  # the split-K reduce (the decode-step kernel reduces in place)


def gemm_grouped(a, b_ptr: int, expert_offsets, E: int, N: int, out, epilogue=EPI_BF16, aux=None, stream=None,
                 variant: int = 0):
    """Grouped expert GEMM; ``b_ptr`` addresses [E, N, K] bf16 weights (e.g. a window slot)."""
    rows, K = a.shape
    _need(a, torch.bfloat16, "a")
    _check(lib().so_gemm_bf16_v(_ptr(a), b_ptr, _ptr(expert_offsets), E, rows, N, K, _ptr(out), out.stride(0),
                                epilogue, _ptr(aux), None, 0, variant, _stream(stream)), "so_gemm_grouped_bf16")


# ---------------------------------------------------------------- K8 ---

def embed(tokens, table, out, stream=None):
    T = tokens.numel()
    H = table.shape[1]
    _check(lib().so_embed(_ptr(tokens), _ptr(table), T, H, _ptr(out), _stream(stream)), "so_embed")


def rmsnorm(x, w, out, eps, stream=None):
    T, H = x.shape
    _check(lib().so_rmsnorm(_ptr(x), _ptr(w), T, H, eps, _ptr(out), _stream(stream)), "so_rmsnorm")


def rope_kv_append(qkv, positions, slots, hq, hkv, dh, theta, page_size, q_out, k_cache, v_cache, stream=None):
    T = qkv.shape[0]
    _check(lib().so_rope_kv_append(_ptr(qkv), _ptr(positions), _ptr(slots), T, hq, hkv, dh, theta, page_size,
                                   _ptr(q_out), _ptr(k_cache), _ptr(v_cache), _stream(stream)),
           "so_rope_kv_append")


# ---------------------------------------------------------------- K6 ---

def attn_paged(q, k_cache, v_cache, block_table, q_start, kv_before, max_q, hq, hkv, dh, page_size, scale, out,
               stream=None, variant: int = 0):
    """``variant`` 0 = auto (TMA-staged K/V tiles where the page size allows), 1 = cp.async staging,
    2 = the tcgen05 kernel K6c (S and O in TMEM), 3 = K6d (decode steps, CUDA-core streaming)."""
    bs = kv_before.numel()
    _check(lib().so_attn_paged_v(_ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(block_table), block_table.shape[1],
                                 _ptr(q_start), _ptr(kv_before), bs, max_q, hq, hkv, dh, page_size, scale,
                                 _ptr(out), variant, _stream(stream)), "so_attn_paged")


# ------------------------------------------- canonical-order arithmetic ---
# Parity mode (csrc/canon.cu): the same ops as the kernels above in a fixed
# IEEE evaluation order that oracle/csrc/canon_oracle.c restates bit for bit.

def canon_gemm(a, b, out, epilogue=EPI_BF16, aux=None, stream=None):
    M, K = a.shape
    N = b.shape[-2]
    _check(lib().so_canon_gemm(_ptr(a), _ptr(b), None, 0, M, N, K, _ptr(out), out.stride(0), epilogue, _ptr(aux),
                               _stream(stream)), "so_canon_gemm")


def canon_gemm_grouped(a, b_ptr: int, expert_offsets, E: int, N: int, out, epilogue=EPI_BF16, aux=None,
                       stream=None):
    rows, K = a.shape
    _check(lib().so_canon_gemm(_ptr(a), b_ptr, _ptr(expert_offsets), E, rows, N, K, _ptr(out), out.stride(0),
                               epilogue, _ptr(aux), _stream(stream)), "so_canon_gemm")


def canon_rmsnorm(x, w, out, eps, stream=None):
    T, H = x.shape
    _check(lib().so_canon_rmsnorm(_ptr(x), _ptr(w), T, H, eps, _ptr(out), _stream(stream)), "so_canon_rmsnorm")


def canon_rope_kv_append(qkv, positions, slots, hq, hkv, dh, table, page_size, q_out, k_cache, v_cache,
                         stream=None):
    """``table`` [rows, dh] fp32: cos(p·f_i) in columns [0, dh/2), sin in [dh/2, dh)."""
    T = qkv.shape[0]
    _need(table, torch.float32, "table")
    _check(lib().so_canon_rope_kv_append(_ptr(qkv), _ptr(positions), _ptr(slots), T, hq, hkv, dh, _ptr(table),
                                         table.shape[0], page_size, _ptr(q_out), _ptr(k_cache), _ptr(v_cache),
                                         _stream(stream)), "so_canon_rope_kv_append")


def canon_attn_paged(q, k_cache, v_cache, block_table, q_start, kv_before, max_q, hq, hkv, dh, page_size, scale,
                     out, stream=None):
    bs = kv_before.numel()
    _check(lib().so_canon_attn_paged(_ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(block_table), block_table.shape[1],
                                     _ptr(q_start), _ptr(kv_before), bs, max_q, hq, hkv, dh, page_size, scale,
                                     _ptr(out), _stream(stream)), "so_canon_attn_paged")


def canon_router_top2(x, w_gate, expert_offsets, perm_token, row_weight, token_rows, x_perm, workspace,
                      topk_idx=None, topk_w=None, stream=None):
    T, H = x.shape
    E = w_gate.shape[0]
    _check(lib().so_canon_router_top2(_ptr(x), _ptr(w_gate), T, H, E, _ptr(topk_idx), _ptr(topk_w),
                                      _ptr(expert_offsets), _ptr(perm_token), _ptr(row_weight), _ptr(token_rows),
                                      _ptr(x_perm), _ptr(workspace), _stream(stream)), "so_canon_router_top2")


# ------------------------------------------------------ stream plumbing ---

def _sp(stream) -> int:
    """Raw handle of a torch stream (or an int handle)."""
    return stream if isinstance(stream, int) else stream.cuda_stream


class Event:
    """A CUDA event driven through the C ABI (GIL released on every call)."""

    __slots__ = ("handle",)

    def __init__(self, timing: bool = False):
        h = c_void_p()
        _check(lib().so_event_create(1 if timing else 0, ctypes.byref(h)), "so_event_create")
        self.handle = h.value

    def record(self, stream) -> "Event":
        _check(lib().so_event_record(self.handle, _sp(stream)), "so_event_record")
        return self

    def wait(self, stream) -> None:
        """Make ``stream`` wait for the most recent record of this event."""
        _check(lib().so_stream_wait_event(_sp(stream), self.handle), "so_stream_wait_event")

    def synchronize(self) -> None:
        _check(lib().so_event_synchronize(self.handle), "so_event_synchronize")

    def query(self) -> int:
        """0 = the last record completed, 600 = pending (never blocks)."""
        return int(lib().so_event_query(self.handle))

    def elapsed_ms(self, end: "Event") -> float:
        ms = c_float()
        _check(lib().so_event_elapsed_ms(self.handle, end.handle, ctypes.byref(ms)), "so_event_elapsed_ms")
        return float(ms.value)

    def __del__(self):
        if _lib is not None and getattr(self, "handle", None):
            _lib.so_event_destroy(self.handle)
            self.handle = None


def stream_query(stream) -> int:
    """0 = the stream is idle, 600 = work pending; other values are sticky errors."""
    return int(lib().so_stream_query(_sp(stream)))


def memcpy_async(dst_ptr: int, src_ptr: int, nbytes: int, stream) -> None:
    _check(lib().so_memcpy_async(dst_ptr, src_ptr, nbytes, _sp(stream)), "so_memcpy_async")


def copy_sm(dst_ptr: int, src_ptr: int, nbytes: int, stream) -> None:
    """Zero-copy transfer by SMs (pinned host ↔ HBM over UVA); for KB-sized data."""
    _check(lib().so_copy_sm(dst_ptr, src_ptr, nbytes, _sp(stream)), "so_copy_sm")


def stream_synchronize(stream) -> None:
    _check(lib().so_stream_synchronize(_sp(stream)), "so_stream_synchronize")


def build_verify_tokens(t_last, drafts, bs: int, n_cand: int, tokens, draft_rows, stream=None):
    _check(lib().so_build_verify_tokens(_ptr(t_last), _ptr(drafts), drafts.shape[1], bs, n_cand, _ptr(tokens),
                                        _ptr(draft_rows), _stream(stream)), "so_build_verify_tokens")


def gather_i32(src, idx, out, stream=None):
    _check(lib().so_gather_i32(_ptr(src), _ptr(idx), idx.numel(), _ptr(out), _stream(stream)), "so_gather_i32")


def scatter_i32(dst, idx, val, stream=None):
    _check(lib().so_scatter_i32(_ptr(dst), _ptr(idx), _ptr(val), idx.numel(), _stream(stream)), "so_scatter_i32")


# ---------------------------------------------------------------- K1 ---

def stream_layer(slot_ptr: int, host_ptr: int, nbytes: int, chunk: int, stream,
                 event: "Event | None" = None) -> None:
    ev = event.handle if event is not None else None
    _check(lib().so_stream_layer(slot_ptr, host_ptr, nbytes, chunk, _sp(stream), ev), "so_stream_layer")


# ---------------------------------------------------------------- K9 ---

class XC4Header(ctypes.Structure):
    """so_xc4_header (include/specoffload_b200.h)."""

    _fields_ = [("magic", ctypes.c_uint32), ("version", ctypes.c_uint32), ("n_elems", ctypes.c_uint64),
                ("frame_elems", ctypes.c_uint32), ("n_frames", ctypes.c_uint32),
                ("exp_of_code", ctypes.c_uint8 * 16), ("total_bytes", ctypes.c_uint64),
                ("n_escapes", ctypes.c_uint64), ("reserved", ctypes.c_uint8 * 8)]


assert ctypes.sizeof(XC4Header) == 64


def xc4_scratch_bytes(n_elems: int, frame_elems: int) -> int:
    return int(lib().so_xc4_scratch_bytes(n_elems, frame_elems))


def xc4_bound(n_elems: int, frame_elems: int) -> int:
    return int(lib().so_xc4_bound(n_elems, frame_elems))


def xc4_encode(src, frame_elems: int, dst, scratch, stream=None, code_bits: int = 0) -> tuple[int, XC4Header]:
    """Encode bf16 ``src`` (device) into ``dst`` (device uint8, or None for a
    size query).  ``code_bits`` 0 = smaller of 3/4-bit codes, else forced.
    Returns (encoded bytes, header).  Synchronises the stream."""
    assert src.dtype in (torch.bfloat16, torch.int16, torch.uint16) and src.is_cuda and src.is_contiguous()
    n = ctypes.c_uint64()
    h = XC4Header()
    cap = dst.numel() if dst is not None else 0
    _check(lib().so_xc4_encode(_ptr(src), src.numel(), frame_elems, code_bits, _ptr(dst), cap, _ptr(scratch),
                               ctypes.byref(n), ctypes.byref(h), _stream(stream)), "so_xc4_encode")
    return int(n.value), h


def xc4_decode(unit_host_ptr: int, unit_dev_ptr: int, frame_begin: int, frame_end: int, dst_ptr: int,
               stream=None) -> None:
    _check(lib().so_xc4_decode(unit_host_ptr, unit_dev_ptr, frame_begin, frame_end, dst_ptr,
                               _sp(stream) if stream is not None else _stream(None)), "so_xc4_decode")
    with _count_lock:
        launches["kernels"] += frame_end - frame_begin


def xc4_stream(slot_ptr: int, unit_ptr: int, frame_begin: int, frame_end: int, ring_ptr: int,
               ring_slot_bytes: int, ring_events, cursor: "ctypes.c_uint64", copy_stream, decode_stream,
               slot_free: "Event | None", done: "Event") -> None:
    evs = (c_void_p * len(ring_events))(*[e.handle for e in ring_events])
    _check(lib().so_xc4_stream(slot_ptr, unit_ptr, frame_begin, frame_end, ring_ptr, ring_slot_bytes,
                               len(ring_events) // 2, evs, ctypes.byref(cursor), _sp(copy_stream),
                               _sp(decode_stream), slot_free.handle if slot_free is not None else None,
                               done.handle), "so_xc4_stream")
    with _count_lock:
        launches["kernels"] += frame_end - frame_begin
        launches["copies"] += frame_end - frame_begin
