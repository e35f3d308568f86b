"""ORACLE — test infrastructure only.  ctypes wrapper of oracle/csrc/xc4_oracle.c,
the scalar restatement of the XC4 weight-unit format (K9, csrc/wcodec.cu).

The streamed payload it must preserve is the reference's per-layer FFN bytes
(placement.py:260-283, costmodel.py:74); parity = decode(encode(w)) == w bit
for bit, and the GPU encoder's bytes == these bytes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_xc4.so")
_lib = None

HEADER_DTYPE = np.dtype([("magic", "<u4"), ("version", "<u4"), ("n_elems", "<u8"), ("frame_elems", "<u4"),
                         ("n_frames", "<u4"), ("exp_of_code", "u1", 16), ("total_bytes", "<u8"),
                         ("n_escapes", "<u8"), ("reserved", "u1", 8)])


def _l():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        _lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        _lib.oracle_xc4_encode.argtypes = [P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, P, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_uint64)]
        _lib.oracle_xc4_decode.argtypes = [P, P]
    return _lib


def encode(w: np.ndarray, frame_elems: int, bits: int = 0) -> np.ndarray:
    """bf16 bit patterns (uint16, 1-D) → encoded unit bytes (uint8); bits 0 =
    the smaller of 3- and 4-bit codes, else forced."""
    w = np.ascontiguousarray(w, dtype=np.uint16)
    n = ctypes.c_uint64()
    rc = _l().oracle_xc4_encode(w.ctypes.data, w.size, frame_elems, bits, None, 0, ctypes.byref(n))
    if rc:
        raise ValueError(f"oracle_xc4_encode: bad geometry (rc {rc})")
    out = np.zeros(n.value, dtype=np.uint8)
    rc = _l().oracle_xc4_encode(w.ctypes.data, w.size, frame_elems, bits, out.ctypes.data, out.size,
                                ctypes.byref(n))
    assert rc == 0
    return out


def header(unit: np.ndarray) -> np.void:
    return np.frombuffer(unit[:HEADER_DTYPE.itemsize].tobytes(), dtype=HEADER_DTYPE)[0]


def decode(unit: np.ndarray) -> np.ndarray:
    unit = np.ascontiguousarray(unit, dtype=np.uint8)
    h = header(unit)
    out = np.empty(int(h["n_elems"]), dtype=np.uint16)
    rc = _l().oracle_xc4_decode(unit.ctypes.data, out.ctypes.data)
    if rc:
        raise ValueError("oracle_xc4_decode: malformed unit")
    return out
