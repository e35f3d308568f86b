"""K9 host side — XC4 lossless exponent-coded weight units (csrc/wcodec.cu).

The streamed unit of one target layer (placement.py:260-283 prefetch op,
ffn_bytes / c2g_bandwidth in costmodel.py:74) is encoded once at load time on
the GPU and kept encoded in pinned host DRAM; every pass moves the encoded
frames over the link and decodes them into the HBM window slot.  The decoded
bytes are bit-identical to the unit, so nothing downstream changes.

Frames are the unit of both copying and multi-GPU slicing: with N ranks,
rank r moves and decodes frames [r·F/N, (r+1)·F/N), which decode to exactly
its 1/N byte slice of the layer (``slice_bounds``), and the NVLink all-gather
rebuilds the rest.
"""
from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import native

MAX_FRAME_ELEMS = 1 << 27   # ≤ 128 Mi weights (≈180 MB encoded) per frame: few copy/decode launches per layer
MIN_FRAME_ELEMS = 4096
SLICE_WORLD = 8             # frames split evenly over 1, 2, 4 or 8 ranks when the unit allows it


def frame_elems_for(n_elems: int, world: int = SLICE_WORLD) -> int:
    """Largest frame (a multiple of 4096 weights, ≤ 32 Mi) that tiles the unit
    into a multiple of ``world`` whole frames — any divisor works, so awkward
    unit sizes (e.g. attention + FFN units, 2^22·597 weights) still get frames
    of tens of MB rather than a power of two small enough to divide them.
    Units that cannot split evenly fall back to world = 1, then to a partial
    last frame (single rank only)."""
    for w in (world, 1):
        if n_elems % w:
            continue
        share = n_elems // w
        k = max(1, -(-share // MAX_FRAME_ELEMS))
        while share // k >= (1 << 20) or (w == 1 and share // k >= MIN_FRAME_ELEMS):
            if share % k == 0 and (share // k) % MIN_FRAME_ELEMS == 0:
                return share // k
            k += 1
    return min(MAX_FRAME_ELEMS, max(MIN_FRAME_ELEMS, (n_elems + MIN_FRAME_ELEMS - 1) // MIN_FRAME_ELEMS
                                    * MIN_FRAME_ELEMS))


@dataclasses.dataclass
class XC4Unit:
    """An encoded unit in (pinned) host memory plus its parsed header."""

    data: torch.Tensor          # uint8, the whole encoded unit
    n_elems: int
    frame_elems: int
    n_frames: int
    frame_off: np.ndarray       # uint64 [n_frames + 1]
    n_escapes: int
    code_bits: int = 4


    @classmethod
    def parse(cls, data: torch.Tensor) -> "XC4Unit":
        raw = bytes(data[:64].numpy()) if data.device.type == "cpu" else bytes(data[:64].cpu().numpy())
        h = native.XC4Header.from_buffer_copy(raw)
        if h.magic != 0x31344358 or h.version not in (1, 2):
            raise ValueError("not an XC4 unit")
        tab = data[64:64 + 8 * (h.n_frames + 1)]
        off = np.frombuffer(bytes(tab.cpu().numpy()), dtype=np.uint64).copy()
        return cls(data, int(h.n_elems), int(h.frame_elems), int(h.n_frames), off, int(h.n_escapes),
                   3 if h.version == 2 else 4)

    @property
    def nbytes(self) -> int:
        return int(self.frame_off[-1])

    @property
    def raw_bytes(self) -> int:
        return 2 * self.n_elems

    @property
    def ratio(self) -> float:
        return self.nbytes / self.raw_bytes

    def frame_range(self, rank: int, world: int) -> tuple[int, int]:
        if self.n_frames % world:
            raise ValueError(f"{self.n_frames} frames do not split over {world} ranks")
        per = self.n_frames // world
        return rank * per, (rank + 1) * per

    def frame_bytes(self, f0: int, f1: int) -> int:
        return int(self.frame_off[f1] - self.frame_off[f0])

    def max_frame_bytes(self) -> int:
        return int(np.max(np.diff(self.frame_off)))


@dataclasses.dataclass
class XC4Parts:
    """A streamed unit encoded as independent XC4 units, one per window segment
    (split window, streamer.py): segment s decodes from its own frame 0 into
    its own slot, so segment boundaries need not fall on frame boundaries."""

    parts: list

    @property
    def nbytes(self) -> int:
        return sum(u.nbytes for u in self.parts)

    @property
    def raw_bytes(self) -> int:
        return sum(u.raw_bytes for u in self.parts)

    @property
    def ratio(self) -> float:
        return self.nbytes / self.raw_bytes

    def max_frame_bytes(self) -> int:
        return max(u.max_frame_bytes() for u in self.parts)


class Encoder:
    """Device-side XC4 encoder with grow-only scratch (setup time only)."""

    def __init__(self, device, world: int = SLICE_WORLD, code_bits: int = 0):
        self.device = torch.device(device)
        self.world = world
        self.code_bits = code_bits  # 0 = per unit, the smaller of 3- and 4-bit codes
        self._scratch = None
        self._dst = None

    def _grow(self, name: str, nbytes: int) -> torch.Tensor:
        t = getattr(self, name)
        if t is None or t.numel() < nbytes:
            t = None
            setattr(self, name, None)
            t = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            setattr(self, name, t)
        return t

    def encode(self, unit: torch.Tensor) -> tuple[torch.Tensor, native.XC4Header]:
        """bf16 device tensor → (device uint8 view of the encoded unit, header)."""
        flat = unit.reshape(-1)
        if flat.dtype != torch.bfloat16:
            flat = flat.view(torch.bfloat16)
        n = flat.numel()
        fe = frame_elems_for(n, self.world)
        scratch = self._grow("_scratch", native.xc4_scratch_bytes(n, fe))
        nbytes, _ = native.xc4_encode(flat, fe, None, scratch, code_bits=self.code_bits)
        dst = self._grow("_dst", nbytes)
        nbytes, h = native.xc4_encode(flat, fe, dst, scratch, code_bits=self.code_bits)
        return dst[:nbytes], h

    def release(self) -> None:
        self._scratch = None
        self._dst = None


def encode_to_host(unit: torch.Tensor, encoder: Encoder, host_alloc=None) -> XC4Unit:
    """Encode a device unit and copy the result into pinned host memory."""
    dev, _ = encoder.encode(unit)
    buf = host_alloc(dev.numel()) if host_alloc is not None else torch.empty(dev.numel(), dtype=torch.uint8,
                                                                             pin_memory=True)
    buf = buf.view(torch.uint8)[: dev.numel()]
    buf.copy_(dev)
    return XC4Unit.parse(buf)


def encode_segments_to_host(unit: torch.Tensor, encoder: Encoder, segments, host_alloc=None):
    """One XC4Unit for the whole unit, or (``segments`` = byte ranges of a split
    window) an XC4Parts with one independently encoded unit per range."""
    if not segments or len(segments) == 1:
        return encode_to_host(unit, encoder, host_alloc)
    flat = unit.reshape(-1).view(torch.uint8)
    return XC4Parts([encode_to_host(flat[lo:hi].view(torch.bfloat16), encoder, host_alloc) for lo, hi in segments])


def decode_unit(u: XC4Unit, out: torch.Tensor) -> None:
    """Test helper: copy a host unit's encoded bytes to the device and decode
    all its frames into ``out`` (device, ≥ 2·n_elems bytes); synchronous."""
    dev = u.data.to(out.device)
    native.xc4_decode(u.data.data_ptr(), dev.data_ptr(), 0, u.n_frames, out.data_ptr())
    torch.cuda.current_stream(out.device).synchronize()
    del dev


# ctypes cursor type re-exported for the streamer
Cursor = ctypes.c_uint64
