"""Paged KV cache in HBM (target and draft).

Layout per model: K and V pools [n_layer, n_pages, n_kv_head, page_size, dh]
bf16, so one page of one KV head is a contiguous [page_size, dh] run — the
unit the verification-attention kernel stages with coalesced 16-B copies.
Sequence s owns the pages listed in row s of ``block_table`` [n_seq, pages].
The reference charges this memory as kv_bytes_per_token_per_layer × tokens ×
n_layer (costmodel.py:106-138; placement.py:120-130 "target/kv") but keeps
target KV on the CPU during decoding; here it is HBM-resident.
"""
from __future__ import annotations

import numpy as np
import torch

from .config import ModelArch


DEFAULT_PAGE = 32  # tokens per page: ≤ 31 slots wasted per sequence; half the TMA page boxes of 16 (profiles/kernels_r2.md)


class PagedKVCache:
    def __init__(self, arch: ModelArch, n_seq: int, max_len: int, device, page_size: int = DEFAULT_PAGE):
        self.arch = arch
        self.page_size = page_size
        self.pages_per_seq = (max_len + page_size - 1) // page_size
        self.n_seq = n_seq
        n_pages = n_seq * self.pages_per_seq
        shape = (arch.n_layer, n_pages, arch.n_kv_head, page_size, arch.head_dim)
        self.k = torch.empty(shape, dtype=torch.bfloat16, device=device)
        self.v = torch.empty(shape, dtype=torch.bfloat16, device=device)
        # contiguous page ranges per sequence (any permutation would do: the
        # kernels only ever read through the table)
        bt = np.arange(n_pages, dtype=np.int32).reshape(n_seq, self.pages_per_seq)
        self._bt_host = bt
        self.block_table = torch.from_numpy(bt).to(device)

    @staticmethod
    def bytes_needed(arch: ModelArch, n_seq: int, max_len: int, page_size: int = DEFAULT_PAGE) -> int:
        pages = n_seq * ((max_len + page_size - 1) // page_size)
        return 2 * arch.n_layer * pages * arch.n_kv_head * page_size * arch.head_dim * 2

    def slots(self, seq_ids: np.ndarray, positions: np.ndarray) -> np.ndarray:
        """Flat slot index page·page_size + offset for each (seq, position)."""
        seq_ids = np.asarray(seq_ids)
        positions = np.asarray(positions)
        pages = self._bt_host[seq_ids, positions // self.page_size]
        return (pages * self.page_size + positions % self.page_size).astype(np.int32)

    def layer(self, li: int, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        return self.k[li], self.v[li]

    def release(self, li: int, stream) -> None:
        """End of layer li's use in a pass (HBM-resident pools: nothing to do)."""

    def set_window(self, lo_seq: int, hi_seq: int) -> None:
        """All sequences are always resident."""

    def join(self, stream) -> None:
        """Make ``stream`` wait for every copy this cache issued (HBM pools: none)."""


class HostPagedKVCache(PagedKVCache):
    """Target KV in pinned host DRAM, one verified batch's pages staged per layer.

    The reference keeps target KV in CPU memory and runs attention there
    (placement.py:120-130 "target/kv" outside the GPU set; attn_cpu,
    costmodel.py:73).  On B200 attention stays on the GPU, but when the HBM
    budget is tiny (configs[1]: 24 GB, most of it the draft) the KV pool moves
    to host DRAM: for layer ℓ of a pass, the current window's pages
    ([page base, base + n)) are copied host → HBM into one of two window slots
    one layer ahead (H2D stream), attention and the KV append run on the slot,
    and the slot is written back (D2H stream — the other direction of the
    full-duplex link) before it is reused.  Block tables and slot indices the
    engine builds are window-relative while a window is set.
    """

    def __init__(self, arch: ModelArch, n_seq: int, max_len: int, device, page_size: int = DEFAULT_PAGE,
                 window_seqs: int | None = None, host_alloc=None):
        from . import native

        self.arch = arch
        self.page_size = page_size
        self.pages_per_seq = (max_len + page_size - 1) // page_size
        self.n_seq = n_seq
        n_pages = n_seq * self.pages_per_seq
        self.page_elems = arch.n_kv_head * page_size * arch.head_dim
        shape = (arch.n_layer, n_pages, arch.n_kv_head, page_size, arch.head_dim)
        nbytes = arch.n_layer * n_pages * self.page_elems * 2

        def pinned():
            if host_alloc is not None:
                return host_alloc(nbytes).view(torch.bfloat16).view(shape)
            return torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)

        self.k, self.v = pinned(), pinned()   # host pools
        bt = np.arange(n_pages, dtype=np.int32).reshape(n_seq, self.pages_per_seq)
        self._bt_global = bt
        self.block_table = torch.from_numpy(bt).to(device)
        self.window_pages = (window_seqs or n_seq) * self.pages_per_seq
        wshape = (self.window_pages, arch.n_kv_head, page_size, arch.head_dim)
        self.wk = [torch.empty(wshape, dtype=torch.bfloat16, device=device) for _ in range(2)]
        self.wv = [torch.empty(wshape, dtype=torch.bfloat16, device=device) for _ in range(2)]
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.loaded = [native.Event() for _ in range(2)]
        self.computed = [native.Event() for _ in range(2)]
        self.written = [native.Event() for _ in range(2)]
        self._native = native
        self.base, self.npages = 0, 0
        self.issued: set[int] = set()
        self.bytes_h2d = 0

    @staticmethod
    def window_bytes_needed(arch: ModelArch, window_seqs: int, max_len: int, page_size: int = DEFAULT_PAGE) -> int:
        return 2 * PagedKVCache.bytes_needed(arch, window_seqs, max_len, page_size) // arch.n_layer

    def set_window(self, lo_seq: int, hi_seq: int) -> None:
        """Sequences [lo, hi) are the ones the next pass touches."""
        n = (hi_seq - lo_seq) * self.pages_per_seq
        if n > self.window_pages:
            raise ValueError(f"KV window holds {self.window_pages} pages, the pass needs {n}")
        self.base, self.npages = lo_seq * self.pages_per_seq, n
        self.issued = set()

    @property
    def _bt_host(self) -> np.ndarray:
        return self._bt_global - self.base

    def slots(self, seq_ids: np.ndarray, positions: np.ndarray) -> np.ndarray:
        seq_ids = np.asarray(seq_ids)
        positions = np.asarray(positions)
        pages = self._bt_global[seq_ids, positions // self.page_size] - self.base
        return (pages * self.page_size + positions % self.page_size).astype(np.int32)

    def _issue(self, li: int) -> None:
        w = li % 2
        self.written[w].wait(self.h2d)  # the slot's previous layer is back in host memory
        n = self.npages * self.page_elems * 2
        for win, pool in ((self.wk[w], self.k), (self.wv[w], self.v)):
            self._native.memcpy_async(win.data_ptr(), pool[li, self.base].data_ptr(), n, self.h2d)
        self.loaded[w].record(self.h2d)
        self.issued.add(li)
        self.bytes_h2d += 2 * n

    def layer(self, li: int, stream=None):
        if li not in self.issued:
            self._issue(li)
        if li + 1 < self.arch.n_layer and li + 1 not in self.issued:
            self._issue(li + 1)  # one layer ahead
        w = li % 2
        self.loaded[w].wait(stream)
        return self.wk[w], self.wv[w]

    def release(self, li: int, stream) -> None:
        w = li % 2
        self.computed[w].record(stream)
        self.computed[w].wait(self.d2h)
        n = self.npages * self.page_elems * 2
        for win, pool in ((self.wk[w], self.k), (self.wv[w], self.v)):
            self._native.memcpy_async(pool[li, self.base].data_ptr(), win.data_ptr(), n, self.d2h)
        self.written[w].record(self.d2h)

    def join(self, stream) -> None:
        """``stream`` waits for both window slots' last write-back (d2h stream)."""
        for ev in self.written:
            ev.wait(stream)

    def fill_random(self, g: torch.Generator, device) -> None:
        """Synthetic prompt KV (decode benchmarks), generated on the GPU per layer."""
        tmp = torch.empty(self.k.shape[1:], dtype=torch.bfloat16, device=device)
        for pool in (self.k, self.v):
            for li in range(self.arch.n_layer):
                tmp.normal_(0.0, 1.0, generator=g)
                pool[li].copy_(tmp)
        torch.cuda.synchronize(device)
