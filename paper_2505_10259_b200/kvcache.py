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


DEFAULT_PAGE = 16  # tokens per page: small pages waste ≤ 15 slots per sequence


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

    def layer(self, li: int) -> tuple[torch.Tensor, torch.Tensor]:
        return self.k[li], self.v[li]
