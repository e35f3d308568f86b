"""Target (Mixtral-style MoE, FFN streamed) and draft (Mistral-style dense,
HBM-resident) models as sequences of C-ABI kernel launches.

The reference defines no model; the interface here is the one
SURVEY.md §8b asks for: ``spec()`` returns the reference ``ModelSpec``;
``forward`` runs new tokens of a set of sequences through the model over the
paged KV cache and returns fp32 logits.  Every op is an sm_100a kernel from
``native`` launched on the caller's stream; nothing here computes on the CPU.

Per layer (simulator.py:168-192):
    xn = RMSNorm(x) → qkv = xn·Wqkvᵀ (tcgen05) → RoPE + KV append →
    paged attention (mma.sync) → h = attn·Woᵀ + x (fused residual epilogue) →
    hn = RMSNorm(h) → [MoE]  top-2 router + permute → grouped gate_up GEMM
    with fused SwiGLU → grouped down GEMM with fused routing-weight scale →
    deterministic two-slot combine + residual
                     [dense] gate_up GEMM + SwiGLU → down GEMM + residual

The loop is layer-major over *chunks*: a verify or draft step is one chunk;
prefill splits the prompts into token-bounded chunks and runs every chunk
through layer ℓ before layer ℓ+1, so each streamed layer crosses the host
link once per prefill (the zig-zag order of PAPER.md:135-136 / FlexGen).
"""
from __future__ import annotations

import math

import torch

from . import native
from .config import ModelArch
from .kvcache import PagedKVCache
from .weights import ModelWeights, ffn_offsets


class Workspace:
    """Grow-only scratch buffers, one set per stream (target / draft)."""

    def __init__(self, device):
        self.device = torch.device(device)
        self._bufs: dict[str, torch.Tensor] = {}

    def get(self, name: str, shape, dtype) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= int(s)
        esize = torch.empty((), dtype=dtype).element_size()
        nbytes = max(n * esize, 16)
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < nbytes:
            # grow with 50% headroom: the re-prefill chunk grows a little every
            # round, and each device allocation risks an allocator reclaim
            # (cudaFree = whole-device synchronisation) inside the round loop
            grown = nbytes if buf is None else max(nbytes, buf.numel() * 3 // 2)
            grown = (grown + (2 << 20) - 1) // (2 << 20) * (2 << 20)
            buf = torch.empty(grown, dtype=torch.uint8, device=self.device)
            self._bufs[name] = buf
        return buf[: n * esize].view(dtype).view(*shape)

    def bytes(self) -> int:
        return sum(b.numel() for b in self._bufs.values())


class ForwardBatch:
    """Device-side metadata of one chunk of a forward call (built by the engine).

    Rows [row0, row0 + T) of the call's hidden-state buffer belong to this
    chunk; its sequences' query rows are given CSR-style by ``q_start``.
    """

    def __init__(self, tokens, positions, slots, q_start, kv_before, block_table, n_seq, max_q,
                 last_rows=None, row0: int = 0, last_pos=None, last_qs=None):
        self.tokens = tokens          # int32 [T]
        self.positions = positions    # int32 [T]
        self.slots = slots            # int32 [T]
        self.q_start = q_start        # int32 [n_seq+1], relative to row0
        self.kv_before = kv_before    # int32 [n_seq]
        self.block_table = block_table  # int32 [n_seq, pages] (view of the cache's table)
        self.n_seq = n_seq
        self.max_q = max_q
        self.last_rows = last_rows    # int32 [k] absolute rows whose logits are wanted (None = all)
        self.row0 = row0
        # with last_rows: the positions of those rows (int32 [k]) and arange(k + 1) (int32) — given,
        # the last layer runs attention onward for those rows only (the rest only feeds the KV cache)
        self.last_pos = last_pos
        self.last_qs = last_qs

    @property
    def T(self) -> int:
        return self.tokens.numel()


class CausalLM:
    """Shared forward of the target and the draft."""

    ARITH = ("tensor", "canonical")

    def __init__(self, weights: ModelWeights, device, streamer=None, arith: str = "tensor"):
        """``arith="tensor"``: the product kernels (tcgen05 GEMMs, mma.sync
        attention).  ``"canonical"``: the parity mode — the same ops at the
        same bf16 rounding points in a fixed IEEE order (csrc/canon.cu) that
        the CPU oracle reproduces bit for bit; CUDA-core code for tiny shapes."""
        if arith not in self.ARITH:
            raise ValueError(f"arith must be one of {self.ARITH}, got {arith!r}")
        self.w = weights
        self.arch: ModelArch = weights.arch
        self.device = torch.device(device)
        self.streamer = streamer
        self.ws = Workspace(device)
        self.hooks = None  # optional callback(layer, phase, stream) used by the tracer
        self.arith = arith
        canon = arith == "canonical"
        self._gemm = native.canon_gemm if canon else native.gemm
        self._gemm_grouped = native.canon_gemm_grouped if canon else native.gemm_grouped
        self._rmsnorm = native.canon_rmsnorm if canon else native.rmsnorm
        self._attn = native.canon_attn_paged if canon else native.attn_paged
        self._router = native.canon_router_top2 if canon else native.router_top2
        self._rope_table = None  # canonical RoPE: host-computed cos/sin rows, grown to the KV capacity

    def spec(self):
        return self.arch.spec()

    # ------------------------------------------------------------------
    def forward(self, chunks: list[ForwardBatch] | ForwardBatch, kv: PagedKVCache, stream: torch.cuda.Stream,
                logits_out: torch.Tensor | None = None, want_logits: bool = True) -> torch.Tensor | None:
        if isinstance(chunks, ForwardBatch):
            chunks = [chunks]
        with torch.cuda.stream(stream):
            return self._forward(chunks, kv, stream, logits_out, want_logits)

    def _forward(self, chunks, kv, stream, logits_out, want_logits):
        a, ws = self.arch, self.ws
        Ttot = sum(c.T for c in chunks)
        Tmax = max(c.T for c in chunks)
        H, dh, hq, hkv = a.hidden, a.head_dim, a.n_head, a.n_kv_head
        # one hidden-state buffer for all chunks, updated in place: a layer reads
        # x only until h = attn·Woᵀ + x exists, so its output can overwrite x
        xa = ws.get("x", (Ttot, H), torch.bfloat16)
        xn = ws.get("xn", (Tmax, H), torch.bfloat16)
        h = ws.get("h", (Tmax, H), torch.bfloat16)
        qkv = ws.get("qkv", (Tmax, a.qkv_rows), torch.bfloat16)
        q = ws.get("q", (Tmax, hq * dh), torch.bfloat16)
        att = ws.get("att", (Tmax, hq * dh), torch.bfloat16)
        scale = 1.0 / math.sqrt(dh)
        for c in chunks:
            native.embed(c.tokens, self.w.embed, xa[c.row0:c.row0 + c.T], stream)
        hook = self.hooks
        q_dim = hq * dh
        c0 = chunks[0]
        # last-layer pruning (a context re-prefill wants one row of logits per sequence): the last
        # layer's K/V need every row, its attention, O, FFN and the LM head only the wanted rows
        prune = (len(chunks) == 1 and c0.row0 == 0 and c0.last_rows is not None and c0.last_pos is not None
                 and c0.last_qs is not None and self.arith == "tensor")
        n_layers = len(self.w.layers)
        x_last = None
        for li, L in enumerate(self.w.layers):
            if hook:
                hook(li, "attn_start", stream)
            kc, vc = kv.layer(li, stream)
            base = None
            split = self._split(li)  # [.. gate_up | down] in two window slots (streamer segments)
            base_dn = None
            wqkv, wo = L.wqkv, L.wo
            ffn_off = 0  # the FFN's byte offset inside the streamed unit
            if wqkv is None:  # attention weights stream with the layer: wait before QKV
                unit = self._ffn_acquire(li, L, stream)
                wqkv = _RawView(unit, (a.qkv_rows, H))
                wo = _RawView(unit + a.qkv_rows * H * 2, (H, q_dim))
                ffn_off = (a.qkv_rows * H + H * q_dim) * 2
                base = unit + ffn_off
            for ci, c in enumerate(chunks):
                T = c.T
                x = xa[c.row0:c.row0 + T]
                out = x  # in place (see above)
                self._rmsnorm(x, L.attn_norm, xn[:T], a.eps, stream)
                self._gemm(xn[:T], wqkv, qkv[:T], native.EPI_BF16, None, stream)
                self._rope(kv, qkv[:T], c.positions, c.slots, q[:T], kc, vc, stream)
                if prune and li == n_layers - 1:  # the wanted rows only from here on
                    k = c.last_rows.numel()
                    q_l = ws.get("q_last", (k, q_dim), torch.bfloat16)
                    x_last = ws.get("x_last", (k, H), torch.bfloat16)
                    native.embed(c.last_rows, q[:T], q_l, stream)
                    native.embed(c.last_rows, xa, x_last, stream)
                    self._attn(q_l, kc, vc, c.block_table, c.last_qs, c.last_pos, 1, hq, hkv, dh, kv.page_size,
                               scale, att[:k], stream)
                    T, x, out = k, x_last, x_last
                else:
                    self._attn(q[:T], kc, vc, c.block_table, c.q_start, c.kv_before, c.max_q, hq, hkv, dh,
                               kv.page_size, scale, att[:T], stream)
                self._gemm(att[:T], wo, h[:T], native.EPI_BF16_RESID, x, stream)
                self._rmsnorm(h[:T], L.ffn_norm, xn[:T], a.eps, stream)
                if ci == 0:
                    if base is None:
                        base = self._ffn_acquire(li, L, stream)
                    if hook:
                        hook(li, "ffn_start", stream)
                if a.is_moe:
                    self._moe_up(L, base, xn[:T], T, stream)
                else:
                    self._mlp_up(base, xn[:T], T, stream)
                if base_dn is None:
                    if split:
                        # one chunk: gate_up's slot goes back to the link before down waits for its own
                        if len(chunks) == 1:
                            self.streamer.release(li, stream, 0)
                        base_dn = self.streamer.acquire(li, stream, 1) + ffn_off
                        if hook:
                            hook(li, "ffn_part", stream)
                    else:
                        base_dn = base
                if a.is_moe:
                    self._moe_down(base_dn, h[:T], out, T, stream)
                else:
                    self._mlp_down(base_dn, h[:T], out, T, stream)
            kv.release(li, stream)  # host-resident KV: write the layer's window back
            if split:
                if len(chunks) > 1:
                    self.streamer.release(li, stream, 0)
                self.streamer.release(li, stream, 1)
            else:
                self._ffn_release(li, stream)
            if hook:
                hook(li, "ffn_end", stream)
        if not want_logits:
            return None
        rows_idx = [c.last_rows for c in chunks if c.last_rows is not None]
        x = xa
        if x_last is not None:  # pruned last layer: the wanted rows are already compact
            x = x_last
        elif rows_idx:
            assert len(rows_idx) == 1, "last_rows are given once, on the first chunk"
            sel = rows_idx[0]
            rows = ws.get("lastx", (sel.numel(), H), torch.bfloat16)
            native.embed(sel, xa, rows, stream)  # row gather: rows[i] = x[sel[i]]
            x = rows
        R = x.shape[0]
        xf = ws.get("xf", (R, H), torch.bfloat16)
        self._rmsnorm(x, self.w.final_norm, xf, a.eps, stream)
        if logits_out is None:
            logits_out = ws.get("logits", (R, a.vocab), torch.float32)
        self._gemm(xf, self.w.lm_head, logits_out, native.EPI_F32, None, stream)
        return logits_out

    def _rope(self, kv, qkv, positions, slots, q, kc, vc, stream):
        a = self.arch
        if self.arith == "tensor":
            native.rope_kv_append(qkv, positions, slots, a.n_head, a.n_kv_head, a.head_dim, a.rope_theta,
                                  kv.page_size, q, kc, vc, stream)
            return
        rows = kv.pages_per_seq * kv.page_size  # every position a sequence of this cache can hold
        if self._rope_table is None or self._rope_table.shape[0] < rows:
            self._rope_table = torch.from_numpy(rope_table(a.head_dim, a.rope_theta, rows)).to(self.device)
        native.canon_rope_kv_append(qkv, positions, slots, a.n_head, a.n_kv_head, a.head_dim, self._rope_table,
                                    kv.page_size, q, kc, vc, stream)

    # ------------------------------------------------------------------
    def _ffn_acquire(self, li, L, stream) -> int:
        if self.streamer is not None:
            return self.streamer.acquire(li, stream)
        return L.ffn.data_ptr()

    def _ffn_release(self, li, stream) -> None:
        if self.streamer is not None:
            self.streamer.release(li, stream)

    def _split(self, li) -> bool:
        st = self.streamer
        return st is not None and len(st.segments) > 1 and li in st.host

    def _moe_up(self, L, base, xn, T, stream):
        """top-2 router + permute, grouped gate_up GEMM with the SwiGLU epilogue
        (reads the unit's gate_up range only)."""
        a, ws = self.arch, self.ws
        E, H, I = a.n_expert, a.hidden, a.inter
        rows = 2 * T
        offs = ws.get("offs", (E + 1,), torch.int32)
        perm = ws.get("perm", (rows,), torch.int32)
        roww = ws.get("roww", (rows,), torch.float32)
        trows = ws.get("trows", (T, 2), torch.int32)
        xperm = ws.get("xperm", (rows, H), torch.bfloat16)
        act = ws.get("act", (rows, I), torch.bfloat16)
        rws = ws.get("router_ws", (native.router_workspace_bytes(T, E),), torch.uint8)
        self._router(xn, L.router, offs, perm, roww, trows, xperm, rws, stream=stream)
        self._gemm_grouped(xperm, base, offs, E, 2 * I, act, native.EPI_SWIGLU, None, stream)

    def _moe_down(self, base, h, out, T, stream):
        """grouped down GEMM with the routing-weight row scale, then the top-2
        combine + residual (reads the unit's down range only)."""
        a, ws = self.arch, self.ws
        E, H, I = a.n_expert, a.hidden, a.inter
        rows = 2 * T
        offs = ws.get("offs", (E + 1,), torch.int32)
        roww = ws.get("roww", (rows,), torch.float32)
        trows = ws.get("trows", (T, 2), torch.int32)
        act = ws.get("act", (rows, I), torch.bfloat16)
        y = ws.get("y", (rows, H), torch.bfloat16)
        gu_elems, _, _ = ffn_offsets(a)
        self._gemm_grouped(act, base + 2 * gu_elems, offs, E, H, y, native.EPI_BF16_ROWSCALE, roww, stream)
        native.moe_combine(y, trows, h, out, stream)

    def _mlp_up(self, base, xn, T, stream):
        a, ws = self.arch, self.ws
        I, H = a.inter, a.hidden
        act = ws.get("act", (T, I), torch.bfloat16)
        gu = _raw_bf16(base, (2 * I, H), self.device)
        self._gemm(xn, gu, act, native.EPI_SWIGLU, None, stream)

    def _mlp_down(self, base, h, out, T, stream):
        a, ws = self.arch, self.ws
        I, H = a.inter, a.hidden
        act = ws.get("act", (T, I), torch.bfloat16)
        gu_elems, _, _ = ffn_offsets(a)
        dn = _raw_bf16(base + 2 * gu_elems, (H, I), self.device)
        self._gemm(act, dn, out, native.EPI_BF16_RESID, h, stream)


def rope_table(dh: int, theta: float, rows: int):
    """cos/sin rows of the canonical RoPE: [rows, dh] fp32, cos(p·f_i) in columns
    [0, dh/2), sin(p·f_i) in [dh/2, dh), f_i = θ^(−2i/dh) — evaluated in float64
    on the host and rounded once (setup-time constants of the parity mode)."""
    import numpy as np

    inv = 1.0 / theta ** (np.arange(0, dh, 2, dtype=np.float64) / dh)
    ang = np.arange(rows, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


class _RawView:
    """Minimal tensor-like view of device memory by address (for native.gemm)."""

    def __init__(self, ptr: int, shape):
        self._ptr = ptr
        self.shape = tuple(shape)
        self.dtype = torch.bfloat16

    def data_ptr(self) -> int:
        return self._ptr


def _raw_bf16(ptr: int, shape, device) -> _RawView:
    return _RawView(ptr, shape)


class SeqState:
    """Decoding state of a set of sequences — the ``state`` argument of the
    model protocol: a paged KV cache, the cache row of each
    sequence, its committed context length (KV positions [0, ctx) are valid)
    and its last committed token (position ctx, KV not yet written).

    One state per model: the target's and the draft's rows may differ (the
    engine gives re-prefilled draft sequences scratch rows)."""

    def __init__(self, kv: PagedKVCache, rows, ctx, t_last, stream: torch.cuda.Stream | None = None):
        import numpy as np

        self.kv = kv
        self.rows = np.asarray(rows, np.int64)
        self.ctx = np.asarray(ctx, np.int64).copy()
        self.t_last = np.asarray(t_last, np.int32).copy()
        self.stream = stream
        if not (self.rows.shape == self.ctx.shape == self.t_last.shape):
            raise ValueError("rows, ctx and t_last need one entry per sequence")

    @property
    def bs(self) -> int:
        return int(self.rows.size)

    def advance(self, counts, tokens) -> None:
        """Commit ``counts[i]`` tokens ``tokens[i, :counts[i]]`` (accept/reject
        output, acceptance.py:1-6): the context grows by the count and the last
        committed token becomes the new t_last.  KV written beyond the new
        context is stale and is overwritten by the next step at that position."""
        import numpy as np

        counts = np.asarray(counts, np.int64)
        tokens = np.asarray(tokens)
        for i, c in enumerate(counts):
            if c > 0:
                self.ctx[i] += c
                self.t_last[i] = tokens[i, c - 1]


def _dev_i32(a, device) -> torch.Tensor:
    import numpy as np

    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.int32))).to(device, non_blocking=False)


def _step_batch(kv, rows, positions, tokens_dev, device, max_q: int) -> ForwardBatch:
    """ForwardBatch of ``max_q`` consecutive positions per sequence starting at
    ``positions[:, 0]`` (verify: t_last + n_cand drafts; draft step: one)."""
    import numpy as np

    n_seq = rows.size
    slots = kv.slots(np.broadcast_to(rows[:, None], positions.shape), positions)
    qs = np.arange(n_seq + 1) * max_q
    bt = _dev_i32(kv._bt_host[rows], device)  # window-relative pages for host-resident KV
    return ForwardBatch(tokens_dev, _dev_i32(positions.ravel(), device), _dev_i32(slots.ravel(), device),
                        _dev_i32(qs, device), _dev_i32(positions[:, 0], device), bt, n_seq, max_q)


class TargetModel(CausalLM):
    """Mixtral-style MoE verifier; FFN layers come through the streamer."""

    def verify(self, state: SeqState, draft_tokens) -> torch.Tensor:
        """Target logits of t_last and the drafted tokens: ``draft_tokens``
        [bs, n_cand] → fp32 logits [bs, n_cand + 1, V] (row j scores the token
        after position ctx + j).  Appends the n_cand + 1
        positions to the KV cache; the accept/reject step decides how many of
        them the context keeps (``SeqState.advance``)."""
        import numpy as np

        dev = self.device
        st = state.stream or torch.cuda.current_stream(dev)
        state.kv.set_window(int(state.rows.min()), int(state.rows.max()) + 1)  # host-resident KV: the pass's pages
        with torch.cuda.stream(st):  # metadata copies ordered before the kernels that read them
            d = torch.as_tensor(draft_tokens, dtype=torch.int32).to(dev)
            bs, n = d.shape
            if bs != state.bs:
                raise ValueError(f"draft_tokens has {bs} rows, the state {state.bs} sequences")
            toks = torch.cat([_dev_i32(state.t_last, dev)[:, None], d], dim=1).contiguous()
            pos = state.ctx[:, None] + np.arange(n + 1)[None, :]
            fb = _step_batch(state.kv, state.rows, pos, toks.view(-1), dev, n + 1)
            out = torch.empty((bs * (n + 1), self.arch.vocab), dtype=torch.float32, device=dev)
            self.forward(fb, state.kv, st, logits_out=out)
        return out.view(bs, n + 1, self.arch.vocab)


class DraftModel(CausalLM):
    """Mistral-style dense drafter, fully HBM-resident."""

    def draft(self, state: SeqState, n_cand: int, bs_draft: int | None = None, uniforms=None,
              temperature: float = 1.0):
        """``n_cand`` draft tokens per sequence from cached-KV decode steps, in
        chunks of ``bs_draft`` sequences (costmodel.py:53-57): tokens
        [bs, n_cand] int32, greedy; with ``uniforms`` [bs, n_cand] (inverse-CDF
        sampling at ``temperature``) also the draft distributions
        [bs, n_cand, V] fp32 the sampling accept step needs.  A last step
        writes the KV of d_n, so after ``advance`` the cache holds every
        committed position (no rollback copies)."""
        import numpy as np

        from . import native

        dev = self.device
        st = state.stream or torch.cuda.current_stream(dev)
        bs = state.bs
        step = bs_draft or bs
        V = self.arch.vocab
        with torch.cuda.stream(st):
            tokens = torch.empty((bs, n_cand), dtype=torch.int32, device=dev)
            probs = torch.empty((bs, n_cand, V), dtype=torch.float32, device=dev) if uniforms is not None else None
            u = None if uniforms is None else torch.as_tensor(uniforms, dtype=torch.float32).to(dev).contiguous()
            logits = torch.empty((step, V), dtype=torch.float32, device=dev)
            for lo in range(0, bs, step):
                hi = min(bs, lo + step)
                rows = state.rows[lo:hi]
                cur = _dev_i32(state.t_last[lo:hi], dev)
                for j in range(n_cand + 1):
                    pos = state.ctx[lo:hi, None] + j
                    fb = _step_batch(state.kv, rows, pos, cur, dev, 1)
                    if j == n_cand:
                        self.forward(fb, state.kv, st, want_logits=False)  # KV of d_n only
                        break
                    lg = self.forward(fb, state.kv, st, logits_out=logits[:hi - lo])
                    out = tokens[lo:hi, j]
                    if u is None:
                        native.sample_tokens(lg, out, stream=st)
                    else:
                        native.sample_tokens(lg, out, uniforms=u[lo:hi, j].contiguous(), out_probs=probs[lo:hi, j],
                                             temperature=temperature, stream=st)
                    cur = out.contiguous()
        return tokens if probs is None else (tokens, probs)
