"""Ping-pong executor: the measured counterpart of the reference's pipeline engine.

Reference: ``simulate_decoding(policy, workload, hw, target, draft, plan, seed)
-> SimResult`` (simulator.py:108-227) *models* barrier-synchronised rounds in
which one batch is verified layer by layer while the other drafts
(simulator.py:155-215).  ``Engine.run_decoding`` keeps that
signature and returns a *measured* ``SimResult``; ``Engine.generate`` is the
user entry the reference lacks.

Physical schedule of round r (b = r mod 2), all enqueued without host syncs:
  copy stream    K1 chunks of the streamed FFN layers, running ahead of compute
                 into the HBM window (streamer.py);
  target stream  verify batch b: per layer attention (KV in HBM) → wait for
                 the layer's FFN slot → MoE → release the slot; LM head; K7
                 accept/reject; device→host copy of the committed tokens;
  draft stream   batch 1−b: n_cand+1 cached-KV decode steps of the resident
                 draft (the extra step fills the KV of d_n so both caches
                 always agree with the committed prefix: no rollback copies);
  barrier        host waits on both streams, reads the committed counts.
Round accounting: one verification per round — the reference
decrements both batches per round.
"""
from __future__ import annotations

import dataclasses
import threading
import time

import numpy as np
import torch

from . import native
from .acceptance import forced_counts, input_uniforms
from .domain import Policy
from .kvcache import HostPagedKVCache, PagedKVCache
from .models import DraftModel, ForwardBatch, TargetModel
from .trace import SimResult, Tracer, busy


@dataclasses.dataclass(frozen=True)
class Forced:
    """Forced-acceptance mode: committed counts drawn from AcceptanceModel(p, n_cand)."""

    p: float


class _Batch:
    def __init__(self, lo: int, hi: int):
        self.lo, self.hi = lo, hi

    @property
    def n(self) -> int:
        return self.hi - self.lo

    @property
    def ids(self) -> np.ndarray:
        return np.arange(self.lo, self.hi)


class _StagingArena:
    """Bump allocator over a pinned host buffer and an HBM buffer of the same size.

    Each ``put`` writes a host array into the next free host slice, copies it
    to the matching device slice with an SM copy on the given stream and
    returns the device view.  Slices are reused only after ``reset`` (called
    at the round barrier, when every copy has completed).  Growth allocates a
    larger pair and retires the old one at the next reset.
    """

    ALIGN = 256

    def __init__(self, device, capacity: int = 8 << 20):
        self.device = device
        self.off = 0
        self.retired: list = []
        self._alloc(capacity)

    def _alloc(self, capacity: int) -> None:
        self.cap = capacity
        self.host = torch.empty(capacity, dtype=torch.uint8, pin_memory=True)
        self.dev = torch.empty(capacity, dtype=torch.uint8, device=self.device)
        self.off = 0

    def put(self, a: np.ndarray, dtype: torch.dtype, stream) -> torch.Tensor:
        nbytes = a.nbytes
        if self.off + nbytes > self.cap:
            self.retired.append((self.host, self.dev))
            self._alloc(max(2 * self.cap, 2 * nbytes))
        lo = self.off
        self.off = (lo + nbytes + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        hv = self.host[lo:lo + nbytes].numpy()
        hv[:] = a.view(np.uint8).reshape(-1)
        native.copy_sm(self.dev.data_ptr() + lo, self.host.data_ptr() + lo, nbytes, stream)
        return self.dev[lo:lo + nbytes].view(dtype).view(a.shape)

    def reset(self) -> None:
        self.off = 0
        self.retired.clear()


class DecodeSession:
    """All per-run state: caches, per-sequence counters, committed tokens."""

    def __init__(self, engine: "Engine", n_seq: int, bs_decoding: int, max_len: int, n_cand: int,
                 mode: str, seed: int, temperature: float, forced_p: float | None, bs_draft: int,
                 draft_kv: str = "cached", draft_cached: int | None = None, prompts: list | None = None,
                 max_new: int = 0, max_admit: int | None = None, kv_host: bool = False):
        self.e = engine
        self.n_seq = n_seq
        self.n_cand = n_cand
        self.mode = mode
        self.seed = seed
        self.temperature = temperature
        self.forced_p = forced_p
        self.bs_draft = bs_draft
        if draft_kv not in ("cached", "reprefill", "mixed"):
            raise ValueError(f"draft_kv must be 'cached', 'reprefill' or 'mixed', got {draft_kv!r}")
        if draft_kv == "mixed" and draft_cached is None:
            raise ValueError("draft_kv='mixed' needs draft_cached (cached sequences per batch)")
        self.draft_kv = draft_kv
        self.batches = [_Batch(0, min(bs_decoding, n_seq)), _Batch(min(bs_decoding, n_seq), n_seq)]
        dev = engine.device
        # target KV in HBM, or (kv_host, for tiny HBM budgets) in pinned host DRAM
        # with one batch's pages staged per layer (kvcache.HostPagedKVCache)
        self.tkv = (HostPagedKVCache(engine.target.arch, n_seq, max_len, dev, engine.page_size,
                                     window_seqs=max(b.n for b in self.batches), host_alloc=engine.host_alloc)
                    if kv_host else PagedKVCache(engine.target.arch, n_seq, max_len, dev, engine.page_size))
        # Draft KV policy (planner choice):
        #   cached    one persistent draft KV row per sequence;
        #   reprefill the paper's draft (costmodel.py:53-57,
        #             132-137): the whole context is re-read each round into a
        #             scratch cache sized for one bs_draft chunk, so HBM goes to
        #             a larger batch instead;
        #   mixed     the first ``draft_cached`` sequences of each batch keep a
        #             row, the rest re-prefill — HBM and tensor time traded
        #             sequence by sequence until both bind.
        if draft_kv == "cached":
            self.n_cached = [b.n for b in self.batches]
        elif draft_kv == "reprefill":
            self.n_cached = [0, 0]
        else:
            self.n_cached = [min(int(draft_cached), b.n) for b in self.batches]
        self.drow = np.full(n_seq, -1, np.int64)   # sequence → persistent draft KV row
        r = 0
        for b, kc in zip(self.batches, self.n_cached):
            self.drow[b.lo:b.lo + kc] = np.arange(r, r + kc)
            r += kc
        self.scratch_row0 = r
        self.any_reprefill = any(kc < b.n for b, kc in zip(self.batches, self.n_cached))
        self.dkv = PagedKVCache(engine.draft.arch, max(1, r + (bs_draft if self.any_reprefill else 0)), max_len,
                                dev, engine.page_size)
        # Slot refill: with ``prompts`` the n_seq slots are a
        # pool; a prompt is admitted into a free slot of the batch about to be
        # verified, prefilled inside that verify pass (the streamed layers are
        # crossing the link anyway), drafted from its context in the next round
        # ("fresh"), and its slot is freed as soon as it has max_new tokens.
        self.refill = prompts is not None
        self.prompts = prompts
        self.max_new = max_new
        self.queue = list(range(len(prompts))) if self.refill else []
        self.queue.reverse()  # pop() from the end = admission in prompt order
        # admissions per round: prefill is the heavy part of a refill round, so
        # spreading it keeps rounds near the link pass instead of alternating
        # prefill-bound and idle-tensor rounds (and keeps finishes staggered)
        self.max_admit = max_admit
        # token history (position-indexed) for every draft that re-reads its context
        self.hist = (torch.zeros((n_seq, max_len), dtype=torch.int32, device=dev)
                     if (self.any_reprefill or self.refill) else None)
        self.max_len = max_len
        self.ctx = np.zeros(n_seq, np.int64)
        self.t_last = np.zeros(n_seq, np.int32)
        self.remaining = np.zeros(n_seq, np.int32)
        self.slot_prompt = np.full(n_seq, -1, np.int64) if self.refill else np.arange(n_seq)
        self.active = np.zeros(n_seq, bool)     # the slot holds a decoding sequence
        self.fresh = np.zeros(n_seq, bool)      # ... whose draft state must be built from its context
        self.dlist = [np.zeros(0, np.int64), np.zeros(0, np.int64)]  # slots drafted for each batch's next verify
        self.pending_new = [np.zeros(0, np.int64), np.zeros(0, np.int64)]  # slots prefilled in the next verify
        self.out: list[list[int]] = [[] for _ in range(len(prompts) if self.refill else n_seq)]
        V = engine.target.arch.vocab
        self.drafts = []
        self.qprobs = []
        for b in self.batches:
            self.drafts.append(torch.zeros((n_cand, max(b.n, 1)), dtype=torch.int32, device=dev))
            self.qprobs.append(torch.zeros((max(b.n, 1), n_cand, V), dtype=torch.float32, device=dev)
                               if mode == "sample" else None)
        self.res_tok = [torch.empty((max(b.n, 1), n_cand + 1), dtype=torch.int32, pin_memory=True)
                        for b in self.batches]
        self.res_cnt = [torch.empty(max(b.n, 1), dtype=torch.int32, pin_memory=True) for b in self.batches]
        self.res_first = [torch.empty(max(b.n, 1), dtype=torch.int32, pin_memory=True) for b in self.batches]
        self.rounds = 0
        self.committed_decode = 0
        self.recycle = None   # (ctx0, t_last0, max_new): finished sequences restart (synthetic_context)
        self.recycled = 0


class Engine:
    FRESH_CHUNK = 64  # sequences per draft context prefill of freshly admitted slots
    prefill_chunk_tokens = 16384  # prompt tokens per chunk of a verify pass that prefills (activation workspace)

    def __init__(self, target: TargetModel, draft: DraftModel, hw=None, device="cuda:0", page_size: int = 32,
                 trace: bool = True):
        self.target = target
        self.draft = draft
        self.hw = hw
        self.device = torch.device(device)
        self.page_size = page_size
        # the verify stream gets the higher priority: each layer's expert GEMMs
        # must release its window slot promptly or the copy engine idles, while
        # the draft's (re-)prefill work only has to finish by the barrier
        self.host_alloc = None   # pinned-host allocator for host-resident KV pools (None: torch's)
        # acceptance probability generate(policy=None) plans with (the reference ships none:
        # presets.py:16-19 — typical well-matched drafts measure 0.6-0.9)
        self.acceptance_p = 0.7
        self.last_policy = None
        self.tgt_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self.drf_stream = torch.cuda.Stream(device=self.device, priority=0)
        self.tracer = Tracer(trace)
        self._cur = (None, None)  # (round, batch) being verified, for trace tags
        self._marks: dict = {}
        self._part: dict = {}  # layers whose FFN ran in two parts (split window)
        self._arenas: dict = {}   # stream handle -> _StagingArena (per-round H2D metadata)
        self.nvtx_range: str | None = None  # mirrored onto the draft-enqueue thread when set
        self._join = native.Event()
        # per-round stream busy times (draft stream start→end, verify start→end), ms
        self._tev = [native.Event(timing=True) for _ in range(4)]
        self.round_times: list[tuple[float, float]] = []
        if trace:
            self.target.hooks = self._layer_hook
            if self.target.streamer is not None:
                self.target.streamer.trace = True
        native.lib()  # fail loudly now if the sm_100a library is missing
        native.set_device(self.device.index or 0)

    def _layer_hook(self, li: int, phase: str, stream) -> None:
        ev = self.tracer.mark(stream)
        rnd, bi = self._cur
        if phase == "attn_start":
            self._marks[li] = ev
        elif phase == "ffn_start":
            self.tracer.add("GPU_TARGET", "attn_gpu", self._marks.get(li), ev, bi, li, rnd)
            self._marks[li] = ev
        elif phase == "ffn_part":  # split window: the down GEMM's part waits for the second segment
            self.tracer.add("GPU_TARGET", "ffn_gpu", self._marks.get(li), ev, bi, li, rnd)
            self._marks[li] = ev
            self._part[li] = True
        else:
            label = "ffn_gpu_part" if self._part.pop(li, False) else "ffn_gpu"
            self.tracer.add("GPU_TARGET", label, self._marks.get(li), ev, bi, li, rnd)
            self._last_ffn_end = ev

    def resolve_trace(self) -> list:
        # the streamer runs ahead across rounds: copies for the next round's
        # layers may still be in flight on the copy stream when the last
        # round's barrier completes — their marks resolve once they land
        torch.cuda.synchronize(self.device)
        st = self.target.streamer
        if st is not None and self.tracer.enabled and self.tracer.t0 is not None:
            tags = {}
            for k, layer, a, b, resource, label in st.copy_marks:
                if a is not None and b is not None:
                    if k not in tags:
                        tags[k] = st.use_tags.pop(k, (None, None))
                    rnd, bi = tags[k]
                    self.tracer.add(resource, label, a, b, bi, layer, rnd)
            st.copy_marks.clear()
        return self.tracer.resolve()

    # ------------------------------------------------------------------ utils
    def _up(self, arr: np.ndarray, stream, dtype=torch.int32) -> torch.Tensor:
        """Host array → device tensor, copied asynchronously on ``stream``.

        Per-stream staging arenas (pinned host + HBM, allocated once, reset at
        every barrier) mean the round loop never calls the device allocator
        (whose reclaim path would cudaFree = synchronise the whole GPU) and
        the copy is done by SMs, never queued behind a layer on the copy
        engine."""
        a = np.ascontiguousarray(arr).astype(torch.empty((), dtype=dtype).numpy().dtype, copy=False)
        arena = self._arenas.get(stream.cuda_stream)
        if arena is None:
            arena = self._arenas[stream.cuda_stream] = _StagingArena(self.device)
        return arena.put(a, dtype, stream)

    def _release_staging(self) -> None:
        for arena in self._arenas.values():
            arena.reset()

    def set_window_slots(self, n_slots: int) -> None:
        """Resize the target's streamed-layer window between passes
        (``LayerStreamer.resize``): e.g. widen a split window to two slots per
        segment before a prefill-heavy ``generate()``, whose multi-chunk
        passes hold a layer's segments together."""
        if self.target.streamer is not None:
            torch.cuda.synchronize(self.device)
            self.target.streamer.resize(n_slots)

    def new_session(self, n_seq: int, bs_decoding: int, max_len: int, n_cand: int, mode: str = "greedy",
                    seed: int = 0, temperature: float = 1.0, forced_p: float | None = None,
                    bs_draft: int | None = None, draft_kv: str = "cached",
                    draft_cached: int | None = None, prompts: list | None = None,
                    max_new: int = 0, max_admit: int | None = None, kv_host: bool = False) -> DecodeSession:
        return DecodeSession(self, n_seq, bs_decoding, max_len, n_cand, mode, seed, temperature, forced_p,
                             bs_draft or bs_decoding, draft_kv, draft_cached, prompts, max_new, max_admit, kv_host)

    def _bt(self, kv: PagedKVCache, rows, stream) -> torch.Tensor:
        """Block-table rows of an arbitrary slot list, staged to the device."""
        return self._up(kv._bt_host[np.asarray(rows, np.int64)], stream)

    def _hist_write(self, s: DecodeSession, seqs, positions, tokens, stream) -> None:
        """Record committed tokens in the device-side history (reprefill drafts)."""
        if s.hist is None or len(seqs) == 0:
            return
        flat = (np.asarray(seqs, np.int64) * s.max_len + np.asarray(positions, np.int64))
        idx = self._up(flat, stream, torch.int64)
        val = self._up(np.asarray(tokens, np.int32), stream)
        native.scatter_i32(s.hist, idx, val, stream)

    # ---------------------------------------------------------------- prefill
    def prefill(self, s: DecodeSession, prompts: list, max_new: int, bs_prefill: int | None = None,
                chunk_tokens: int = 16384) -> None:
        """Layer-major prefill of every prompt through both models; emits token 1."""
        lens = np.array([len(p) for p in prompts], np.int64)
        assert len(prompts) == s.n_seq and lens.max() + max_new + s.n_cand + 1 <= s.max_len
        bs_prefill = bs_prefill or s.n_seq
        # chunk = consecutive sequences, ≤ bs_prefill of them and ≤ chunk_tokens
        groups, cur, cur_tok = [], [], 0
        for i, L in enumerate(lens):
            if cur and (len(cur) >= bs_prefill or cur_tok + L > chunk_tokens):
                groups.append(cur)
                cur, cur_tok = [], 0
            cur.append(i)
            cur_tok += int(L)
        groups.append(cur)
        if isinstance(s.tkv, HostPagedKVCache):  # one target pass per batch: the KV window holds one batch
            models = [(self.target, s.tkv, self.tgt_stream,
                       [[i for i in g if b.lo <= i < b.hi] for g in groups if any(b.lo <= i < b.hi for i in g)],
                       np.arange(s.n_seq), b) for b in s.batches if b.n]
        else:
            models = [(self.target, s.tkv, self.tgt_stream, groups, np.arange(s.n_seq), None)]
        if s.any_reprefill:  # the re-prefilling draft only needs the prompt tokens
            seqs = np.concatenate([np.full(L, i) for i, L in enumerate(lens)])
            pos = np.concatenate([np.arange(L) for L in lens])
            self._hist_write(s, seqs, pos, np.concatenate([np.asarray(p, np.int32) for p in prompts]),
                             self.drf_stream)
        # sequences with a persistent draft KV row prefill the draft too (rows
        # are consecutive in sequence order, so a group maps to a row range)
        dgroups = [[i for i in g if s.drow[i] >= 0] for g in groups]
        dgroups = [g for g in dgroups if g]
        if dgroups:
            models.append((self.draft, s.dkv, self.drf_stream, dgroups, s.drow, None))
        first = torch.empty(s.n_seq, dtype=torch.int32, device=self.device)
        first_h = None
        for model, kv, stream, mgroups, rowmap, window in models:
            if window is not None:
                kv.set_window(window.lo, window.hi)
            chunks = []
            row0 = 0
            last = []
            for g in mgroups:
                toks = np.concatenate([np.asarray(prompts[i], np.int32) for i in g])
                pos = np.concatenate([np.arange(lens[i]) for i in g])
                seq = np.concatenate([np.full(lens[i], rowmap[i]) for i in g])
                qs = np.concatenate([[0], np.cumsum(lens[g])]).astype(np.int32)
                meta = self._up(np.concatenate([toks, pos.astype(np.int32), kv.slots(seq, pos), qs,
                                                np.zeros(len(g), np.int32)]), stream)
                T = len(toks)
                o = 0
                r0, r1 = int(rowmap[g[0]]), int(rowmap[g[-1]])
                bt = (self._bt(kv, rowmap[g], stream) if isinstance(kv, HostPagedKVCache)
                      else kv.block_table[r0:r1 + 1])  # host KV: window-relative pages
                fb = ForwardBatch(meta[o:o + T], meta[o + T:o + 2 * T], meta[o + 2 * T:o + 3 * T],
                                  meta[o + 3 * T:o + 3 * T + len(g) + 1], meta[o + 3 * T + len(g) + 1:],
                                  bt, len(g), int(lens[g].max()), None, row0)
                last.extend(row0 + qs[1:] - 1)
                chunks.append(fb)
                row0 += T
            lr = self._up(np.asarray(last, np.int32), stream)
            chunks[0].last_rows = lr
            if model is self.target:
                logits = model.forward(chunks, kv, stream)
                lo = 0 if window is None else window.lo  # logits rows = this pass's sequences
                with torch.cuda.stream(stream):
                    for bi, b in enumerate(s.batches):
                        if b.n == 0 or (window is not None and b is not window):
                            continue
                        u = None
                        if s.mode == "sample":
                            u = self._up(input_uniforms(s.seed, -2, bi, 3, b.n), stream, torch.float32)
                        native.sample_tokens(logits[b.lo - lo:b.hi - lo], first[b.lo:b.hi], uniforms=u,
                                             temperature=s.temperature, stream=stream)
                    if window is None or window is s.batches[-1] or s.batches[-1].n == 0:
                        first_h = first.to("cpu", non_blocking=True)
            else:
                model.forward(chunks, kv, stream, want_logits=False)
        s.tkv.join(self.tgt_stream)
        self.tgt_stream.synchronize()
        self.drf_stream.synchronize()
        first_np = first_h.numpy()
        for i in range(s.n_seq):
            s.out[i].append(int(first_np[i]))
        s.t_last[:] = first_np
        s.ctx[:] = lens
        s.remaining[:] = max_new - 1
        s.active[:] = True
        self._hist_write(s, np.arange(s.n_seq), lens, first_np, self.drf_stream)
        self.drf_stream.synchronize()
        self._release_staging()

    def synthetic_context(self, s: DecodeSession, ctx_len: int, max_new: int, seed: int = 0,
                          recycle: bool = False) -> None:
        """Decode-only benchmark input: caches hold ``ctx_len`` random KV rows per
        sequence (as if prefilled), t_last random.  The prompt KV is an input
        of the decode metric, resident in HBM before timing starts.

        ``recycle``: the steady state of a pool serving ``max_new``-token
        requests (the reference's Workload, commits clamped to what is left,
        simulator.py:213-214): a sequence that has generated ``max_new``
        tokens restarts as a new request for the same ``ctx_len``-token prompt,
        whose KV is still cached (a prefix-cache hit: its context rows are
        kept, everything past them is overwritten).  Prefill is not decode
        work; ``generate()`` times it end to end."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for kv in (s.tkv, s.dkv):
            if isinstance(kv, HostPagedKVCache):
                kv.fill_random(g, self.device)
                continue
            kv.k.normal_(0.0, 1.0, generator=g)
            kv.v.normal_(0.0, 1.0, generator=g)
        rng = np.random.default_rng(seed)
        s.t_last[:] = rng.integers(0, self.target.arch.vocab, s.n_seq)
        s.ctx[:] = ctx_len
        s.remaining[:] = max_new
        s.active[:] = True
        if recycle:
            s.recycle = (s.ctx.copy(), s.t_last.copy(), int(max_new))
        if s.hist is not None:
            s.hist.random_(0, self.target.arch.vocab, generator=g)
            self._hist_write(s, np.arange(s.n_seq), s.ctx, s.t_last, self.drf_stream)
        torch.cuda.synchronize(self.device)
        self._release_staging()

    # ------------------------------------------------------------------ draft
    def _draft(self, s: DecodeSession, bi: int, rnd: int) -> None:
        """Draft n_cand tokens for every active slot of batch ``bi``.

        Slots are ordered [cached rows | fresh rows | re-prefilled] and that
        order (``s.dlist[bi]``) indexes the draft buffers and the next verify
        of the batch.  Cached rows run n+1 decode steps; fresh rows (a prompt
        just prefilled by the target) and slots without a row re-read their
        whole context (the paper's re-prefill, into their own row or the
        scratch rows)."""
        b = s.batches[bi]
        slots = np.arange(b.lo, b.hi)
        act = slots[s.active[slots]]
        has_row = s.drow[act] >= 0
        fresh = s.fresh[act]
        cached, fresh_rows, rp = act[has_row & ~fresh], act[has_row & fresh], act[~has_row]
        order = np.concatenate([cached, fresh_rows, rp])
        s.dlist[bi] = order
        if order.size == 0:
            return
        st = self.drf_stream
        n = s.n_cand
        tr = self.tracer
        ev0 = tr.mark(st)
        u_all = input_uniforms(s.seed, rnd, bi, 0, (order.size, n)) if s.mode == "sample" else None
        cstep = s.bs_draft if s.draft_kv == "cached" else max(cached.size, 1)
        for c_lo in range(0, cached.size, cstep):
            c_hi = min(cached.size, c_lo + cstep)
            self._draft_chunk_cached(s, bi, c_lo, order[c_lo:c_hi], u_all)
        base = cached.size
        fstep = min(s.bs_draft, self.FRESH_CHUNK)  # context prefills: bounded activation workspace
        for c_lo in range(0, fresh_rows.size, fstep):
            seqs = fresh_rows[c_lo:c_lo + fstep]
            self._draft_chunk_reprefill(s, bi, base + c_lo, seqs, u_all, rows=s.drow[seqs], kv_dn=True)
        base += fresh_rows.size
        for c_lo in range(0, rp.size, s.bs_draft):
            seqs = rp[c_lo:c_lo + s.bs_draft]
            self._draft_chunk_reprefill(s, bi, base + c_lo, seqs, u_all,
                                        rows=s.scratch_row0 + np.arange(seqs.size), kv_dn=False)
        s.fresh[act] = False
        tr.add("GPU_DRAFT", "draft_decode", ev0, tr.mark(st), batch=bi, rnd=rnd)

    def _draft_chunk_cached(self, s: DecodeSession, bi: int, p0: int, seqs, u_all) -> None:
        """n+1 cached-KV decode steps for slots ``seqs`` (draft positions p0..)."""
        st = self.drf_stream
        n = s.n_cand
        cm = seqs.size
        ctx = s.ctx[seqs]
        rows = s.drow[seqs]
        pos = ctx[None, :] + np.arange(n + 1)[:, None]                  # [n+1, cm]
        slots = s.dkv.slots(np.broadcast_to(rows, pos.shape), pos)
        qs = np.arange(cm + 1, dtype=np.int32)
        parts = [s.t_last[seqs], pos.astype(np.int32).ravel(), slots.ravel(), qs, pos.astype(np.int32).ravel()]
        if u_all is not None:
            parts.append(u_all[p0:p0 + cm].T.ravel().view(np.int32))
        meta = self._up(np.concatenate(parts), st)
        o = cm
        P = (n + 1) * cm
        pos_d, slot_d = meta[o:o + P], meta[o + P:o + 2 * P]
        qs_d = meta[o + 2 * P:o + 2 * P + cm + 1]
        kvb_d = meta[o + 2 * P + cm + 1:o + 3 * P + cm + 1]
        u_d = meta[o + 3 * P + cm + 1:].view(torch.float32) if u_all is not None else None
        bt = self._bt(s.dkv, rows, st)
        for j in range(n + 1):
            toks = meta[:cm] if j == 0 else s.drafts[bi][j - 1, p0:p0 + cm]
            fb = ForwardBatch(toks, pos_d[j * cm:(j + 1) * cm], slot_d[j * cm:(j + 1) * cm], qs_d,
                              kvb_d[j * cm:(j + 1) * cm], bt, cm, 1)
            if j == n:
                self.draft.forward(fb, s.dkv, st, want_logits=False)  # KV of d_n only
                break
            logits = self.draft.forward(fb, s.dkv, st)
            out_tok = s.drafts[bi][j, p0:p0 + cm]
            if s.mode == "sample":
                qp = s.qprobs[bi][p0:p0 + cm, j, :]
                native.sample_tokens(logits, out_tok, uniforms=u_d[j * cm:(j + 1) * cm], out_probs=qp,
                                     temperature=s.temperature, stream=st)
            else:
                native.sample_tokens(logits, out_tok, stream=st)

    def _draft_chunk_reprefill(self, s: DecodeSession, bi: int, p0: int, seqs, u_all, rows, kv_dn: bool) -> None:
        """The paper's draft for slots ``seqs``: prefill the whole context
        (prompt + committed tokens + t_last) into draft KV rows ``rows``, take
        d_1 from its last row, then n_cand−1 cached decode steps.  ``kv_dn``
        (a fresh slot with a persistent row) adds the step that writes d_n's
        KV, after which the row follows the cached invariant."""
        st = self.drf_stream
        n = s.n_cand
        cm = seqs.size
        ctx = s.ctx[seqs]
        rows = np.asarray(rows, np.int64)
        lens = ctx + 1                                    # positions 0..ctx (t_last at ctx)
        T = int(lens.sum())
        flat = np.concatenate([seq * s.max_len + np.arange(L) for seq, L in zip(seqs, lens)])
        pos = np.concatenate([np.arange(L) for L in lens])
        slots = s.dkv.slots(np.repeat(rows, lens), pos)
        qs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        steps = n if kv_dn else n - 1                     # decode steps j = 1..steps
        dpos = ctx[None, :] + np.arange(1, steps + 1)[:, None]
        dslots = s.dkv.slots(np.broadcast_to(rows, dpos.shape), dpos)
        parts = [pos.astype(np.int32), slots, qs, np.zeros(cm, np.int32), (qs[1:] - 1).astype(np.int32),
                 dpos.astype(np.int32).ravel(), dslots.ravel(), np.arange(cm + 1, dtype=np.int32),
                 ctx.astype(np.int32)]
        if u_all is not None:
            parts.append(u_all[p0:p0 + cm].T.ravel().view(np.int32))
        meta = self._up(np.concatenate(parts), st)
        idx = self._up(flat, st, torch.int64)
        o = 0
        pos_d = meta[o:o + T]; o += T
        slot_d = meta[o:o + T]; o += T
        qs_d = meta[o:o + cm + 1]; o += cm + 1
        zero_d = meta[o:o + cm]; o += cm
        last_d = meta[o:o + cm]; o += cm
        D = steps * cm
        dpos_d = meta[o:o + D]; o += D
        dslot_d = meta[o:o + D]; o += D
        dqs_d = meta[o:o + cm + 1]; o += cm + 1
        ctx_d = meta[o:o + cm]; o += cm                   # position of each sequence's last context row
        u_d = meta[o:].view(torch.float32) if u_all is not None else None
        toks = self.draft.ws.get("rp_tokens", (T,), torch.int32)
        native.gather_i32(s.hist, idx, toks, st)
        bt = self._bt(s.dkv, rows, st)
        for j in range(steps + 1):
            if j == 0:
                # the last layer runs attention onward for the last rows only (one per sequence)
                fb = ForwardBatch(toks, pos_d, slot_d, qs_d, zero_d, bt, cm, int(lens.max()), last_d,
                                  last_pos=ctx_d, last_qs=dqs_d)
            else:
                sl = slice((j - 1) * cm, j * cm)
                fb = ForwardBatch(s.drafts[bi][j - 1, p0:p0 + cm], dpos_d[sl], dslot_d[sl], dqs_d, dpos_d[sl], bt,
                                  cm, 1)
            if j == n:
                self.draft.forward(fb, s.dkv, st, want_logits=False)  # KV of d_n only
                break
            logits = self.draft.forward(fb, s.dkv, st)
            out_tok = s.drafts[bi][j, p0:p0 + cm]
            if s.mode == "sample":
                native.sample_tokens(logits, out_tok, uniforms=u_d[j * cm:(j + 1) * cm],
                                     out_probs=s.qprobs[bi][p0:p0 + cm, j, :], temperature=s.temperature, stream=st)
            else:
                native.sample_tokens(logits, out_tok, stream=st)

    # ----------------------------------------------------------------- verify
    def _verify(self, s: DecodeSession, bi: int, rnd: int) -> None:
        """Verify batch ``bi``: the drafted slots (``s.dlist[bi]``, n_cand+1
        query tokens each) and, with slot refill, prefill the prompts admitted
        into its free slots (``s.pending_new[bi]``) in the same layer pass —
        layer-major over token-bounded chunks, so each streamed layer still
        crosses the link once.  LM-head rows: every verify row, then the last
        prompt row of each admitted slot (its first token)."""
        st = self.tgt_stream
        n = s.n_cand
        tr = self.tracer
        act = s.dlist[bi]
        new = s.pending_new[bi]
        na, nn = act.size, new.size
        s.tkv.set_window(s.batches[bi].lo, s.batches[bi].hi)  # host-resident KV: this batch's pages
        T = na * (n + 1)
        ctx = s.ctx[act]
        pos = ctx[:, None] + np.arange(n + 1)[None, :]
        slots = s.tkv.slots(np.broadcast_to(act[:, None], pos.shape), pos)
        qs = (np.arange(na + 1) * (n + 1)).astype(np.int32)
        forced = None
        if s.forced_p is not None and s.mode == "greedy":
            forced = forced_counts(s.seed, rnd, bi, s.forced_p, n, na)
        parts = [s.t_last[act], pos.astype(np.int32).ravel(), slots.ravel(), qs, ctx.astype(np.int32),
                 s.remaining[act]]
        if forced is not None:
            parts.append(forced)
        if s.mode == "sample":
            parts.append(input_uniforms(s.seed, rnd, bi, 1, (na, n)).ravel().view(np.int32))
            parts.append(input_uniforms(s.seed, rnd, bi, 2, na).view(np.int32))
        meta = self._up(np.concatenate(parts), st)
        o = 0
        t_last_d = meta[o:o + na]; o += na
        pos_d = meta[o:o + T]; o += T
        slot_d = meta[o:o + T]; o += T
        qs_d = meta[o:o + na + 1]; o += na + 1
        kvb_d = meta[o:o + na]; o += na
        rem_d = meta[o:o + na]; o += na
        forced_d = None
        if forced is not None:
            forced_d = meta[o:o + na]; o += na
        ev0 = tr.mark(st)
        chunks, last = [], []
        if na:
            toks = self.target.ws.get("vtok", (na, n + 1), torch.int32)
            draft_rows = self.target.ws.get("vdraft", (na, n), torch.int32)
            native.build_verify_tokens(t_last_d, s.drafts[bi], na, n, toks, draft_rows, st)
            chunks.append(ForwardBatch(toks.view(-1), pos_d, slot_d, qs_d, kvb_d, self._bt(s.tkv, act, st), na,
                                       n + 1, None, 0))
            last.append(np.arange(T, dtype=np.int32))
        row0 = T
        lo = 0
        chunk_tokens = self.prefill_chunk_tokens
        while lo < nn:  # admitted prompts, ≤ chunk_tokens per chunk
            hi, tok = lo, 0
            while hi < nn and (hi == lo or tok + len(s.prompts[s.slot_prompt[new[hi]]]) <= chunk_tokens):
                tok += len(s.prompts[s.slot_prompt[new[hi]]])
                hi += 1
            g = new[lo:hi]
            lens = np.array([len(s.prompts[s.slot_prompt[i]]) for i in g], np.int64)
            ptok = np.concatenate([np.asarray(s.prompts[s.slot_prompt[i]], np.int32) for i in g])
            ppos = np.concatenate([np.arange(L) for L in lens])
            pq = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
            pm = self._up(np.concatenate([ptok, ppos.astype(np.int32), s.tkv.slots(np.repeat(g, lens), ppos), pq,
                                          np.zeros(g.size, np.int32)]), st)
            Tg = int(lens.sum())
            chunks.append(ForwardBatch(pm[:Tg], pm[Tg:2 * Tg], pm[2 * Tg:3 * Tg], pm[3 * Tg:3 * Tg + g.size + 1],
                                       pm[3 * Tg + g.size + 1:], self._bt(s.tkv, g, st), g.size, int(lens.max()),
                                       None, row0))
            last.append((row0 + pq[1:] - 1).astype(np.int32))
            row0 += Tg
            lo = hi
        if len(chunks) > 1 or nn:
            chunks[0].last_rows = self._up(np.concatenate(last), st)
        if self.target.streamer is not None:
            self.target.streamer.pass_tag = (rnd, bi)
        logits = self.target.forward(chunks, s.tkv, st)
        if self.target.streamer is not None:
            self.target.streamer.pass_tag = None
        ev1 = tr.mark(st)
        if na:
            out_tok = self.target.ws.get("acc_tok", (na, n + 1), torch.int32)
            out_cnt = self.target.ws.get("acc_cnt", (na,), torch.int32)
            vlog = logits[:T]
            if s.mode == "sample":
                u_acc = meta[o:o + na * n].view(torch.float32); o += na * n
                u_res = meta[o:o + na].view(torch.float32); o += na
                native.accept_sample(draft_rows, vlog, s.qprobs[bi][:na], u_acc, u_res, rem_d, out_tok, out_cnt,
                                     s.temperature, st)
            else:
                native.accept_greedy(draft_rows, vlog, rem_d, out_tok, out_cnt, forced_d, st)
            # device → host: the round's result (committed tokens and counts)
            native.copy_sm(s.res_tok[bi].data_ptr(), out_tok.data_ptr(), out_tok.numel() * 4, st)
            native.copy_sm(s.res_cnt[bi].data_ptr(), out_cnt.data_ptr(), out_cnt.numel() * 4, st)
        if nn:  # first tokens of the admitted prompts
            first = self.target.ws.get("first_tok", (nn,), torch.int32)
            u = (self._up(input_uniforms(s.seed, rnd, bi, 3, nn), st, torch.float32)
                 if s.mode == "sample" else None)
            native.sample_tokens(logits[T:T + nn], first, uniforms=u, temperature=s.temperature, stream=st)
            native.copy_sm(s.res_first[bi].data_ptr(), first.data_ptr(), nn * 4, st)
        ev2 = tr.mark(st)
        if self.target.hooks is not None and getattr(self, "_last_ffn_end", None) is not None:
            # per-layer events cover the pass (one event at a time per resource, _checks.py:7-18):
            # only the final norm + LM head remain
            tr.add("GPU_TARGET", "lm_head", self._last_ffn_end, ev1, batch=bi, rnd=rnd)
            self._last_ffn_end = None
        else:
            tr.add("GPU_TARGET", "verify", ev0, ev1, batch=bi, rnd=rnd)
        tr.add("GPU_TARGET", "accept", ev1, ev2, batch=bi, rnd=rnd)

    def _commit(self, s: DecodeSession, bi: int) -> int:
        act, new = s.dlist[bi], s.pending_new[bi]
        cnt = s.res_cnt[bi][:act.size].numpy()
        tok = s.res_tok[bi][:act.size].numpy()
        total = 0
        hs, hp, hv = [], [], []
        for j, i in enumerate(act):
            c = int(cnt[j])
            if c > 0:
                s.out[s.slot_prompt[i]].extend(int(x) for x in tok[j, :c])
                if s.hist is not None:  # committed tokens land at positions ctx+1 .. ctx+c
                    hs.append(np.full(c, i))
                    hp.append(s.ctx[i] + 1 + np.arange(c))
                    hv.append(tok[j, :c])
                s.remaining[i] -= c
                s.t_last[i] = tok[j, c - 1]
                s.ctx[i] += c
                total += c
            if s.refill and s.remaining[i] <= 0:  # done: free the slot for the next prompt
                s.active[i] = False
                s.slot_prompt[i] = -1
            elif s.recycle is not None and s.remaining[i] <= 0:  # done: the same prompt again (cached prefix)
                ctx0, t0, new_tokens = s.recycle
                s.ctx[i], s.t_last[i], s.remaining[i] = ctx0[i], t0[i], new_tokens
                s.recycled += 1
        if new.size:
            first = s.res_first[bi][:new.size].numpy()
            for k, i in enumerate(new):
                pid = s.slot_prompt[i]
                s.out[pid].append(int(first[k]))
                L = len(s.prompts[pid])
                s.ctx[i] = L
                s.t_last[i] = first[k]
                s.remaining[i] = s.max_new - 1
                hs.append(np.array([i]))
                hp.append(np.array([L]))
                hv.append(first[k:k + 1])
                if s.remaining[i] > 0:
                    s.active[i] = True
                    s.fresh[i] = True   # its draft state is built from the context next round
                else:
                    s.slot_prompt[i] = -1
            s.pending_new[bi] = np.zeros(0, np.int64)
        if hs and s.hist is not None:
            self._hist_write(s, np.concatenate(hs), np.concatenate(hp), np.concatenate(hv), self.drf_stream)
        return total

    def _admit(self, s: DecodeSession, bi: int) -> None:
        """Slot refill: queued prompts take the free slots of batch ``bi``
        (prompt order); their tokens go to the draft's history now, their
        target prefill runs inside this round's verify."""
        b = s.batches[bi]
        free = [i for i in range(b.lo, b.hi) if s.slot_prompt[i] < 0]
        if s.max_admit is not None:
            free = free[:s.max_admit]
        take = []
        for i in free:
            if not s.queue:
                break
            s.slot_prompt[i] = s.queue.pop()
            take.append(i)
        s.pending_new[bi] = np.asarray(take, np.int64)
        if take and s.hist is not None:
            lens = [len(s.prompts[s.slot_prompt[i]]) for i in take]
            self._hist_write(s, np.repeat(take, lens), np.concatenate([np.arange(L) for L in lens]),
                             np.concatenate([np.asarray(s.prompts[s.slot_prompt[i]], np.int32) for i in take]),
                             self.drf_stream)

    # ----------------------------------------------------------------- rounds
    def first_draft(self, s: DecodeSession) -> None:
        self._draft(s, 0, -1)
        native.stream_synchronize(self.drf_stream)
        self._release_staging()

    def round(self, s: DecodeSession) -> int:
        """One barrier-synchronised round; returns tokens committed."""
        rnd = s.rounds
        bi = rnd % 2
        b, o = s.batches[bi], s.batches[1 - bi]
        if s.refill:
            self._admit(s, bi)
            verify = s.dlist[bi].size > 0 or s.pending_new[bi].size > 0
            draft = bool(s.active[o.lo:o.hi].any())
        else:
            verify = b.n > 0 and (s.remaining[b.lo:b.hi] > 0).any()
            draft = o.n > 0 and (s.remaining[o.lo:o.hi] > 0).any()
        # Two host enqueuers: the verify's launches drain only as fast as its
        # layers arrive over PCIe, so a single thread would block on a full
        # launch queue and enqueue the draft late (serialising the streams).
        worker = None
        err: list = []
        if draft:
            def run_draft():
                try:
                    torch.cuda.set_device(self.device)
                    native.set_device(self.device.index or 0)
                    if self.nvtx_range:  # NVTX ranges are per thread (ncu --nvtx-include)
                        torch.cuda.nvtx.range_push(self.nvtx_range)
                    try:
                        self._draft(s, 1 - bi, rnd)
                    finally:
                        if self.nvtx_range:
                            torch.cuda.nvtx.range_pop()
                except BaseException as exc:  # re-raised on the caller's thread
                    err.append(exc)

            self._tev[0].record(self.drf_stream)
            worker = threading.Thread(target=run_draft, name="draft-enqueue", daemon=True)
            worker.start()
        try:
            self._tev[2].record(self.tgt_stream)
            if verify:
                self._cur = (rnd, bi)
                self._verify(s, bi, rnd)
            self._tev[3].record(self.tgt_stream)
        finally:
            if worker is not None:  # never leave the draft enqueue running past an error
                worker.join()
        if worker is not None:
            if err:
                raise err[0]
            self._tev[1].record(self.drf_stream)
        # barrier (simulator.py:209-211): device-side join, then the host reads counts.
        # Host-resident KV: the last layers' write-backs (d2h stream) join too, so
        # no DMA into the pinned pool outlives the round and its time is counted.
        self._join.record(self.drf_stream)
        self._join.wait(self.tgt_stream)
        s.tkv.join(self.tgt_stream)
        bev = self.tracer.mark(self.tgt_stream)
        self.tracer.add("GPU_TARGET", "barrier", bev, bev, rnd=rnd)
        native.stream_synchronize(self.tgt_stream)
        self.round_times.append((self._tev[0].elapsed_ms(self._tev[1]) if draft else 0.0,
                                 self._tev[2].elapsed_ms(self._tev[3])))
        self._release_staging()
        c = self._commit(s, bi) if verify else 0
        s.rounds += 1
        s.committed_decode += c
        return c

    def decode(self, s: DecodeSession, max_rounds: int | None = None) -> None:
        if s.refill:
            while s.queue or s.active.any() or any(p.size for p in s.pending_new):
                if max_rounds is not None and s.rounds >= max_rounds:
                    break
                self.round(s)
            return
        while (s.remaining > 0).any():
            if max_rounds is not None and s.rounds >= max_rounds:
                break
            self.round(s)

    # ------------------------------------------------------------ public API
    def generate(self, prompts: list, max_new_tokens: int, policy: Policy | None = None, seed: int = 0,
                 mode: str = "greedy", temperature: float = 1.0, forced_p: float | None = None,
                 draft_kv: str = "cached", draft_cached: int | None = None,
                 refill: bool | None = None, max_admit: int | None = None,
                 kv_host: bool = False) -> list[list[int]]:
        """prompts (token id lists) → committed continuations, max_new_tokens each.

        With more prompts than the two batches hold (or ``refill=True``), the
        2·bs_decoding sequences are slots of a pool refilled as sequences
        finish: no straggler rounds and no separate prefill
        pass; otherwise every prompt is prefilled layer-major first."""
        S = len(prompts)
        if policy is None:  # the reference's planner picks it (planner.py:161-184)
            p = forced_p if forced_p is not None else self.acceptance_p
            policy = self.plan_policy(S, max(len(q) for q in prompts), max_new_tokens, p)
            self.last_policy = policy
        max_len = max(len(p) for p in prompts) + max_new_tokens + policy.n_cand + 2
        if refill is None:
            refill = S > 2 * policy.bs_decoding
        if refill:
            slots = min(S, 2 * policy.bs_decoding)
            s = self.new_session(slots, min(policy.bs_decoding, slots), max_len, policy.n_cand, mode, seed,
                                 temperature, forced_p, policy.bs_draft, draft_kv, draft_cached,
                                 prompts=[np.asarray(p, np.int32) for p in prompts], max_new=max_new_tokens,
                                 max_admit=max_admit, kv_host=kv_host)
            self.decode(s)
            self.last_session = s
            return [o[:max_new_tokens] for o in s.out]
        s = self.new_session(S, policy.bs_decoding, max_len, policy.n_cand, mode, seed, temperature, forced_p,
                             policy.bs_draft, draft_kv, draft_cached, kv_host=kv_host)
        self.prefill(s, prompts, max_new_tokens, policy.bs_prefill)
        if (s.remaining > 0).any():
            self.first_draft(s)
            self.decode(s)
        self.last_session = s
        return [o[:max_new_tokens] for o in s.out]

    def b200_profile(self, l_input: int):
        """``self.hw``, or a B200 HardwareProfile of this device for the pair
        (presets.b200_profile): HBM = the device's total, host = MemAvailable,
        the streamed units' encoded/raw ratio when they are XC4-coded."""
        if self.hw is not None:
            return self.hw
        from .presets import b200_profile

        _, total = torch.cuda.mem_get_info(self.device)
        host = 0
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    host = int(line.split()[1]) * 1024
        st = self.target.streamer
        ratio = 1.0
        if st is not None and st.coded and st.host:
            units = [u for u in st.host.values() if hasattr(u, "ratio")]
            ratio = max((u.ratio for u in units), default=1.0)
        return b200_profile(self.target.arch, self.draft.arch, ctx=l_input, gpu_mem=total, cpu_mem=max(host, 1),
                            stream_ratio=ratio)

    def plan_policy(self, n_prompts: int, l_input: int, max_new: int, acceptance_p: float, space=None):
        """``planner.search`` over ``space`` (default: a grid sized to the
        prompt count) for this pair on ``b200_profile``; returns the best Policy."""
        from .domain import Workload
        from .planner import SearchSpace, search

        if space is None:
            half = max(1, (n_prompts + 1) // 2)
            bs = sorted({min(half, b) for b in (8, 16, 32, 64, 128, 256, 384, 512)})
            space = SearchSpace(bs_prefill_values=tuple(sorted({min(n_prompts, 2 * b) for b in bs})),
                                bs_decoding_values=tuple(bs),
                                bs_draft_values=tuple(sorted({min(half, b) for b in (8, 16, 32, 64)})),
                                n_cand_values=(2, 4, 6, 8))
        wl = Workload(total_sequences=n_prompts, l_input=l_input, max_new_tokens=max_new,
                      acceptance_p=float(acceptance_p))
        return search(space, wl, self.b200_profile(l_input), self.target.spec(), self.draft.spec()).best

    def run_decoding(self, policy, workload, plan=None, seed: int = 0, acceptance="greedy", prompts=None,
                     max_rounds: int | None = None, draft_kv: str = "cached",
                     draft_cached: int | None = None) -> SimResult:
        """Measured counterpart of simulate_decoding (simulator.py:108-116).

        Runs workload.total_sequences sequences (two batches of
        policy.bs_decoding) for workload.max_new_tokens tokens each and returns
        the measured trace.  ``acceptance`` = "greedy" | "sample" | Forced(p);
        without prompts the context is synthetic (l_input random KV rows).
        """
        mode = "sample" if acceptance == "sample" else "greedy"
        forced_p = acceptance.p if isinstance(acceptance, Forced) else None
        S = workload.total_sequences
        max_len = workload.l_input + workload.max_new_tokens + policy.n_cand + 2
        s = self.new_session(S, policy.bs_decoding, max_len, policy.n_cand, mode, seed, 1.0, forced_p,
                             policy.bs_draft, draft_kv, draft_cached)
        if prompts is not None:
            self.prefill(s, prompts, workload.max_new_tokens, policy.bs_prefill)
        else:
            self.synthetic_context(s, workload.l_input, workload.max_new_tokens, seed)
        self.first_draft(s)
        torch.cuda.synchronize(self.device)
        if self.target.streamer is not None:
            self.target.streamer.copy_marks.clear()
        self.tracer.origin(self.tgt_stream)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(self.tgt_stream)
        wall0 = time.perf_counter()
        self.decode(s, max_rounds)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(self.tgt_stream)
        t1.synchronize()
        wall = time.perf_counter() - wall0
        total = t0.elapsed_time(t1) * 1e-3
        events = self.resolve_trace()
        tokens = s.committed_decode
        self.last_session = s
        return SimResult(trace=events, total_time=total, tokens_generated=tokens,
                         throughput=tokens / total if total > 0 else 0.0,
                         peak_gpu_bytes=int(torch.cuda.max_memory_allocated(self.device)),
                         rounds_executed=s.rounds, per_resource_busy=busy(events),
                         extra={"wall_s": wall})
