"""Measurement-side fp32 reference of the full-depth verify pass (bench.py parity).

The headline bench runs with forced acceptance, so the committed tokens do
not depend on the logits; this module checks the logits themselves after the
timed rounds: a few sequences are verified through the product path
(``TargetModel.verify``: tcgen05 GEMMs, paged attention, fused router, XC4
streamed units) and through a plain PyTorch fp32 restatement of the same
Mixtral block (modeling_mixtral.py arithmetic: RMSNorm, rotate-half RoPE, GQA
softmax attention, fp32 top-2 routing renormalised over the pair, SwiGLU
experts), layer by layer, reading each streamed layer from the same window
slot the streamer fills (so the pass also consumes the streamer in order).
Activations stay fp32 (no bf16 re-rounding), so differences are the product
path's bf16 storage rounding accumulated over the layers; the report gives
max |Δlogit|, its ratio to the logit scale and argmax agreement.

Test/measurement infrastructure: never imported by the product package.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from paper_2505_10259_b200.models import SeqState
from paper_2505_10259_b200.weights import SWIGLU_BLOCK, ffn_offsets, unit_layout


def _rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w.float()


def _rope(x, pos, theta):
    dh = x.shape[-1]
    inv = 1.0 / theta ** (torch.arange(0, dh, 2, device=x.device, dtype=torch.float64) / dh)
    ang = pos.double()[:, None] * inv[None, :]
    c, s = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    x0, x1 = x[..., : dh // 2], x[..., dh // 2:]
    return torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], dim=-1)


def _kv_rows(pool_layer, bt_row, ctx, ps, dev):
    """Cached K or V of one sequence, positions [0, ctx): [ctx, hkv, dh] fp32 on
    the GPU (the pool may be HBM or pinned host DRAM)."""
    n_pages = -(-ctx // ps)
    pages = torch.as_tensor(np.asarray(bt_row[:n_pages], np.int64), device=pool_layer.device)
    blk = pool_layer[pages].to(dev)              # [pages, hkv, ps, dh]
    blk = blk.permute(0, 2, 1, 3).reshape(-1, blk.shape[1], blk.shape[3])
    return blk[:ctx].float()


def _layer_fp32(eng, li, L, unit, streamed, x, pos, state, bs, T, routing=None):
    """One Mixtral/Mistral block in fp32 on input ``x`` [bs·T, H] (fp32).
    ``routing``: optional bool [bs·T, E] expert choice to force (the product
    path's own top-2); the pair weights are always the fp32 renormalised
    softmax of this pass's router logits.  Returns (x_out, router_logits)."""
    tm = eng.target
    a, w = tm.arch, tm.w
    dev = tm.device
    H, dh, hq, hkv, E = a.hidden, a.head_dim, a.n_head, a.n_kv_head, a.n_expert
    stream_attn = any(M.wqkv is None for M in w.layers)
    ffn_off = unit_layout(a, stream_attn)[0] // 2
    gu_el, dn_el, _ = ffn_offsets(a)
    kv = state.kv
    if L.wqkv is None:
        wqkv = unit[: a.qkv_rows * H].view(a.qkv_rows, H)
        wo = unit[a.qkv_rows * H: a.qkv_rows * H + H * hq * dh].view(H, hq * dh)
    else:
        wqkv, wo = L.wqkv, L.wo
    xn = _rms(x, L.attn_norm, a.eps)
    qkv = xn @ wqkv.float().T
    q = qkv[:, : hq * dh].view(-1, hq, dh)
    k = qkv[:, hq * dh:(hq + hkv) * dh].view(-1, hkv, dh)
    v = qkv[:, (hq + hkv) * dh:].view(-1, hkv, dh)
    p = pos.reshape(-1)
    q, k = _rope(q, p, a.rope_theta), _rope(k, p, a.rope_theta)
    att = torch.empty_like(q)
    pk, pv = kv.k[li], kv.v[li]
    for i in range(bs):
        c = int(state.ctx[i])
        bt_row = kv._bt_global[state.rows[i]] if hasattr(kv, "_bt_global") else kv._bt_host[state.rows[i]]
        Kc = _kv_rows(pk, bt_row, c, kv.page_size, dev)
        Vc = _kv_rows(pv, bt_row, c, kv.page_size, dev)
        sl = slice(i * T, (i + 1) * T)
        K = torch.cat([Kc, k[sl]], 0).repeat_interleave(hq // hkv, dim=1)  # [c+T, hq, dh]
        V = torch.cat([Vc, v[sl]], 0).repeat_interleave(hq // hkv, dim=1)
        s = torch.einsum("thd,khd->htk", q[sl], K) / math.sqrt(dh)
        mask = torch.arange(c + T, device=dev)[None, :] > (c + torch.arange(T, device=dev))[:, None]
        s = s.masked_fill(mask[None], float("-inf"))
        att[sl] = torch.einsum("htk,khd->thd", torch.softmax(s, -1), V)
    h = att.reshape(-1, hq * dh) @ wo.float().T + x
    hn = _rms(h, L.ffn_norm, a.eps)
    ffn = unit[ffn_off:] if (streamed and stream_attn) else unit
    if not E:
        g = ffn[: 2 * a.inter * H].view(a.inter // SWIGLU_BLOCK, 2, SWIGLU_BLOCK, H)
        gate = hn @ g[:, 0].reshape(a.inter, H).float().T
        up = hn @ g[:, 1].reshape(a.inter, H).float().T
        return h + (torch.nn.functional.silu(gate) * up) @ ffn[2 * a.inter * H:3 * a.inter * H].view(H, a.inter).float().T, None
    lr = hn @ L.router.float().T
    if routing is None:
        top = torch.topk(lr, 2, dim=-1).indices
        sel = torch.zeros_like(lr, dtype=torch.bool).scatter_(1, top, True)
    else:
        sel = routing
    # softmax over all E renormalised over the chosen pair == softmax over the pair
    lp = lr.masked_fill(~sel, float("-inf"))
    wts = torch.softmax(lp, -1)
    gu = ffn[:gu_el].view(E, 2 * a.inter, H)
    dn = ffn[gu_el:gu_el + dn_el].view(E, H, a.inter)
    y = torch.zeros_like(h)
    for e in range(E):
        rows = sel[:, e].nonzero().squeeze(-1)
        if rows.numel() == 0:
            continue
        g = gu[e].view(a.inter // SWIGLU_BLOCK, 2, SWIGLU_BLOCK, H)
        gate = hn[rows] @ g[:, 0].reshape(a.inter, H).float().T
        up = hn[rows] @ g[:, 1].reshape(a.inter, H).float().T
        y[rows] += (torch.nn.functional.silu(gate) * up) @ dn[e].float().T * wts[rows, e][:, None]
    return h + y, lr


class _SegUnit:
    """A streamed unit held as several window slots (split window): element
    slices map to the segment that holds them (a slice never spans two)."""

    def __init__(self, parts, off=0):
        self.parts, self.off = parts, off  # [(first element, bf16 view)]

    def __getitem__(self, sl):
        a = (sl.start or 0) + self.off
        if sl.stop is None:  # an open-ended view: re-based, still resolved per slice
            return _SegUnit(self.parts, a)
        b = sl.stop + self.off
        for lo, t in self.parts:
            if lo <= a < lo + t.numel():
                assert b <= lo + t.numel(), "slice spans two window segments"
                return t[a - lo:b - lo]
        raise IndexError(sl)


def _unit(eng, li, L, stream):
    st = eng.target.streamer
    streamed = st is not None and li in st.streamed
    if streamed:
        parts = []
        for sg, (lo, _) in enumerate(st.segments):
            st.acquire(li, stream, sg)  # the stream waits for the slot; k_acq - 1 indexes it
            parts.append((lo // 2, st.slots[(st.k_acq - 1) % st.n_slots].view(torch.bfloat16)))
        return (parts[0][1] if len(parts) == 1 else _SegUnit(parts)), True
    return L.ffn, False


def _release(eng, li, stream):
    st = eng.target.streamer
    for sg in range(len(st.segments)):
        st.release(li, stream, sg)


def verify_fp32(eng, state: SeqState, draft_tokens: torch.Tensor, stream) -> torch.Tensor:
    """Free-running fp32 logits [bs, n+1, V] of t_last + drafts at positions ctx..ctx+n."""
    tm = eng.target
    w, st, dev = tm.w, tm.streamer, tm.device
    bs, n = draft_tokens.shape
    T = n + 1
    with torch.cuda.stream(stream):
        toks = torch.cat([torch.as_tensor(state.t_last, device=dev)[:, None].int(), draft_tokens.to(dev).int()], 1)
        pos = torch.as_tensor(state.ctx, device=dev)[:, None] + torch.arange(T, device=dev)[None, :]
        x = w.embed[toks.reshape(-1).long()].float()                      # [bs·T, H]
        for li, L in enumerate(w.layers):
            unit, streamed = _unit(eng, li, L, stream)
            x, _ = _layer_fp32(eng, li, L, unit, streamed, x, pos, state, bs, T)
            if streamed:
                _release(eng, li, stream)
        xf = _rms(x, w.final_norm, tm.arch.eps)
        return (xf @ w.lm_head.float().T).view(bs, T, -1)


def verify_teacher_forced(eng, state: SeqState, draft_tokens: torch.Tensor, stream) -> dict:
    """Layer-local parity of the product verify pass: the product path runs
    once with a hook that snapshots each layer's input hidden state and its
    router's token → expert choice; then every layer is recomputed in fp32
    FROM THE PRODUCT'S OWN INPUT (with the product's expert choice forced and
    the pair weights from fp32 router logits), and the LM head from the
    product's last hidden state.  A random-weight 56-layer MoE is chaotic in
    its routing (a bf16 rounding flips a near-tied expert choice, and a flipped
    expert replaces a whole FFN contribution), so free-running logits diverge
    without any kernel error; this check isolates the kernels' error per layer."""
    tm = eng.target
    a, w, st, dev = tm.arch, tm.w, tm.streamer, tm.device
    H, E = a.hidden, a.n_expert
    bs, n = draft_tokens.shape
    T = n + 1
    R = bs * T
    nL = len(w.layers)
    xs, routes = [None] * (nL + 1), [None] * nL

    def hook(li, phase, s):
        xa = tm.ws.get("x", (R, H), torch.bfloat16)
        if phase == "attn_start":
            xs[li] = xa.clone()
        elif phase == "ffn_end":
            if E:
                offs = tm.ws.get("offs", (E + 1,), torch.int32).clone()
                perm = tm.ws.get("perm", (2 * R,), torch.int32).clone()
                routes[li] = (offs, perm)
            if li == nL - 1:
                xs[nL] = xa.clone()

    prev = tm.hooks
    tm.hooks = hook
    try:
        got = tm.verify(state, draft_tokens)
    finally:
        tm.hooks = prev
    state.kv.join(stream)
    stream.synchronize()
    per_layer = []
    with torch.cuda.stream(stream):
        pos = torch.as_tensor(state.ctx, device=dev)[:, None] + torch.arange(T, device=dev)[None, :]
        for li, L in enumerate(w.layers):
            unit, streamed = _unit(eng, li, L, stream)
            sel = None
            if E:
                offs, perm = routes[li]
                o = offs.cpu().numpy()
                sel = torch.zeros((R, E), dtype=torch.bool, device=dev)
                for e in range(E):
                    sel[perm[int(o[e]):int(o[e + 1])].long(), e] = True
            x_in = xs[li].float()
            ref, lr = _layer_fp32(eng, li, L, unit, streamed, x_in, pos, state, bs, T, routing=sel)
            if streamed:
                _release(eng, li, stream)
            out = xs[li + 1].float()
            d = (out - ref).abs()
            upd = ref - x_in
            rec = {"layer": li, "max_abs": d.max().item(),
                   "rel": (d / (ref.abs() + ref.pow(2).mean().sqrt())).max().item(),
                   "rms_err_over_rms_update": (d.pow(2).mean().sqrt() / upd.pow(2).mean().sqrt()).item()}
            if E:
                top = torch.topk(lr, 3, dim=-1)
                ref_sel = torch.zeros_like(sel).scatter_(1, top.indices[:, :2], True)
                rec["route_agree"] = (ref_sel == sel).all(-1).float().mean().item()
                rec["route_min_gap"] = (top.values[:, 1] - top.values[:, 2]).min().item()
            per_layer.append(rec)
        xf = _rms(xs[nL].float(), w.final_norm, a.eps)
        want = (xf @ w.lm_head.float().T).view(bs, T, -1)
        # the same final norm + LM head re-run through the native ops on the snapshot
        from paper_2505_10259_b200 import native
        xf_n = torch.empty((R, H), dtype=torch.bfloat16, device=dev)
        native.rmsnorm(xs[nL], w.final_norm, xf_n, a.eps, stream)
        lg_n = torch.empty((R, a.vocab), dtype=torch.float32, device=dev)
        native.gemm(xf_n, w.lm_head, lg_n, native.EPI_F32, None, stream)
        xf_prod = tm.ws.get("xf", (R, H), torch.bfloat16).clone()
    stream.synchronize()
    got = got.float()
    d = (got - want).abs()
    row_max = d.amax(-1).reshape(-1)
    diag = {"native_rerun_vs_fp32_max": (lg_n.view_as(want) - want).abs().max().item(),
            "native_rerun_vs_product_max": (lg_n.view_as(got) - got).abs().max().item(),
            "xf_product_vs_rerun_max": (xf_prod.float() - xf_n.float()).abs().max().item(),
            "lm_head_ptr_aligned": w.lm_head.data_ptr() % 16 == 0, "lm_head_shape": list(w.lm_head.shape),
            "lm_head_contig": w.lm_head.is_contiguous()}
    scale = want.abs().max().item()
    top2 = torch.topk(want, 2, dim=-1).values
    decisive = (top2[..., 0] - top2[..., 1]) > 0.02 * scale
    agree = got.argmax(-1) == want.argmax(-1)
    worst = max(per_layer, key=lambda r: r["rms_err_over_rms_update"])
    res = {"layers": nL, "max_layer_rel": max(r["rel"] for r in per_layer),
           "max_layer_rms_err_over_rms_update": worst["rms_err_over_rms_update"], "worst_layer": worst["layer"],
           "lm_head_max_abs_dlogit": d.max().item(), "lm_head_rel_max": d.max().item() / scale if scale else None,
           "argmax_agree": agree.float().mean().item(),
           "argmax_agree_decisive": agree[decisive].float().mean().item() if decisive.any() else None,
           "decisive_rows": int(decisive.sum().item()), "per_layer": per_layer,
           "lm_head_row_max_abs": [round(v, 4) for v in row_max.tolist()],
           "got_zero_rows": int((got.reshape(-1, got.shape[-1]).abs().amax(-1) == 0).sum().item()), "diag": diag}
    if E:
        res["route_agree_min"] = min(r["route_agree"] for r in per_layer)
    return res


def parity_report(eng, session, n_seq: int = 2, seed: int = 0) -> dict:
    """Verify ``n_seq`` sequences of batch 0 through the product path and the
    fp32 restatement: layer-local (teacher-forced, the kernel check) and
    free-running (end to end, chaotic in the routing on random weights)."""
    s = session
    b = s.batches[0]
    rows = np.arange(b.lo, b.lo + min(n_seq, b.n))
    rng = np.random.default_rng(seed)
    drafts = torch.from_numpy(rng.integers(0, eng.target.arch.vocab, (rows.size, s.n_cand)).astype(np.int32))
    st = eng.tgt_stream
    s.tkv.set_window(b.lo, b.hi)
    state = SeqState(s.tkv, rows, s.ctx[rows], s.t_last[rows], st)
    forced = verify_teacher_forced(eng, state, drafts, st)
    got = eng.target.verify(state, drafts)
    s.tkv.join(st)
    st.synchronize()
    want = verify_fp32(eng, state, drafts, st)
    st.synchronize()
    got, want = got.float(), want.float()
    d = (got - want).abs()
    scale = want.abs().max().item()
    top2 = torch.topk(want, 2, dim=-1).values
    decisive = (top2[..., 0] - top2[..., 1]) > 0.02 * scale
    agree = (got.argmax(-1) == want.argmax(-1))
    free = {"max_abs_dlogit": d.max().item(), "rms_dlogit": d.pow(2).mean().sqrt().item(),
            "logit_scale_max_abs": scale, "rel_max": d.max().item() / scale if scale else None,
            "argmax_agree": agree.float().mean().item(),
            "argmax_agree_decisive": agree[decisive].float().mean().item() if decisive.any() else None,
            "decisive_rows": int(decisive.sum().item())}
    per_layer = forced.pop("per_layer")
    return {"sequences": int(rows.size), "rows": int(rows.size * (s.n_cand + 1)),
            "teacher_forced": forced, "free_running": free,
            "per_layer_rms_err_over_rms_update": [round(r["rms_err_over_rms_update"], 5) for r in per_layer],
            "per_layer_route_agree": [round(r.get("route_agree", 1.0), 4) for r in per_layer],
            "reference": "PyTorch fp32 restatement (tools/fp32_ref.py) over the same streamed weights and KV; "
                         "teacher_forced = every layer (and the LM head) recomputed in fp32 from the product's own "
                         "input hidden state with the product's expert choice; free_running = 56 fp32 layers "
                         "end to end (random-weight MoE routing is chaotic: near-tied expert choices flip)"}
