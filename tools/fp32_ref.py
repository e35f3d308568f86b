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


def verify_fp32(eng, state: SeqState, draft_tokens: torch.Tensor, stream) -> torch.Tensor:
    """fp32 logits [bs, n+1, V] of t_last + drafts at positions ctx..ctx+n."""
    tm = eng.target
    a, w, st = tm.arch, tm.w, tm.streamer
    dev = tm.device
    H, dh, hq, hkv, E = a.hidden, a.head_dim, a.n_head, a.n_kv_head, a.n_expert
    bs, n = draft_tokens.shape
    T = n + 1
    stream_attn = any(L.wqkv is None for L in w.layers)
    ffn_off = unit_layout(a, stream_attn)[0] // 2
    gu_el, dn_el, _ = ffn_offsets(a)
    kv = state.kv
    with torch.cuda.stream(stream):
        toks = torch.cat([torch.as_tensor(state.t_last, device=dev)[:, None].int(), draft_tokens.to(dev).int()], 1)
        pos = torch.as_tensor(state.ctx, device=dev)[:, None] + torch.arange(T, device=dev)[None, :]
        x = w.embed[toks.reshape(-1).long()].float()                      # [bs·T, H]
        for li, L in enumerate(w.layers):
            streamed = st is not None and li in st.streamed
            if streamed:
                st.acquire(li, stream)  # the stream waits for the slot; k_use indexes it until release
                unit = st.slots[st.k_use % st.n_slots].view(torch.bfloat16)
            else:
                unit = L.ffn
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
            if E:
                lr = hn @ L.router.float().T
                top = torch.topk(lr, 2, dim=-1)
                w1 = torch.sigmoid(top.values[:, 1] - top.values[:, 0])
                wts = torch.stack([1.0 - w1, w1], -1)
                gu = ffn[:gu_el].view(E, 2 * a.inter, H)
                dn = ffn[gu_el:gu_el + dn_el].view(E, H, a.inter)
                y = torch.zeros_like(h)
                for e in range(E):
                    sel = (top.indices == e)
                    rows = sel.any(-1).nonzero().squeeze(-1)
                    if rows.numel() == 0:
                        continue
                    we = (wts * sel).sum(-1)[rows]
                    g = gu[e].view(a.inter // SWIGLU_BLOCK, 2, SWIGLU_BLOCK, H)
                    gate = hn[rows] @ g[:, 0].reshape(a.inter, H).float().T
                    up = hn[rows] @ g[:, 1].reshape(a.inter, H).float().T
                    y[rows] += (torch.nn.functional.silu(gate) * up) @ dn[e].float().T * we[:, None]
                x = h + y
            else:
                g = ffn[: 2 * a.inter * H].view(a.inter // SWIGLU_BLOCK, 2, SWIGLU_BLOCK, H)
                gate = hn @ g[:, 0].reshape(a.inter, H).float().T
                up = hn @ g[:, 1].reshape(a.inter, H).float().T
                x = h + (torch.nn.functional.silu(gate) * up) @ ffn[2 * a.inter * H:].view(H, a.inter).float().T
            if streamed:
                st.release(li, stream)
        xf = _rms(x, w.final_norm, a.eps)
        return (xf @ w.lm_head.float().T).view(bs, T, -1)


def parity_report(eng, session, n_seq: int = 2, seed: int = 0) -> dict:
    """Verify ``n_seq`` sequences of batch 0 through the product path and the
    fp32 restatement; compare the logits."""
    s = session
    b = s.batches[0]
    rows = np.arange(b.lo, b.lo + min(n_seq, b.n))
    rng = np.random.default_rng(seed)
    drafts = torch.from_numpy(rng.integers(0, eng.target.arch.vocab, (rows.size, s.n_cand)).astype(np.int32))
    st = eng.tgt_stream
    s.tkv.set_window(b.lo, b.hi)
    state = SeqState(s.tkv, rows, s.ctx[rows], s.t_last[rows], st)
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
    return {"sequences": int(rows.size), "rows": int(rows.size * (s.n_cand + 1)),
            "max_abs_dlogit": d.max().item(), "rms_dlogit": d.pow(2).mean().sqrt().item(),
            "logit_scale_max_abs": scale, "rel_max": d.max().item() / scale if scale else None,
            "argmax_agree": agree.float().mean().item(),
            "argmax_agree_decisive": agree[decisive].float().mean().item() if decisive.any() else None,
            "decisive_rows": int(decisive.sum().item()),
            "reference": "PyTorch fp32 restatement (tools/fp32_ref.py) over the same streamed weights and KV"}
