"""Parity-mode kernels (csrc/canon.cu) against the canonical CPU oracle
(oracle/csrc/canon_oracle.c) on random inputs: every output must be EQUAL bit
for bit — these are the ops through which the engine's ``arith="canonical"``
reproduces the oracle's tokens (tests/test_engine_gpu.py)."""
import math

import numpy as np
import pytest
import torch

from oracle import canon_ref
from paper_2505_10259_b200 import native
from paper_2505_10259_b200.models import rope_table
from paper_2505_10259_b200.weights import interleave_gate_up

pytestmark = pytest.mark.gpu


def rand_bf16(shape, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * scale).to(torch.bfloat16)


def bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def same(a: np.ndarray, b: np.ndarray) -> bool:
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("epi", [native.EPI_BF16, native.EPI_F32, native.EPI_BF16_RESID, native.EPI_BF16_ROWSCALE])
@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (37, 256, 320), (130, 1024, 256)])
def test_canon_gemm_dense(M, N, K, epi):
    a, b = rand_bf16((M, K), 1), rand_bf16((N, K), 2, 0.1)
    aux_t = None
    if epi == native.EPI_BF16_RESID:
        aux_t = rand_bf16((M, N), 3)
    elif epi == native.EPI_BF16_ROWSCALE:
        aux_t = torch.rand(M, generator=torch.Generator().manual_seed(4))
    out = torch.empty((M, N), dtype=torch.float32 if epi == native.EPI_F32 else torch.bfloat16, device="cuda")
    native.canon_gemm(a.cuda(), b.cuda(), out, epi, aux_t.cuda() if aux_t is not None else None)
    aux = None if aux_t is None else (aux_t.numpy() if epi == native.EPI_BF16_ROWSCALE else bits(aux_t))
    want = canon_ref.gemm(bits(a), bits(b), epi, aux)
    got = out.cpu().numpy() if epi == native.EPI_F32 else bits(out)
    assert same(got, want)


@pytest.mark.parametrize("counts", [[5, 0, 9, 1, 0, 3, 7, 2], [0, 0, 0, 16, 0, 0, 0, 0], [33, 1, 1, 1, 1, 1, 1, 1]])
def test_canon_gemm_grouped_swiglu_and_rowscale(counts):
    """Grouped expert GEMMs: SwiGLU over the interleaved gate/up window layout,
    then the routing-weight-scaled down projection, rows routed by offsets."""
    E, H, I = len(counts), 128, 192
    rows = sum(counts)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    x = rand_bf16((rows, H), 5)
    wg, wu, wd = rand_bf16((E, I, H), 6, 0.1), rand_bf16((E, I, H), 7, 0.1), rand_bf16((E, H, I), 8, 0.1)
    gu = interleave_gate_up(wg, wu).contiguous().cuda()
    act = torch.empty((rows, I), dtype=torch.bfloat16, device="cuda")
    offs_d = torch.from_numpy(offs).cuda()
    native.canon_gemm_grouped(x.cuda(), gu.data_ptr(), offs_d, E, 2 * I, act, native.EPI_SWIGLU)
    scale = torch.rand(rows, generator=torch.Generator().manual_seed(9))
    y = torch.empty((rows, H), dtype=torch.bfloat16, device="cuda")
    wd_d = wd.contiguous().cuda()
    native.canon_gemm_grouped(act, wd_d.data_ptr(), offs_d, E, H, y, native.EPI_BF16_ROWSCALE, scale.cuda())
    xa, ga, ua, da = bits(x), bits(wg), bits(wu), bits(wd)
    want_act = np.zeros((rows, I), np.uint16)
    want_y = np.zeros((rows, H), np.uint16)
    for e in range(E):
        lo, hi = offs[e], offs[e + 1]
        if hi == lo:
            continue
        want_act[lo:hi] = canon_ref.swiglu(xa[lo:hi], ga[e], ua[e])
        want_y[lo:hi] = canon_ref.gemm(want_act[lo:hi], da[e], canon_ref.EPI_BF16_ROWSCALE, scale.numpy()[lo:hi])
    assert same(bits(act), want_act)
    assert same(bits(y), want_y)


@pytest.mark.parametrize("T,H", [(1, 64), (29, 256), (7, 4096)])
def test_canon_rmsnorm(T, H):
    x, w = rand_bf16((T, H), 10, 3.0), rand_bf16((H,), 11)
    out = torch.empty((T, H), dtype=torch.bfloat16, device="cuda")
    native.canon_rmsnorm(x.cuda(), w.cuda(), out, 1e-5)
    assert same(bits(out), canon_ref.rmsnorm(bits(x), bits(w), 1e-5))


def test_canon_rope_table_matches_oracle_table():
    assert np.array_equal(rope_table(64, 1e6, 300), canon_ref.rope_table(64, 1e6, 300))


@pytest.mark.parametrize("hq,hkv,dh", [(4, 2, 64), (6, 1, 128)])
def test_canon_rope_kv_append(hq, hkv, dh):
    T, ps, n_pages = 23, 16, 8
    qkv = rand_bf16((T, (hq + 2 * hkv) * dh), 12)
    rng = np.random.default_rng(13)
    pos = rng.integers(0, 120, T).astype(np.int32)
    slots = rng.permutation(n_pages * ps)[:T].astype(np.int32)
    table = rope_table(dh, 1e6, 128)
    q = torch.empty((T, hq, dh), dtype=torch.bfloat16, device="cuda")
    kc = torch.zeros((n_pages, hkv, ps, dh), dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    native.canon_rope_kv_append(qkv.cuda(), torch.from_numpy(pos).cuda(), torch.from_numpy(slots).cuda(), hq, hkv,
                                dh, torch.from_numpy(table).cuda(), ps, q, kc, vc)
    qa = bits(qkv).reshape(T, hq + 2 * hkv, dh)
    assert same(bits(q), canon_ref.rope(qa[:, :hq], pos, table))
    kw = canon_ref.rope(qa[:, hq:hq + hkv], pos, table)
    kg, vg = bits(kc), bits(vc)
    for t in range(T):
        pg, off = divmod(int(slots[t]), ps)
        assert same(kg[pg, :, off], kw[t])
        assert same(vg[pg, :, off], qa[t, hq + hkv:])


@pytest.mark.parametrize("hq,hkv,dh,ps", [(4, 2, 64, 16), (8, 1, 128, 8)])
def test_canon_attn_paged(hq, hkv, dh, ps):
    """Per sequence: query rows at positions kv_before + j attend keys
    [0, kv_before + j] through a shuffled block table."""
    qlens, kvb = [5, 1, 9], [40, 0, 17]
    bs, max_pages = len(qlens), 8
    n_pages = bs * max_pages
    rng = np.random.default_rng(14)
    bt = rng.permutation(n_pages).astype(np.int32).reshape(bs, max_pages)
    kc, vc = rand_bf16((n_pages, hkv, ps, dh), 15), rand_bf16((n_pages, hkv, ps, dh), 16)
    rows = sum(qlens)
    q = rand_bf16((rows, hq, dh), 17)
    qs = np.concatenate([[0], np.cumsum(qlens)]).astype(np.int32)
    out = torch.empty((rows, hq * dh), dtype=torch.bfloat16, device="cuda")
    scale = 1.0 / math.sqrt(dh)
    native.canon_attn_paged(q.cuda(), kc.cuda(), vc.cuda(), torch.from_numpy(bt).cuda(), torch.from_numpy(qs).cuda(),
                            torch.tensor(kvb, dtype=torch.int32).cuda(), max(qlens), hq, hkv, dh, ps, scale, out)
    ka, va, qa = bits(kc), bits(vc), bits(q)
    got = bits(out).reshape(rows, hq, dh)
    for s in range(bs):
        n_keys = kvb[s] + qlens[s]
        pages = bt[s, :(n_keys + ps - 1) // ps]
        kseq = ka[pages].transpose(0, 2, 1, 3).reshape(-1, hkv, dh)[:n_keys]
        vseq = va[pages].transpose(0, 2, 1, 3).reshape(-1, hkv, dh)[:n_keys]
        want = canon_ref.attn(qa[qs[s]:qs[s + 1]], kseq, vseq, kvb[s], np.float32(scale))
        assert same(got[qs[s]:qs[s + 1]], want)


@pytest.mark.parametrize("T,H,E", [(1, 64, 8), (50, 256, 8), (9, 128, 4)])
def test_canon_router_top2(T, H, E):
    x, wg = rand_bf16((T, H), 18), rand_bf16((E, H), 19, 0.2)
    idx = torch.empty((T, 2), dtype=torch.int32, device="cuda")
    w = torch.empty((T, 2), dtype=torch.float32, device="cuda")
    offs = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    perm = torch.empty(2 * T, dtype=torch.int32, device="cuda")
    roww = torch.empty(2 * T, dtype=torch.float32, device="cuda")
    trows = torch.empty((T, 2), dtype=torch.int32, device="cuda")
    xperm = torch.empty((2 * T, H), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(native.router_workspace_bytes(T, E), dtype=torch.uint8, device="cuda")
    native.canon_router_top2(x.cuda(), wg.cuda(), offs, perm, roww, trows, xperm, ws, topk_idx=idx, topk_w=w)
    want_i, want_w = canon_ref.route(bits(x), bits(wg))
    assert np.array_equal(idx.cpu().numpy(), want_i)
    assert same(w.cpu().numpy(), want_w)
    # stable expert-major permutation: rows of expert e in token order
    order = sorted(range(2 * T), key=lambda p: (want_i.reshape(-1)[p], p))
    assert perm.cpu().tolist() == [p // 2 for p in order]
    assert same(bits(xperm), bits(x)[[p // 2 for p in order]])
    inv = np.empty(2 * T, np.int64)
    inv[order] = np.arange(2 * T)
    assert trows.cpu().numpy().reshape(-1).tolist() == inv.tolist()
