"""GPU parity at the headline shapes (configs[2]: Mixtral-8x22B target,
Mistral-7B-v0.3 draft).

The headline bench runs with forced acceptance, so these tests pin the
numerics the benchmark exercises, at the production shapes:

* the grouped MoE GEMMs at gate_up N = 2·16384, K = 6144 and down N = 6144,
  K = 16384 over full 8-expert slabs addressed through the 3-D tensor maps,
  with skewed expert row counts (empty experts, experts spanning more than
  one 16-m-tile raster band) — against an fp32 torch reference on sampled
  output columns;
* one full Mixtral-8x22B layer + final norm + LM head (V = 32768) for a
  verify batch of 32 sequences × 9 tokens at context 503, its FFN streamed
  from pinned host DRAM as an XC4 unit through a window slot, against the
  CPU oracle (oracle/model_ref.forward, bf16 rounding points mirrored);
* one full Mistral-7B-v0.3 draft layer + LM head the same way (HBM-resident).

Tolerances (written here, SURVEY.md north star "within a stated bf16/fp32
tolerance"): GEMM outputs within 1.5 % of |ref| + rms(ref) (one bf16 rounding
after fp32 accumulation in a different order); layer logits within
0.05 + 2 % of |ref| except for tokens whose top-2 routing is a near-tie in the
oracle (router-logit gap < 1e-3 — a rounding difference may legitimately pick
the other expert there), and the argmax equal wherever the oracle's top-1/top-2
logit gap exceeds 0.1."""
import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import model_ref
from paper_2505_10259_b200 import MIXTRAL_8X22B, MISTRAL_7B_V3, native
from paper_2505_10259_b200.api import build_engine
from paper_2505_10259_b200.models import SeqState
from paper_2505_10259_b200.weights import ffn_offsets

pytestmark = pytest.mark.gpu
DEV = "cuda"
ROWS_8X22B = 8064  # 2 experts × bs 448 × (n_cand 8 + 1) tokens: the headline verify pass


def _bf16_close(got, want, rel=1.5e-2):
    got, want = got.float(), want.float()
    scale = want.abs() + want.pow(2).mean().sqrt()
    bad = ((got - want).abs() > rel * scale).sum().item()
    assert bad == 0, f"{bad} elements off; max err {(got - want).abs().max().item()}"


def _counts():
    # skewed: two empty experts, two spanning > 16 m-tiles (> 2048 rows), a 1-row expert
    c = [2600, 0, 2100, 130, 1, 0, 1000, 0]
    c[7] = ROWS_8X22B - sum(c)
    return c


@pytest.fixture(scope="module")
def expert_slab():
    """One 8x22B FFN unit in HBM in the streamed layout [gate_up interleaved | down], N(0, 0.02²)."""
    a = MIXTRAL_8X22B
    gu, dn, total = ffn_offsets(a)
    g = torch.Generator(device=DEV).manual_seed(22)
    unit = torch.empty(total // 2, dtype=torch.bfloat16, device=DEV).normal_(0.0, 0.02, generator=g)
    return unit, gu, dn


def _offs(counts):
    return torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=DEV)


@pytest.mark.parametrize("variant", [0, 1, 2, 3], ids=["auto", "cta1", "cta_pair", "one_tile_per_cta"])
def test_grouped_gateup_swiglu_production_shape(expert_slab, variant):
    a = MIXTRAL_8X22B
    E, H, I = a.n_expert, a.hidden, a.inter
    unit, gu, _ = expert_slab
    counts = _counts()
    g = torch.Generator(device=DEV).manual_seed(1)
    x = torch.randn(ROWS_8X22B, H, device=DEV, generator=g).to(torch.bfloat16)
    act = torch.empty(ROWS_8X22B, I, dtype=torch.bfloat16, device=DEV)
    native.gemm_grouped(x, unit.data_ptr(), _offs(counts), E, 2 * I, act, native.EPI_SWIGLU, variant=variant)
    torch.cuda.synchronize()
    w = unit[:gu].view(E, 2 * I, H)
    # sampled output columns: first / last of the tile grid and a spread in between
    cols = torch.tensor(sorted({0, 1, 63, 64, 127, 128, I - 1, I - 64} | set(range(97, I, 613))), device=DEV)
    p, j = cols // 64, cols % 64
    g_rows, u_rows = 128 * p + j, 128 * p + 64 + j
    o = np.concatenate([[0], np.cumsum(counts)])
    ref = torch.zeros(ROWS_8X22B, cols.numel(), device=DEV)
    for e in range(E):
        if counts[e] == 0:
            continue
        xe = x[o[e]:o[e + 1]].float()
        gate = xe @ w[e, g_rows].float().T
        up = xe @ w[e, u_rows].float().T
        ref[o[e]:o[e + 1]] = torch.nn.functional.silu(gate) * up
    _bf16_close(act[:, cols], ref)


@pytest.mark.parametrize("variant", [0, 1, 2, 3], ids=["auto", "cta1", "cta_pair", "one_tile_per_cta"])
def test_grouped_down_rowscale_production_shape(expert_slab, variant):
    a = MIXTRAL_8X22B
    E, H, I = a.n_expert, a.hidden, a.inter
    unit, gu, dn = expert_slab
    counts = _counts()
    g = torch.Generator(device=DEV).manual_seed(2)
    act = (torch.randn(ROWS_8X22B, I, device=DEV, generator=g) * 0.5).to(torch.bfloat16)
    wts = torch.rand(ROWS_8X22B, device=DEV, generator=g)
    y = torch.empty(ROWS_8X22B, H, dtype=torch.bfloat16, device=DEV)
    native.gemm_grouped(act, unit.data_ptr() + 2 * gu, _offs(counts), E, H, y, native.EPI_BF16_ROWSCALE, wts,
                        variant=variant)
    torch.cuda.synchronize()
    w = unit[gu:gu + dn].view(E, H, I)
    cols = torch.tensor(sorted({0, 1, 127, 128, 255, 256, H - 1} | set(range(41, H, 97))), device=DEV)
    o = np.concatenate([[0], np.cumsum(counts)])
    ref = torch.zeros(ROWS_8X22B, cols.numel(), device=DEV)
    for e in range(E):
        if counts[e]:
            ref[o[e]:o[e + 1]] = (act[o[e]:o[e + 1]].float() @ w[e, cols].float().T) * wts[o[e]:o[e + 1], None]
    _bf16_close(y[:, cols], ref)


# ------------------------------------------------------------------ full layer vs the CPU oracle


def _logical(arch, seed):
    """Logical (HF-shaped) bf16 weights of a 1-layer model on the GPU, drawn as
    SURVEY.md §8d prescribes (N(0, 0.02²); norms ≈ 1; embeddings std 1 and an
    LM head scaled like oracle.model_ref.init_weights)."""
    g = torch.Generator(device=DEV).manual_seed(seed)
    H, I, E, dh = arch.hidden, arch.inter, arch.n_expert, arch.head_dim

    def w(*shape, s=0.02):
        return torch.empty(*shape, device=DEV).normal_(0.0, s, generator=g).to(torch.bfloat16)

    def norm():
        return (1.0 + 0.1 * torch.randn(H, device=DEV, generator=g)).to(torch.bfloat16)

    L = {"attn_norm": norm(), "wq": w(arch.n_head * dh, H), "wk": w(arch.n_kv_head * dh, H),
         "wv": w(arch.n_kv_head * dh, H), "wo": w(H, arch.n_head * dh), "ffn_norm": norm()}
    if E:
        L.update(router=w(E, H, s=0.1), w_gate=w(E, I, H), w_up=w(E, I, H), w_down=w(E, H, I))
    else:
        L.update(w_gate=w(I, H), w_up=w(I, H), w_down=w(H, I))
    return {"embed": w(arch.vocab, H, s=1.0), "final_norm": norm(),
            "lm_head": w(arch.vocab, H, s=4.0 / math.sqrt(H)), "layers": [L]}


def _np(W):
    out = {k: v.float().cpu().numpy() for k, v in W.items() if k != "layers"}
    out["layers"] = [{k: v.float().cpu().numpy() for k, v in L.items()} for L in W["layers"]]
    return out


def _oracle_arch(a):
    return model_ref.Arch(vocab=a.vocab, hidden=a.hidden, inter=a.inter, n_layer=a.n_layer, n_head=a.n_head,
                          n_kv_head=a.n_kv_head, head_dim=a.head_dim, n_expert=a.n_expert, top_k=a.top_k,
                          rope_theta=a.rope_theta, eps=a.eps)


def _layer_parity(arch, model_of, stream_layers, codec, n_seq=32, n_cand=8, ctx=503, seed=7, stream_attn=False,
                  draft=None, split_window=False):
    """Verify pass of n_seq sequences × (n_cand + 1) tokens over ctx positions of
    shared random KV, engine vs oracle.  Returns (got, want, router_gap, want_fp32):
    ``want`` mirrors the kernels' bf16 rounding points, ``want_fp32`` keeps fp32."""
    W = _logical(arch, seed)
    rng = np.random.default_rng(seed)
    tokens = rng.integers(0, arch.vocab, (n_seq, n_cand + 1)).astype(np.int32)
    max_len = ctx + n_cand + 2
    # shared context KV, bf16-representable
    kv_np = model_ref.KV(_oracle_arch(arch), n_seq, max_len)
    g = torch.Generator(device=DEV).manual_seed(seed + 1)
    shape = (n_seq, ctx, arch.n_kv_head, arch.head_dim)
    k_ctx = torch.randn(shape, device=DEV, generator=g).to(torch.bfloat16)
    v_ctx = torch.randn(shape, device=DEV, generator=g).to(torch.bfloat16)
    kv_np.k[0, :, :ctx] = k_ctx.float().cpu().numpy()
    kv_np.v[0, :, :ctx] = v_ctx.float().cpu().numpy()
    if arch.is_moe:
        eng = build_engine(arch, draft or MISTRAL_7B_V3_1L, W, None, stream_layers=stream_layers, codec=codec,
                           trace=False, stream_attn=stream_attn, split_window=split_window)
    else:
        eng = build_engine(MIXTRAL_1L_TINYFFN, arch, None, W, stream_layers=set(), trace=False)
    model = model_of(eng)
    s = eng.new_session(n_seq, n_seq, max_len, n_cand)
    kv = s.tkv if arch.is_moe else s.dkv
    rows = np.arange(n_seq) if arch.is_moe else s.drow[:n_seq]
    # write the context KV into the paged cache: position p of row r → slot
    for r in range(n_seq):
        pos = np.arange(ctx)
        slots = torch.from_numpy(kv.slots(np.full(ctx, rows[r]), pos).astype(np.int64)).to(DEV)
        pages, off = slots // kv.page_size, slots % kv.page_size
        kv.k[0][pages, :, off] = k_ctx[r]
        kv.v[0][pages, :, off] = v_ctx[r]
    torch.cuda.synchronize()
    state = SeqState(kv, rows, np.full(n_seq, ctx), tokens[:, 0], eng.tgt_stream if arch.is_moe else eng.drf_stream)
    logits = model.verify(state, torch.from_numpy(tokens[:, 1:])) if arch.is_moe else \
        _dense_verify(model, state, tokens)
    torch.cuda.synchronize()
    got = logits.reshape(n_seq, n_cand + 1, -1).cpu().numpy()
    Wn = _np(W)
    cap = {}
    orig = model_ref.rmsnorm
    if arch.is_moe:  # capture the oracle's router input to find near-tie routings
        def spy(x, w, eps, mirror):
            y = orig(x, w, eps, mirror)
            if w is Wn["layers"][0]["ffn_norm"]:
                cap["hn"] = y
            return y

        model_ref.rmsnorm = spy
    try:
        want = model_ref.forward(_oracle_arch(arch), Wn, kv_np, list(range(n_seq)), list(tokens), [ctx] * n_seq,
                                 True, "all")
    finally:
        model_ref.rmsnorm = orig
    want = np.stack(want)
    # the same oracle without bf16 rounding points: exact arithmetic, for the calibration bar
    want32 = np.stack(model_ref.forward(_oracle_arch(arch), Wn, kv_np, list(range(n_seq)), list(tokens),
                                        [ctx] * n_seq, False, "all"))
    gap = None
    if arch.is_moe:  # min(top1 − top2, top2 − top3) router-logit gap per token
        lr = cap["hn"].astype(np.float64) @ Wn["layers"][0]["router"].T.astype(np.float64)
        srt = -np.sort(-lr, axis=1)
        gap = np.minimum(srt[:, 0] - srt[:, 1], srt[:, 1] - srt[:, 2]).reshape(tokens.shape)
    return got, want, gap, want32


def _dense_verify(model, state, tokens):
    """DraftModel has no verify(); run its forward over the same n_cand+1 rows."""
    from paper_2505_10259_b200.models import TargetModel

    return TargetModel.verify(model, state, torch.from_numpy(tokens[:, 1:]))


MISTRAL_7B_V3_1L = dataclasses.replace(MISTRAL_7B_V3, n_layer=1)
MIXTRAL_1L_TINYFFN = dataclasses.replace(MIXTRAL_8X22B, n_layer=1, inter=128)


def _check_logits(got, want, exclude=None, want32=None):
    """Logits tolerance.  Every intermediate hidden state is stored in bf16 (the
    kernels' and the mirroring oracle's rounding points), and a 1-ulp rounding
    disagreement anywhere in the 6144- (4096-) wide state moves every logit by
    ≈ ulp·|w_lm|, so the bar is stated relative to the logit scale:
      * rms(Δ) ≤ 1 % of rms(want) and max |Δ| ≤ 0.15·rms(want);
      * argmax equal wherever the oracle's top-1/top-2 gap exceeds 0.25·rms(want);
      * calibration: the GPU is no further from exact fp32 arithmetic than the
        bf16-mirroring oracle itself, within 2× (rms(got − fp32) ≤ 2·rms(want − fp32)).
    Tokens whose top-2 routing is a near-tie in the oracle (``exclude``) are
    skipped: a rounding difference may legitimately pick the other expert."""
    n_seq, T, V = want.shape
    mask = np.ones((n_seq, T), bool) if exclude is None else ~exclude
    assert mask.mean() > 0.9, f"too many near-tie routed tokens excluded ({(~mask).sum()})"
    d = np.abs(got - want)[mask]
    scale = float(np.sqrt((want[mask] ** 2).mean()))
    rms = float(np.sqrt((d ** 2).mean()))
    assert rms <= 0.01 * scale, f"rms |Δ| {rms:.4f} > 1% of rms logit {scale:.3f}"
    assert d.max() <= 0.15 * scale, f"max |Δ| {d.max():.4f} > 0.15·rms logit {scale:.3f}"
    top2 = -np.sort(-want, axis=-1)[..., :2]
    decisive = (top2[..., 0] - top2[..., 1] > 0.25 * scale) & mask
    assert (got.argmax(-1) == want.argmax(-1))[decisive].all()
    if want32 is not None:
        e_gpu = float(np.sqrt(((got - want32)[mask] ** 2).mean()))
        e_orc = float(np.sqrt(((want - want32)[mask] ** 2).mean()))
        assert e_gpu <= 2.0 * e_orc + 1e-4 * scale, f"GPU {e_gpu:.4f} vs oracle {e_orc:.4f} from exact fp32"
    return float(d.max()), float(decisive.mean())


@pytest.mark.parametrize("split", [False, True])
def test_mixtral_8x22b_layer_and_lm_head_vs_oracle(split):
    """``split``: the unit streams through the split window ([gate_up | down], one XC4 unit per
    segment) — the same oracle bar."""
    a = dataclasses.replace(MIXTRAL_8X22B, n_layer=1)
    got, want, gap, want32 = _layer_parity(a, lambda e: e.target, {0}, "xc4", split_window=split)
    near = gap < 1e-3
    maxd, dec = _check_logits(got, want, exclude=near, want32=want32)
    print(f"8x22B layer (split {split}): max |Δlogit| {maxd:.4f}, decisive rows {dec:.2f}, "
          f"near-tie routed tokens {near.sum()}")


def test_mistral_7b_draft_layer_and_lm_head_vs_oracle():
    a = MISTRAL_7B_V3_1L
    got, want, _, want32 = _layer_parity(a, lambda e: e.draft, set(), "none", n_seq=32, n_cand=4)
    maxd, dec = _check_logits(got, want, want32=want32)
    print(f"Mistral-7B layer: max |Δlogit| {maxd:.4f}, decisive rows {dec:.2f}")


def test_mixtral_8x7b_streamed_attention_layer_vs_oracle():
    """configs[1]'s layout (HBM capped at 24 GiB): the attention projections travel
    inside the streamed XC4 unit with the FFN (H3) through the split window
    ([Wqkv | Wo | gate_up] | down), Mixtral-8x7B shapes."""
    from paper_2505_10259_b200 import MIXTRAL_8X7B, MISTRAL_7B

    a = dataclasses.replace(MIXTRAL_8X7B, n_layer=1)
    d = dataclasses.replace(MISTRAL_7B, n_layer=1)
    got, want, gap, want32 = _layer_parity(a, lambda e: e.target, {0}, "xc4", n_seq=16, stream_attn=True, draft=d,
                                           split_window=True)
    near = gap < 1e-3
    maxd, dec = _check_logits(got, want, exclude=near, want32=want32)
    print(f"8x7B streamed-attention layer: max |Δlogit| {maxd:.4f}, decisive rows {dec:.2f}")
