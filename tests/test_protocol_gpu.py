"""GPU: the model protocol of SURVEY.md §8b (``TargetModel.verify`` /
``DraftModel.draft`` over a ``SeqState``), ``generate(policy=None)`` through
the reference-signature planner, and the measured-trace / HBM contracts
(reference _checks.py invariants, costmodel.py:106-138 memory accounting)."""
import dataclasses

import numpy as np
import pytest
import torch

from _trace_checks import assert_causality, assert_dual_batch_overlap, assert_resource_exclusive
from oracle import accept_ref, decode_ref, tiny
from paper_2505_10259_b200 import MIXTRAL_8X22B, MISTRAL_7B_V3, TINY_DRAFT, TINY_TARGET, Policy, Workload, native
from paper_2505_10259_b200.api import build_engine
from paper_2505_10259_b200.engine import Forced
from paper_2505_10259_b200.models import SeqState
from paper_2505_10259_b200.trace import export_trace, parse_trace

pytestmark = pytest.mark.gpu
CANON = "canonical"


@pytest.fixture(scope="module")
def pair():
    return tiny.weights()


def _prefilled(tw, dw, prompts, max_new, n_cand, arith=CANON):
    eng = build_engine(TINY_TARGET, TINY_DRAFT, tw, dw, stream_layers={1, 3}, codec="xc4", arith=arith)
    S = len(prompts)
    s = eng.new_session(S, S, max(len(p) for p in prompts) + max_new + n_cand + 2, n_cand, draft_kv="cached")
    eng.prefill(s, prompts, max_new)
    tstate = SeqState(s.tkv, np.arange(S), s.ctx, s.t_last, eng.tgt_stream)
    dstate = SeqState(s.dkv, s.drow[:S], s.ctx, s.t_last, eng.drf_stream)
    return eng, s, tstate, dstate


@pytest.mark.parametrize("n_cand,bs_draft", [(4, 8), (3, 3)])
def test_protocol_loop_is_bit_exact_to_the_oracle(pair, n_cand, bs_draft):
    """A caller-written speculative loop over the protocol — draft, verify,
    accept/reject (K7), advance — in the parity mode: committed tokens EQUAL
    the canonical oracle's (north star: bit-exact accepted tokens)."""
    tw, dw = pair
    prompts = tiny.prompts(8, seed=5)
    max_new = 12
    eng, s, ts, ds = _prefilled(tw, dw, prompts, max_new, n_cand)
    out = [list(o) for o in s.out]
    dev = eng.device
    while min(len(o) for o in out) < max_new:
        drafts = eng.draft.draft(ds, n_cand, bs_draft)
        assert drafts.shape == (8, n_cand) and drafts.dtype == torch.int32
        torch.cuda.synchronize()
        logits = eng.target.verify(ts, drafts)
        assert logits.shape == (8, n_cand + 1, TINY_TARGET.vocab) and logits.dtype == torch.float32
        rem = torch.tensor([max_new - len(o) for o in out], dtype=torch.int32, device=dev)
        tok = torch.empty((8, n_cand + 1), dtype=torch.int32, device=dev)
        cnt = torch.empty(8, dtype=torch.int32, device=dev)
        native.accept_greedy(drafts, logits, rem, tok, cnt, stream=eng.tgt_stream)
        torch.cuda.synchronize()
        tok_h, cnt_h = tok.cpu().numpy(), cnt.cpu().numpy()
        # the accept kernel is the oracle's decision on the same logits
        want_t, want_c = accept_ref.accept_greedy(drafts.cpu().numpy(), logits.cpu().numpy(), rem.cpu().numpy())
        assert (cnt_h == want_c).all() and all((tok_h[i, :c] == want_t[i, :c]).all() for i, c in enumerate(cnt_h))
        for i, c in enumerate(cnt_h):
            out[i].extend(int(x) for x in tok_h[i, :c])
        ts.advance(cnt_h, tok_h)
        ds.advance(cnt_h, tok_h)
    want, _ = decode_ref.generate(tiny.TARGET, tw, tiny.DRAFT, dw, prompts, max_new, n_cand, 8, arith=CANON)
    assert out == want


def test_draft_sampling_returns_distributions(pair):
    tw, dw = pair
    prompts = tiny.prompts(4, seed=9)
    eng, s, ts, ds = _prefilled(tw, dw, prompts, 8, 3)
    u = np.random.default_rng(0).random((4, 3)).astype(np.float32)
    tok, probs = eng.draft.draft(ds, 3, 2, uniforms=u)
    torch.cuda.synchronize()
    assert probs.shape == (4, 3, TINY_DRAFT.vocab)
    p = probs.cpu().numpy()
    np.testing.assert_allclose(p.sum(-1), 1.0, atol=1e-4)
    t = tok.cpu().numpy()
    assert all(p[i, j, t[i, j]] > 0 for i in range(4) for j in range(3))


def test_generate_without_policy_plans_and_matches_oracle(pair):
    """generate(policy=None) calls planner.search (planner.py:161-184) on the
    device's B200 profile; the chosen policy changes rounds, not tokens."""
    tw, dw = pair
    prompts = tiny.prompts(8, seed=3)
    eng = build_engine(TINY_TARGET, TINY_DRAFT, tw, dw, stream_layers={1, 3}, codec="xc4", arith=CANON)
    got = eng.generate(prompts, 12)
    pol = eng.last_policy
    assert isinstance(pol, Policy) and 2 * pol.bs_decoding >= 8
    want, _ = decode_ref.generate(tiny.TARGET, tw, tiny.DRAFT, dw, prompts, 12, pol.n_cand, pol.bs_decoding,
                                  arith=CANON)
    assert got == want


@pytest.mark.parametrize("split", [False, True])
def test_measured_trace_invariants_8x22b_shapes(split):
    """The reference's three trace invariants (_checks.py:7-52) on a measured
    trace at Mixtral-8x22B layer shapes (3 layers, 2 streamed XC4 units) with
    a 2-layer Mistral-7B draft; plus the json/csv round trip of that trace.
    ``split``: the units move as [gate_up | down] segments, each its own XC4
    unit (16 + 8 frames)."""
    t = dataclasses.replace(MIXTRAL_8X22B, n_layer=3)
    d = dataclasses.replace(MISTRAL_7B_V3, n_layer=2)
    eng = build_engine(t, d, stream_layers={1, 2}, codec="xc4", trace=True, split_window=split)
    if split:
        st = eng.target.streamer
        assert [st.frames[(1, sg)] for sg in (0, 1)] == [(0, 16), (0, 8)]  # gate_up | down, own XC4 units
    res = eng.run_decoding(Policy(32, 16, 16, 4), Workload(32, 128, 12, 0.8), acceptance=Forced(0.8),
                           max_rounds=6)
    assert res.rounds_executed == 6 and res.tokens_generated > 0
    assert_resource_exclusive(res.trace)
    assert assert_causality(res.trace) >= 2 * 6  # every streamed layer's ffn_gpu after its load, every round
    assert_dual_batch_overlap(res.trace)
    loads = [e for e in res.trace if e.label == "ffn_load" and e.round is not None]
    assert {e.layer for e in loads} == {1, 2}
    for fmt in ("json", "csv"):
        back = parse_trace(export_trace(res, fmt), fmt)
        assert len(back.trace) == len(res.trace)
        assert_causality(back.trace)


@pytest.mark.parametrize("split", [False, True])
def test_hbm_contract_capped_plan(split):
    """a10: the measured allocator peak of a plan-built engine at the configs[1]
    cap (24 GiB, 8x7B-shaped, 4 layers) stays within the plan's hbm_bytes —
    with the whole window and with the split window the plan charges one unit for."""
    from paper_2505_10259_b200 import MIXTRAL_8X7B, MISTRAL_7B
    from paper_2505_10259_b200.planner_b200 import B200Rates, plan_offload

    t = dataclasses.replace(MIXTRAL_8X7B, n_layer=4)
    d = dataclasses.replace(MISTRAL_7B, n_layer=4)
    cap = 12 * 2**30
    n_cand, ctx, max_new = 4, 256, 20
    plan = plan_offload(t, d, cap, int(40e9), n_cand, 0.8, ctx, max_new, B200Rates(), bs_candidates=[32, 64],
                        kv_host_modes=(False,), draft_kv_modes=("cached",), split_window=split)
    assert plan.split_window == split
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated()
    eng = build_engine(t, d, stream_layers=set(plan.stream_layers), stream_attn=plan.stream_attn, trace=False,
                       split_window=plan.split_window)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()  # decoding peak: weights + window + KV + workspaces (not init scratch)
    S = 2 * plan.bs_decoding
    s = eng.new_session(S, plan.bs_decoding, ctx + max_new + n_cand + 2, n_cand, forced_p=0.8,
                        bs_draft=plan.bs_draft, draft_kv=plan.draft_kv)
    eng.synthetic_context(s, ctx, max_new)
    eng.first_draft(s)
    for _ in range(4):
        eng.round(s)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    planned = sum(plan.hbm_bytes.values())
    assert peak <= planned, (peak, plan.hbm_bytes)
