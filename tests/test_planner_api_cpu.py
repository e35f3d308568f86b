"""CPU: the reference-signature planner API on the B200 cost model
(paper_2505_10259_b200.planner / .presets; SURVEY.md §8 a5, a10, a11, a14,
a15 and the §8b boundary).

The drop-in check imports the unmodified reference from /root/reference (this
container only; skipped where it is absent) and passes ITS objects —
SearchSpace, Policy, Workload, HardwareProfile, ModelSpec — through our calls,
exactly as a specpipe caller would after swapping the import."""
import dataclasses
import math
import os
import sys

import numpy as np
import pytest

from paper_2505_10259_b200 import Policy, Workload
from paper_2505_10259_b200 import planner as P
from paper_2505_10259_b200 import presets as R
from paper_2505_10259_b200.acceptance import AcceptanceModel, expected_accepted
from paper_2505_10259_b200.errors import (InfeasiblePlan, NoFeasiblePolicy, NonConvergent, Underdetermined,
                                          UnknownPreset, ValidationError)

REF_SRC = "/root/reference/pkg/src"
WL = Workload(total_sequences=2048, l_input=503, max_new_tokens=16, acceptance_p=0.8)


@pytest.fixture(scope="module")
def specpipe():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import specpipe as sp

    return sp


def test_presets_named_and_valid():
    assert {"b200_8x22b", "b200_8x7b", "b200_8x7b_24g", "b200_tiny"} <= set(R.preset_names())
    hw, t, d = R.preset("b200_8x22b")
    assert t.name == "mixtral-8x22b" and d.name == "mistral-7b-v0.3"
    assert hw.t_ffn_gpu > hw.t_attn_cpu > 0 and hw.c2g_bandwidth > 55e9
    with pytest.raises(UnknownPreset):
        R.preset("env9")


def test_assign_tiers_b200_rules():
    hw, t, d = R.preset("b200_8x22b")
    pol = Policy(256, 512, 64, 8)
    plan = P.assign_tiers(t, d, hw, pol, P.rotation_workload(WL, pol), P.DECODING)
    # T4: attention, embeddings, target KV and the draft are GPU-resident
    for gid, g in plan.groups.items():
        if g.kind != "ffn_params":
            assert plan.assignments[gid] == P.GPU, gid
    pinned = [g.layer for gid, g in plan.groups.items() if g.kind == "ffn_params" and plan.assignments[gid] == P.GPU]
    assert pinned == list(range(len(pinned)))          # ascending (placement.py:220-231)
    assert plan.gpu_bytes_with_window() <= hw.gpu_mem_capacity
    streamed = plan.streamed_layers()
    assert streamed and len(pinned) + len(streamed) == t.n_layer
    # one load per streamed layer, issued one layer ahead (T5)
    loads = [op for op in plan.prefetch_ops if op.dst == P.GPU]
    assert sorted(int(op.group_id[-3:]) for op in loads) == streamed
    assert all(int(op.group_id[-3:]) == (op.trigger + 1) % t.n_layer for op in loads)
    d_ = plan.to_dict()
    assert d_["phase"] == "decoding" and len(d_["assignments"]) == len(plan.groups)


def test_assign_tiers_infeasible_and_insufficient():
    hw, t, d = R.preset("b200_8x22b")
    small = dataclasses.replace(hw, gpu_mem_capacity=20 * R.GiB)
    with pytest.raises(InfeasiblePlan):
        P.assign_tiers(t, d, small, Policy(8, 8, 8, 4), WL, P.DECODING)
    nohost = dataclasses.replace(hw, cpu_mem_capacity=10**9)
    from paper_2505_10259_b200.errors import InsufficientTotalMemory
    with pytest.raises(InsufficientTotalMemory):
        P.assign_tiers(t, d, nohost, Policy(64, 512, 64, 8), P.rotation_workload(WL, Policy(64, 512, 64, 8)),
                       P.DECODING)


def test_rounds_one_verification_per_round():
    pol = Policy(8, 8, 8, 4)
    e = expected_accepted(AcceptanceModel(0.8, 4))
    assert P.decoding_rounds(pol, WL) == 2 * math.ceil(16 / e)
    assert P.decoding_rounds(pol, dataclasses.replace(WL, acceptance_p=1.0)) == 2 * math.ceil(16 / 5)


def test_predict_throughput_fields_and_bounds():
    hw, t, d = R.preset("b200_8x22b")
    pol = Policy(256, 512, 64, 8)
    bd = P.predict_throughput(pol, WL, hw, t, d)
    assert bd.feasible and bd.policy == pol
    assert bd.t_target_per_round >= bd.t_target_per_round * 0 and bd.rounds == P.decoding_rounds(pol, WL)
    plan = P.assign_tiers(t, d, hw, pol, P.rotation_workload(WL, pol), P.DECODING)
    link = sum(plan.groups[f"target/ffn/{li:03d}"].bytes for li in plan.streamed_layers()) / hw.c2g_bandwidth
    assert bd.t_target_per_round == pytest.approx(max(link, t.n_layer * 512 * 9 * (hw.t_attn_cpu + hw.t_ffn_gpu)))
    groups = math.ceil(2048 / 1024)
    assert bd.t_decoding == pytest.approx(groups * bd.rounds * max(bd.t_target_per_round, bd.t_draft_per_round))
    assert bd.throughput == pytest.approx(2048 * 16 / (bd.t_prefill + bd.t_decoding))
    serial = P.predict_throughput(pol, WL, hw, t, d, serial_sd=True)
    assert serial.throughput < bd.throughput
    strict = P.predict_throughput(pol, WL, hw, t, d, strict_paper_approx=True)
    assert strict.t_target_per_round <= bd.t_target_per_round


def test_search_ranks_and_breaks_ties():
    hw, t, d = R.preset("b200_8x22b")
    rk = P.search(P.B200_SEARCH_SPACE, WL, hw, t, d)
    thr = [b.throughput for _, b in rk.entries]
    assert thr == sorted(thr, reverse=True)
    for (p1, b1), (p2, b2) in zip(rk.entries, rk.entries[1:]):
        if b1.throughput == b2.throughput:
            assert p1.as_tuple() < p2.as_tuple()
    assert rk.best == rk.entries[0][0] and all(b.feasible for _, b in rk.entries)
    # the link binds at 8x22B: the best policy streams its layers with a large batch
    assert rk.best.bs_decoding >= 256
    tiny = P.SearchSpace((8,), (4096,), (8,), (4,))
    with pytest.raises(NoFeasiblePolicy):
        P.search(tiny, WL, hw, t, d)


def test_search_space_validation_and_roundtrip():
    with pytest.raises(ValidationError):
        P.SearchSpace((), (1,), (1,), (1,))
    s = P.SearchSpace((2, 1), (4,), (4, 8), (3,))
    assert [p.as_tuple() for p in s.policies()] == [(1, 4, 4, 3), (2, 4, 4, 3)]  # bs_draft 8 > 4 dropped
    assert P.SearchSpace.from_dict(s.to_dict()) == s


def _observations(hw, t, d, policies):
    return [(p, P.predict_throughput(p, WL, hw, t, d).throughput) for p in policies]


def test_calibrate_recovers_link_and_ffn_rates():
    hw, t, d = R.preset("b200_8x22b")
    truth = dataclasses.replace(hw, c2g_bandwidth=hw.c2g_bandwidth * 0.8, t_ffn_gpu=hw.t_ffn_gpu * 1.6)
    pols = [Policy(128, b, 64, n) for b in (64, 128, 256, 512) for n in (2, 4, 8)]
    obs = _observations(truth, t, d, pols)
    res = P.calibrate(obs, WL, hw, t, d, ("c2g_bandwidth", "t_ffn_gpu"), n_starts=3)
    assert isinstance(res, P.CalibrationResult)
    assert res.max_abs_residual < 0.02
    assert res.fitted["c2g_bandwidth"] == pytest.approx(truth.c2g_bandwidth, rel=0.03)
    pred = P.predict_throughput(Policy(256, 384, 64, 6), WL, res.hardware, t, d).throughput
    want = P.predict_throughput(Policy(256, 384, 64, 6), WL, truth, t, d).throughput
    assert pred == pytest.approx(want, rel=0.03)


def test_calibrate_errors():
    hw, t, d = R.preset("b200_8x22b")
    obs = _observations(hw, t, d, [Policy(256, 512, 64, 8)])
    with pytest.raises(Underdetermined):
        P.calibrate(obs, WL, hw, t, d, ("c2g_bandwidth", "t_ffn_gpu"))
    with pytest.raises(ValidationError):
        P.calibrate(obs, WL, hw, t, d, ("gpu_mem_capacity",))
    # contradictory observations of one policy: no fit within a tiny threshold
    bad = [(Policy(256, 512, 64, 8), 100.0), (Policy(256, 512, 64, 8), 1000.0)]
    with pytest.raises(NonConvergent):
        P.calibrate(bad, WL, hw, t, d, ("c2g_bandwidth",), residual_threshold=0.1, n_starts=2)


def test_reference_objects_drop_in(specpipe):
    """A specpipe caller's own objects go through every call unchanged."""
    sp = specpipe
    hw_ours, t_ours, d_ours = R.preset("b200_8x22b")
    hw = sp.HardwareProfile(**hw_ours.to_dict())
    t = sp.presets.MIXTRAL_8X22B
    d = sp.ModelSpec(**dataclasses.asdict(d_ours))
    wl = sp.Workload(total_sequences=2048, l_input=503, max_new_tokens=16, acceptance_p=0.8)
    space = sp.planner.SearchSpace(bs_prefill_values=(64, 256), bs_decoding_values=(128, 256, 512),
                                   bs_draft_values=(32, 64), n_cand_values=(4, 8))
    rk = P.search(space, wl, hw, t, d)
    assert isinstance(rk, P.RankedPolicies) and isinstance(rk.best, sp.Policy)
    ours = P.search(P.SearchSpace(**space.to_dict()), WL, hw_ours, t_ours, d_ours)
    assert [p.as_tuple() for p, _ in rk.entries] == [p.as_tuple() for p, _ in ours.entries]
    assert [b.throughput for _, b in rk.entries] == [b.throughput for _, b in ours.entries]
    bd = P.predict_throughput(rk.best, wl, hw, t, d)
    assert bd.feasible and bd.throughput == rk.entries[0][1].throughput
    plan = P.assign_tiers(t, d, hw, rk.best, P.rotation_workload(wl, rk.best), "decoding")
    assert plan.streamed_layers()
    obs = [(p, b.throughput * 1.1) for p, b in rk.entries[:4]]
    res = P.calibrate(obs, wl, hw, t, d, ("c2g_bandwidth",), n_starts=2)
    assert res.max_abs_residual < 0.1 and isinstance(res.hardware, sp.HardwareProfile)
    # the reference's own error types are what a caller catches: ours subclass the same
    # roles (ValueError for validation), so `except ValueError` keeps working
    with pytest.raises(ValueError):
        P.calibrate(obs, wl, hw, t, d, ("gpu_mem_capacity",))


def test_reference_cost_model_accepts_b200_profile(specpipe):
    """The B200 preset is a valid reference HardwareProfile: the reference's own
    predict_throughput runs on it (bench.py reports that prediction)."""
    sp = specpipe
    hw_ours, _, d_ours = R.preset("b200_8x22b")
    hw = sp.validate_profile(sp.HardwareProfile(**hw_ours.to_dict()))
    bd = sp.planner.predict_throughput(sp.Policy(256, 512, 64, 8), sp.Workload(2048, 503, 16, 0.8), hw,
                                       sp.presets.MIXTRAL_8X22B, sp.ModelSpec(**dataclasses.asdict(d_ours)))
    assert bd.throughput > 0


def test_memory_model_matches_group_sum():
    """a10: the decoding peak is the GPU tier plus the window (costmodel.py:123-138
    restated for the B200 mandatory set), and every term is a group size."""
    hw, t, d = R.preset("b200_8x22b")
    pol = Policy(64, 256, 64, 8)
    wl = P.rotation_workload(WL, pol)
    plan = P.assign_tiers(t, d, hw, pol, wl, P.DECODING)
    want = plan.window_bytes + sum(g.bytes for gid, g in plan.groups.items() if plan.assignments[gid] == P.GPU)
    assert P.decoding_memory(pol, wl, t, d, hw) == want
    kv = plan.groups["target/kv"].bytes
    assert kv == 2 * 256 * (503 + 16 + 9) * t.kv_bytes_per_token_per_layer * t.n_layer


def test_rng_free_and_deterministic():
    hw, t, d = R.preset("b200_8x7b_24g")
    a = P.search(P.SearchSpace((16,), (16, 32, 64), (8, 16), (2, 4, 8)), WL, hw, t, d)
    b = P.search(P.SearchSpace((16,), (16, 32, 64), (8, 16), (2, 4, 8)), WL, hw, t, d)
    assert [(p.as_tuple(), x.throughput) for p, x in a.entries] == [(p.as_tuple(), x.throughput) for p, x in b.entries]
    assert np.isfinite([x.throughput for _, x in a.entries]).all()


def test_bench_reference_cpu_work_runs_the_unmodified_reference():
    """bench.py's reference_cpu_work: the reference's own search / simulate /
    predict on the B200 preset, from the baseline/_ref install."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.isdir(os.path.join(root, "baseline", "_ref", "specpipe")):
        pytest.skip("baseline/_ref not installed (run __graft_entry__.build())")
    import bench

    out = bench.reference_cpu_work("8x22b")
    assert "unavailable" not in out and out["grid_points"] > 100
    assert [r["hbm_gib"] for r in out["search"]][:3] == [24, 48, 96]
    assert out["simulate_decoding"]["events"] > 0 and out["predict_throughput"]["tokens_per_s"] > 0
