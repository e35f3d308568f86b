"""CPU: the B200 planner (placement + cost model re-fit, SURVEY.md §8 a5–a11, a14–a15)."""
import dataclasses

import pytest

from paper_2505_10259_b200 import MIXTRAL_8X7B, MIXTRAL_8X22B, MISTRAL_7B, MISTRAL_7B_V3, Policy, Workload
from paper_2505_10259_b200.errors import InfeasiblePlan, NoFeasiblePolicy, Underdetermined
from paper_2505_10259_b200.planner_b200 import (B200Rates, calibrate, plan_offload, predict_throughput,
                                                roofline_tokens_per_s, search)
from paper_2505_10259_b200.weights import ffn_offsets

GiB = 1 << 30
RATES = B200Rates(h2d_bytes_per_s=55.5e9)


class Space:
    """Minimal SearchSpace (planner.py:42-76 shape): lexicographic valid grid."""

    def __init__(self, *axes):
        self.axes = axes

    def policies(self):
        import itertools

        out = []
        for c in itertools.product(*[sorted(a) for a in self.axes]):
            try:
                out.append(Policy(*c))
            except Exception:
                continue
        return out


def test_plan_respects_both_budgets():
    p = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9), 8, 0.8, 503, 45, RATES)
    assert sum(p.hbm_bytes.values()) <= 190e9
    assert p.host_bytes <= 191e9
    assert len(p.stream_layers) + len(p.pinned_layers) == 56
    # the pinned layers are the first ones (placement.py:220-231 ascending order)
    assert p.pinned_layers == tuple(range(len(p.pinned_layers)))
    assert p.t_round_s >= p.t_stream_s


def test_capped_8x7b_needs_attention_streaming():
    """at 24 GiB the resident set leaves no room unless attention streams."""
    with pytest.raises(InfeasiblePlan):
        plan_offload(MIXTRAL_8X7B, MISTRAL_7B, 24 * GiB, int(180e9), 4, 0.8, 503, 45, RATES, stream_attn_modes=(False,))
    p = plan_offload(MIXTRAL_8X7B, MISTRAL_7B, 24 * GiB, int(180e9), 4, 0.8, 503, 45, RATES)
    assert p.stream_attn and len(p.stream_layers) == 32
    assert sum(p.hbm_bytes.values()) <= 24 * GiB


def test_more_host_memory_never_hurts():
    a = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(150e9), 4, 0.8, 503, 45, RATES)
    b = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(250e9), 4, 0.8, 503, 45, RATES)
    assert b.tokens_per_s >= a.tokens_per_s


def test_reprefill_draft_frees_kv_for_a_bigger_batch():
    c = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9), 8, 0.8, 503, 45, RATES,
                     draft_kv_modes=("cached",))
    r = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9), 8, 0.8, 503, 45, RATES,
                     draft_kv_modes=("reprefill",))
    assert r.bs_decoding > c.bs_decoding and r.tokens_per_s > c.tokens_per_s


def test_search_ranks_and_rejects():
    wl = Workload(464, 503, 16, 0.8)
    ranked = search(Space((64,), (64, 128, 232), (32, 64), (2, 4, 8)), wl, RATES, MIXTRAL_8X22B, MISTRAL_7B_V3,
                    int(190e9), int(191e9))
    tps = [b.throughput for _, b in ranked]
    assert tps == sorted(tps, reverse=True)
    with pytest.raises(NoFeasiblePolicy):
        search(Space((64,), (64,), (32,), (4,)), wl, RATES, MIXTRAL_8X22B, MISTRAL_7B_V3, int(20e9), int(10e9))


def test_rounds_follow_one_verification_per_round():
    wl = Workload(2 * 64, 503, 17, 1.0)  # E = n+1 = 5 at p = 1 → ceil(16/5) = 4 verifies per batch
    bd = predict_throughput(Policy(64, 64, 64, 4), wl, RATES, MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9))
    assert bd.rounds == 2 * 4


def test_calibrate_recovers_link_rate():
    wl = Workload(464, 503, 16, 0.8)
    truth = dataclasses.replace(RATES, h2d_bytes_per_s=61e9)
    pols = [Policy(64, b, 32, n) for b in (64, 128, 232) for n in (2, 4, 8)]
    obs = [(p, predict_throughput(p, wl, truth, MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9),
                                  include_prefill=False).throughput) for p in pols]
    fit = calibrate(obs, wl, dataclasses.replace(RATES, h2d_bytes_per_s=40e9), MIXTRAL_8X22B, MISTRAL_7B_V3,
                    int(190e9), int(191e9), free_params=("h2d_bytes_per_s",))
    assert abs(fit.h2d_bytes_per_s / 61e9 - 1) < 0.02
    with pytest.raises(Underdetermined):
        calibrate(obs[:1], wl, RATES, MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(191e9))


def test_roofline_definition():
    # SURVEY.md §8d worked example: 270.58 GB streamed at 55 GB/s, 256·3.3616 tokens → 174.9 tok/s
    S = 56 * ffn_offsets(MIXTRAL_8X22B)[2]
    r = roofline_tokens_per_s(256 * 3.3616, S, 73e-3 * 1375.5e12, 55e9, 1375.5e12)
    assert abs(r - 174.9) < 0.5


def test_multi_gpu_plan_uses_hbm_shards():
    """§8 e/f3: at N GPUs each rank pulls 1/N of the host-streamed bytes and the
    planner moves layers into the N GPUs' aggregate HBM (1/N each) when that
    beats the host link; every layer is pinned, sharded or host-streamed."""
    one = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(193e9), 8, 0.8, 503, 45, RATES,
                       stream_ratio=0.7, ring_bytes=800 << 20, bs_candidates=list(range(64, 1025, 32)))
    prev = one.tokens_per_s
    for world in (2, 8):
        p = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(193e9), 8, 0.8, 503, 45, RATES,
                         stream_ratio=0.7, ring_bytes=800 << 20, world=world, bs_candidates=list(range(64, 1025, 32)))
        assert len(p.pinned_layers) + len(p.stream_layers) + len(p.shard_layers) == 56
        assert set(p.pinned_layers).isdisjoint(p.shard_layers) and set(p.stream_layers).isdisjoint(p.shard_layers)
        assert p.shard_layers and p.world == world
        assert sum(p.hbm_bytes.values()) <= 190e9
        assert p.t_round_s >= max(p.t_stream_s, p.t_nvlink_s, p.t_compute_s)
        assert p.tokens_per_s > prev  # per-GPU tokens/s grows: the host link stops binding alone
        prev = p.tokens_per_s
    no = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(193e9), 8, 0.8, 503, 45, RATES,
                      stream_ratio=0.7, ring_bytes=800 << 20, world=8, allow_shards=False,
                      bs_candidates=list(range(64, 1025, 32)))
    assert not no.shard_layers and no.tokens_per_s < prev


def test_disk_tier_spill():
    """§8 f4 (placement.py:241-243): with too little host DRAM the planner
    spills streamed units to disk instead of failing, and the pass pays the
    disk read time; without a disk budget the same budgets are infeasible."""
    kw = dict(stream_ratio=0.7, ring_bytes=800 << 20, bs_candidates=list(range(64, 1025, 32)))
    with pytest.raises(InfeasiblePlan):
        plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(60e9), 8, 0.8, 503, 45, RATES, **kw)
    p = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(190e9), int(60e9), 8, 0.8, 503, 45, RATES,
                     disk_budget=int(2e12), **kw)
    assert p.disk_layers and set(p.disk_layers) <= set(p.stream_layers)
    host_units = len(p.stream_layers) - len(p.disk_layers)
    assert (host_units + 2) * p.host_bytes / len(p.stream_layers) <= 60e9 * 1.001
    assert p.t_disk_s > 0 and p.t_round_s >= p.t_disk_s


def test_split_window_frees_one_unit_of_hbm_for_kv():
    """A split window ([gate_up | down] segments, one slot each) holds one
    unit instead of two: the fixed HBM drops by a unit and the planner spends
    it on the batch."""
    kw = dict(stream_ratio=0.7, ring_bytes=800 << 20, stream_attn_modes=(False,))
    whole = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(178e9), int(193e9), 8, 0.8, 503, 16, RATES, **kw)
    split = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(178e9), int(193e9), 8, 0.8, 503, 16, RATES,
                         split_window=True, **kw)
    unit = ffn_offsets(MIXTRAL_8X22B)[2]
    assert split.split_window and not whole.split_window
    assert whole.hbm_bytes["fixed"] - split.hbm_bytes["fixed"] == unit
    assert split.bs_decoding >= whole.bs_decoding and split.tokens_per_s >= whole.tokens_per_s
    with pytest.raises(ValueError):
        plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, int(178e9), int(193e9), 8, 0.8, 503, 16, RATES,
                     split_window=True, world=2)
