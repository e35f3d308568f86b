"""B200 re-fit of the reference's placement + cost model (north-star item 4).

Reference pieces and what changes on B200:
  * assign_tiers (placement.py:167-257): mandatory GPU set = 2-slot FFN window
    + draft params + draft KV, then FFN layers pinned in ascending order while
    they fit.  Target KV and attention weights are *not* in its GPU set
    because the paper runs attention on the CPU.  Here
    attention runs on the GPU, so target attention weights, embeddings, the
    router and the paged target KV join the mandatory set, and the host DRAM
    budget caps how many layers can be streamed.
  * target_round_time (costmodel.py:60-76): n_layer·(max(attn_cpu, load) +
    ffn_gpu) assumes no prefetch-ahead (T5).  The streamer keeps the copy
    engine busy across layers and rounds, so a verification pass costs
    max(streamed_bytes / B_h2d, compute) plus a per-round host overhead.
  * decoding_rounds (costmodel.py:79-81): one verification per round (T1).
"""
from __future__ import annotations

import dataclasses
import math

from .acceptance import AcceptanceModel, expected_accepted
from .config import ModelArch
from .errors import InfeasiblePlan
from .kvcache import HostPagedKVCache, PagedKVCache
from .weights import attn_elems, ffn_offsets, unit_layout

GB = 1e9


@dataclasses.dataclass(frozen=True)
class B200Rates:
    """Measured rates of one B200 box (defaults: this pool)."""

    h2d_bytes_per_s: float = 55.5e9        # pinned H2D, measured 55.5 GB/s
    hbm_bytes_per_s: float = 6552e9        # MEASURED_PEAKS.json
    tensor_flops: float = 1375.5e12        # sustained bf16, MEASURED_PEAKS.json
    # achieved fraction of the sustained peak for a round's mixed compute (verify MoE + draft re-prefill,
    # the two streams concurrent, power-capped): 0.68 measured with the persistent GEMMs
    # (profiles/planner_sweep_r1.md, bs 440 / 48 cached: 3.3 PFLOP in 3.5 s), 0.69 after the split-K
    # decode steps and the RoPE rewrite (bs 472 / 112 cached: 2.92 PFLOP in 3.1 s).  Planned at 0.65:
    # with 0.68 the planner chose bs 480 / 90 cached, whose draft stream (3.50-3.63 s at a 1.22 GHz
    # power-capped clock) overran the 3.46 s link pass: 589.8 tok/s instead of 598 — a compute
    # overrun costs linearly, a margin only a few sequences
    # Round 2 (K5c decode-step GEMMs, fused router, 16-token steady state): bs 504 / 135 cached planned
    # at 0.65 predicted 3.52 s of compute; the draft stream measured 3.06–3.08 s at 1.35 GHz (0.74
    # effective).  Planned at 0.70: a 6 % margin under that
    tensor_efficiency: float = 0.70
    round_overhead_s: float = 0.004        # host enqueue + barrier per round
    # a draft decode step is a pass over the draft's weights: K5c's whole-launch rate at decode shapes
    # (O 14.8 µs, down 31.3 µs = 3.75 TB/s, profiles/kernels_r2.md) ≈ 0.57 of the HBM peak
    decode_hbm_efficiency: float = 0.57
    # NVLink 5 all-gather bus bandwidth per GPU (B200_PROFILING.md: 770 GB/s measured peer copy
    # per direction, 725 GB/s 8-rank all-reduce bus bandwidth); planning value with margin
    nvlink_bytes_per_s: float = 650e9
    disk_bytes_per_s: float = 12e9         # NVMe Gen5 sequential read (disk tier, §8 f4); no drive on the test box


@dataclasses.dataclass(frozen=True)
class OffloadPlan:
    bs_decoding: int
    n_cand: int
    draft_kv: str          # "cached" | "reprefill"
    bs_draft: int
    stream_layers: tuple[int, ...]
    pinned_layers: tuple[int, ...]
    n_slots: int
    hbm_bytes: dict
    host_bytes: int
    streamed_bytes_per_pass: int
    t_stream_s: float
    t_compute_s: float
    t_round_s: float
    expected_tokens_per_round: float
    tokens_per_s: float
    stream_attn: bool = False  # attention projections streamed with each layer (H3)
    stream_ratio: float = 1.0  # encoded / raw bytes of a streamed unit (K9 XC4 ≈ 0.75; 1 = raw)
    draft_cached: int = 0      # draft_kv == "mixed": sequences per batch with a persistent draft KV row
    shard_layers: tuple[int, ...] = ()  # f3 (world > 1): 1/N per GPU in HBM, NVLink all-gather each pass
    world: int = 1
    t_nvlink_s: float = 0.0
    disk_layers: tuple[int, ...] = ()   # f4: streamed layers kept on disk (subset of stream_layers)
    t_disk_s: float = 0.0
    kv_host: bool = False               # target KV in pinned host DRAM, one batch staged per layer
    split_window: bool = False  # units move as [.. gate_up | down] segments: n_slots / 2 units of window

    def as_dict(self) -> dict:
        d = dataclasses.asdict(self)
        d["stream_layers"] = len(self.stream_layers)
        d["pinned_layers"] = len(self.pinned_layers)
        d["shard_layers"] = len(self.shard_layers)
        d["disk_layers"] = len(self.disk_layers)
        return d


def resident_bytes(arch: ModelArch, include_ffn: bool) -> int:
    """HBM bytes of a model's always-resident tensors."""
    per_layer = (arch.qkv_rows * arch.hidden + arch.hidden * arch.n_head * arch.head_dim) * 2
    small = arch.small_resident_bytes()
    b = arch.embed_bytes() + arch.n_layer * per_layer + small
    if include_ffn:
        b += arch.n_layer * ffn_offsets(arch)[2]
    return b


def _act_bytes(a: ModelArch, T: int, moe: bool) -> int:
    rows = 2 * T if moe else T
    return (T * (6 * a.hidden + a.qkv_rows + 2 * a.n_head * a.head_dim) + rows * (2 * a.hidden + a.inter)) * 2


def workspace_bytes(target: ModelArch, draft: ModelArch, bs: int, n_cand: int, draft_tokens: int | None = None) -> int:
    """Scratch of one verify pass + one draft call (draft_tokens = prefill chunk size)."""
    T = bs * (n_cand + 1)
    tgt = _act_bytes(target, T, True) + T * target.vocab * 4
    dt = bs if draft_tokens is None else draft_tokens
    drf = _act_bytes(draft, dt, False) + bs * draft.vocab * 4
    return tgt + drf + (1 << 30)  # + allocator slack


def verify_flops(target: ModelArch, bs: int, n_cand: int, ctx: int) -> float:
    return bs * (n_cand + 1) * target.verify_flops_per_token(ctx)


def draft_flops(draft: ModelArch, bs: int, n_cand: int, ctx: int, draft_kv: str, draft_cached: int = 0) -> float:
    """One batch's draft work per round: n+1 cached steps per cached sequence, a
    context re-prefill + n−1 steps per re-prefilled one ("mixed": the first
    ``draft_cached`` sequences are cached)."""
    kc = bs if draft_kv == "cached" else (0 if draft_kv == "reprefill" else min(draft_cached, bs))
    cached = kc * (n_cand + 1) * draft.verify_flops_per_token(ctx)
    # a context re-prefill: every position through every layer, except that the LM head runs for
    # the last row only, and so do the last layer's attention, O projection and FFN (models.py
    # last-layer pruning: the other rows only feed that layer's K/V)
    H, q_dim = draft.hidden, draft.n_head * draft.head_dim
    lm = 2 * H * draft.vocab
    ffn = 2 * draft.top_k * 3 * H * draft.inter if draft.is_moe else 2 * 3 * H * draft.inter
    last_layer_rest = 2 * q_dim * H + ffn + 4 * q_dim * (ctx // 2)
    prefill = ctx * (draft.verify_flops_per_token(ctx // 2) - lm) + lm - (ctx - 1) * last_layer_rest
    rp = (bs - kc) * (prefill + (n_cand - 1) * draft.verify_flops_per_token(ctx))
    return cached + rp


def plan_offload(target: ModelArch, draft: ModelArch, hbm_budget: int, host_budget: int, n_cand: int,
                 acceptance_p: float, ctx_len: int, max_new: int, rates: B200Rates = B200Rates(),
                 n_slots: int = 2, bs_candidates=None, page_size: int = 32,
                 draft_kv_modes=("cached", "reprefill", "mixed"),
                 max_draft_chunk: int = 64, stream_attn_modes=(False, True), stream_ratio: float = 1.0,
                 ring_bytes: int = 0, max_pinned: int | None = None, draft_cached_candidates=None,
                 world: int = 1, allow_shards: bool = True, disk_budget: int = 0,
                 kv_host_modes=(False,), tokens_per_verify: float | None = None,
                 split_window: bool = False) -> OffloadPlan:
    """Choose bs_decoding, the draft-KV policy and the pinned / streamed split that
    maximise predicted decode tokens/s under both memory budgets.

    ``stream_ratio`` < 1: streamed units are kept XC4-encoded (K9) — host DRAM
    and the link carry ratio × the layer bytes, HBM adds the ``ring_bytes``
    staging ring and each pass pays the decode's HBM traffic (1.5 B read +
    2 B written per weight).

    ``world`` = N > 1 (per-GPU plan; every GPU runs its own batches, SURVEY.md
    §8e): host-streamed layers cost each rank 1/N of their bytes on its own
    link plus an NVLink all-gather; with ``allow_shards`` (§8 f3) layers may
    instead live 1/N per GPU in HBM and cross only NVLink — the aggregate HBM
    of N GPUs holds what one GPU's cannot.  Per layer and pass each rank
    receives (N−1)/N of the layer over NVLink either way.

    ``disk_budget`` > 0 (§8 f4, placement.py:241-243): streamed units beyond
    host DRAM (less two pinned staging units) live on disk and are read once
    per pass, so the pass also costs disk bytes / disk_bytes_per_s.

    ``kv_host_modes`` containing True lets the target KV live in host DRAM (the
    reference's CPU-resident KV, placement.py:120-130): HBM keeps a 2-slot
    window of one batch's per-layer KV, host DRAM the pool, and every pass also
    moves the verified batch's KV host → GPU (the write-back uses the other
    link direction).

    ``split_window`` (single GPU): units stream as [(attention +) gate_up | down]
    segments, one slot each, so the window costs n_slots / 2 units of HBM
    (streamer.py)."""
    if split_window and (world > 1 or n_slots % 2):
        raise ValueError("split_window needs world == 1 and an even slot count")
    # commits per verification: E[k], or the caller's steady-state figure (clamped requests,
    # acceptance.committed_per_verify) — a constant factor of every candidate's rate
    e_tok = tokens_per_verify or expected_accepted(AcceptanceModel(acceptance_p, n_cand))
    max_len = ctx_len + max_new + n_cand + 2
    draft_w = resident_bytes(draft, True)
    best = None
    cands = bs_candidates or [b for b in range(8, 2049, 4)]  # 4-sequence steps: 1 GB of 8x22B KV per step
    attn_layer = attn_elems(target) * 2
    for stream_attn, mode, kv_host in [(sa, m, kh) for sa in stream_attn_modes for m in draft_kv_modes
                                        for kh in kv_host_modes]:
        # unit = bytes of one streamed (or pinned) layer; with stream_attn the
        # attention projections travel with the FFN and leave the resident set
        layer_bytes = unit_layout(target, stream_attn)[1]
        window_units = n_slots // 2 if split_window else n_slots
        fixed = (resident_bytes(target, False) - (target.n_layer * attn_layer if stream_attn else 0)
                 + resident_bytes(draft, True) + window_units * layer_bytes
                 + (ring_bytes if stream_ratio < 1 else 0))
        host_unit = int(math.ceil(layer_bytes * stream_ratio))
        for bs in cands:
            if mode == "mixed":  # interior split points; the endpoints are the pure modes
                step = max(8, bs // 32)
                kcs = list(range(step, bs, step)) if draft_cached_candidates is None else [
                    k for k in draft_cached_candidates if 0 < k < bs]
            else:
                kcs = [bs if mode == "cached" else 0]
            for kc in kcs:
                # re-prefill scratch chunk: max_draft_chunk sequences; with host-resident
                # KV (tiny HBM budgets) the largest of it, ½ and ¼ that fits (half-size chunks
                # at full HBM were measured draft-bound: profiles/bench_r2.json r2mm)
                chunks = [bs] if mode == "cached" else sorted(
                    {min(bs, max_draft_chunk >> k) for k in range(3 if kv_host else 1)}, reverse=True)
                for bs_draft in chunks:
                    draft_rows = 2 * kc + (bs_draft if kc < bs else 0)
                    tkv_bytes = PagedKVCache.bytes_needed(target, 2 * bs, max_len, page_size)
                    kv_link = 0  # KV bytes the verified batch moves host → GPU per pass
                    host_kv = 0
                    if kv_host:
                        host_kv = tkv_bytes
                        kv_link = tkv_bytes // 2
                        tkv_bytes = HostPagedKVCache.window_bytes_needed(target, bs, max_len, page_size)
                    kv = tkv_bytes + PagedKVCache.bytes_needed(draft, draft_rows, max_len, page_size)
                    ws = workspace_bytes(target, draft, bs, n_cand, None if kc == bs else max(bs_draft * max_len, kc))
                    free = hbm_budget - fixed - kv - ws
                    if free >= 0:
                        break
                if free < 0:
                    continue
                L = target.n_layer
                cap = L if max_pinned is None else max_pinned
                eff = rates.tensor_flops * rates.tensor_efficiency
                t_base = (verify_flops(target, bs, n_cand, ctx_len)
                          + draft_flops(draft, bs, n_cand, ctx_len, "mixed", kc)) / eff
                # each draft chunk's decode steps stream the draft's weights from HBM
                # (weight-bound at these row counts).  The re-fit tensor efficiency was
                # measured with max_draft_chunk-sized chunks and absorbs their passes;
                # the smaller chunks of host-KV plans pay the extra passes explicitly
                if bs_draft < min(bs, max_draft_chunk) and kc < bs:
                    extra = -(-(bs - kc) // bs_draft) - -(-(bs - kc) // max_draft_chunk)
                    t_base += n_cand * extra * draft_w / (rates.hbm_bytes_per_s * rates.decode_hbm_efficiency)
                p0 = min(L, int(free // layer_bytes), cap)
                for n_sh in (range(0, L - p0 + 1) if (world > 1 and allow_shards) else (0,)):
                    room = free - n_sh * layer_bytes / world
                    if room < 0:
                        break
                    pinned = min(L - n_sh, int(room // layer_bytes), cap)
                    streamed = L - pinned - n_sh
                    n_disk = 0
                    if host_kv and streamed * host_unit + host_kv > host_budget:
                        continue
                    if streamed * host_unit > host_budget:
                        if disk_budget <= 0 or world > 1:
                            continue
                        n_host = max(0, (host_budget - 2 * host_unit) // host_unit)  # 2 staging units
                        n_disk = streamed - n_host
                        if n_disk * host_unit > disk_budget:
                            continue
                    S = streamed * host_unit // world + kv_link  # this rank's link bytes per pass
                    t_stream = max(S / rates.h2d_bytes_per_s, n_disk * host_unit / rates.disk_bytes_per_s)
                    t_nvl = ((streamed + n_sh) * layer_bytes * (world - 1) / world / rates.nvlink_bytes_per_s
                             if world > 1 else 0.0)
                    t_comp = t_base + (streamed * layer_bytes / world * 1.75 / rates.hbm_bytes_per_s
                                       if stream_ratio < 1 else 0.0)
                    t_round = max(t_stream, t_nvl, t_comp) + rates.round_overhead_s
                    tps = bs * e_tok / t_round
                    if best is None or tps > best[0] * 1.001:
                        best = (tps, bs, mode, bs_draft, pinned, streamed, kv, ws, S, t_stream, t_comp, t_round,
                                stream_attn, fixed, layer_bytes, kc, n_sh, t_nvl, host_unit, n_disk, kv_host)
    if best is None:
        raise InfeasiblePlan("no batch size fits the HBM and host budgets")
    (tps, bs, mode, bs_draft, pinned, streamed, kv, ws, S, t_stream, t_comp, t_round, sa, fixed, layer_bytes, kc,
     n_sh, t_nvl, host_unit, n_disk, kv_host) = best
    # pin the first layers (ascending order, placement.py:220-231); among the
    # rest, host-streamed layers are spread evenly between the sharded ones so
    # the PCIe link keeps a layer in flight while NVLink gathers the others
    pinned_l = tuple(range(pinned))
    rest = list(range(pinned, target.n_layer))
    host_pos = {int((i + 0.5) * len(rest) / streamed) for i in range(streamed)} if streamed else set()
    stream_l = tuple(li for j, li in enumerate(rest) if j in host_pos)
    shard_l = tuple(li for j, li in enumerate(rest) if j not in host_pos)
    disk_pos = {int((i + 0.5) * streamed / n_disk) for i in range(n_disk)} if n_disk else set()
    disk_l = tuple(li for j, li in enumerate(stream_l) if j in disk_pos)  # spread among the DRAM-streamed ones
    return OffloadPlan(bs, n_cand, mode, bs_draft, stream_l, pinned_l, n_slots if rest else 0,
                       {"fixed": fixed, "kv": kv, "workspace": ws, "pinned_layers": pinned * layer_bytes,
                        "shards": int(n_sh * layer_bytes / world)},
                       streamed * host_unit, S, t_stream, t_comp, t_round, bs * e_tok, tps, sa, stream_ratio,
                       kc if mode == "mixed" else 0, shard_l, world, t_nvl, disk_l,
                       n_disk * host_unit / rates.disk_bytes_per_s, kv_host, split_window)


def roofline_tokens_per_s(committed_per_round: float, streamed_bytes: int, flops: float,
                          h2d_peak: float, tensor_peak: float) -> float:
    """C / max(S / B_h2d, F / peak)."""
    t = max(streamed_bytes / h2d_peak, flops / tensor_peak)
    return committed_per_round / t if t > 0 else math.inf


# ---------------------------------------------------------------------------
# Planner API on the B200 cost model (same shapes as planner.py:117-319)
# ---------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class B200CostBreakdown:
    """Fields of the reference's CostBreakdown (costmodel.py:19-31) plus the plan."""

    policy: object
    t_prefill: float
    t_decoding: float
    t_draft_per_round: float
    t_target_per_round: float
    rounds: int
    v_prefill: int
    v_decoding: int
    expected_tokens: float
    throughput: float
    feasible: bool
    plan: OffloadPlan | None = None


def prefill_time(target: ModelArch, draft: ModelArch, n_seq: int, ctx_len: int, streamed_bytes: int,
                 rates: B200Rates) -> float:
    """Layer-major (zig-zag) prefill: every streamed layer crosses the link once
    while all prompts run through it; bound by max(stream, compute)."""
    flops = n_seq * ctx_len * (target.verify_flops_per_token(ctx_len // 2) + draft.verify_flops_per_token(ctx_len // 2))
    return max(streamed_bytes / rates.h2d_bytes_per_s, flops / (rates.tensor_flops * rates.tensor_efficiency))


def predict_throughput(policy, workload, rates: B200Rates, target: ModelArch, draft: ModelArch, hbm_budget: int,
                       host_budget: int, draft_kv_modes=("cached", "reprefill"), stream_attn_modes=(False, True),
                       include_prefill: bool = True) -> B200CostBreakdown:
    """Predicted end-to-end tokens/s of ``workload`` under ``policy`` on one B200.

    Round accounting: one verification per round, so each
    dual-batch group needs 2·ceil(max_new / E[k]) rounds; groups of
    2·bs_decoding sequences run one after another (planner.py:131-135).
    """
    p = policy
    try:
        plan = plan_offload(target, draft, hbm_budget, host_budget, p.n_cand, workload.acceptance_p,
                            workload.l_input, workload.max_new_tokens, rates, bs_candidates=[p.bs_decoding],
                            draft_kv_modes=draft_kv_modes, stream_attn_modes=stream_attn_modes,
                            max_draft_chunk=p.bs_draft)
    except InfeasiblePlan:
        return B200CostBreakdown(p, math.inf, math.inf, 0.0, 0.0, 0, 0, 0, 0.0, 0.0, False, None)
    e = expected_accepted(AcceptanceModel(workload.acceptance_p, p.n_cand))
    per_batch_rounds = math.ceil(max(workload.max_new_tokens - 1, 1) / e)
    groups = max(1, math.ceil(workload.total_sequences / (2 * p.bs_decoding)))
    rounds = 2 * per_batch_rounds * groups
    t_dec = rounds * plan.t_round_s
    t_pf = prefill_time(target, draft, workload.total_sequences, workload.l_input, plan.streamed_bytes_per_pass,
                        rates) if include_prefill else 0.0
    tokens = float(workload.total_sequences * workload.max_new_tokens)
    v_dec = sum(plan.hbm_bytes.values()) + plan.n_slots * 0
    return B200CostBreakdown(p, t_pf, t_dec, plan.t_compute_s, plan.t_stream_s, rounds, v_dec, v_dec, tokens,
                             tokens / (t_pf + t_dec), True, plan)


def search(space, workload, rates: B200Rates, target: ModelArch, draft: ModelArch, hbm_budget: int,
           host_budget: int, **kw) -> list[tuple[object, B200CostBreakdown]]:
    """Exhaustive sweep (planner.py:161-184): drop infeasible, rank by throughput,
    ties broken by the policy tuple."""
    from .errors import NoFeasiblePolicy

    entries = []
    for policy in space.policies():
        bd = predict_throughput(policy, workload, rates, target, draft, hbm_budget, host_budget, **kw)
        if bd.feasible:
            entries.append((policy, bd))
    if not entries:
        raise NoFeasiblePolicy("every policy in the grid violates the memory budgets")
    entries.sort(key=lambda e: (-e[1].throughput, e[0].as_tuple()))
    return entries


CALIBRATABLE = ("h2d_bytes_per_s", "tensor_efficiency", "round_overhead_s")


def calibrate(observations, workload, rates: B200Rates, target: ModelArch, draft: ModelArch, hbm_budget: int,
              host_budget: int, free_params=CALIBRATABLE, include_prefill: bool = False, **kw) -> B200Rates:
    """Fit the B200 rates to measured (policy, tokens/s) pairs (planner.py:215-319
    restated for this cost model): log-space least squares on relative error."""
    import numpy as np
    from scipy.optimize import least_squares

    from .errors import Underdetermined, ValidationError

    for name in free_params:
        if name not in CALIBRATABLE:
            raise ValidationError(f"'{name}' is not a calibratable rate")
    if len(observations) < len(free_params):
        raise Underdetermined(f"{len(observations)} observations cannot identify {len(free_params)} parameters")
    measured = np.array([t for _, t in observations], dtype=np.float64)
    z0 = np.log([getattr(rates, n) for n in free_params])

    def with_z(z):
        return dataclasses.replace(rates, **{n: float(np.exp(v)) for n, v in zip(free_params, z)})

    def resid(z):
        r = with_z(z)
        pred = np.array([predict_throughput(p, workload, r, target, draft, hbm_budget, host_budget,
                                            include_prefill=include_prefill, **kw).throughput
                         for p, _ in observations])
        return np.concatenate([pred / measured - 1.0, 0.05 * (z - z0)])

    sol = least_squares(resid, z0, method="lm", max_nfev=400)
    return with_z(sol.x)


def predict_round_s(rates: B200Rates, target: ModelArch, draft: ModelArch, bs: int, n_cand: int, ctx: int,
                    draft_kv: str, streamed_bytes: int, draft_cached: int = 0) -> float:
    """Round time of one measured configuration (fixed streamed split)."""
    eff = rates.tensor_flops * rates.tensor_efficiency
    comp = (verify_flops(target, bs, n_cand, ctx) + draft_flops(draft, bs, n_cand, ctx, draft_kv, draft_cached)) / eff
    return max(streamed_bytes / rates.h2d_bytes_per_s, comp) + rates.round_overhead_s


def calibrate_rounds(points, target: ModelArch, draft: ModelArch, rates: B200Rates, ctx: int,
                     free_params=("h2d_bytes_per_s", "round_overhead_s")) -> B200Rates:
    """Re-fit rates to measured rounds: points = [{policy: (bs_prefill, bs, bs_draft, n),
    draft_kv, streamed_bytes, round_s}] (tools/sweep.py output); log-space LM on
    relative round-time error with a weak pull to the prior (planner.py:251-274)."""
    import numpy as np
    from scipy.optimize import least_squares

    meas = np.array([p["round_s"] for p in points])
    z0 = np.log([getattr(rates, n) for n in free_params])

    def with_z(z):
        return dataclasses.replace(rates, **{n: float(np.exp(v)) for n, v in zip(free_params, z)})

    def resid(z):
        r = with_z(z)
        pred = np.array([predict_round_s(r, target, draft, p["policy"][1], p["policy"][3], ctx, p["draft_kv"],
                                         p["streamed_bytes"]) for p in points])
        return np.concatenate([pred / meas - 1.0, 0.01 * (z - z0)])

    return with_z(least_squares(resid, z0, method="lm", max_nfev=400).x)
