"""The reference's planner API, on the B200 cost model (drop-in for specpipe).

Same entry points, argument meanings, return types and errors as the
reference, so a ``specpipe`` caller swaps the import and keeps its objects
(either package's ``Policy`` / ``Workload`` / ``HardwareProfile`` /
``ModelSpec`` / ``SearchSpace`` work — only attribute access is used):

  predict_throughput  planner.py:117-158    -> CostBreakdown
  search              planner.py:161-184    -> RankedPolicies
  calibrate           planner.py:187-319    -> CalibrationResult (NonConvergent, Underdetermined)
  evaluate            costmodel.py:157-197  -> CostBreakdown
  assign_tiers        placement.py:167-257  -> PlacementPlan
  prefetch_schedule   placement.py:260-283  -> list[PrefetchOp]
  tensor_groups       placement.py:92-164

What is re-fit for B200, in the reference's
``HardwareProfile`` vocabulary so its presets, JSON files and calibration
keep working:

  * attention runs on the GPU (T4): target attention weights, embeddings and
    the paged target KV are in the mandatory GPU set; FFN layers are pinned in
    ascending order while they fit, the rest are streamed (CPU tier) or staged
    from disk.  ``t_attn_cpu`` keeps its field name but is read as the GPU
    attention-block seconds per verified token per layer, ``t_ffn_gpu`` as the
    GPU MoE seconds per verified token per layer (the verify pass carries
    bs·(n_cand+1) tokens).
  * prefetch-ahead (T5): the copy engine runs across layers and rounds, so a
    verification pass costs max(streamed bytes / c2g, compute), not
    Σ_layers max(attn, load) + ffn (costmodel.py:60-76).
  * one verification per round (T1): each of the two batches needs
    ceil(max_new / E[k]) verifications, so a group runs 2·ceil(...) rounds.
  * the draft keeps the reference's policy semantics (costmodel.py:53-57):
    ceil(bs_decoding / bs_draft) chunks of one context re-prefill plus
    n_cand − 1 decode steps, its KV sized for one bs_draft chunk.

``presets.b200_profile`` derives the time fields of a B200 box from the
architecture and the measured rates; ``calibrate`` re-fits any of them to
measured (policy, tokens/s) rows exactly as the reference does (damped
Levenberg-Marquardt in log / logit space, seeded multi-start).
"""
from __future__ import annotations

import dataclasses
import itertools
import math
from dataclasses import dataclass, field

import numpy as np

from .acceptance import AcceptanceModel, expected_accepted
from .domain import Policy
from .errors import InfeasiblePlan, InsufficientTotalMemory, NoFeasiblePolicy, NonConvergent, Underdetermined, \
    ValidationError

GPU = "GPU"
CPU = "CPU"
DISK = "DISK"
PREFILL = "prefill"
DECODING = "decoding"
KINDS = ("attention_params", "ffn_params", "kv_cache", "draft_params", "draft_kv", "other")
_KIND_ORDER = {k: i for i, k in enumerate(KINDS)}

_HW_FLOAT_FIELDS = ("c2g_bandwidth", "g2c_bandwidth", "disk_read_bandwidth", "disk_write_bandwidth", "t_attn_cpu",
                    "t_ffn_gpu", "t_draft_prefill_gpu", "t_draft_decode_gpu", "t_target_prefill_gpu")
ACCEPTANCE_PARAM = "acceptance_p"


# --------------------------------------------------------------------------- search space
@dataclass(frozen=True)
class SearchSpace:
    """Explicit policy grid (planner.py:42-83)."""

    bs_prefill_values: tuple
    bs_decoding_values: tuple
    bs_draft_values: tuple
    n_cand_values: tuple

    def __post_init__(self):
        for name in ("bs_prefill_values", "bs_decoding_values", "bs_draft_values", "n_cand_values"):
            values = tuple(getattr(self, name))
            object.__setattr__(self, name, values)
            if not values:
                raise ValidationError(f"{name} must be non-empty")
            if any(v < 1 for v in values):
                raise ValidationError(f"{name} values must be >= 1")

    def policies(self) -> list:
        """All valid grid points, in lexicographic order."""
        out = []
        for combo in itertools.product(sorted(self.bs_prefill_values), sorted(self.bs_decoding_values),
                                       sorted(self.bs_draft_values), sorted(self.n_cand_values)):
            try:
                out.append(Policy(*combo))
            except ValidationError:
                continue
        return out

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)

    @classmethod
    def from_dict(cls, data: dict) -> "SearchSpace":
        names = {f.name for f in dataclasses.fields(cls)}
        extra = sorted(set(data) - names)
        if extra:
            from .errors import ConfigError
            raise ConfigError(f"unknown key '{extra[0]}' for {cls.__name__}")
        return cls(**{k: tuple(v) for k, v in data.items()})


# the C5 sweep of SURVEY.md §8d (draft length 2-8 × batch), bs_draft = the re-prefill chunk
B200_SEARCH_SPACE = SearchSpace(bs_prefill_values=(64, 128, 256), bs_decoding_values=(32, 64, 128, 256, 384, 512, 640),
                                bs_draft_values=(16, 32, 64), n_cand_values=(2, 3, 4, 5, 6, 7, 8))


def _policies(space) -> list:
    return list(space.policies())


@dataclass(frozen=True)
class CostBreakdown:
    """Fields of costmodel.py:19-31."""

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


@dataclass
class RankedPolicies:
    entries: list

    @property
    def best(self):
        return self.entries[0][0]


@dataclass
class CalibrationResult:
    hardware: object
    workload: object
    free_params: tuple
    fitted: dict
    residuals: np.ndarray
    cost: float

    @property
    def max_abs_residual(self) -> float:
        return float(np.max(np.abs(self.residuals)))


# --------------------------------------------------------------------------- placement
@dataclass(frozen=True)
class TensorGroup:
    id: str
    kind: str
    layer: int | None
    bytes: int
    phase_relevance: str

    def sort_key(self) -> tuple:
        return (self.layer if self.layer is not None else -1, _KIND_ORDER[self.kind], self.id)


@dataclass(frozen=True)
class PrefetchOp:
    trigger: int
    group_id: str
    src: str
    dst: str


@dataclass
class PlacementPlan:
    phase: str
    assignments: dict
    groups: dict
    pinned_gpu: set
    window_bytes: int
    prefetch_ops: list = field(default_factory=list)

    def tier_bytes(self, tier: str) -> int:
        return sum(self.groups[g].bytes for g, t in self.assignments.items() if t == tier)

    def gpu_bytes_with_window(self) -> int:
        return self.tier_bytes(GPU) + self.window_bytes

    def streamed_layers(self) -> list[int]:
        """FFN layers the pass streams (CPU or DISK tier), ascending."""
        return sorted(g.layer for gid, g in self.groups.items()
                      if g.kind == "ffn_params" and self.assignments.get(gid) != GPU)

    def to_dict(self) -> dict:
        return {"phase": self.phase, "window_bytes": self.window_bytes,
                "assignments": {g: self.assignments[g] for g in sorted(self.assignments)},
                "pinned_gpu": sorted(self.pinned_gpu),
                "prefetch_ops": [{"trigger": o.trigger, "group_id": o.group_id, "from": o.src, "to": o.dst}
                                 for o in self.prefetch_ops]}


def kv_tokens(policy, workload) -> int:
    """Positions one sequence's KV holds: prompt, generated tokens and the
    n_cand + 1 verification rows of its last round."""
    return workload.l_input + workload.max_new_tokens + policy.n_cand + 1


def _workspace_bytes(policy, workload, target, draft) -> int:
    """Activation scratch of one verify pass and one re-prefill draft chunk
    when both architectures are known (planner_b200.workspace_bytes), else 0."""
    from .config import arch_for_spec
    from .planner_b200 import workspace_bytes

    ta, da = arch_for_spec(target), arch_for_spec(draft)
    if ta is None or da is None:
        return 0
    return workspace_bytes(ta, da, policy.bs_decoding, policy.n_cand, policy.bs_draft * kv_tokens(policy, workload))


def tensor_groups(target, draft, policy, workload, phase: str) -> list[TensorGroup]:
    """Every group the plan places (placement.py:92-164 ids).  B200 (T4): the
    target KV covers both interleaved batches (2·bs_decoding sequences), and
    the draft, HBM-resident through prefill and decoding, appears in both."""
    groups = []
    for layer in range(target.n_layer):
        groups.append(TensorGroup(f"target/attn/{layer:03d}", "attention_params", layer,
                                  target.attn_bytes_per_layer, "both"))
        groups.append(TensorGroup(f"target/ffn/{layer:03d}", "ffn_params", layer, target.ffn_bytes_per_layer,
                                  "both"))
    groups.append(TensorGroup("target/other", "other", None, target.other_bytes, "both"))
    seqs = min(workload.total_sequences, 2 * policy.bs_decoding)
    toks = kv_tokens(policy, workload) if phase == DECODING else workload.l_input
    groups.append(TensorGroup("target/kv", "kv_cache", None,
                              seqs * toks * target.kv_bytes_per_token_per_layer * target.n_layer, "both"))
    groups.append(TensorGroup("draft/params", "draft_params", None, draft.total_bytes(), "both"))
    groups.append(TensorGroup("draft/kv", "draft_kv", None,
                              policy.bs_draft * kv_tokens(policy, workload) * draft.kv_bytes_per_token_per_layer
                              * draft.n_layer, "decoding"))
    return sorted(groups, key=TensorGroup.sort_key)


def assign_tiers(target, draft, hw, policy, workload, phase: str) -> PlacementPlan:
    """B200 placement (placement.py:167-257 with SURVEY.md T4 / H3).

    Priorities: (1) the two-slot layer window (``window_bytes``; it also
    carries the activation workspace when the architectures are known), the
    draft weights and KV, the embeddings / LM head; (2) the target attention
    weights and the paged target KV, GPU-resident while they fit — attention
    runs on the GPU either way, so when they do not, first the attention
    weights stream with their FFN layer (the window slots grow to attention +
    FFN), then the target KV moves to pinned host DRAM with a two-slot
    one-layer window of the verified batch in HBM; (3) FFN layers pinned by
    ascending layer index while they fit; (4) the rest streamed from pinned
    host DRAM; (5) overflow to disk.  Raises InfeasiblePlan when even the
    smallest mandatory set exceeds ``hw.gpu_mem_capacity`` and
    InsufficientTotalMemory when a group fits no tier."""
    if phase not in (PREFILL, DECODING):
        raise ValueError(f"unknown phase '{phase}'")
    groups = tensor_groups(target, draft, policy, workload, phase)
    by_id = {g.id: g for g in groups}
    ws = _workspace_bytes(policy, workload, target, draft)
    base = [g for g in groups if g.kind in ("other", "draft_params", "draft_kv")
            and (phase == DECODING or g.phase_relevance != "decoding")]
    attn = [g for g in groups if g.kind == "attention_params"]
    kv = by_id["target/kv"]
    toks = kv_tokens(policy, workload) if phase == DECODING else workload.l_input
    kv_win = 2 * policy.bs_decoding * toks * target.kv_bytes_per_token_per_layer
    need = None
    for stream_attn, kv_host in ((False, False), (True, False), (True, True)):
        window = 2 * (target.ffn_bytes_per_layer + (target.attn_bytes_per_layer if stream_attn else 0)) + ws
        resident = base + ([] if stream_attn else attn) + ([] if kv_host else [kv])
        used = window + (kv_win if kv_host else 0) + sum(g.bytes for g in resident)
        need = used if need is None else min(need, used)
        if used <= hw.gpu_mem_capacity:
            break
    else:
        raise InfeasiblePlan(f"mandatory GPU-resident set ({need} B) exceeds capacity ({hw.gpu_mem_capacity} B) "
                             f"in {phase}")
    assignments = {g.id: GPU for g in resident}
    pinned = set(assignments)
    for g in groups:  # low-yield pinning, ascending layer order (placement.py:220-231)
        if g.kind == "ffn_params" and used + g.bytes <= hw.gpu_mem_capacity:
            assignments[g.id] = GPU
            pinned.add(g.id)
            used += g.bytes
    cpu_used = disk_used = 0
    for g in groups:
        if g.id in assignments:
            continue
        if cpu_used + g.bytes <= hw.cpu_mem_capacity:
            assignments[g.id] = CPU
            cpu_used += g.bytes
        elif hw.disk_capacity > 0 and disk_used + g.bytes <= hw.disk_capacity and g.kind == "ffn_params":
            assignments[g.id] = DISK
            disk_used += g.bytes
        else:
            raise InsufficientTotalMemory(f"group '{g.id}' ({g.bytes} B) does not fit in any tier")
    plan = PlacementPlan(phase, assignments, by_id, pinned, window + (kv_win if kv_host else 0))
    plan.prefetch_ops = prefetch_schedule(plan, target, phase)
    return plan


def prefetch_schedule(plan: PlacementPlan, target, phase: str) -> list[PrefetchOp]:
    """Copy order of the streamer (placement.py:260-283).  B200 (T5): a layer's
    load is issued when layer ℓ−1 starts (one layer ahead; the window's two
    slots keep the copy engine busy across layers and into the next pass), and
    a disk-tier layer is staged into DRAM two layers ahead."""
    ops: list[PrefetchOp] = []
    L = target.n_layer
    for layer in range(L):
        nxt = (layer + 1) % L  # the last layer prefetches the next pass's first one
        gid = f"target/ffn/{nxt:03d}"
        if plan.assignments.get(gid) != GPU:
            ops.append(PrefetchOp(layer, gid, CPU, GPU))
        aid = f"target/attn/{nxt:03d}"
        if plan.assignments.get(aid) == CPU:  # streamed attention travels with its layer
            ops.append(PrefetchOp(layer, aid, CPU, GPU))
        stage = f"target/ffn/{(layer + 2) % L:03d}"
        if plan.assignments.get(stage) == DISK:
            ops.append(PrefetchOp(layer, stage, DISK, CPU))
    return ops


# --------------------------------------------------------------------------- cost model
def decoding_rounds(policy, workload) -> int:
    """Rounds of one dual-batch group: one verification per round (T1), so
    each batch's ceil(max_new / E[k]) verifications take two rounds apiece."""
    e = expected_accepted(AcceptanceModel(p=workload.acceptance_p, n_cand=policy.n_cand))
    return 2 * math.ceil(workload.max_new_tokens / e)


def _streamed(target, plan: PlacementPlan) -> tuple[int, int]:
    """(bytes streamed host → HBM per pass, of which staged from disk).  A
    host-resident target KV adds the verified batch's pages (half the pool)."""
    s = d = 0
    if plan.assignments.get("target/kv") == CPU:
        s += plan.groups["target/kv"].bytes // 2
    for gid, g in plan.groups.items():
        if g.kind in ("ffn_params", "attention_params"):
            tier = plan.assignments.get(gid)
            if tier in (CPU, DISK):
                s += g.bytes
                d += g.bytes if tier == DISK else 0
    return s, d


def target_round_time(policy, workload, hw, target, plan: PlacementPlan, strict_paper_approx: bool = False) -> float:
    """One verification pass of one batch: max(link, disk, GPU compute) with
    prefetch-ahead; ``strict_paper_approx`` keeps only the transfer terms."""
    s, d = _streamed(target, plan)
    load = s / hw.c2g_bandwidth
    if d:
        load = max(load, d / hw.disk_read_bandwidth)
    if strict_paper_approx:
        return load
    tokens = policy.bs_decoding * (policy.n_cand + 1)
    return max(load, target.n_layer * tokens * (hw.t_attn_cpu + hw.t_ffn_gpu))


def draft_round_time(policy, workload, hw) -> float:
    """costmodel.py:53-57 unchanged: ceil(bs / bs_draft) re-prefill chunks."""
    chunks = math.ceil(policy.bs_decoding / policy.bs_draft)
    return chunks * (hw.t_draft_prefill_gpu + (policy.n_cand - 1) * hw.t_draft_decode_gpu)


def prefill_time(policy, workload, hw, target, plan: PlacementPlan) -> float:
    """Layer-major prefill: every streamed layer crosses the link once while
    ceil(S / bs_prefill) micro-batches run through it; the KV stays in HBM
    (no G2C offload on B200 — it is in the mandatory set)."""
    s, d = _streamed(target, plan)
    micro = math.ceil(workload.total_sequences / policy.bs_prefill)
    return max(micro * hw.t_target_prefill_gpu, s / hw.c2g_bandwidth,
               d / hw.disk_read_bandwidth if d else 0.0)


def decoding_memory(policy, workload, target, draft, hw=None) -> int:
    """Peak HBM of decoding: the GPU tier of ``assign_tiers`` plus the window."""
    hw = hw if hw is not None else _unbounded()
    return assign_tiers(target, draft, hw, policy, workload, DECODING).gpu_bytes_with_window()


def prefill_memory(policy, workload, target, draft=None, hw=None) -> int:
    hw = hw if hw is not None else _unbounded()
    draft = draft if draft is not None else target
    return assign_tiers(target, draft, hw, policy, workload, PREFILL).gpu_bytes_with_window()


def _unbounded():
    from .domain import HardwareProfile

    return HardwareProfile(1 << 62, 1 << 62, 0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0)


def evaluate(policy, workload, hw, target, draft, strict_paper_approx: bool = False,
             serial_sd: bool = False) -> CostBreakdown:
    """One dual-batch group of ``workload`` (costmodel.py:157-197 fields).
    Infeasible (mandatory set over capacity, or a group in no tier) ⇒
    throughput 0."""
    try:
        dec = assign_tiers(target, draft, hw, policy, workload, DECODING)
        pre = assign_tiers(target, draft, hw, policy, workload, PREFILL)
    except (InfeasiblePlan, InsufficientTotalMemory):
        return CostBreakdown(policy, math.inf, math.inf, 0.0, 0.0, 0, 0, 0,
                             float(workload.total_sequences * workload.max_new_tokens), 0.0, False)
    t_tgt = target_round_time(policy, workload, hw, target, dec, strict_paper_approx)
    t_drf = draft_round_time(policy, workload, hw)
    rounds = decoding_rounds(policy, workload)
    per_round = t_tgt + t_drf if serial_sd else max(t_tgt, t_drf)
    t_dec = rounds * per_round
    t_pf = prefill_time(policy, workload, hw, target, pre)
    tokens = float(workload.total_sequences * workload.max_new_tokens)
    return CostBreakdown(policy, t_pf, t_dec, t_drf, t_tgt, rounds, pre.gpu_bytes_with_window(),
                         dec.gpu_bytes_with_window(), tokens, tokens / (t_pf + t_dec), True)


def rotation_workload(workload, policy):
    """planner.py:108-114: 2·bs_decoding sequences in flight."""
    return dataclasses.replace(workload, total_sequences=2 * policy.bs_decoding)


def predict_throughput(policy, workload, hw, target, draft, strict_paper_approx: bool = False,
                       serial_sd: bool = False) -> CostBreakdown:
    """Whole-workload cost under ``policy`` (planner.py:117-158): successive
    dual-batch groups of 2·bs_decoding sequences, a partial last group paying
    for full batches, prefill once over the workload."""
    bd = evaluate(policy, rotation_workload(workload, policy), hw, target, draft, strict_paper_approx, serial_sd)
    if not bd.feasible:
        return bd
    groups = max(1, math.ceil(workload.total_sequences / (2 * policy.bs_decoding)))
    plan = assign_tiers(target, draft, hw, policy, rotation_workload(workload, policy), PREFILL)
    t_prefill = prefill_time(policy, workload, hw, target, plan)
    t_decoding = groups * bd.t_decoding
    tokens = float(workload.total_sequences * workload.max_new_tokens)
    return dataclasses.replace(bd, t_prefill=t_prefill, t_decoding=t_decoding, expected_tokens=tokens,
                               throughput=tokens / (t_prefill + t_decoding))


def search(space, workload, hw, target, draft, strict_paper_approx: bool = False) -> RankedPolicies:
    """planner.py:161-184: every grid point, infeasible dropped, ranked by
    throughput, ties broken by the policy tuple."""
    entries = []
    for policy in _policies(space):
        bd = predict_throughput(policy, workload, hw, target, draft, strict_paper_approx)
        if bd.feasible:
            entries.append((policy, bd))
    if not entries:
        raise NoFeasiblePolicy("every policy in the grid violates the memory constraint")
    entries.sort(key=lambda e: (-e[1].throughput, tuple(e[0].as_tuple())))
    return RankedPolicies(entries=entries)


def _apply(hw, workload, names, values):
    upd = {}
    for n, v in zip(names, values):
        if n == ACCEPTANCE_PARAM:
            workload = dataclasses.replace(workload, acceptance_p=float(v))
        else:
            upd[n] = float(v)
    return (dataclasses.replace(hw, **upd) if upd else hw), workload


def calibrate(observations, workload, hw_template, target, draft, free_params, residual_threshold: float = 2.0,
              n_starts: int = 8, damping: float = 0.08) -> CalibrationResult:
    """Fit hardware primitives (and optionally acceptance_p) to measured
    (policy, tokens/s) pairs — the reference's procedure (planner.py:215-319)
    over this module's B200 predict_throughput: log-space positives, logit
    acceptance, weak quadratic pull to the template, seeded multi-start
    (rng 20240501) with one start per acceptance plateau."""
    from scipy.optimize import least_squares

    free_params = tuple(free_params)
    for name in free_params:
        if name != ACCEPTANCE_PARAM and name not in _HW_FLOAT_FIELDS:
            raise ValidationError(f"'{name}' is not a calibratable parameter")
    if len(observations) < len(free_params):
        raise Underdetermined(f"{len(observations)} observations cannot identify {len(free_params)} parameters")
    measured = np.array([t for _, t in observations], dtype=np.float64)
    if np.any(measured <= 0):
        raise ValidationError("measured throughputs must be > 0")
    policies = [p for p, _ in observations]

    def decode(z):
        out = np.empty_like(z)
        for i, name in enumerate(free_params):
            zi = min(max(z[i], -60.0), 60.0)
            out[i] = 1.0 / (1.0 + math.exp(-zi)) if name == ACCEPTANCE_PARAM else math.exp(zi)
        return out

    def data_residuals(z):
        hw, wl = _apply(hw_template, workload, free_params, decode(z))
        return np.array([predict_throughput(p, wl, hw, target, draft).throughput for p in policies]) / measured - 1.0

    z0 = np.empty(len(free_params))
    for i, name in enumerate(free_params):
        if name == ACCEPTANCE_PARAM:
            p0 = min(max(workload.acceptance_p, 0.05), 0.95)
            z0[i] = math.log(p0 / (1.0 - p0))
        else:
            base = getattr(hw_template, name)
            z0[i] = math.log(base if base > 0 else 1e-3)

    def residual_fn(z):
        return np.concatenate([data_residuals(z), math.sqrt(damping) * (z - z0)])

    rng = np.random.default_rng(20240501)
    starts = [z0] + [z0 + rng.normal(0.0, 1.0, size=z0.shape) for _ in range(n_starts - 1)]
    if ACCEPTANCE_PARAM in free_params:
        ip = free_params.index(ACCEPTANCE_PARAM)
        for ps in (0.3, 0.5, 0.65, 0.75, 0.8, 0.85, 0.9, 0.95):
            z = z0.copy()
            z[ip] = math.log(ps / (1.0 - ps))
            starts.append(z)
    best = None
    for st in starts:
        sol = least_squares(residual_fn, st, method="lm", max_nfev=2000)
        if best is None or sol.cost < best.cost:
            best = sol
    values = decode(best.x)
    hw, wl = _apply(hw_template, workload, free_params, values)
    res = CalibrationResult(hw, wl, free_params, {n: float(v) for n, v in zip(free_params, values)},
                            data_residuals(best.x), float(best.cost))
    if res.max_abs_residual > residual_threshold:
        raise NonConvergent(f"max relative residual {res.max_abs_residual:.3f} exceeds threshold "
                            f"{residual_threshold}")
    return res
