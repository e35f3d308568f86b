"""B200 hardware presets in the reference's ``HardwareProfile`` vocabulary.

The reference ships two workstation profiles (presets.py:72-111: RTX 4090 on
PCIe 3/4) behind ``preset(name) -> (hardware, target, draft)``.  This module
keeps that entry point and adds one B200 box per offloaded pair, with the time
fields derived from the architecture and the measured rates of this pool
(``planner_b200.B200Rates``; MEASURED_PEAKS.json) in the B200 reading of
planner.py: ``t_attn_cpu`` / ``t_ffn_gpu`` are GPU seconds per verified token
per layer, the draft times are per ``bs_draft`` chunk (re-prefill of the
context; one decode step), ``t_target_prefill_gpu`` per ``bs_prefill``
micro-batch of prompts.  ``calibrate`` re-fits them to measured runs.

The same profiles can be fed to the reference's own cost model (its
``predict_throughput`` reads the fields with its CPU-attention semantics);
bench.py reports that prediction beside the measurement.
"""
from __future__ import annotations

from .config import MIXTRAL_8X7B, MIXTRAL_8X22B, MISTRAL_7B, MISTRAL_7B_V3, TINY_DRAFT, TINY_TARGET, ModelArch
from .domain import HardwareProfile, validate_profile
from .errors import UnknownPreset
from .planner_b200 import B200Rates, resident_bytes

GiB = 1 << 30
# torch.cuda.mem_get_info total of a B200 on this pool, less the CUDA context
B200_HBM_BYTES = 178 * GiB
# pinned host DRAM a planner may spend on streamed layers (of ~2 TiB per 8-GPU box: 1/8, less headroom)
B200_HOST_BYTES = 180 * 10**9


def b200_profile(target: ModelArch, draft: ModelArch, rates: B200Rates = B200Rates(), ctx: int = 503,
                 bs_draft: int = 64, bs_prefill: int = 64, gpu_mem: int = B200_HBM_BYTES,
                 cpu_mem: int = B200_HOST_BYTES, stream_ratio: float = 1.0) -> HardwareProfile:
    """A B200 ``HardwareProfile`` for the pair at context ``ctx``.

    ``stream_ratio`` < 1 (XC4-encoded streamed units, K9): the link and the
    pinned DRAM hold ratio × the weight bytes, so the profile — which counts
    weight bytes, like the reference's ModelSpec — carries the effective
    c2g bandwidth h2d / ratio and host capacity cpu_mem / ratio."""
    eff = rates.tensor_flops * rates.tensor_efficiency
    H, dh = target.hidden, target.head_dim
    q_dim, kv_dim = target.n_head * dh, target.n_kv_head * dh
    attn = 2 * (H * q_dim + 2 * H * kv_dim + q_dim * H) + 4 * q_dim * ctx
    ffn = (2 * target.top_k * 3 * H * target.inter + 2 * H * target.n_expert) if target.is_moe else 2 * 3 * H * target.inter
    d_tok = draft.verify_flops_per_token(ctx)
    step = max(resident_bytes(draft, True) / rates.hbm_bytes_per_s, bs_draft * d_tok / eff)
    return HardwareProfile(
        gpu_mem_capacity=int(gpu_mem),
        cpu_mem_capacity=int(cpu_mem / stream_ratio),
        disk_capacity=0,
        c2g_bandwidth=rates.h2d_bytes_per_s / stream_ratio,
        g2c_bandwidth=rates.h2d_bytes_per_s,
        disk_read_bandwidth=0.0,
        disk_write_bandwidth=0.0,
        t_attn_cpu=attn / eff,
        t_ffn_gpu=ffn / eff,
        t_draft_prefill_gpu=bs_draft * ctx * draft.verify_flops_per_token(ctx // 2) / eff,
        t_draft_decode_gpu=step,
        t_target_prefill_gpu=bs_prefill * ctx * target.verify_flops_per_token(ctx // 2) / eff,
    )


# XC4 ratio the planner assumes for N(0, 0.02²) bf16 weights (measured 0.6986, BENCH_r01 codec line)
XC4_RATIO = 0.70
B200_8X22B = b200_profile(MIXTRAL_8X22B, MISTRAL_7B_V3, stream_ratio=XC4_RATIO)
B200_8X22B_RAW = b200_profile(MIXTRAL_8X22B, MISTRAL_7B_V3)
B200_8X7B = b200_profile(MIXTRAL_8X7B, MISTRAL_7B, stream_ratio=XC4_RATIO)
# configs[1]: the same box with HBM capped at 24 GiB (the reference's 4090 budget, presets.py:76)
B200_8X7B_24G = b200_profile(MIXTRAL_8X7B, MISTRAL_7B, gpu_mem=24 * GiB, bs_draft=16, stream_ratio=XC4_RATIO)
B200_TINY = b200_profile(TINY_TARGET, TINY_DRAFT, ctx=64, bs_draft=4, bs_prefill=8)

_PRESETS = {
    "b200_8x22b": (B200_8X22B, MIXTRAL_8X22B.spec(), MISTRAL_7B_V3.spec()),
    "b200_8x22b_raw": (B200_8X22B_RAW, MIXTRAL_8X22B.spec(), MISTRAL_7B_V3.spec()),
    "b200_8x7b": (B200_8X7B, MIXTRAL_8X7B.spec(), MISTRAL_7B.spec()),
    "b200_8x7b_24g": (B200_8X7B_24G, MIXTRAL_8X7B.spec(), MISTRAL_7B.spec()),
    "b200_tiny": (B200_TINY, TINY_TARGET.spec(), TINY_DRAFT.spec()),
}


def preset_names() -> list[str]:
    return sorted(_PRESETS)


def preset(name: str):
    """``(hardware, target_model, draft_model)`` for a named setup (presets.py:114-126)."""
    try:
        hw, target, draft = _PRESETS[name]
    except KeyError:
        raise UnknownPreset(f"unknown preset '{name}'; available: {', '.join(preset_names())}") from None
    return validate_profile(hw), target, draft
