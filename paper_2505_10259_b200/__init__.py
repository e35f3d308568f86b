"""B200-native offloaded speculative decoding (SpecOffload, arXiv 2505.10259).

The hot path the reference (`specpipe`) models — dual-batch speculative
decoding of an offloaded MoE target with an HBM-resident draft — executed on
sm_100a: C-ABI kernels (include/specoffload_b200.h) under a Python host layer
that keeps the reference's API shapes (Policy / Workload / ModelSpec /
HardwareProfile, SimEvent / SimResult, planner functions) and adds the
``Engine.generate`` / ``Engine.run_decoding`` entry points.
"""
from .acceptance import AcceptanceModel, expected_accepted, pmf, sample_accepted
from .config import MIXTRAL_8X7B, MIXTRAL_8X22B, MISTRAL_7B, MISTRAL_7B_V3, PAIRS, TINY_DRAFT, TINY_TARGET, ModelArch
from .domain import HardwareProfile, ModelSpec, Policy, Workload, validate_profile
from .errors import SpecPipeError

__version__ = "0.2.0"


def reserve_work_queues(n: int = 32) -> bool:
    """Ask the CUDA runtime for ``n`` hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS)
    before the CUDA context exists.  The engine drives up to eight streams per
    device (verify, draft, weight copy, XC4 decode, KV h2d/d2h, torch's own);
    with the default 8 queues two can share one, which serialises them.  This
    is a mitigation for the intermittent host-KV + slot-refill stall
    (DESIGN.md robustness notes; cause unconfirmed) that bench.py and the tools
    apply explicitly — importing the package changes no process state.
    Returns False (and leaves the environment alone) when a value is already
    set or the context already exists."""
    import os
    import sys

    if "CUDA_DEVICE_MAX_CONNECTIONS" in os.environ:
        return False
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        import warnings

        warnings.warn("reserve_work_queues() after the CUDA context was created has no effect", RuntimeWarning,
                      stacklevel=2)
        return False
    os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = str(int(n))
    return True

__all__ = [
    "AcceptanceModel", "expected_accepted", "pmf", "sample_accepted",
    "ModelArch", "MIXTRAL_8X7B", "MIXTRAL_8X22B", "MISTRAL_7B", "MISTRAL_7B_V3", "TINY_TARGET", "TINY_DRAFT",
    "PAIRS", "HardwareProfile", "ModelSpec", "Policy", "Workload", "validate_profile", "SpecPipeError",
    "build_engine", "Engine", "Forced", "reserve_work_queues",
]


def __getattr__(name):  # torch-dependent pieces load lazily
    if name == "build_engine":
        from .api import build_engine
        return build_engine
    if name in ("Engine", "Forced"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
