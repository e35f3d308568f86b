"""B200-native offloaded speculative decoding (SpecOffload, arXiv 2505.10259).

The hot path the reference (`specpipe`) models — dual-batch speculative
decoding of an offloaded MoE target with an HBM-resident draft — executed on
sm_100a: C-ABI kernels (include/specoffload_b200.h) under a Python host layer
that keeps the reference's API shapes (Policy / Workload / ModelSpec /
HardwareProfile, SimEvent / SimResult, planner functions) and adds the
``Engine.generate`` / ``Engine.run_decoding`` entry points.
"""
import os as _os

# The engine runs up to eight streams per device (verify, draft, weight copy,
# XC4 decode, KV h2d/d2h, torch's own).  With the default 8 hardware work
# queues two of them can share a queue, and a cross-stream event wait at the
# head of one can block the other's runnable work.  One queue per stream rules
# that false dependency out (mitigation for the intermittent host-KV + refill
# stall, DESIGN.md robustness notes; cause unconfirmed).  Must be set before
# the CUDA context exists.
if "CUDA_DEVICE_MAX_CONNECTIONS" not in _os.environ:
    _os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
    import sys as _sys
    _torch = _sys.modules.get("torch")
    if _torch is not None and _torch.cuda.is_initialized():
        import warnings as _warnings
        _warnings.warn("paper_2505_10259_b200 imported after the CUDA context was created: set "
                       "CUDA_DEVICE_MAX_CONNECTIONS=32 in the environment (host-resident KV can stall with 8 "
                       "hardware work queues)", RuntimeWarning, stacklevel=2)

from .acceptance import AcceptanceModel, expected_accepted, pmf, sample_accepted
from .config import MIXTRAL_8X7B, MIXTRAL_8X22B, MISTRAL_7B, MISTRAL_7B_V3, PAIRS, TINY_DRAFT, TINY_TARGET, ModelArch
from .domain import HardwareProfile, ModelSpec, Policy, Workload, validate_profile
from .errors import SpecPipeError

__version__ = "0.1.0"

__all__ = [
    "AcceptanceModel", "expected_accepted", "pmf", "sample_accepted",
    "ModelArch", "MIXTRAL_8X7B", "MIXTRAL_8X22B", "MISTRAL_7B", "MISTRAL_7B_V3", "TINY_TARGET", "TINY_DRAFT",
    "PAIRS", "HardwareProfile", "ModelSpec", "Policy", "Workload", "validate_profile", "SpecPipeError",
    "build_engine", "Engine", "Forced",
]


def __getattr__(name):  # torch-dependent pieces load lazily
    if name == "build_engine":
        from .api import build_engine
        return build_engine
    if name in ("Engine", "Forced"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
