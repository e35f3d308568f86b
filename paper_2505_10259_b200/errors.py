"""Error hierarchy of the B200 path.

Keeps the reference's convention — one ``SpecPipeError`` base with typed
subclasses (pkg/src/specpipe/errors.py:4-49) — so callers catching the
reference's errors keep working; adds the native-layer failures.
"""
from __future__ import annotations


class SpecPipeError(Exception):
    """Base class of every error raised by this package."""


class ValidationError(SpecPipeError, ValueError):
    """An argument violates a documented invariant."""


class NonPositiveBandwidth(ValidationError):
    pass


class NegativeLatency(ValidationError):
    pass


class ZeroGpuMemory(ValidationError):
    pass


class ConfigError(SpecPipeError, ValueError):
    pass


class UnknownPreset(SpecPipeError, KeyError):
    pass


class InsufficientTotalMemory(SpecPipeError):
    """Weights + KV do not fit in HBM + host DRAM."""


class NoFeasiblePolicy(SpecPipeError):
    pass


class Underdetermined(SpecPipeError):
    pass


class NonConvergent(SpecPipeError):
    pass


class InfeasiblePlan(SpecPipeError):
    """The HBM budget cannot hold the mandatory resident set of a plan."""


class NativeLibraryMissing(SpecPipeError, RuntimeError):
    """The sm_100a shared library has not been built (there is no fallback)."""


class NativeError(SpecPipeError, RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, message: str, status: int):
        super().__init__(message)
        self.status = status
