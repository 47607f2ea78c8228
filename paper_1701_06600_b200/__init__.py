"""paper_1701_06600_b200 — B200-native CPRAND / CPRAND-MIX hot path.

The compute lives in libcprand_b200.so (sm_100a CUDA + C++ host runtime,
C ABI in include/cprand_b200.h); this package is the Python mirror of the
reference's entry points (see api.py).
"""
from ._lib import (CprandError, CudaRuntimeError, InvalidArgument, NumericalConsistencyError,
                   UnsupportedOnDevice, LIB_PATH, EXPORTS, lib)
from .api import (Comm, DeviceTensor, LoopbackGroup, PinnedBuffer, Session, SolveOptions, SolveResult, cprand, cprand_mix,
                  cprand_premix, debug_normal_stream, default_sample_count, device_count,
                  estimate_fit, exact_fit, fit_values, gather_fibers, mix_factor, mix_tensor, mode_update,
                  skr, solve, unmix_factor, unmix_sampled_rhs, STOP_REASONS)

__all__ = [
    "CprandError", "CudaRuntimeError", "InvalidArgument", "NumericalConsistencyError",
    "UnsupportedOnDevice", "LIB_PATH", "EXPORTS", "lib", "Comm", "LoopbackGroup", "DeviceTensor", "PinnedBuffer", "Session",
    "SolveOptions", "SolveResult", "cprand", "cprand_mix", "cprand_premix",
    "debug_normal_stream", "default_sample_count", "device_count", "estimate_fit", "exact_fit",
    "fit_values", "gather_fibers", "mix_factor", "mix_tensor", "mode_update", "skr", "solve",
    "unmix_factor", "unmix_sampled_rhs", "STOP_REASONS",
]
