"""ctypes binding of libcprand_b200.so (the C ABI in include/cprand_b200.h).

The shared library is built in-tree by `make lib` (or __graft_entry__.build()).
There is no fallback: if the library is missing or fails to load, every call
raises. Device work only happens inside the library.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPRAND_LIB") or os.path.join(HERE, "libcprand_b200.so")

OK, ERR_INTERNAL, ERR_INVALID, ERR_NUMERICAL, ERR_CUDA, ERR_UNSUPPORTED = 0, 1, 2, 3, 4, 5


class CprandError(RuntimeError):
    """Base error; .status carries the C ABI status code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class InvalidArgument(CprandError, ValueError):
    """std::invalid_argument / std::out_of_range in the reference."""


class NumericalConsistencyError(CprandError):
    """cprand::numerical_consistency_error in the reference."""


class CudaRuntimeError(CprandError):
    pass


class UnsupportedOnDevice(CprandError, NotImplementedError):
    """Valid reference input that the B200 path does not cover (yet)."""


class Options(C.Structure):
    _fields_ = [
        ("max_iters", C.c_int32), ("fit_tolerance", C.c_double),
        ("has_fit_threshold", C.c_int32), ("fit_threshold", C.c_double),
        ("rng_seed", C.c_uint64), ("init", C.c_int32), ("fit_sample_count", C.c_int64),
        ("stall_limit", C.c_int32), ("transform", C.c_int32), ("bench_mode", C.c_int32),
        ("exhaustive_samples", C.c_int32), ("exact_fit_trace", C.c_int32),
        ("device", C.c_int32), ("x_is_device", C.c_int32), ("x_mutable", C.c_int32),
        ("comm", C.c_void_p), ("replicas", C.c_int32), ("fused", C.c_int32),
        ("shard_total", C.c_int64),
        ("atomic_gram", C.c_int32),
    ]


class TraceRecord(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("elapsed_seconds", C.c_double), ("fit", C.c_double),
                ("fit_is_estimate", C.c_int32), ("best_fit_so_far", C.c_double)]


class Result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("reason", C.c_int32), ("setup_seconds", C.c_double),
                ("total_seconds", C.c_double), ("trace_len", C.c_int32),
                ("loop_seconds_device", C.c_double)]


EXPORTS = [
    "cprand_options_init", "cprand_last_error", "cprand_device_count",
    "cprand_default_sample_count", "cprand_build_info", "cprand_solve",
    "cprand_tensor_create", "cprand_tensor_upload", "cprand_tensor_download",
    "cprand_tensor_synth", "cprand_tensor_device_ptr", "cprand_tensor_destroy",
    "cprand_session_create", "cprand_session_run", "cprand_session_enqueue",
    "cprand_session_sync", "cprand_session_timed_enqueue", "cprand_host_alloc_pinned",
    "cprand_host_free_pinned", "cprand_device_cache_release", "cprand_session_stream", "cprand_session_set_kernel_timing",
    "cprand_session_kernel_stats", "cprand_session_phase_us", "cprand_session_gram_fallbacks", "cprand_session_gather_bench",
    "cprand_tensor_exact_fit", "cprand_exact_fit",
    "cprand_session_result", "cprand_session_destroy",
    "cprand_gather_fibers", "cprand_skr", "cprand_mode_update", "cprand_fit_values",
    "cprand_estimate_fit", "cprand_mix_tensor", "cprand_mix_factor", "cprand_unmix_factor",
    "cprand_unmix_rows", "cprand_debug_normal_stream", "cprand_comm_unique_id",
    "cprand_comm_create", "cprand_comm_destroy", "cprand_tensor_synth_slab", "cprand_tensor_mix",
    "cprand_tensor_mix_modes", "cprand_tensor_read_fibers", "cprand_session_fused",
    "cprand_loopback_group_create", "cprand_loopback_group_destroy", "cprand_comm_create_loopback",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.cprand_last_error.restype = C.c_char_p
    L.cprand_build_info.restype = C.c_char_p
    L.cprand_default_sample_count.restype = C.c_int64
    L.cprand_default_sample_count.argtypes = [C.c_int64]
    L.cprand_tensor_device_ptr.restype = C.c_void_p
    L.cprand_tensor_device_ptr.argtypes = [C.c_void_p]
    L.cprand_tensor_destroy.argtypes = [C.c_void_p]
    L.cprand_tensor_destroy.restype = None
    L.cprand_session_destroy.argtypes = [C.c_void_p]
    L.cprand_session_destroy.restype = None
    L.cprand_session_stream.restype = C.c_void_p
    L.cprand_session_stream.argtypes = [C.c_void_p]
    L.cprand_comm_destroy.argtypes = [C.c_void_p]
    L.cprand_comm_destroy.restype = None
    L.cprand_loopback_group_destroy.argtypes = [C.c_void_p]
    L.cprand_loopback_group_destroy.restype = None
    L.cprand_options_init.restype = None
    L.cprand_host_alloc_pinned.restype = C.c_void_p
    L.cprand_host_alloc_pinned.argtypes = [C.c_uint64]
    L.cprand_host_free_pinned.argtypes = [C.c_void_p]
    L.cprand_host_free_pinned.restype = None
    L.cprand_device_cache_release.argtypes = []
    L.cprand_device_cache_release.restype = None
    _lib = L
    return L


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().cprand_last_error().decode(errors="replace")
    cls = {ERR_INVALID: InvalidArgument, ERR_NUMERICAL: NumericalConsistencyError,
           ERR_CUDA: CudaRuntimeError, ERR_UNSUPPORTED: UnsupportedOnDevice}.get(status, CprandError)
    raise cls(status, msg)
