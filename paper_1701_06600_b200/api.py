"""Python mirror of the reference interface for the B200 path.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/cprand/): `cprand(x, r, s, opts)`
(sampling.hpp:257), `cprand_mix` (mixing.hpp:326/340), `cprand_premix`
(mixing.hpp:351/372), `SolveOptions` (solver.hpp:40-64), `SolveResult`
(solver.hpp:83-90), plus the kernel-level operators (gather_fibers, skr, ...).
Every call goes through libcprand_b200.so; numpy arrays are the host
containers (column-major matrices, tensors in storage order = Fortran order).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import Options, Result, TraceRecord, check, lib

METHODS = {"als": 0, "rand": 1, "mix": 2, "premix": 3}
TRANSFORMS = {None: -1, "fft": 0, "dct": 1, "wht": 2, "identity": 3}
INITS = {"random": 0, "hosvd": 1, "given": 2}
STOP_REASONS = ["max_iterations", "fit_stagnation", "fit_threshold", "best_fit_stall",
                "zero_tensor", "bench_complete"]


@dataclass
class SolveOptions:
    """SolveOptions (solver.hpp:40-64), reference defaults, + device fields."""
    max_iters: int = 200
    fit_tolerance: float = 1e-4
    fit_threshold: float | None = None
    rng_seed: int = 0
    init: str = "random"
    init_model: tuple | None = None  # (lambda, [factors]) for init="given"
    fit_sample_count: int = 1 << 14
    stall_limit: int = 10
    transform: str | None = None
    bench_mode: bool = False
    exhaustive_samples: bool = False
    exact_fit_trace: bool = False
    device: int = -1
    x_mutable: bool = False
    replicas: int = -1  # mode-major replicas of strided modes: -1 auto, 0 off, 1 on
    fused: int = -1  # persistent per-iteration kernel: -1 auto, 0 off
    comm: object | None = None  # Comm: slab-sharded run (tensor = this rank's slab)
    shard_total: int = 0  # with comm: global length of the last mode
    atomic_gram: bool = False  # fused CPRAND kernel: Gram via L2 fp64 atomics (not bitwise reproducible)

    def to_c(self) -> Options:
        o = Options()
        lib().cprand_options_init(C.byref(o))
        o.max_iters = self.max_iters
        o.fit_tolerance = self.fit_tolerance
        o.has_fit_threshold = int(self.fit_threshold is not None)
        o.fit_threshold = float(self.fit_threshold or 0.0)
        o.rng_seed = self.rng_seed
        o.init = INITS[self.init]
        o.fit_sample_count = self.fit_sample_count
        o.stall_limit = self.stall_limit
        o.transform = TRANSFORMS[self.transform]
        o.bench_mode = int(self.bench_mode)
        o.exhaustive_samples = int(self.exhaustive_samples)
        o.exact_fit_trace = int(self.exact_fit_trace)
        o.device = self.device
        o.x_mutable = int(self.x_mutable)
        o.replicas = self.replicas
        o.fused = self.fused
        o.atomic_gram = int(self.atomic_gram)
        if self.comm is not None:
            o.comm = self.comm.h
            o.shard_total = int(self.shard_total)
        return o


@dataclass
class SolveResult:
    """SolveResult (solver.hpp:83-90): model = (lam, factors)."""
    lam: np.ndarray
    factors: list
    trace: list = field(default_factory=list)  # (iteration, elapsed_s, fit, is_estimate, best)
    iterations: int = 0
    reason: str = "max_iterations"
    setup_seconds: float = 0.0
    total_seconds: float = 0.0
    loop_seconds_device: float = 0.0


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims(d) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(d, dtype=np.int64))


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _flat(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, order="F"))


def _ptrs(mats):
    arr = (C.c_void_p * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = m.ctypes.data
    return arr


def device_count() -> int:
    return int(lib().cprand_device_count())


def default_sample_count(r: int) -> int:
    v = lib().cprand_default_sample_count(r)
    if v < 0:
        from ._lib import InvalidArgument
        raise InvalidArgument(2, lib().cprand_last_error().decode())
    return int(v)


def _init_arrays(opts: SolveOptions, dims, r):
    if opts.init != "given" or opts.init_model is None:
        return None, None, None
    lam = np.ascontiguousarray(np.asarray(opts.init_model[0], dtype=np.float64))
    fs = [_f64(f) for f in opts.init_model[1]]
    return lam, fs, _ptrs(fs)


def _unpack(lam, fs, trace, res) -> SolveResult:
    tr = [(t.iteration, t.elapsed_seconds, t.fit, bool(t.fit_is_estimate), t.best_fit_so_far)
          for t in trace[: min(res.trace_len, len(trace))]]
    return SolveResult(lam, fs, tr, res.iterations, STOP_REASONS[res.reason], res.setup_seconds,
                       res.total_seconds, res.loop_seconds_device)


def solve(method: str, x: np.ndarray, r: int, s: int, opts: SolveOptions | None = None) -> SolveResult:
    """One-shot drop-in solve from a host tensor (cprand_solve)."""
    opts = opts or SolveOptions()
    dims = x.shape
    xf = _flat(x)
    lam = np.empty(r, dtype=np.float64)
    fs = [np.empty((d, r), dtype=np.float64, order="F") for d in dims]
    cap = opts.max_iters + 2
    trace = (TraceRecord * cap)()
    res = Result()
    il, ifs, iptr = _init_arrays(opts, dims, r)
    check(lib().cprand_solve(METHODS[method], _p(xf), _p(_dims(dims)), len(dims), C.c_int64(r),
                             C.c_int64(s), C.byref(opts.to_c()),
                             _p(il) if il is not None else None, iptr, _p(lam), _ptrs(fs),
                             trace, cap, C.byref(res)))
    return _unpack(lam, fs, trace, res)


def cprand(x, r, s, opts=None):
    """CPRAND (sampling.hpp:257)."""
    return solve("rand", x, r, s, opts)


def cprand_mix(x, r, s, opts=None):
    """CPRAND-MIX (mixing.hpp:340; default transform FFT as in the reference)."""
    return solve("mix", x, r, s, opts)


def cprand_premix(x, r, s, opts=None):
    """CPRAND-PREMIX (mixing.hpp:372; default transform DCT-II)."""
    return solve("premix", x, r, s, opts)


class DeviceTensor:
    """A tensor resident in HBM (cprand_tensor_*)."""

    def __init__(self, dims, device: int = -1):
        self.dims = tuple(int(d) for d in dims)
        self.h = C.c_void_p()
        check(lib().cprand_tensor_create(_p(_dims(self.dims)), len(self.dims), device,
                                         C.byref(self.h)))

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))

    def upload(self, x: np.ndarray) -> None:
        check(lib().cprand_tensor_upload(self.h, _p(_flat(x))))

    def upload_flat(self, flat: np.ndarray) -> None:
        assert flat.dtype == np.float64 and flat.flags.c_contiguous and flat.size == self.size
        check(lib().cprand_tensor_upload(self.h, _p(flat)))

    def download(self) -> np.ndarray:
        out = np.empty(self.size, dtype=np.float64)
        check(lib().cprand_tensor_download(self.h, _p(out)))
        return out.reshape(self.dims, order="F")

    def download_into(self, flat: np.ndarray) -> None:
        """Copy the tensor (column-major) into a caller-owned float64 buffer."""
        if flat.dtype != np.float64 or flat.size != self.size or not flat.flags["C_CONTIGUOUS"]:
            raise ValueError("download_into needs a contiguous float64 buffer of the tensor's size")
        check(lib().cprand_tensor_download(self.h, _p(flat)))

    def exact_fit(self, lam, factors) -> float:
        """exact_fit (solver.hpp:161-181) of the model (lam, factors) to this tensor."""
        lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
        fs = [_f64(f) for f in factors]
        out = C.c_double()
        check(lib().cprand_tensor_exact_fit(self.h, _p(lam), _ptrs(fs), C.c_int64(lam.size), C.byref(out)))
        return out.value

    def synth(self, r: int, collinearity: float, eta: float, seed: int, want_factors=False):
        fs = [np.empty((d, r), dtype=np.float64, order="F") for d in self.dims] if want_factors else None
        check(lib().cprand_tensor_synth(self.h, C.c_int64(r), C.c_double(collinearity),
                                        C.c_double(eta), C.c_uint64(seed),
                                        _ptrs(fs) if fs else None))
        return fs

    def mix(self, transform: str = "dct", seed: int = 0) -> list:
        """mix_tensor in place (device); returns the per-mode pass times in ms."""
        ms = np.zeros(len(self.dims), dtype=np.float64)
        check(lib().cprand_tensor_mix(self.h, TRANSFORMS[transform], C.c_uint64(seed), _p(ms)))
        return [float(v) for v in ms]

    def mix_modes(self, transform: str, seed: int, mode_begin: int, mode_end: int) -> list:
        """The passes of modes [mode_begin, mode_end) of mix_tensor, in place."""
        ms = np.zeros(len(self.dims), dtype=np.float64)
        check(lib().cprand_tensor_mix_modes(self.h, TRANSFORMS[transform], C.c_uint64(seed), mode_begin,
                                            mode_end, _p(ms)))
        return [float(v) for v in ms[mode_begin:mode_end]]

    def read_fibers(self, mode: int, idxs: np.ndarray) -> np.ndarray:
        """gather_fibers of the device tensor by plain strided copies (I_n x S)."""
        idxs = np.asfortranarray(idxs, dtype=np.int64)
        out = np.empty((self.dims[mode], idxs.shape[0]), dtype=np.float64, order="F")
        check(lib().cprand_tensor_read_fibers(self.h, mode, _p(idxs), C.c_int64(idxs.shape[0]), _p(out)))
        return out

    def synth_slab(self, r: int, collinearity: float, eta: float, seed: int, shard_total: int, comm,
                   want_factors=False):
        """This rank's slab of the BASELINE.json tensor (last dim shard_total)."""
        gd = list(self.dims[:-1]) + [int(shard_total)]
        fs = [np.empty((d, r), dtype=np.float64, order="F") for d in gd] if want_factors else None
        check(lib().cprand_tensor_synth_slab(self.h, C.c_int64(r), C.c_double(collinearity), C.c_double(eta),
                                             C.c_uint64(seed), C.c_int64(shard_total), comm.h,
                                             _ptrs(fs) if fs else None))
        return fs

    def close(self):
        if self.h:
            lib().cprand_tensor_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """Solver session over a DeviceTensor (setup once, iterate, read result)."""

    def __init__(self, method: str, t: DeviceTensor, r: int, s: int, opts: SolveOptions):
        # the model's shape: a sharded session's tensor is a slab of the last mode
        dims = t.dims
        if opts.comm is not None and opts.shard_total > 0:
            dims = tuple(dims[:-1]) + (int(opts.shard_total),)
        self.t, self.r, self.dims, self.opts = t, r, dims, opts
        self.h = C.c_void_p()
        il, ifs, iptr = _init_arrays(opts, dims, r)
        self._keep = (il, ifs)
        check(lib().cprand_session_create(METHODS[method], t.h, C.c_int64(r), C.c_int64(s),
                                          C.byref(opts.to_c()), _p(il) if il is not None else None,
                                          iptr, C.byref(self.h)))

    def run(self, n: int) -> int:
        ran = C.c_int32()
        check(lib().cprand_session_run(self.h, n, C.byref(ran)))
        return ran.value

    def enqueue(self, n: int) -> None:
        check(lib().cprand_session_enqueue(self.h, n))

    def sync(self) -> None:
        check(lib().cprand_session_sync(self.h))

    def timed_enqueue(self, n: int) -> float:
        """Enqueue n bench-mode iterations between CUDA events; returns ms."""
        ms = C.c_double()
        check(lib().cprand_session_timed_enqueue(self.h, n, C.byref(ms)))
        return ms.value

    @property
    def stream(self) -> int:
        return int(lib().cprand_session_stream(self.h) or 0)

    def set_kernel_timing(self, on: bool) -> None:
        check(lib().cprand_session_set_kernel_timing(self.h, int(on)))

    def kernel_stats(self, mode: int, kind: int = 0):
        """(launches, total ms, work) of the gather (kind 0, B_min bytes) or
        the RHS GEMM (kind 1, flops) over timed launches."""
        n, ms, b = C.c_int64(), C.c_double(), C.c_double()
        check(lib().cprand_session_kernel_stats(self.h, mode, kind, C.byref(n), C.byref(ms),
                                                C.byref(b)))
        return n.value, ms.value, b.value

    def phase_us(self) -> list:
        out = (C.c_double * 16)()
        n = C.c_int32()
        check(lib().cprand_session_phase_us(self.h, out, 16, C.byref(n)))
        return [out[i] for i in range(min(n.value, 16))]

    @property
    def fused(self) -> bool:
        """True when one persistent kernel runs each outer iteration."""
        v = C.c_int32()
        check(lib().cprand_session_fused(self.h, C.byref(v)))
        return bool(v.value)

    def gram_fallbacks(self) -> int:
        """Gram solves so far that took the pivoted-Cholesky min-norm path."""
        n = C.c_int64()
        check(lib().cprand_session_gram_fallbacks(self.h, C.byref(n)))
        return n.value

    def gather_bench(self, iters: int, replicas: bool) -> tuple:
        """Batched sampled-fiber gather of iterations 1..iters (every mode):
        (ms, useful bytes, minimum-traffic bytes)."""
        ms, bu, bm = C.c_double(), C.c_double(), C.c_double()
        check(lib().cprand_session_gather_bench(self.h, iters, int(replicas), C.byref(ms), C.byref(bu),
                                                C.byref(bm)))
        return ms.value, bu.value, bm.value

    def result(self) -> SolveResult:
        lam = np.empty(self.r, dtype=np.float64)
        fs = [np.empty((d, self.r), dtype=np.float64, order="F") for d in self.dims]
        cap = self.opts.max_iters + 2
        trace = (TraceRecord * cap)()
        res = Result()
        check(lib().cprand_session_result(self.h, _p(lam), _ptrs(fs), trace, cap, C.byref(res)))
        return _unpack(lam, fs, trace, res)

    def close(self):
        if self.h:
            lib().cprand_session_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host float64 buffer (cprand_host_alloc_pinned)."""

    def __init__(self, n: int):
        self.n = int(n)
        self.ptr = lib().cprand_host_alloc_pinned(self.n * 8)
        if not self.ptr:
            raise MemoryError(f"pinned allocation of {self.n * 8} bytes failed")
        self.array = np.ctypeslib.as_array((C.c_double * self.n).from_address(self.ptr))

    def close(self):
        if self.ptr:
            self.array = None
            lib().cprand_host_free_pinned(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- operator-level entry points (reference free functions) ------------------
def gather_fibers(x: np.ndarray, mode: int, idxs: np.ndarray) -> np.ndarray:
    """gather_fibers (tensor.hpp:188-212) -> I_n x S."""
    idxs = np.asfortranarray(np.asarray(idxs, dtype=np.int64))
    if idxs.ndim != 2 or idxs.shape[1] != x.ndim - 1:
        from ._lib import InvalidArgument
        raise InvalidArgument(2, "gather_fibers: table must have order-1 columns")
    s = idxs.shape[0]
    out = np.empty((x.shape[mode], s), dtype=np.float64, order="F")
    check(lib().cprand_gather_fibers(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, mode, _p(idxs),
                                     C.c_int64(s), _p(out)))
    return out


def skr(idxs: np.ndarray, factors, mode: int) -> np.ndarray:
    """skr (sampling.hpp:74-92) -> S x R."""
    idxs = np.asfortranarray(np.asarray(idxs, dtype=np.int64))
    fs = [_f64(f) for f in factors]
    r = fs[0].shape[1]
    out = np.empty((idxs.shape[0], r), dtype=np.float64, order="F")
    check(lib().cprand_skr(_p(idxs), C.c_int64(idxs.shape[0]), _p(_dims([f.shape[0] for f in fs])),
                           len(fs), mode, C.c_int64(r), _ptrs(fs), _p(out)))
    return out


def mode_update(x: np.ndarray, mode: int, idxs: np.ndarray, factors, lam, first_of_pass: bool,
                transform: str | None = None, mixing_seed: int = 0):
    """One fused mode step = skr + gather + sampled_update + normalize_columns
    (sampling.hpp:283-290); with transform="dct", the MIX step of
    mixing.hpp:286-296 on an already-mixed x. Returns (factor, lam, rank)."""
    idxs = np.asfortranarray(np.asarray(idxs, dtype=np.int64))
    fs = [_f64(f) for f in factors]
    r = fs[0].shape[1]
    lam = np.array(lam, dtype=np.float64)
    out = np.empty((x.shape[mode], r), dtype=np.float64, order="F")
    rank = C.c_int32()
    check(lib().cprand_mode_update(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, mode, _p(idxs),
                                   C.c_int64(idxs.shape[0]), C.c_int64(r), _ptrs(fs), _p(lam),
                                   int(first_of_pass), TRANSFORMS[transform] if transform else -1,
                                   C.c_uint64(mixing_seed), _p(out), C.byref(rank)))
    return out, lam, rank.value


def fit_values(x: np.ndarray, offsets) -> tuple:
    """Estimator entry values x[offsets] (bit-exact) and ||X|| (sampling.hpp:163-177)."""
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    vals = np.empty(off.size, dtype=np.float64)
    nrm = C.c_double()
    check(lib().cprand_fit_values(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, _p(off),
                                  C.c_int64(off.size), _p(vals), C.byref(nrm)))
    return vals, nrm.value


def estimate_fit(lam, factors, idxs, values, x_norm: float, total: int) -> float:
    """estimate_fit (sampling.hpp:191-210)."""
    fs = [_f64(f) for f in factors]
    lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
    idxs = np.asfortranarray(np.asarray(idxs, dtype=np.int64))
    vals = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    out = C.c_double()
    check(lib().cprand_estimate_fit(_p(lam), _ptrs(fs), _p(_dims([f.shape[0] for f in fs])),
                                    len(fs), C.c_int64(lam.size), _p(idxs), _p(vals),
                                    C.c_int64(vals.size), C.c_double(x_norm), C.c_int64(total),
                                    C.byref(out)))
    return out.value


def exact_fit(x: np.ndarray, lam, factors, device: int = -1) -> float:
    """exact_fit (solver.hpp:161-181) on the device from a host tensor."""
    lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
    fs = [_f64(f) for f in factors]
    out = C.c_double()
    check(lib().cprand_exact_fit(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, _p(lam), _ptrs(fs),
                                 C.c_int64(lam.size), device, C.byref(out)))
    return out.value


def mix_tensor(x: np.ndarray, kind: str, seed: int) -> np.ndarray:
    """mix_tensor<double> (mixing.hpp:130-156)."""
    out = np.empty(x.size, dtype=np.float64)
    check(lib().cprand_mix_tensor(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, TRANSFORMS[kind],
                                  C.c_uint64(seed), _p(out)))
    return out.reshape(x.shape, order="F")


def mix_factor(a, dims, kind: str, seed: int, mode: int) -> np.ndarray:
    """mix_factor<double> (mixing.hpp:159-174)."""
    a = _f64(a)
    out = np.empty_like(a, order="F")
    check(lib().cprand_mix_factor(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                  _p(_dims(dims)), len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                  mode, _p(out)))
    return out


def unmix_factor(a, dims, kind: str, seed: int, mode: int) -> np.ndarray:
    """unmix_factor (mixing.hpp:190-212), real kinds."""
    a = _f64(a)
    out = np.empty_like(a, order="F")
    check(lib().cprand_unmix_factor(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                    _p(_dims(dims)), len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                    mode, _p(out)))
    return out


def unmix_sampled_rhs(g, dims, kind: str, seed: int, mode: int) -> np.ndarray:
    """unmix_sampled_rhs<double> (mixing.hpp:218-236) on G (S x I_n)."""
    g = _f64(g)
    out = np.empty_like(g, order="F")
    check(lib().cprand_unmix_rows(_p(g), C.c_int64(g.shape[0]), C.c_int64(g.shape[1]),
                                  _p(_dims(dims)), len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                  mode, _p(out)))
    return out


def debug_normal_stream(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    check(lib().cprand_debug_normal_stream(C.c_uint64(seed), n, _p(out)))
    return out


class Comm:
    """NCCL communicator for slab-sharded runs (one process per GPU). Rank 0
    creates the id (unique_id()), every rank passes it to Comm(...).
    Comm.loopback(group, rank) makes a rank of a LoopbackGroup instead."""

    def __init__(self, uid: bytes | None, rank: int, nranks: int, device: int, _group=None):
        self.rank, self.nranks, self.device = rank, nranks, device
        self.h = C.c_void_p()
        self._group = _group  # keeps a loopback group alive
        if _group is not None:
            check(lib().cprand_comm_create_loopback(_group.h, rank, device, C.byref(self.h)))
            return
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        check(lib().cprand_comm_create(buf, rank, nranks, device, C.byref(self.h)))

    @staticmethod
    def loopback(group: "LoopbackGroup", rank: int, device: int = 0) -> "Comm":
        return Comm(None, rank, group.nranks, device, _group=group)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().cprand_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.h:
            lib().cprand_comm_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """P ranks of one process on one device (cprand_loopback_*): each rank's
    host thread creates Comm.loopback(group, rank), its slab tensor and its
    session; collectives meet at host barriers and sum in rank order. For
    running the sharded path with one GPU (tests), not for performance."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.h = C.c_void_p()
        check(lib().cprand_loopback_group_create(nranks, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().cprand_loopback_group_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

