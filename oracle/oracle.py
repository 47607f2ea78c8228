"""TEST INFRASTRUCTURE — ctypes front end of the CPU oracle (oracle/liborc.so).

The oracle restates the reference CPRAND path on the CPU (see
cprand_oracle.hpp). Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs may import this module; the product never does.

Arrays follow the reference's Eigen convention: column-major (Fortran order)
float64; index tables are int64 S x (N-1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liborc.so")

METHODS = {"als": 0, "rand": 1, "mix": 2, "premix": 3}
TRANSFORMS = {None: -1, "fft": 0, "dct": 1, "wht": 2, "identity": 3}
INITS = {"random": 0, "hosvd": 1, "given": 2}
STOP_REASONS = ["max_iterations", "fit_stagnation", "fit_threshold", "best_fit_stall",
                "zero_tensor", "bench_complete"]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


class InvalidArgument(OracleError, ValueError):
    pass


class NumericalConsistencyError(OracleError):
    pass


def build() -> str:
    subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_engine_new.restype = C.c_void_p
        _lib.orc_engine_new.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        _lib.orc_engine_free.argtypes = [C.c_void_p]
        _lib.orc_default_sample_count.restype = C.c_int64
        _lib.orc_stable_norm.restype = C.c_double
        _lib.orc_tensor_norm.restype = C.c_double
        for name in ("orc_engine_next",):
            getattr(_lib, name).restype = None
        _lib.orc_philox_gaussian.restype = None
    return _lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().orc_last_error().decode()
    if status == 2:
        raise InvalidArgument(status, msg)
    if status == 3:
        raise NumericalConsistencyError(status, msg)
    raise OracleError(status, msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _i64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.int64))


def _dims(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


def _ptrs(mats):
    arr = (C.c_void_p * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = m.ctypes.data
    return arr


def _flat(x: np.ndarray) -> np.ndarray:
    """Tensor values in storage order (mode-1 fastest)."""
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, order="F"))


class Engine:
    """mt19937_64 from seeded_engine(seed, stream) (rng.hpp:19-34), or the
    raw std::mt19937_64(seed) the reference's test fixtures use."""

    def __init__(self, seed: int, stream: int = 0, raw: bool = False):
        self.h = lib().orc_engine_new(C.c_uint64(seed), C.c_uint64(stream), int(raw))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_engine_free(C.c_void_p(self.h))
            self.h = None

    def next(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        lib().orc_engine_next(C.c_void_p(self.h), C.c_int64(n), _p(out))
        return out

    def uniform_int(self, a: int, b: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        _check(lib().orc_engine_uniform_int(C.c_void_p(self.h), C.c_int64(a), C.c_int64(b),
                                            C.c_int64(n), _p(out)))
        return out

    def uniform_real(self, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        _check(lib().orc_engine_uniform_real(C.c_void_p(self.h), C.c_double(lo), C.c_double(hi),
                                             C.c_int64(n), _p(out)))
        return out

    def normal(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        _check(lib().orc_engine_normal(C.c_void_p(self.h), C.c_int64(n), _p(out)))
        return out

    def bernoulli(self, p: float, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int32)
        _check(lib().orc_engine_bernoulli(C.c_void_p(self.h), C.c_double(p), C.c_int64(n), _p(out)))
        return out

    def matrix(self, rows: int, cols: int, lo=-1.0, hi=1.0) -> np.ndarray:
        """testutil::random_matrix (test_util.hpp:21-28): column-major fill."""
        return self.uniform_real(lo, hi, rows * cols).reshape(rows, cols, order="F")


def random_tensor(dims, seed: int) -> np.ndarray:
    """testutil::random_tensor (test_util.hpp:38-41): U[-1,1) in storage order."""
    g = Engine(seed, raw=True)
    p = int(np.prod(dims))
    return g.uniform_real(-1.0, 1.0, p).reshape(tuple(dims), order="F")


def default_sample_count(r: int) -> int:
    v = lib().orc_default_sample_count(C.c_int64(r))
    if v < 0:
        raise InvalidArgument(2, lib().orc_last_error().decode())
    return int(v)


def unfold_column_index(mode: int, idx, dims) -> int:
    out = C.c_int64()
    _check(lib().orc_unfold_column_index(C.c_int64(mode), _p(_dims(idx)), _p(_dims(dims)),
                                         len(dims), C.byref(out)))
    return out.value


def draw_samples(engine: Engine, dims, mode: int, count: int) -> np.ndarray:
    out = np.empty((count, len(dims) - 1), dtype=np.int64, order="F")
    _check(lib().orc_draw_samples(C.c_void_p(engine.h), _p(_dims(dims)), len(dims),
                                  C.c_int64(mode), C.c_int64(count), _p(out)))
    return out


def sample_tables(dims, s: int, seed: int, iters: int) -> list:
    """Tables in solver order: [(it, mode)] for it in 1..iters, mode in 0..N-1,
    all from one sampling stream (sampling.hpp:269, :283-286)."""
    g = Engine(seed, 2)
    return [[draw_samples(g, dims, n, s) for n in range(len(dims))] for _ in range(iters)]


def exhaustive_samples(dims, mode: int) -> np.ndarray:
    rows = int(np.prod(dims)) // dims[mode]
    out = np.empty((rows, len(dims) - 1), dtype=np.int64, order="F")
    _check(lib().orc_exhaustive_samples(_p(_dims(dims)), len(dims), C.c_int64(mode), _p(out)))
    return out


def gather_fibers(x: np.ndarray, mode: int, idxs: np.ndarray) -> np.ndarray:
    dims = x.shape
    xf = _flat(x)
    idxs = _i64(idxs)
    s = idxs.shape[0]
    out = np.empty((dims[mode], s), dtype=np.float64, order="F")
    _check(lib().orc_gather_fibers(_p(xf), _p(_dims(dims)), len(dims), C.c_int64(mode), _p(idxs),
                                   C.c_int64(s), C.c_int64(idxs.shape[1]), _p(out)))
    return out


def skr(idxs: np.ndarray, factors, mode: int) -> np.ndarray:
    idxs = _i64(idxs)
    fs = [_f64(f) for f in factors]
    dims = [f.shape[0] for f in fs]
    r = fs[0].shape[1]
    out = np.empty((idxs.shape[0], r), dtype=np.float64, order="F")
    _check(lib().orc_skr(_p(idxs), C.c_int64(idxs.shape[0]), _p(_dims(dims)), len(dims),
                         C.c_int64(mode), C.c_int64(r), _ptrs(fs), _p(out)))
    return out


def least_squares(a, b):
    a, b = _f64(a), _f64(b)
    if b.ndim == 1:
        b = b.reshape(-1, 1, order="F")
    out = np.empty((a.shape[1], b.shape[1]), dtype=np.float64, order="F")
    rank = C.c_int()
    _check(lib().orc_least_squares(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), _p(b),
                                   C.c_int64(b.shape[1]), _p(out), C.byref(rank)))
    return out, rank.value


def sampled_update(zs, xs):
    zs, xs = _f64(zs), _f64(xs)
    s, r = zs.shape
    out = np.empty((xs.shape[0], r), dtype=np.float64, order="F")
    _check(lib().orc_sampled_update(_p(zs), _p(xs), C.c_int64(s), C.c_int64(r),
                                    C.c_int64(xs.shape[0]), C.c_int64(xs.shape[1]), _p(out)))
    return out


def normalize_columns(factors, lam, mode: int, first: bool, engine: Engine):
    fs = [_f64(f).copy(order="F") for f in factors]
    lam = np.ascontiguousarray(np.array(lam, dtype=np.float64))
    dims = [f.shape[0] for f in fs]
    _check(lib().orc_normalize_columns(_ptrs(fs), _p(_dims(dims)), len(dims),
                                       C.c_int64(lam.size), _p(lam), C.c_int64(mode), int(first),
                                       C.c_void_p(engine.h)))
    return fs, lam


def stable_norm(v) -> float:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    return lib().orc_stable_norm(_p(v), C.c_int64(v.size))


def fit_offsets(total: int, want: int, seed: int) -> np.ndarray:
    g = Engine(seed, 3)
    out = np.empty(min(total, want), dtype=np.int64)
    n = C.c_int64()
    _check(lib().orc_fit_offsets(C.c_int64(total), C.c_int64(want), C.c_void_p(g.h), _p(out),
                                 C.byref(n)))
    return out[: n.value]


@dataclass
class FitEstimator:
    idxs: np.ndarray
    x_values: np.ndarray
    x_norm: float
    total_count: int


def make_fit_estimator(x: np.ndarray, count: int, engine: Engine, stall: int = 10) -> FitEstimator:
    dims = x.shape
    xf = _flat(x)
    p = min(count, xf.size)
    idxs = np.empty((p, len(dims)), dtype=np.int64, order="F")
    vals = np.empty(p, dtype=np.float64)
    n = C.c_int64()
    nrm = C.c_double()
    _check(lib().orc_make_fit_estimator(_p(xf), _p(_dims(dims)), len(dims), C.c_int64(count),
                                        int(stall), C.c_void_p(engine.h), _p(idxs), _p(vals),
                                        C.byref(n), C.byref(nrm)))
    return FitEstimator(idxs, vals, nrm.value, xf.size)


def estimate_fit(lam, factors, est: FitEstimator) -> float:
    fs = [_f64(f) for f in factors]
    lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
    dims = [f.shape[0] for f in fs]
    out = C.c_double()
    _check(lib().orc_estimate_fit(_p(lam), _ptrs(fs), _p(_dims(dims)), len(dims),
                                  C.c_int64(lam.size), _p(_i64(est.idxs)),
                                  _p(np.ascontiguousarray(est.x_values)),
                                  C.c_int64(est.idxs.shape[0]), C.c_double(est.x_norm),
                                  C.c_int64(est.total_count), C.byref(out)))
    return out.value


def exact_fit(x: np.ndarray, lam, factors) -> float:
    fs = [_f64(f) for f in factors]
    lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
    out = C.c_double()
    _check(lib().orc_exact_fit(_p(_flat(x)), _p(_dims(x.shape)), x.ndim, _p(lam), _ptrs(fs),
                               C.c_int64(lam.size), C.byref(out)))
    return out.value


def tensor_norm(x: np.ndarray) -> float:
    return lib().orc_tensor_norm(_p(_flat(x)), _p(_dims(x.shape)), x.ndim)


def should_stop(state: dict, fit: float, iteration: int, max_iters: int, fit_threshold=None):
    best = C.c_double(state["best_fit"])
    stall = C.c_int(state["stall_count"])
    stop = C.c_int()
    reason = C.c_int()
    _check(lib().orc_should_stop(C.byref(best), C.byref(stall), int(state["stall_limit"]),
                                 C.c_double(fit), int(iteration), int(max_iters),
                                 int(fit_threshold is not None),
                                 C.c_double(fit_threshold or 0.0), C.byref(stop), C.byref(reason)))
    state["best_fit"] = best.value
    state["stall_count"] = stall.value
    return bool(stop.value), STOP_REASONS[reason.value]


def init_random(dims, r: int, seed: int):
    lam = np.empty(r, dtype=np.float64)
    fs = [np.empty((d, r), dtype=np.float64, order="F") for d in dims]
    _check(lib().orc_init_random(_p(_dims(dims)), len(dims), C.c_int64(r), C.c_uint64(seed),
                                 _p(lam), _ptrs(fs)))
    return lam, fs


class OrcOptions(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("fit_tolerance", C.c_double),
                ("has_fit_threshold", C.c_int32), ("fit_threshold", C.c_double),
                ("rng_seed", C.c_uint64), ("init", C.c_int32),
                ("fit_sample_count", C.c_int64), ("stall_limit", C.c_int32),
                ("transform", C.c_int32), ("bench_mode", C.c_int32),
                ("exhaustive_samples", C.c_int32), ("exact_fit_trace", C.c_int32)]


class OrcTrace(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("elapsed_seconds", C.c_double), ("fit", C.c_double),
                ("fit_is_estimate", C.c_int32), ("best_fit_so_far", C.c_double)]


class OrcResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("reason", C.c_int32), ("setup_seconds", C.c_double),
                ("total_seconds", C.c_double), ("trace_len", C.c_int32)]


@dataclass
class SolveOptions:
    """SolveOptions (solver.hpp:40-64) with the reference defaults."""
    max_iters: int = 200
    fit_tolerance: float = 1e-4
    fit_threshold: float | None = None
    rng_seed: int = 0
    init: str = "random"
    init_model: tuple | None = None  # (lambda, [factors])
    fit_sample_count: int = 1 << 14
    stall_limit: int = 10
    transform: str | None = None
    bench_mode: bool = False
    exhaustive_samples: bool = False
    exact_fit_trace: bool = False


@dataclass
class SolveResult:
    lam: np.ndarray
    factors: list
    trace: list = field(default_factory=list)
    iterations: int = 0
    reason: str = "max_iterations"
    setup_seconds: float = 0.0
    total_seconds: float = 0.0


def _opts(o: SolveOptions) -> OrcOptions:
    return OrcOptions(o.max_iters, o.fit_tolerance, int(o.fit_threshold is not None),
                      o.fit_threshold or 0.0, o.rng_seed, INITS[o.init], o.fit_sample_count,
                      o.stall_limit, TRANSFORMS[o.transform], int(o.bench_mode),
                      int(o.exhaustive_samples), int(o.exact_fit_trace))


def solve(method: str, x: np.ndarray, r: int, s: int, opts: SolveOptions | None = None) -> SolveResult:
    """cp_als / cprand / cprand_mix / cprand_premix on the CPU oracle."""
    opts = opts or SolveOptions()
    dims = x.shape
    xf = _flat(x)
    lam = np.empty(r, dtype=np.float64)
    fs = [np.empty((d, r), dtype=np.float64, order="F") for d in dims]
    cap = opts.max_iters + 2
    trace = (OrcTrace * cap)()
    res = OrcResult()
    il, ifs = None, None
    if opts.init_model is not None:
        il = np.ascontiguousarray(np.asarray(opts.init_model[0], dtype=np.float64))
        ifs = [_f64(f) for f in opts.init_model[1]]
    _check(lib().orc_solve(METHODS[method], _p(xf), _p(_dims(dims)), len(dims), C.c_int64(r),
                           C.c_int64(s), C.byref(_opts(opts)),
                           _p(il) if il is not None else None,
                           _ptrs(ifs) if ifs is not None else None,
                           _p(lam), _ptrs(fs), trace, cap, C.byref(res)))
    tr = [(t.iteration, t.elapsed_seconds, t.fit, bool(t.fit_is_estimate), t.best_fit_so_far)
          for t in trace[: min(res.trace_len, cap)]]
    return SolveResult(lam, fs, tr, res.iterations, STOP_REASONS[res.reason], res.setup_seconds,
                       res.total_seconds)


def cprand(x, r, s, opts=None):
    return solve("rand", x, r, s, opts)


def cprand_mix(x, r, s, opts=None):
    return solve("mix", x, r, s, opts)


def cprand_premix(x, r, s, opts=None):
    return solve("premix", x, r, s, opts)


def cp_als(x, r, opts=None):
    return solve("als", x, r, 1, opts)


def mixing_signs(dims, kind: str, seed: int) -> list:
    out = np.empty(int(sum(dims)), dtype=np.float64)
    _check(lib().orc_mixing_signs(_p(_dims(dims)), len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                  _p(out)))
    res, o = [], 0
    for d in dims:
        res.append(out[o:o + d].copy())
        o += d
    return res


def mix_tensor(x: np.ndarray, kind: str, seed: int) -> np.ndarray:
    xf = _flat(x)
    re = np.empty_like(xf)
    if kind == "fft":
        im = np.empty_like(xf)
        _check(lib().orc_mix_tensor(_p(xf), _p(_dims(x.shape)), x.ndim, 0, C.c_uint64(seed),
                                    _p(re), _p(im)))
        return (re + 1j * im).reshape(x.shape, order="F")
    _check(lib().orc_mix_tensor(_p(xf), _p(_dims(x.shape)), x.ndim, TRANSFORMS[kind],
                                C.c_uint64(seed), _p(re), None))
    return re.reshape(x.shape, order="F")


def mix_factor(a, dims, kind: str, seed: int, mode: int):
    a = _f64(a)
    re = np.empty_like(a, order="F")
    if kind == "fft":
        im = np.empty_like(a, order="F")
        _check(lib().orc_mix_factor(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                    _p(_dims(dims)), len(dims), 0, C.c_uint64(seed),
                                    C.c_int64(mode), _p(re), _p(im)))
        return re + 1j * im
    _check(lib().orc_mix_factor(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                _p(_dims(dims)), len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                C.c_int64(mode), _p(re), None))
    return re


def unmix_factor(a_hat, dims, kind: str, seed: int, mode: int):
    out = np.empty(a_hat.shape, dtype=np.float64, order="F")
    if np.iscomplexobj(a_hat):
        re, im = _f64(a_hat.real), _f64(a_hat.imag)
        _check(lib().orc_unmix_factor(_p(re), _p(im), C.c_int64(a_hat.shape[0]),
                                      C.c_int64(a_hat.shape[1]), _p(_dims(dims)), len(dims),
                                      TRANSFORMS[kind], C.c_uint64(seed), C.c_int64(mode), _p(out)))
    else:
        re = _f64(a_hat)
        _check(lib().orc_unmix_factor(_p(re), None, C.c_int64(a_hat.shape[0]),
                                      C.c_int64(a_hat.shape[1]), _p(_dims(dims)), len(dims),
                                      TRANSFORMS[kind], C.c_uint64(seed), C.c_int64(mode), _p(out)))
    return out


def unmix_sampled_rhs(g, dims, kind: str, seed: int, mode: int):
    s, n = g.shape
    if np.iscomplexobj(g):
        re, im = _f64(g.real), _f64(g.imag)
        ore = np.empty((s, n), dtype=np.float64, order="F")
        oim = np.empty((s, n), dtype=np.float64, order="F")
        _check(lib().orc_unmix_sampled_rhs(_p(re), _p(im), C.c_int64(s), C.c_int64(n),
                                           _p(_dims(dims)), len(dims), TRANSFORMS[kind],
                                           C.c_uint64(seed), C.c_int64(mode), _p(ore), _p(oim)))
        return ore + 1j * oim
    re = _f64(g)
    ore = np.empty((s, n), dtype=np.float64, order="F")
    _check(lib().orc_unmix_sampled_rhs(_p(re), None, C.c_int64(s), C.c_int64(n), _p(_dims(dims)),
                                       len(dims), TRANSFORMS[kind], C.c_uint64(seed),
                                       C.c_int64(mode), _p(ore), None))
    return ore


def transform(kind: str, v, forward: bool = True):
    """Single-vector DCT-II/III ('dct'), WHT ('wht') or unnormalized FFT ('fft')."""
    if kind == "fft":
        v = np.asarray(v, dtype=np.complex128)
        re, im = np.ascontiguousarray(v.real.copy()), np.ascontiguousarray(v.imag.copy())
        _check(lib().orc_transform(0, int(forward), _p(re), _p(im), C.c_int64(v.size)))
        return re + 1j * im
    re = np.ascontiguousarray(np.array(v, dtype=np.float64))
    _check(lib().orc_transform(TRANSFORMS[kind], int(forward), _p(re), None, C.c_int64(re.size)))
    return re


def gen_baseline(dims, r: int, collinearity: float, eta: float, seed: int, want_tensor=True):
    """BASELINE.json synthetic generator (see cprand_oracle.cpp)."""
    fs = [np.empty((d, r), dtype=np.float64, order="F") for d in dims]
    if not want_tensor:
        _check(lib().orc_gen_baseline(_p(_dims(dims)), len(dims), C.c_int64(r),
                                      C.c_double(collinearity), C.c_double(eta), C.c_uint64(seed),
                                      None, _ptrs(fs)))
        return None, fs
    x = np.empty(int(np.prod(dims)), dtype=np.float64)
    _check(lib().orc_gen_baseline(_p(_dims(dims)), len(dims), C.c_int64(r),
                                  C.c_double(collinearity), C.c_double(eta), C.c_uint64(seed),
                                  _p(x), _ptrs(fs)))
    return x.reshape(tuple(dims), order="F"), fs


def philox_gaussian(seed: int, counter0: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().orc_philox_gaussian(C.c_uint64(seed), C.c_uint64(counter0), C.c_int64(n), _p(out))
    return out


def gen_problem(dims, rank: int, collinearity: float, noise: float, seed: int):
    """Reference gen_problem (synth.hpp:60-85), restated."""
    x = np.empty(int(np.prod(dims)), dtype=np.float64)
    lam = np.empty(rank, dtype=np.float64)
    fs = [np.empty((d, rank), dtype=np.float64, order="F") for d in dims]
    _check(lib().orc_gen_problem(_p(_dims(dims)), len(dims), C.c_int64(rank),
                                 C.c_double(collinearity), C.c_double(noise), C.c_uint64(seed),
                                 _p(x), _p(lam), _ptrs(fs)))
    return x.reshape(tuple(dims), order="F"), lam, fs


def score(fa, fb) -> float:
    fa = [_f64(f) for f in fa]
    fb = [_f64(f) for f in fb]
    out = C.c_double()
    _check(lib().orc_score(_ptrs(fa), _ptrs(fb), _p(_dims([f.shape[0] for f in fa])), len(fa),
                           C.c_int64(fa[0].shape[1]), C.byref(out)))
    return out.value


def bench_mix_premixed(x_hat_flat: np.ndarray, dims, r: int, s: int, kind: str, seed: int, iters: int) -> float:
    """Seconds of `iters` bench-mode cprand_mix iterations on an already-mixed
    tensor (column-major flat buffer, read in place)."""
    out = C.c_double()
    _check(lib().orc_bench_mix_premixed(_p(x_hat_flat), _p(_dims(dims)), len(dims), C.c_int64(r), C.c_int64(s),
                                        TRANSFORMS[kind], C.c_uint64(seed), int(iters), C.byref(out)))
    return out.value

