"""The sampled least-squares step across conditioning (kr_linalg.hpp:105-118).

The reference solves min ||Z_S A^T - X_S^T|| with Eigen's column-pivoted
Householder QR (rank threshold max(S,R) eps on |R_kk| / max pivot) and the
complete orthogonal decomposition when that rank is short. The device solves
the normal equations while every Gauss-Jordan pivot of the Gram exceeds
kNeTol = 1e-6 of its largest diagonal and otherwise runs the same pivoted QR
/ COD on the device (qr.cuh). These tests drive Z_S through the band where
the normal equations would lose the reference's answer:

* near-collinear factor columns give cond(Z_S) from 1e3 to 1e11 on a
  consistent system (the tensor is built from the same factors, so the exact
  solution is known and both QR solutions agree to ~cond * eps);
* cond(Z_S) ~ 1e14 and exactly duplicated / zero columns make the reference
  rank deficient: the device must return the same minimum-norm solution;
* every execution path: the operator-level chain (cprand_mode_update), the
  multi-kernel session chain, the persistent CPRAND kernel and the
  persistent CPRAND-MIX kernel.

Tolerances: relative Frobenius difference of the normalized factor below
max(1e-10, 200 * cond(Z_S) * eps) for full-rank systems, 1e-8 for the
rank-deficient minimum-norm solutions.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def pb():
    import paper_1701_06600_b200 as pb
    assert pb.device_count() > 0, "GPU tests need a visible CUDA device"
    return pb


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def collinear_factors(g, dims, r, delta, zero_col=None):
    """Random factors whose last two columns differ by delta (relative) in
    every mode; optionally one exactly zero column in mode 1."""
    fs = []
    for d in dims:
        f = g.matrix(d, r)
        f[:, r - 1] = f[:, r - 2] + delta * g.matrix(d, 1)[:, 0]
        fs.append(np.asfortranarray(f))
    if zero_col is not None:
        fs[1][:, zero_col] = 0.0
    return fs


def model_tensor(lam, fs):
    x = np.einsum("r,ir,jr,kr->ijk", lam, *fs)
    return np.asfortranarray(x)


def oracle_update(orc, x, mode, idx, fs, lam, first, mix=None, seed=0):
    dims = x.shape
    if mix is None:
        zs = orc.skr(idx, fs, mode)
        a = orc.sampled_update(zs, orc.gather_fibers(x, mode, idx))
    else:
        xh = orc.mix_tensor(x, mix, seed)
        mixed = [orc.mix_factor(f, dims, mix, seed, m) for m, f in enumerate(fs)]
        zs = orc.skr(idx, mixed, mode)
        rhs = orc.unmix_sampled_rhs(np.asfortranarray(orc.gather_fibers(xh, mode, idx).T), dims, mix, seed, mode)
        sol, _ = orc.least_squares(zs, rhs)
        a = np.asfortranarray(sol.T)
    f2 = list(fs)
    f2[mode] = a
    want, wlam = orc.normalize_columns(f2, lam, mode, first, orc.Engine(seed, 8))
    return want[mode], wlam, zs


def tol_for(zs):
    return max(1e-10, 200.0 * np.linalg.cond(zs) * EPS)


DELTAS = [1e-3, 1e-5, 1e-7, 1e-9, 1e-11]


@pytest.mark.parametrize("delta", DELTAS)
def test_operator_chain_conditioning_band(pb, orc, delta):
    """cprand_mode_update (Z, Gram, Gauss-Jordan / QR, RHS, apply) on a
    consistent system with cond(Z_S) ~ 1 / delta."""
    dims, r, s = (40, 30, 20), 6, 150
    g = orc.Engine(4100, raw=True)
    fs = collinear_factors(g, dims, r, delta)
    x = model_tensor(np.ones(r), fs)
    lam = np.ones(r)
    idx = orc.draw_samples(g, dims, 0, s)
    want, wlam, zs = oracle_update(orc, x, 0, idx, fs, lam, True)
    got, glam, rank = pb.mode_update(x, 0, idx, fs, lam, True)
    assert rank == r
    d = rel(got, want)
    print(f"delta {delta:.0e}: cond(Z_S) {np.linalg.cond(zs):.2e}, relative difference {d:.2e}")
    assert d < tol_for(zs)
    assert rel(glam, wlam) < tol_for(zs)


def test_operator_chain_rank_deficient_cod(pb, orc):
    """cond(Z_S) ~ 1e14 is rank deficient for the reference's threshold: the
    COD minimum-norm solution (kr_linalg.hpp:113-117)."""
    dims, r, s = (40, 30, 20), 6, 150
    g = orc.Engine(4200, raw=True)
    fs = collinear_factors(g, dims, r, 1e-14)
    x = model_tensor(np.ones(r), fs)
    idx = orc.draw_samples(g, dims, 0, s)
    zs = orc.skr(idx, fs, 0)
    xs = orc.gather_fibers(x, 0, idx)
    want, wrank = orc.least_squares(zs, np.asfortranarray(xs.T))
    assert wrank < r
    got, glam, rank = pb.mode_update(x, 0, idx, fs, np.ones(r), False)
    assert rank == wrank
    assert rel(got * glam[None, :], want.T) < 1e-8


def session_first_mode(pb, orc, method, fused, delta, zero_col=None, transform=None, seed=7):
    """One iteration of a session from a given collinear init on the tensor
    built from that init (mode 0's LS is consistent); returns the GPU's
    factors after it and the oracle's teacher-forced updates of every mode."""
    dims, r, s = (48, 40, 36), 6, 120
    g = orc.Engine(4300 + seed, raw=True)
    fs = collinear_factors(g, dims, r, delta, zero_col)
    # consistent for mode 0 (the tensor is built from the init's modes 1, 2);
    # with a zero init column, mode 1 of the truth is a full random factor so
    # the refilled component is determined by the data in the next mode
    truth = [np.asfortranarray(g.matrix(dims[0], r))]
    truth += fs[1:] if zero_col is None else [np.asfortranarray(g.matrix(dims[1], r)), fs[2]]
    x = model_tensor(np.ones(r), truth)
    init = (np.ones(r), fs)
    opts = pb.SolveOptions(rng_seed=seed, max_iters=1, bench_mode=True, init="given", init_model=init,
                           transform=transform, fused=fused, device=0)
    t = pb.DeviceTensor(dims, device=0)
    t.upload(x)
    sess = pb.Session(method, t, r, s, opts)
    assert sess.fused == (fused != 0)
    assert sess.run(1) == 1
    res = sess.result()
    sess.close()
    t.close()
    tables = orc.sample_tables(dims, s, seed, 1)[0]
    out = []
    cur = [f.copy(order="F") for f in fs]
    lam = np.ones(r)
    for n in range(3):
        inp = [res.factors[m] if m < n else cur[m] for m in range(3)]
        want, wlam, zs = oracle_update(orc, x, n, tables[n], inp, lam if n == 0 else res.lam, n == 0,
                                       mix=transform, seed=seed)
        out.append((res.factors[n], want, zs))
        lam = wlam
    return res, out, lam


PATHS = [("rand", 0, None), ("rand", -1, None), ("mix", -1, "dct"), ("mix", 0, "dct")]


@pytest.mark.parametrize("method,fused,transform", PATHS)
@pytest.mark.parametrize("delta", [1e-2, 1e-6, 1e-10])
def test_session_paths_conditioning_band(pb, orc, method, fused, transform, delta):
    """Mode 0 of the first iteration through each execution path (chain,
    persistent CPRAND kernel, persistent / chain CPRAND-MIX)."""
    _, out, _ = session_first_mode(pb, orc, method, fused, delta, transform=transform)
    got, want, zs = out[0]
    d = rel(got, want)
    print(f"{method} fused={fused} delta {delta:.0e}: cond {np.linalg.cond(zs):.2e}, diff {d:.2e}")
    assert d < tol_for(zs)


@pytest.mark.parametrize("method,fused,transform", PATHS)
def test_session_paths_zero_column_refill(pb, orc, method, fused, transform):
    """A zero factor column in mode 1 makes mode 0's Z_S rank deficient: the
    COD gives a zero solution column, normalize_columns refills it from the
    normalize stream with lambda 0 (kruskal.hpp:57-63), and the next mode
    uses the refilled column. The persistent CPRAND kernel forms mode 0's
    norms while mode 1's tiles already run: mode 1 takes the QR path on a
    Z_S rebuilt from the refilled factor."""
    res, out, lam = session_first_mode(pb, orc, method, fused, 0.3, zero_col=2, transform=transform)
    for n, (got, want, zs) in enumerate(out):
        d = rel(got, want)
        print(f"{method} fused={fused} mode {n}: diff {d:.2e}")
        assert d < 1e-8, (n, d)
    assert rel(res.lam, lam) < 1e-8
