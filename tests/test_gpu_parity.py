"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): gathered fibers, Z_S and sampled entries
bit-exact given identical sample tables; solved factors 1e-10 relative
(fp64); end-to-end final fit within 1e-3 of the oracle over seeded runs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_1701_06600_b200 as pb
    assert pb.device_count() > 0, "GPU tests need a visible CUDA device"
    return pb


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


SHAPES = [(3, 4, 5), (17, 9, 13), (64, 33, 20), (9, 7, 6, 5), (100, 100, 100)]


@pytest.mark.parametrize("dims", SHAPES)
def test_gather_bit_exact(pb, orc, dims):
    x = orc.random_tensor(dims, 37)
    g = orc.Engine(38, raw=True)
    for mode in range(len(dims)):
        idxs = orc.draw_samples(g, dims, mode, 257)
        assert np.array_equal(pb.gather_fibers(x, mode, idxs), orc.gather_fibers(x, mode, idxs))


@pytest.mark.parametrize("dims,r", [((4, 5, 3, 2), 3), ((30, 20, 10), 10), ((50, 40, 30), 50),
                                    ((8, 9, 10), 17)])
def test_skr_bit_exact(pb, orc, dims, r):
    g = orc.Engine(807, raw=True)
    fs = [g.matrix(d, r) for d in dims]
    for mode in range(len(dims)):
        idxs = orc.draw_samples(g, dims, mode, 301)
        assert np.array_equal(pb.skr(idxs, fs, mode), orc.skr(idxs, fs, mode))
        if np.prod(dims) // dims[mode] <= 4000:
            ex = orc.exhaustive_samples(dims, mode)
            assert np.array_equal(pb.skr(ex, fs, mode), orc.skr(ex, fs, mode))


def oracle_mode_update(orc, x, mode, idxs, fs, lam, first, seed=0):
    zs = orc.skr(idxs, fs, mode)
    xs = orc.gather_fibers(x, mode, idxs)
    a = orc.sampled_update(zs, xs)
    f2 = list(fs)
    f2[mode] = a
    return orc.normalize_columns(f2, lam, mode, first, orc.Engine(seed, 8))


@pytest.mark.parametrize("dims,r,s", [((30, 25, 20), 5, 80), ((64, 50, 40), 10, 300),
                                      ((40, 30, 20, 10), 20, 200), ((120, 90, 70), 50, 700),
                                      ((300, 300, 30), 10, 300)])
def test_mode_update_teacher_forced(pb, orc, dims, r, s):
    """One GPU mode step from the oracle's factors vs oracle skr+gather+
    sampled_update+normalize (sampling.hpp:283-290): 1e-10 relative."""
    x = orc.random_tensor(dims, 901)
    g = orc.Engine(902, raw=True)
    fs = [g.matrix(d, r) for d in dims]
    lam = g.uniform_real(0.5, 2.0, r)
    for mode in range(len(dims)):
        idxs = orc.draw_samples(g, dims, mode, s)
        for first in (True, False):
            got, glam, rank = pb.mode_update(x, mode, idxs, fs, lam, first)
            want_fs, wlam = oracle_mode_update(orc, x, mode, idxs, fs, lam, first)
            assert rank == r
            assert rel(got, want_fs[mode]) < 1e-10
            assert rel(glam, wlam) < 1e-10


def test_mode_update_exhaustive_is_dense_solve(pb, orc):
    """test_sampling.cpp:97-115 on the GPU: all rows -> the dense normal solve."""
    dims = (4, 5, 3)
    x = orc.random_tensor(dims, 811)
    g = orc.Engine(813, raw=True)
    fs = [g.matrix(d, 2) for d in dims]
    for mode in range(3):
        ex = orc.exhaustive_samples(dims, mode)
        got, _, _ = pb.mode_update(x, mode, ex, fs, np.ones(2), True)
        want, _ = oracle_mode_update(orc, x, mode, ex, fs, np.ones(2), True)
        assert rel(got, want[mode]) < 1e-10


def test_mode_update_rank_deficient_min_norm(pb, orc):
    """A duplicated factor column makes Z_S rank deficient: min-norm path
    (kr_linalg.hpp:113-117) -> same minimum-norm update as the oracle."""
    dims = (12, 10, 8)
    x = orc.random_tensor(dims, 5)
    g = orc.Engine(6, raw=True)
    fs = [g.matrix(d, 3) for d in dims]
    for f in fs:
        f[:, 2] = f[:, 1]
    idxs = orc.draw_samples(g, dims, 0, 60)
    got, glam, rank = pb.mode_update(x, 0, idxs, fs, np.ones(3), False)
    assert rank == 2
    zs = orc.skr(idxs, fs, 0)
    xs = orc.gather_fibers(x, 0, idxs)
    want = orc.sampled_update(zs, xs)
    # compare before normalization: unnormalize with lambda
    assert rel(got * glam[None, :], want) < 1e-8


def test_fit_values_and_estimate(pb, orc):
    dims = (20, 15, 12)
    x = orc.random_tensor(dims, 823)
    est = orc.make_fit_estimator(x, 500, orc.Engine(824, raw=True))
    offs = [int(np.ravel_multi_index(tuple(i), dims, order="F")) for i in est.idxs]
    vals, nrm = pb.fit_values(x, offs)
    assert np.array_equal(vals, est.x_values)
    assert nrm == pytest.approx(est.x_norm, rel=1e-13)
    g = orc.Engine(828, raw=True)
    lam = g.uniform_real(0.2, 1.0, 3)
    fs = [g.matrix(d, 3) for d in dims]
    got = pb.estimate_fit(lam, fs, est.idxs, est.x_values, est.x_norm, est.total_count)
    assert got == pytest.approx(orc.estimate_fit(lam, fs, est), rel=1e-12, abs=1e-13)


def test_device_normalize_rng_matches_libstdcxx(pb, orc):
    """Zero-column refill draws (kruskal.hpp:53-63) come from a device
    mt19937_64 + polar normal that must replay seeded_engine(seed, 8)."""
    for seed in (0, 3, 17):
        want = orc.Engine(seed, 8).normal(501)
        got = pb.debug_normal_stream(seed, 501)
        assert np.max(np.abs(got - want)) <= 4e-16 * np.max(np.abs(want))


@pytest.mark.parametrize("dims", [(4, 3, 5), (80, 16, 12), (20, 7, 9, 11), (320, 6, 5), (1, 5, 3)])
def test_mix_tensor_matches_oracle(pb, orc, dims):
    x = orc.random_tensor(dims, 901)
    got = pb.mix_tensor(x, "dct", 9)
    want = orc.mix_tensor(x, "dct", 9)
    assert rel(got, want) < 1e-12
    assert np.array_equal(pb.mix_tensor(x, "identity", 9), x)


def test_mix_unmix_factor_and_rows(pb, orc):
    dims = (7, 80, 320)
    g = orc.Engine(911, raw=True)
    for mode in range(3):
        a = g.matrix(dims[mode], 5)
        m = pb.mix_factor(a, dims, "dct", 13, mode)
        assert rel(m, orc.mix_factor(a, dims, "dct", 13, mode)) < 1e-12
        assert rel(pb.unmix_factor(m, dims, "dct", 13, mode), a) < 1e-12
        gg = np.asfortranarray(m.T)
        assert rel(pb.unmix_sampled_rhs(gg, dims, "dct", 13, mode),
                   orc.unmix_sampled_rhs(gg, dims, "dct", 13, mode)) < 1e-12


def test_mode_update_mix_teacher_forced(pb, orc):
    """The MIX mode step (mixing.hpp:286-296) on an oracle-mixed tensor."""
    dims = (16, 12, 10, 8)
    x = orc.random_tensor(dims, 3)
    xh = orc.mix_tensor(x, "dct", 21)
    g = orc.Engine(4, raw=True)
    fs = [g.matrix(d, 4) for d in dims]
    lam = np.ones(4)
    for mode in range(4):
        idxs = orc.draw_samples(g, dims, mode, 90)
        got, glam, _ = pb.mode_update(xh, mode, idxs, fs, lam, mode == 0, "dct", 21)
        mixed = [orc.mix_factor(f, dims, "dct", 21, m) for m, f in enumerate(fs)]
        zs = orc.skr(idxs, mixed, mode)
        gathered = orc.gather_fibers(xh, mode, idxs)
        rhs = orc.unmix_sampled_rhs(np.asfortranarray(gathered.T), dims, "dct", 21, mode)
        a, _ = orc.least_squares(zs, rhs)
        f2 = list(fs)
        f2[mode] = np.asfortranarray(a.T)
        want, wlam = orc.normalize_columns(f2, lam, mode, mode == 0, orc.Engine(0, 8))
        assert rel(got, want[mode]) < 1e-10
        assert rel(glam, wlam) < 1e-10


# ---------------------------------------------------------------- end to end
def c1_problem(orc, seed=1):
    """configs[0]: 100^3, rank-5 N(0,1) factors, 1% noise, seeded N(0,1) init."""
    x, _ = orc.gen_baseline((100, 100, 100), 5, 0.0, 0.01, seed)
    init = orc.Engine(seed, 1)
    fs0 = [init.normal(100 * 5).reshape(100, 5, order="F") for _ in range(3)]
    return x, (np.ones(5), fs0)


def test_config1_end_to_end_matches_oracle(pb, orc):
    x, init = c1_problem(orc)
    opts = dict(rng_seed=1, max_iters=20, fit_sample_count=4096, init="given", init_model=init,
                stall_limit=1000)
    ref = orc.cprand(x, 5, 100, orc.SolveOptions(**opts))
    got = pb.cprand(x, 5, 100, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations == 20
    assert got.reason == ref.reason
    fits_g = np.array([t[2] for t in got.trace])
    fits_r = np.array([t[2] for t in ref.trace])
    assert np.max(np.abs(fits_g - fits_r)) < 1e-8
    assert abs(fits_g[-1] - fits_r[-1]) < 1e-3
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6
    assert rel(got.lam, ref.lam) < 1e-6


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_free_running_stop_rule_matches_oracle(pb, orc, seed):
    """Default stopping (best-fit stall, sampling.hpp:237-251) on a 40^3
    collinear problem: same stop iteration and reason, fit within 1e-3."""
    x, _ = orc.gen_baseline((40, 40, 40), 4, 0.5, 0.01, seed)
    opts = dict(rng_seed=seed, max_iters=200)
    ref = orc.cprand(x, 4, 60, orc.SolveOptions(**opts))
    got = pb.cprand(x, 4, 60, pb.SolveOptions(**opts))
    assert abs(got.trace[-1][2] - ref.trace[-1][2]) < 1e-3
    assert got.iterations == ref.iterations
    assert got.reason == ref.reason
    assert abs(orc.exact_fit(x, got.lam, got.factors) - orc.exact_fit(x, ref.lam, ref.factors)) < 1e-3


def test_readme_run_on_gpu(pb, orc):
    """proj/README.md:58-65 through the B200 path."""
    x, lam, fs = orc.gen_problem([50, 50, 50], 5, 0.5, 0.01, 3)
    res = pb.cprand(x, 5, 80, pb.SolveOptions(rng_seed=3))
    assert res.iterations == 53 and res.reason == "best_fit_stall"
    assert f"{res.trace[-1][2]:.5f}" == "0.98870"
    assert orc.score(res.factors, fs) > 0.9999


def test_exhaustive_gpu_reproduces_cp_als(pb, orc):
    """acceptance.cpp:175-203 on the GPU: exhaustive CPRAND == CP-ALS iterates."""
    x, _, _ = orc.gen_problem([6, 7, 8], 3, 0.3, 0.1, 4)
    opts = dict(rng_seed=4, fit_tolerance=1e-300, stall_limit=1 << 20, max_iters=20,
                exhaustive_samples=True, exact_fit_trace=True)
    als = orc.cp_als(x, 3, orc.SolveOptions(**opts))
    rnd = pb.cprand(x, 3, 3, pb.SolveOptions(**opts))
    for fa, fb in zip(als.factors, rnd.factors):
        assert rel(fb, fa) <= 1e-8
    assert abs(als.trace[-1][2] - rnd.trace[-1][2]) <= 1e-8
    assert not rnd.trace[-1][3]  # exact fit in the trace


def test_identity_mix_is_bit_identical_on_gpu(pb, orc):
    """test_mixing.cpp:254-277: identity mixing == plain cprand, bitwise."""
    x = orc.random_tensor((6, 5, 4), 929)
    base = dict(rng_seed=31, max_iters=12, stall_limit=6)
    plain = pb.cprand(x, 2, 20, pb.SolveOptions(**base))
    mixed = pb.cprand_mix(x, 2, 20, pb.SolveOptions(transform="identity", **base))
    pre = pb.cprand_premix(x, 2, 20, pb.SolveOptions(transform="identity", **base))
    assert [t[2] for t in plain.trace] == [t[2] for t in mixed.trace] == [t[2] for t in pre.trace]
    for a, b, c in zip(plain.factors, mixed.factors, pre.factors):
        assert np.array_equal(a, b) and np.array_equal(a, c)
    ref = orc.cprand(x, 2, 20, orc.SolveOptions(**base))
    assert abs(plain.trace[-1][2] - ref.trace[-1][2]) < 1e-8


@pytest.mark.parametrize("method", ["mix", "premix"])
def test_dct_mix_end_to_end_matches_oracle(pb, orc, method):
    x, _ = orc.gen_baseline((16, 12, 10, 8), 3, 0.9, 0.01, 5)
    opts = dict(rng_seed=5, max_iters=15, transform="dct", stall_limit=1000)
    ref = orc.solve(method, x, 3, 60, orc.SolveOptions(**opts))
    got = pb.solve(method, x, 3, 60, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations
    fg = np.array([t[2] for t in got.trace])
    fr = np.array([t[2] for t in ref.trace])
    assert np.max(np.abs(fg - fr)) < 1e-7
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(16, 12, 10, 8), (21, 10, 15), (12, 9, 7, 11)])
def test_mix_kernel_strided_in_place_reads(pb, orc, dims):
    """The persistent MIX kernel reads a strided mode that has no mode-major
    replica straight from the tensor (one 8-byte load per element, C5's
    modes 2-3). Same GEMM inputs as through the replicas, so the two runs
    agree bitwise; both follow the oracle trajectory."""
    x, _ = orc.gen_baseline(dims, 3, 0.9, 0.01, 7)
    opts = dict(rng_seed=7, max_iters=12, transform="dct", stall_limit=1000)
    rep = pb.cprand_mix(x, 3, 60, pb.SolveOptions(replicas=1, **opts))
    strided = pb.cprand_mix(x, 3, 60, pb.SolveOptions(replicas=0, **opts))
    assert np.array_equal(rep.lam, strided.lam)
    for a, b in zip(rep.factors, strided.factors):
        assert np.array_equal(a, b)
    ref = orc.solve("mix", x, 3, 60, orc.SolveOptions(**opts))
    assert strided.iterations == ref.iterations
    assert max(abs(a[2] - b[2]) for a, b in zip(strided.trace, ref.trace)) < 1e-7
    for a, b in zip(strided.factors, ref.factors):
        assert rel(a, b) < 1e-6


@pytest.mark.parametrize("dims,r,s,transform", [((16, 12, 10, 8), 3, 60, None), ((21, 10, 15), 3, 40, "fft"),
                                                 ((14, 9, 25), 4, 50, "fft"), ((40, 36, 30), 5, 100, None)])
def test_fft_mix_end_to_end_matches_oracle(pb, orc, dims, r, s, transform):
    """cprand_mix with the reference's default transform, the unitary FFT
    (complex X_hat and mixed factors, real-constrained stacked solve,
    cfft.cu): same iterations and fit trace as the oracle's
    cprand_mix_impl<Complex>, factors to round-off. Lengths with factors
    2, 3, 5, 7 (Stockham radices) and 4-way."""
    x, _ = orc.gen_baseline(dims, r, 0.7, 0.01, 13)
    opts = dict(rng_seed=13, max_iters=15, transform=transform, stall_limit=1000)
    ref = orc.solve("mix", x, r, s, orc.SolveOptions(**opts))
    got = pb.cprand_mix(x, r, s, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations
    fg = np.array([t[2] for t in got.trace])
    fr = np.array([t[2] for t in ref.trace])
    assert np.max(np.abs(fg - fr)) < 1e-7
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6
    assert rel(got.lam, ref.lam) < 1e-6


def test_fft_mix_free_running_stop_rule(pb, orc):
    """FFT-kind CPRAND-MIX with the reference's stop rule (default options):
    the device stops at the same iteration for the same reason."""
    x, _ = orc.gen_baseline((30, 24, 20), 4, 0.5, 0.01, 21)
    opts = dict(rng_seed=21)
    ref = orc.solve("mix", x, 4, 80, orc.SolveOptions(**opts))
    got = pb.cprand_mix(x, 4, 80, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations and got.reason == ref.reason
    assert abs(got.trace[-1][2] - ref.trace[-1][2]) < 1e-6


@pytest.mark.parametrize("method", ["mix", "premix"])
def test_wht_mix_end_to_end_matches_oracle(pb, orc, method):
    """Walsh-Hadamard mixing (power-of-two modes): the real MIX / PREMIX path
    with the WHT kind follows the oracle's trajectory."""
    x, _ = orc.gen_baseline((16, 8, 32, 4), 3, 0.8, 0.01, 17)
    opts = dict(rng_seed=17, max_iters=15, transform="wht", stall_limit=1000)
    ref = orc.solve(method, x, 3, 60, orc.SolveOptions(**opts))
    got = pb.solve(method, x, 3, 60, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations
    assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, ref.trace)) < 1e-7
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6


def test_wht_operators_bit_exact(pb, orc):
    """WHT mix_tensor / mix_factor / unmix: the reference's butterfly order and
    scale, so the device results equal the oracle's bit for bit."""
    dims = (32, 16, 64)
    x = orc.random_tensor(dims, 4)
    assert np.array_equal(pb.mix_tensor(x, "wht", 9), orc.mix_tensor(x, "wht", 9))
    a = np.asfortranarray(np.random.default_rng(1).standard_normal((16, 5)))
    assert np.array_equal(pb.mix_factor(a, dims, "wht", 9, 1), orc.mix_factor(a, dims, "wht", 9, 1))
    assert np.array_equal(pb.unmix_factor(a, dims, "wht", 9, 1), orc.unmix_factor(a, dims, "wht", 9, 1))
    with pytest.raises(pb.InvalidArgument):
        pb.cprand_mix(orc.random_tensor((6, 8, 8), 2), 2, 10, pb.SolveOptions(transform="wht"))


def test_mixed_solver_recovers(pb, orc):
    g = orc.Engine(931, raw=True)
    fs = [g.matrix(d, 2, 0.1, 1.0) for d in (10, 9, 8)]
    x = np.einsum("ir,jr,kr->ijk", *fs)
    res = pb.cprand_mix(x, 2, 60, pb.SolveOptions(rng_seed=37, max_iters=100, stall_limit=30,
                                                  transform="dct"))
    assert orc.exact_fit(x, res.lam, res.factors) >= 0.99


def test_zero_tensor_and_validation(pb, orc):
    res = pb.cprand(np.zeros((4, 4, 4)), 2, 14)
    ref = orc.cprand(np.zeros((4, 4, 4)), 2, 14)
    assert res.reason == "zero_tensor" and np.linalg.norm(res.lam) == 0.0
    for a, b in zip(res.factors, ref.factors):
        assert np.array_equal(a, b)
    x = orc.random_tensor((6, 5, 4), 833)
    with pytest.raises(pb.InvalidArgument):
        pb.cprand(x, 3, 2)
    with pytest.raises(pb.InvalidArgument):
        pb.cprand(x, 2, 4, pb.SolveOptions(max_iters=0))
    with pytest.raises(pb.InvalidArgument):
        pb.cprand_premix(x, 1, 4, pb.SolveOptions(transform="fft"))
    with pytest.raises(pb.InvalidArgument):
        pb.gather_fibers(x, 0, np.zeros((2, 5), dtype=np.int64))
    with pytest.raises(pb.UnsupportedOnDevice):
        pb.cprand(x, 129, 200)
    with pytest.raises(pb.UnsupportedOnDevice):  # R > 64: cprand / premix on one GPU only
        pb.cprand_mix(x, 65, 100, pb.SolveOptions(transform="dct"))


def test_deterministic_bitwise(pb, orc):
    x, _ = orc.gen_baseline((30, 30, 30), 4, 0.5, 0.01, 9)
    a = pb.cprand(x, 4, 50, pb.SolveOptions(rng_seed=23, max_iters=10))
    b = pb.cprand(x, 4, 50, pb.SolveOptions(rng_seed=23, max_iters=10))
    assert np.array_equal(a.lam, b.lam)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    assert [t[2] for t in a.trace] == [t[2] for t in b.trace]


def test_device_synth_matches_oracle_generator(pb, orc):
    dims = (30, 20, 10)
    t = pb.DeviceTensor(dims)
    fs = t.synth(4, 0.5, 0.01, 7, want_factors=True)
    x = t.download()
    xo, fo = orc.gen_baseline(dims, 4, 0.5, 0.01, 7)
    for a, b in zip(fs, fo):
        assert np.array_equal(a, b)
    assert rel(x, xo) < 1e-13


def test_session_bench_mode_and_kernel_stats(pb, orc):
    dims = (60, 50, 40)
    t = pb.DeviceTensor(dims)
    t.synth(5, 0.5, 0.01, 11)
    x = t.download()
    s = pb.Session("rand", t, 5, 80, pb.SolveOptions(rng_seed=11, max_iters=30, bench_mode=True,
                                                     replicas=0))
    s.set_kernel_timing(True)
    s.enqueue(10)
    s.sync()
    assert s.run(20) == 20
    for m in range(3):
        n, ms, b = s.kernel_stats(m, 1)  # RHS GEMM, every mode
        assert n == 30 and ms > 0 and b > 0
    for m in (1, 2):  # strided modes go through the gather ring when replicas are off
        n, ms, b = s.kernel_stats(m, 0)
        assert n == 30 and ms > 0 and b > 0
    res = s.result()
    assert res.iterations == 30 and res.reason == "bench_complete" and res.trace == []
    ref = orc.cprand(x, 5, 80, orc.SolveOptions(rng_seed=11, max_iters=30, bench_mode=True))
    for a, b_ in zip(res.factors, ref.factors):
        assert rel(a, b_) < 1e-6


def test_cpp_dropin_program(pb):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "dropin_smoke")
    subprocess.run(["make", "-s", "-C", root, "dropin"], check=True)  # no-op when up to date
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    kv = dict(p.split("=") for p in out.strip().split(","))
    assert float(kv["fit"]) > 0.999 - 1e-3 and kv["invalid_caught"] == "1" and kv["dsc5"] == "80"


@pytest.mark.parametrize("dims,r,s", [((30, 28, 26), 4, 60), ((17, 9, 13), 3, 40), ((9, 8, 7, 6), 3, 40)])
def test_execution_paths_agree(pb, orc, dims, r, s):
    """The three device paths -- persistent fused iteration kernel (replicas),
    multi-kernel chain on in-place fibers, multi-kernel chain on the gather
    ring -- agree with each other and with the oracle trajectory (even and
    odd mode lengths). The in-place and ring GEMM inputs are identical, so
    the two multi-kernel paths agree bitwise."""
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 3)
    base = dict(rng_seed=3, max_iters=12, stall_limit=1000)
    fused = pb.cprand(x, r, s, pb.SolveOptions(replicas=1, **base))
    chain = pb.cprand(x, r, s, pb.SolveOptions(replicas=1, fused=0, **base))
    ring = pb.cprand(x, r, s, pb.SolveOptions(replicas=0, **base))
    assert np.array_equal(chain.lam, ring.lam)
    for a, b in zip(chain.factors, ring.factors):
        assert np.array_equal(a, b)
    atom = pb.cprand(x, r, s, pb.SolveOptions(replicas=1, atomic_gram=True, **base))
    for res in (fused, atom):
        for a, b in zip(res.factors, ring.factors):
            assert rel(a, b) < 1e-12
    ref = orc.cprand(x, r, s, orc.SolveOptions(**base))
    for res in (fused, chain, atom):
        assert max(abs(a[2] - b[2]) for a, b in zip(res.trace, ref.trace)) < 1e-8


@pytest.mark.gpu
def test_sharded_session_single_rank(pb, orc):
    """The slab-sharded session path (NCCL communicator, local-sample RHS,
    RHS allreduce, mode-N slab rows + column-sum allreduce + allgather) with
    one rank reproduces the unsharded run; the slab generator with one rank
    reproduces the unsharded generator."""
    dims, r, s = (24, 20, 22), 4, 60
    comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
    t1 = pb.DeviceTensor(dims)
    t1.synth(r, 0.5, 0.01, 9)
    t2 = pb.DeviceTensor(dims)
    t2.synth_slab(r, 0.5, 0.01, 9, dims[-1], comm)
    x1, x2 = t1.download(), t2.download()
    assert rel(x2, x1) < 1e-14
    base = dict(rng_seed=9, max_iters=15, stall_limit=1000)
    full = pb.Session("rand", t1, r, s, pb.SolveOptions(fused=0, **base))
    full.run(15)
    ref = full.result()
    sh = pb.Session("rand", t2, r, s, pb.SolveOptions(comm=comm, shard_total=dims[-1], **base))
    sh.run(15)
    got = sh.result()
    assert got.iterations == ref.iterations
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-10
    assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, ref.trace)) < 1e-10
    o = orc.cprand(x1, r, s, orc.SolveOptions(**base))
    assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, o.trace)) < 1e-8
    for h in (sh, full):
        h.close()
    comm.close()


@pytest.mark.gpu
def test_sharded_session_stops_with_the_unsharded_run(pb, orc):
    """A sharded run that stops early (fit threshold / stall stop): the host
    decides each enqueue from the per-iteration stop mark of iteration
    k - kInFlight, the same on every rank, so the ranks issue the same
    collectives; one rank: same stop iteration and reason as unsharded."""
    dims, r, s = (24, 20, 22), 4, 60
    comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
    t1 = pb.DeviceTensor(dims)
    t1.synth(r, 0.5, 0.01, 9)
    t2 = pb.DeviceTensor(dims)
    t2.synth_slab(r, 0.5, 0.01, 9, dims[-1], comm)
    for extra in (dict(fit_threshold=0.97), dict(stall_limit=3)):
        base = dict(rng_seed=9, max_iters=120, **extra)
        full = pb.Session("rand", t1, r, s, pb.SolveOptions(fused=0, **base))
        full.run(120)
        ref = full.result()
        sh = pb.Session("rand", t2, r, s, pb.SolveOptions(comm=comm, shard_total=dims[-1], **base))
        sh.run(120)
        got = sh.result()
        assert got.reason == ref.reason and got.iterations == ref.iterations < 120
        for h in (sh, full):
            h.close()
    comm.close()


@pytest.mark.gpu
def test_sharded_session_rejects_bad_slab(pb):
    comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
    t = pb.DeviceTensor((10, 9, 8))
    t.synth(3, 0.0, 0.0, 1)
    with pytest.raises(pb.InvalidArgument):
        pb.Session("rand", t, 3, 20, pb.SolveOptions(comm=comm, shard_total=20))
    with pytest.raises(pb.UnsupportedOnDevice):  # complex mixing is not sharded
        pb.Session("mix", t, 3, 20, pb.SolveOptions(comm=comm, shard_total=8, transform="fft"))
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("transform", ["dct", "wht"])
def test_sharded_mix_session_single_rank(pb, orc, transform):
    """Slab-sharded CPRAND-MIX through NCCL with one rank: the distributed
    mixing pass (block pack, send/recv group, last-mode transform, reverse
    exchange, unpack), local-sample RHS + allreduce, the last mode's RHS
    slab rows allgathered and unmixed, replicated solve and mixed factors.
    Reproduces the unsharded chain and tracks the oracle's cprand_mix."""
    dims, r, s = (16, 8, 32), 3, 60
    comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
    t1 = pb.DeviceTensor(dims)
    t1.synth(r, 0.5, 0.01, 9)
    t2 = pb.DeviceTensor(dims)
    t2.synth_slab(r, 0.5, 0.01, 9, dims[-1], comm)
    base = dict(rng_seed=9, max_iters=12, stall_limit=1000, transform=transform)
    full = pb.Session("mix", t1, r, s, pb.SolveOptions(fused=0, **base))
    full.run(12)
    ref = full.result()
    sh = pb.Session("mix", t2, r, s, pb.SolveOptions(comm=comm, shard_total=dims[-1], **base))
    sh.run(12)
    got = sh.result()
    assert got.iterations == ref.iterations
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-10
    assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, ref.trace)) < 1e-10
    o = orc.solve("mix", t1.download(), r, s, orc.SolveOptions(**base))
    assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, o.trace)) < 1e-8
    for h in (sh, full):
        h.close()
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(24, 30, 20), (96, 100, 90), (90, 100, 96), (64, 70, 77), (640, 70, 60),
                                  (320, 37, 120), (33, 320, 130), (50, 256, 90), (40, 1000, 110),
                                  (256, 17, 16, 2)])
def test_device_tensor_mix_matches_oracle(pb, orc, dims):
    """Whole-tensor mixing pass on the device. The larger shapes have >= 4096
    fibers per mode, so they run the persistent pass kernels: lengths 96 /
    100 / 90 (first radix 8 / 5 / 5; 16-32 sequences per group; fiber pairs
    adjacent or straddling a stride boundary), 640 contiguous (2 sequences,
    two CTAs per SM), and 77 = 7 * 11 (the generic per-CTA transform). The
    v4 register kernels (mixreg.cu): n = 320 / 256 contiguous with a partial
    last tile of odd width, n = 320 / 256 / 1000 strided at strides 33 / 50 /
    40 (partial tiles, a tile holding one unpaired fiber)."""
    x = orc.random_tensor(dims, 5)
    t = pb.DeviceTensor(dims)
    t.upload(x)
    ms = t.mix("dct", 7)
    assert len(ms) == len(dims) and all(m > 0 for m in ms)
    got = t.download()
    want = orc.mix_tensor(x, "dct", 7)
    assert rel(got, want) < 1e-12


@pytest.mark.parametrize("dims", [(200, 120, 64), (80, 80, 80, 80), (320, 32, 48), (100, 24, 40, 16)])
def test_tma_mix_pass_matches_v2(pb, orc, dims):
    """The TMA-fed mixing pass (mixtma.cu: bulk / tensor-map tile loads and
    stores, in-place Stockham passes) against the v2 pass kernel
    (CPRAND_MIX_V2=1, oracle-checked above): the same butterflies, twiddles
    and epilogue formulas; only the compiler's FMA contraction differs, so
    the mixed tensors agree to a few ulp (1e-14 relative). Strided modes with
    64-512 B rows, one or several TMA boxes per tile (n > 256), mode 1 with
    whole-fiber bulk copies."""
    import os
    t = pb.DeviceTensor(dims)
    t.synth(4, 0.3, 0.01, 11)
    x = t.download()
    os.environ["CPRAND_MIX_TMA"] = "1"  # also for n < 512, where it is not the default
    try:
        new = t.mix("dct", 3)
    finally:
        del os.environ["CPRAND_MIX_TMA"]
    got = t.download()
    t.upload(x)
    os.environ["CPRAND_MIX_V2"] = "1"
    try:
        old = t.mix("dct", 3)
    finally:
        del os.environ["CPRAND_MIX_V2"]
    want = t.download()
    t.close()
    assert len(new) == len(old) == len(dims)
    assert rel(got, want) < 1e-14


def test_tma_mix_pass_matches_oracle(pb, orc):
    """TMA pass against the oracle's mix_tensor (Bluestein DCT) on a shape
    whose every mode has >= 4096 fibers."""
    import os
    dims = (64, 40, 48, 32)
    x = orc.random_tensor(dims, 9)
    t = pb.DeviceTensor(dims)
    t.upload(x)
    os.environ["CPRAND_MIX_TMA"] = "1"
    try:
        t.mix("dct", 5)
    finally:
        del os.environ["CPRAND_MIX_TMA"]
    got = t.download()
    t.close()
    assert rel(got, orc.mix_tensor(x, "dct", 5)) < 1e-12


@pytest.mark.gpu
def test_atomic_gram_many_tiles(pb, orc):
    """SolveOptions(atomic_gram=True) on a problem that spreads every mode's
    Gram over hundreds of tiles (L2 fp64 adds from many CTAs into each
    element): same trajectory as the reproducible fused kernel to round-off."""
    dims, r, s = (400, 300, 350), 24, 1500
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.5, 0.01, 17)
    base = dict(rng_seed=17, max_iters=8, stall_limit=1000, bench_mode=True)
    runs = []
    for atomic in (False, True):
        sess = pb.Session("rand", t, r, s, pb.SolveOptions(atomic_gram=atomic, **base))
        sess.run(8)
        runs.append(sess.result())
        sess.close()
    t.close()
    assert np.all(np.isfinite(runs[1].lam))
    np.testing.assert_allclose(runs[1].lam, runs[0].lam, rtol=1e-9)
    for a, b in zip(runs[1].factors, runs[0].factors):
        assert rel(a, b) < 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["rand", "mix"])
def test_fused_gram_sum_on_inverse_cta_wide_rank(pb, orc, method):
    """More tiles than CTAs (CPRAND kernel: every Gram block's split partials
    are summed on the inverse CTA) at a rank whose Gram has more than 2048
    block entries (r = 60: 36 8 x 8 blocks): the persistent kernels match
    the multi-kernel chain."""
    dims, r, s = (700, 600, 500), 60, 6000
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.5, 0.01, 23)
    base = dict(rng_seed=23, max_iters=3, stall_limit=1000, bench_mode=True)
    if method == "mix":
        base["transform"] = "dct"
    runs = []
    for fused in (-1, 0):
        sess = pb.Session(method, t, r, s, pb.SolveOptions(fused=fused, **base))
        sess.run(3)
        runs.append(sess.result())
        sess.close()
    t.close()
    np.testing.assert_allclose(runs[0].lam, runs[1].lam, rtol=1e-9)
    for a, b in zip(runs[0].factors, runs[1].factors):
        assert rel(a, b) < 1e-9


def test_session_gather_bench_bytes(pb, orc):
    """The batched sampled-gather measurement moves exactly the fibers of
    the requested iterations: useful bytes 8 * iters * sum_n S I_n; B_min
    counts 32 B per element for strided modes read from the tensor."""
    dims, r, s = (40, 30, 20), 3, 50
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.0, 0.0, 3)
    sess = pb.Session("rand", t, r, s, pb.SolveOptions(rng_seed=3, max_iters=40, bench_mode=True, replicas=1))
    ms, useful, bmin = sess.gather_bench(10, True)
    assert ms > 0 and useful == 8.0 * 10 * s * sum(dims) and bmin == useful
    ms, useful, bmin = sess.gather_bench(10, False)
    assert useful == 8.0 * 10 * s * sum(dims)
    assert bmin == 8.0 * 10 * s * dims[0] + 32.0 * 10 * s * (dims[1] + dims[2])
    sess.close()
    t.close()


@pytest.mark.parametrize("dims,r", [((30, 24, 20), 4), ((12, 10, 8, 6), 3), ((64, 40, 50), 20)])
def test_exact_fit_matches_oracle(pb, orc, dims, r):
    """exact_fit (solver.hpp:161-181) on the device (mode-1 MTTKRP through the
    split-K GEMM, Gram expansion) against the oracle's, for a solved model
    and for a random one; zero tensor -> 1."""
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 6)
    res = orc.cprand(x, r, 60, orc.SolveOptions(rng_seed=6, max_iters=10, stall_limit=1000))
    want = orc.exact_fit(x, res.lam, res.factors)
    assert abs(pb.exact_fit(x, res.lam, res.factors) - want) < 1e-10
    t = pb.DeviceTensor(dims)
    t.upload(x)
    assert abs(t.exact_fit(res.lam, res.factors) - want) < 1e-10
    g = np.random.default_rng(2)
    lam = g.standard_normal(r)
    fs = [g.standard_normal((d, r)) for d in dims]
    assert abs(t.exact_fit(lam, fs) - orc.exact_fit(x, lam, fs)) < 1e-10
    t.close()
    assert pb.exact_fit(np.zeros(dims), lam, fs) == 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(101, 67, 40), (67, 12, 101)])
def test_prime_length_mixing_matches_oracle(pb, orc, dims):
    """Mode lengths with prime factors above 61 (the reference's Bluestein
    FFT, transforms.hpp:27-118; here the generic-radix Stockham pass): the
    device mixing pass, and DCT / FFT CPRAND-MIX end to end, against the
    oracle."""
    x = orc.random_tensor(dims, 17)
    t = pb.DeviceTensor(dims)
    t.upload(x)
    t.mix("dct", 3)
    assert rel(t.download(), orc.mix_tensor(x, "dct", 3)) < 1e-12
    t.close()
    xb, _ = orc.gen_baseline(dims, 3, 0.5, 0.01, 4)
    for transform in ("dct", None):
        opts = dict(rng_seed=4, max_iters=6, transform=transform, stall_limit=1000)
        ref = orc.solve("mix", xb, 3, 60, orc.SolveOptions(**opts))
        got = pb.solve("mix", xb, 3, 60, pb.SolveOptions(**opts))
        assert max(abs(a[2] - b[2]) for a, b in zip(got.trace, ref.trace)) < 1e-8
        for a, b in zip(got.factors, ref.factors):
            assert rel(a, b) < 1e-6


@pytest.mark.parametrize("dims,r,s,method", [((90, 80, 70), 80, 400, "rand"), ((40, 36, 30, 28), 128, 700, "rand"),
                                              ((70, 66, 64), 72, 300, "premix")])
def test_wide_rank_chain_matches_oracle(pb, orc, dims, r, s, method):
    """64 < R <= 128 (the reference has no rank cap): the multi-kernel chain
    with RT = 128 buckets (Z_S, Gram, 512-thread Gauss-Jordan inverse, split-K
    RHS GEMM, apply) and the sampled fit, against the oracle's pivoted-QR loop."""
    x, _ = orc.gen_baseline(dims, r, 0.0, 0.01, 31)
    opts = dict(rng_seed=31, max_iters=6, stall_limit=1000)
    if method == "premix":
        opts["transform"] = "dct"
    ref = orc.solve(method, x, r, s, orc.SolveOptions(**opts))
    got = pb.solve(method, x, r, s, pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations == 6
    fg = np.array([t[2] for t in got.trace])
    fr = np.array([t[2] for t in ref.trace])
    assert np.max(np.abs(fg - fr)) < 1e-8
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6
    assert rel(got.lam, ref.lam) < 1e-6
