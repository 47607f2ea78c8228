"""The reference's own hot-path tests, re-expressed
against the CPU oracle. Each test names the reference test it mirrors."""
import numpy as np
import pytest


def matricize(x, mode):
    """Mode-n unfolding under the layout law (tensor.hpp:123-163)."""
    return np.reshape(np.moveaxis(x, mode, 0), (x.shape[mode], -1), order="F")


def kr_explicit(factors, skip):
    seq = [factors[m] for m in range(len(factors) - 1, -1, -1) if m != skip]
    out = seq[0]
    for b in seq[1:]:
        out = np.einsum("ir,jr->ijr", out, b).reshape(-1, out.shape[1])
    return out


def test_gather_picks_unfolding_columns(orc):  # test_tensor.cpp:200-231
    dims = (3, 4, 5)
    x = orc.random_tensor(dims, 37)
    g = orc.Engine(38, raw=True)
    for mode in range(3):
        other = [dims[k] for k in range(3) if k != mode]
        idxs = np.empty((9, 2), dtype=np.int64, order="F")
        for row in range(9):
            for c in range(2):
                idxs[row, c] = g.uniform_int(0, other[c] - 1, 1)[0]
        got = orc.gather_fibers(x, mode, idxs)
        xm = matricize(x, mode)
        for row in range(9):
            full = [0, 0, 0]
            c = 0
            for k in range(3):
                if k != mode:
                    full[k] = idxs[row, c]
                    c += 1
            j = orc.unfold_column_index(mode, full, dims)
            assert np.array_equal(got[:, row], xm[:, j])
    with pytest.raises(orc.InvalidArgument):
        orc.gather_fibers(x, 0, np.zeros((2, 5), dtype=np.int64))


def test_draw_samples_range_and_replay(orc):  # test_sampling.cpp:33-53
    dims = (3, 4, 5)
    g = orc.Engine(801, raw=True)
    s = orc.draw_samples(g, dims, 1, 50)
    assert s.shape == (50, 2)
    assert s[:, 0].min() >= 0 and s[:, 0].max() < 3
    assert s[:, 1].min() >= 0 and s[:, 1].max() < 5
    s2 = orc.draw_samples(g, dims, 1, 50)
    assert np.abs(s - s2).sum() > 0
    s3 = orc.draw_samples(orc.Engine(801, raw=True), dims, 1, 50)
    assert np.array_equal(s, s3)
    with pytest.raises(orc.InvalidArgument):
        orc.draw_samples(g, dims, 3, 5)
    with pytest.raises(orc.InvalidArgument):
        orc.draw_samples(g, dims, 0, 0)


def test_exhaustive_samples_order(orc):  # test_sampling.cpp:55-69
    dims = (3, 4, 2)
    for mode in range(3):
        s = orc.exhaustive_samples(dims, mode)
        for j in range(s.shape[0]):
            full = [0, 0, 0]
            c = 0
            for k in range(3):
                if k != mode:
                    full[k] = s[j, c]
                    c += 1
            assert orc.unfold_column_index(mode, full, dims) == j


def test_skr_matches_explicit_khatri_rao(orc):  # test_sampling.cpp:71-95
    dims = (4, 5, 3, 2)
    g = orc.Engine(807, raw=True)
    fs = [g.matrix(d, 3) for d in dims]
    for mode in range(4):
        z = kr_explicit(fs, mode)
        zs = orc.skr(orc.exhaustive_samples(dims, mode), fs, mode)
        assert np.linalg.norm(zs - z) <= 1e-14 * np.linalg.norm(z)


def test_sampled_update_full_rows_is_dense_solve(orc):  # test_sampling.cpp:97-115
    dims = (4, 5, 3)
    x = orc.random_tensor(dims, 811)
    g = orc.Engine(813, raw=True)
    fs = [g.matrix(d, 2) for d in dims]
    for mode in range(3):
        all_rows = orc.exhaustive_samples(dims, mode)
        zs = orc.skr(all_rows, fs, mode)
        xs = orc.gather_fibers(x, mode, all_rows)
        a = orc.sampled_update(zs, xs)
        z = kr_explicit(fs, mode)
        v = z.T @ z
        w = matricize(x, mode) @ z
        ref = np.linalg.solve(v, w.T).T
        assert np.linalg.norm(a - ref) <= 1e-10 * (np.linalg.norm(ref) + 1)
    with pytest.raises(orc.InvalidArgument):
        orc.sampled_update(np.ones((2, 3)), np.ones((4, 2)))
    with pytest.raises(orc.InvalidArgument):
        orc.sampled_update(np.ones((5, 3)), np.ones((4, 4)))


def test_least_squares_rank_deficient_is_min_norm(orc):  # test_kr_linalg.cpp:163-175
    g = orc.Engine(5, raw=True)
    a = g.matrix(12, 4)
    a[:, 3] = a[:, 0] + a[:, 1]  # rank 3
    b = g.matrix(12, 2)
    got, rank = orc.least_squares(a, b)
    assert rank == 3
    ref = np.linalg.pinv(a) @ b
    assert np.linalg.norm(got - ref) <= 1e-10 * (np.linalg.norm(ref) + 1)
    full = g.matrix(12, 4)
    got, rank = orc.least_squares(full, b)
    assert rank == 4
    assert np.allclose(got, np.linalg.lstsq(full, b, rcond=None)[0], atol=1e-12)


def test_fit_estimator_full_and_distinct(orc):  # test_sampling.cpp:117-145
    x = orc.random_tensor((3, 4, 2), 821)
    est = orc.make_fit_estimator(x, 1000, orc.Engine(822, raw=True))
    assert est.idxs.shape[0] == x.size and est.total_count == x.size
    for j in range(x.size):
        assert est.x_values[j] == x[tuple(est.idxs[j])]
    x = orc.random_tensor((6, 6, 6), 823)
    est = orc.make_fit_estimator(x, 50, orc.Engine(824, raw=True))
    offs = [int(np.ravel_multi_index(tuple(i), x.shape, order="F")) for i in est.idxs]
    assert len(set(offs)) == 50 and offs == sorted(offs)


def test_estimate_fit_exhaustive_equals_exact(orc):  # test_sampling.cpp:147-157
    dims = (4, 3, 5)
    x = orc.random_tensor(dims, 827)
    g = orc.Engine(828, raw=True)
    lam = g.uniform_real(0.2, 1.0, 2)
    fs = [g.matrix(d, 2) for d in dims]
    est = orc.make_fit_estimator(x, x.size, orc.Engine(0, 3))
    assert orc.estimate_fit(lam, fs, est) == pytest.approx(orc.exact_fit(x, lam, fs), rel=1e-12)


def test_exhaustive_cprand_reproduces_cp_als(orc):  # test_sampling.cpp:234-252
    x = orc.random_tensor((5, 4, 3), 831)
    opts = orc.SolveOptions(rng_seed=17, max_iters=6, fit_tolerance=1e-300, stall_limit=1000,
                            exhaustive_samples=True, exact_fit_trace=True)
    als = orc.cp_als(x, 2, opts)
    rnd = orc.cprand(x, 2, 2, opts)
    assert len(als.trace) == len(rnd.trace)
    for a, b in zip(als.trace, rnd.trace):
        assert a[2] == pytest.approx(b[2], rel=1e-9)
    for fa, fb in zip(als.factors, rnd.factors):
        assert np.linalg.norm(fa - fb) <= 1e-8 * np.linalg.norm(fa)


def test_acceptance_exhaustive_degeneracy(orc):  # acceptance.cpp:175-203
    x, _, _ = orc.gen_problem([6, 7, 8], 3, 0.3, 0.1, 4)
    opts = orc.SolveOptions(rng_seed=4, fit_tolerance=1e-300, stall_limit=1 << 20, max_iters=20,
                            exhaustive_samples=True, exact_fit_trace=True)
    als = orc.cp_als(x, 3, opts)
    rnd = orc.cprand(x, 3, 3, opts)
    for fa, fb in zip(als.factors, rnd.factors):
        assert np.linalg.norm(fa - fb) <= 1e-8 * np.linalg.norm(fa)
    assert abs(als.trace[-1][2] - rnd.trace[-1][2]) <= 1e-8


def test_cprand_deterministic_and_validates(orc):  # test_sampling.cpp:254-271
    x = orc.random_tensor((6, 5, 4), 833)
    opts = orc.SolveOptions(rng_seed=23, max_iters=10, stall_limit=5)
    a = orc.cprand(x, 2, 20, opts)
    b = orc.cprand(x, 2, 20, opts)
    assert np.array_equal(a.lam, b.lam)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    assert [t[2] for t in a.trace] == [t[2] for t in b.trace]
    assert all(t[3] for t in a.trace)
    with pytest.raises(orc.InvalidArgument):
        orc.cprand(x, 3, 2, opts)


def test_cprand_recovers_clean_tensor(orc):  # test_sampling.cpp:273-288
    g = orc.Engine(837, raw=True)
    fs = [g.matrix(d, 2, 0.1, 1.0) for d in (12, 11, 10)]
    x = np.einsum("ir,jr,kr->ijk", *fs)
    res = orc.cprand(x, 2, 60, orc.SolveOptions(rng_seed=7, max_iters=100, stall_limit=30))
    assert orc.exact_fit(x, res.lam, res.factors) >= 0.999


def test_zero_tensor_short_circuit(orc):  # test_sampling.cpp:290-296
    res = orc.cprand(np.zeros((4, 4, 4)), 2, 14)
    assert res.reason == "zero_tensor"
    assert np.linalg.norm(res.lam) == 0.0


def dct_matrix(n):
    k = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    c = np.cos(np.pi * k * (2 * j + 1) / (2 * n))
    c[0] *= np.sqrt(1.0 / n)
    c[1:] *= np.sqrt(2.0 / n)
    return c


def multi_ttm(x, mats):
    y = x.astype(np.result_type(x, *mats))
    for m, u in enumerate(mats):
        y = np.moveaxis(np.tensordot(u, y, axes=([1], [m])), 0, m)
    return y


@pytest.mark.parametrize("kind", ["dct", "fft", "wht", "identity"])
def test_mix_tensor_matches_dense_oracle(orc, kind):  # test_mixing.cpp:90-137
    dims = (4, 2, 8) if kind == "wht" else (4, 3, 5)
    x = orc.random_tensor(dims, 901)
    got = orc.mix_tensor(x, kind, 9)
    signs = orc.mixing_signs(dims, kind, 9)
    if kind == "identity":
        assert np.array_equal(got, x)
        return
    mats = []
    for m, d in enumerate(dims):
        if kind == "dct":
            f = dct_matrix(d)
        elif kind == "fft":
            f = np.fft.fft(np.eye(d), axis=0) / np.sqrt(d)
        else:
            h = np.array([[1.0]])
            while h.shape[0] < d:
                h = np.block([[h, h], [h, -h]])
            f = h / np.sqrt(d)
        mats.append(f * signs[m][None, :])
    ref = multi_ttm(x, mats)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_mixing_preserves_norm_and_roundtrips(orc):  # test_mixing.cpp:139-186
    dims = (5, 6, 7)
    x = orc.random_tensor(dims, 907)
    for kind in ("dct", "fft"):
        assert np.linalg.norm(orc.mix_tensor(x, kind, 3)) == pytest.approx(np.linalg.norm(x), rel=1e-10)
    g = orc.Engine(911, raw=True)
    for kind in ("dct", "fft", "identity"):
        for mode in range(3):
            a = g.matrix(dims[mode], 3)
            back = orc.unmix_factor(orc.mix_factor(a, dims, kind, 13, mode), dims, kind, 13, mode)
            assert np.linalg.norm(back - a) <= 1e-12 * (np.linalg.norm(a) + 1)
    a = g.matrix(8, 2)
    rot = 1j * orc.mix_factor(a, (8, 5), "fft", 17, 0)
    with pytest.raises(orc.NumericalConsistencyError):
        orc.unmix_factor(rot, (8, 5), "fft", 17, 0)


def test_unmix_sampled_rhs_inverts_row_mixing(orc):  # test_mixing.cpp:188-213
    dims = (7, 5, 4)
    g = orc.Engine(917, raw=True)
    for kind in ("fft", "dct"):
        for mode in range(3):
            a = g.matrix(dims[mode], 6)
            mixed = orc.mix_factor(a, dims, kind, 19, mode)
            back = orc.unmix_sampled_rhs(np.asfortranarray(mixed.T), dims, kind, 19, mode)
            assert np.linalg.norm(back - a.T) <= 1e-12 * (np.linalg.norm(a) + 1)


def test_identity_mixing_is_bit_identical_to_cprand(orc):  # test_mixing.cpp:254-277
    x = orc.random_tensor((6, 5, 4), 929)
    opts = orc.SolveOptions(rng_seed=31, max_iters=12, stall_limit=6, transform="identity")
    plain = orc.cprand(x, 2, 20, opts)
    mixed = orc.cprand_mix(x, 2, 20, opts)
    pre = orc.cprand_premix(x, 2, 20, opts)
    assert [t[2] for t in plain.trace] == [t[2] for t in mixed.trace] == [t[2] for t in pre.trace]
    assert np.array_equal(plain.lam, mixed.lam) and np.array_equal(plain.lam, pre.lam)
    for a, b, c in zip(plain.factors, mixed.factors, pre.factors):
        assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("variant", ["fft_mix", "dct_mix", "dct_premix"])
def test_mixed_solvers_recover(orc, variant):  # test_mixing.cpp:279-308
    g = orc.Engine(931, raw=True)
    fs = [g.matrix(d, 2, 0.1, 1.0) for d in (10, 9, 8)]
    x = np.einsum("ir,jr,kr->ijk", *fs)
    opts = orc.SolveOptions(rng_seed=37, max_iters=100, stall_limit=30)
    if variant == "fft_mix":
        res = orc.cprand_mix(x, 2, 60, opts)
    elif variant == "dct_mix":
        opts.transform = "dct"
        res = orc.cprand_mix(x, 2, 60, opts)
    else:
        res = orc.cprand_premix(x, 2, 60, opts)
        for a in res.factors:
            assert np.allclose(np.linalg.norm(a, axis=0), 1.0, rtol=1e-10)
    assert orc.exact_fit(x, res.lam, res.factors) >= 0.99


def test_mix_validation(orc):  # test_mixing.cpp:311-322
    x = orc.random_tensor((4, 4), 937)
    with pytest.raises(orc.InvalidArgument):
        orc.cprand_premix(x, 1, 4, orc.SolveOptions(transform="fft"))
    with pytest.raises(orc.InvalidArgument):
        orc.cprand_mix(x, 2, 1)
    with pytest.raises(orc.InvalidArgument):
        orc.mixing_signs((4, 6), "wht", 1)


def test_baseline_generator_shape_and_noise(orc):
    """BASELINE generator: factor congruence via L = chol((1-C)I + C11^T) and
    realized noise ratio exactly eta (synth.hpp:76-84 scaling)."""
    dims, r, c, eta = (20, 18, 16), 4, 0.5, 0.01
    x, fs = orc.gen_baseline(dims, r, c, eta, 7)
    xt = np.einsum("ir,jr,kr->ijk", *fs)
    ratio = np.linalg.norm(x - xt) / np.linalg.norm(xt)
    assert ratio == pytest.approx(eta, rel=1e-9)
    _, fs2 = orc.gen_baseline(dims, r, c, eta, 7, want_tensor=False)
    for a, b in zip(fs, fs2):
        assert np.array_equal(a, b)
    z = orc.philox_gaussian(7, 0, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
