"""Oracle parity at the BASELINE.json configurations (C2-C5), on the tensors
the bench measures (generated in HBM by the same generator).

* C2 (300^3, CPRAND) and C3 (80^4, DCT CPRAND-MIX): free-running solves
  through the C ABI against the oracle's `cprand` / `cprand_mix_impl`
  (sampling.hpp:257-310, mixing.hpp:258-318): every fit of the trace within
  1e-8, factors within 1e-6, final fit within 1e-3.
* C4 (1000^3, R=50, S=2000): the persistent CPRAND kernel teacher-forced mode
  by mode. The session runs one outer iteration per call; mode n of
  iteration k is recomputed by the oracle (skr + gather + pivoted-QR
  sampled_update + normalize_columns, sampling.hpp:281-290) from the GPU's
  own factors (modes < n of iteration k, modes > n of iteration k-1) and
  compared at 1e-10. Then 10 free-running iterations with the fit: final fit
  within 1e-3 of the oracle's.
* C5 (320^4, R=20, S=1200, DCT MIX, 84 GB): the device mixing pass checked
  pass by pass on 1000 random fibers per mode against the oracle's sign +
  DCT-II (mixing.hpp:130-156) at 1e-12; then the persistent CPRAND-MIX kernel
  teacher-forced mode by mode (mixing.hpp:284-298) from fibers of the mixed
  tensor read back by plain strided copies, at 1e-10.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 1


@pytest.fixture(scope="module")
def pb():
    import paper_1701_06600_b200 as pb
    assert pb.device_count() > 0, "GPU tests need a visible CUDA device"
    return pb


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def snapshots(pb, sess, iters):
    """(lambda, factors) after each of `iters` single-iteration runs."""
    out = []
    for _ in range(iters):
        assert sess.run(1) == 1
        res = sess.result()
        out.append((res.lam.copy(), [f.copy(order="F") for f in res.factors]))
    return out


def teacher_forced(orc, dims, r, seed, tables, init, snaps, fibers, mix=None):
    """Max relative difference of every mode update of every snapshot
    iteration against the oracle's update from the GPU's own inputs."""
    worst = 0.0
    prev = init
    for k, (lam_k, fs_k) in enumerate(snaps):
        for n in range(len(dims)):
            fs = [fs_k[m] if m < n else prev[1][m] for m in range(len(dims))]
            idx = tables[k][n]
            xs = fibers(n, idx)  # I_n x S
            if mix is None:
                zs = orc.skr(idx, fs, n)
                a = orc.sampled_update(zs, xs)
            else:
                mixed = [orc.mix_factor(f, dims, mix, seed, m) for m, f in enumerate(fs)]
                zs = orc.skr(idx, mixed, n)
                rhs = orc.unmix_sampled_rhs(np.asfortranarray(xs.T), dims, mix, seed, n)
                sol, _ = orc.least_squares(zs, rhs)
                a = np.asfortranarray(sol.T)
            f2 = list(fs)
            f2[n] = a
            want, wlam = orc.normalize_columns(f2, prev[0] if n == 0 else lam_k, n, n == 0,
                                               orc.Engine(seed, 8))
            d = rel(fs_k[n], want[n])
            worst = max(worst, d)
            assert d < 1e-10, f"iteration {k + 1} mode {n}: {d:.3e}"
            if n == len(dims) - 1:
                dl = rel(lam_k, wlam)
                assert dl < 1e-10, f"iteration {k + 1} lambda: {dl:.3e}"
        prev = (lam_k, fs_k)
    return worst


@pytest.mark.parametrize("cfg", [
    dict(name="c2", dims=(300, 300, 300), r=10, s=300, phat=1 << 14, c=0.5, eta=0.01, method="rand",
         transform=None),
    dict(name="c3", dims=(80, 80, 80, 80), r=10, s=300, phat=1 << 14, c=0.9, eta=0.01, method="mix",
         transform="dct"),
])
def test_config_free_running_matches_oracle(pb, orc, cfg):
    t = pb.DeviceTensor(cfg["dims"], device=0)
    t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
    x = t.download()
    t.close()
    opts = dict(rng_seed=SEED, max_iters=25, fit_sample_count=cfg["phat"], stall_limit=1000,
                transform=cfg["transform"])
    ref = orc.solve(cfg["method"], x, cfg["r"], cfg["s"], orc.SolveOptions(**opts))
    got = pb.solve(cfg["method"], x, cfg["r"], cfg["s"], pb.SolveOptions(**opts))
    assert got.iterations == ref.iterations == 25
    fg = np.array([tr[2] for tr in got.trace])
    fr = np.array([tr[2] for tr in ref.trace])
    assert np.max(np.abs(fg - fr)) < 1e-8, np.max(np.abs(fg - fr))
    assert abs(fg[-1] - fr[-1]) < 1e-3
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-6
    assert rel(got.lam, ref.lam) < 1e-6


def test_c4_persistent_kernel_teacher_forced_and_free_running(pb, orc):
    dims, r, s = (1000, 1000, 1000), 50, 2000
    t = pb.DeviceTensor(dims, device=0)
    t.synth(r, 0.9, 0.01, SEED)
    iters = 3
    sess = pb.Session("rand", t, r, s, pb.SolveOptions(rng_seed=SEED, max_iters=iters, bench_mode=True,
                                                       device=0))
    assert sess.fused, "C4 must run the persistent CPRAND kernel"
    snaps = snapshots(pb, sess, iters)
    # modes whose Gauss-Jordan pivots fell below kNeTol took the QR path
    print(f"C4: {sess.gram_fallbacks()} of {3 * iters} mode updates on the QR path")
    sess.close()
    x = t.download()
    tables = orc.sample_tables(dims, s, SEED, iters)
    init = orc.init_random(dims, r, SEED)
    worst = teacher_forced(orc, dims, r, SEED, tables, init, snaps,
                           lambda n, idx: orc.gather_fibers(x, n, idx))
    print(f"C4 teacher-forced worst relative difference {worst:.3e}")
    # free running with the sampled fit (P_hat = 2^16) and the stop rule
    opts = dict(rng_seed=SEED, max_iters=10, fit_sample_count=1 << 16, stall_limit=1000)
    sess = pb.Session("rand", t, r, s, pb.SolveOptions(device=0, **opts))
    sess.run(10)
    got = sess.result()
    sess.close()
    t.close()
    ref = orc.cprand(x, r, s, orc.SolveOptions(**opts))
    assert got.iterations == ref.iterations == 10
    fg = np.array([tr[2] for tr in got.trace])
    fr = np.array([tr[2] for tr in ref.trace])
    print(f"C4 free-running max trace difference {np.max(np.abs(fg - fr)):.3e}")
    assert abs(fg[-1] - fr[-1]) < 1e-3
    assert np.max(np.abs(fg - fr)) < 1e-6
    for a, b in zip(got.factors, ref.factors):
        assert rel(a, b) < 1e-4


def test_c5_mixing_pass_and_mix_kernel_teacher_forced(pb, orc):
    dims, r, s = (320, 320, 320, 320), 20, 1200
    t = pb.DeviceTensor(dims, device=0)
    t.synth(r, 0.5, 0.001, SEED)
    # ---- the whole-tensor pass, mode by mode, on 1000 random fibers per mode
    signs = orc.mixing_signs(dims, "dct", SEED)
    g = orc.Engine(77, raw=True)
    for m in range(4):
        idx = orc.draw_samples(g, dims, m, 1000)
        before = t.read_fibers(m, idx)
        t.mix_modes("dct", SEED, m, m + 1)
        after = t.read_fibers(m, idx)
        want = np.stack([orc.transform("dct", signs[m] * before[:, j]) for j in range(idx.shape[0])], axis=1)
        worst = max(np.linalg.norm(after[:, j] - want[:, j]) / np.linalg.norm(want[:, j])
                    for j in range(idx.shape[0]))
        print(f"C5 mixing pass mode {m}: worst fiber relative difference {worst:.3e}")
        assert worst < 1e-12, (m, worst)
    # ---- the persistent CPRAND-MIX kernel on a fresh tensor, mixed in place
    # by the session itself (x_mutable: no 84 GB private copy)
    t.synth(r, 0.5, 0.001, SEED)
    iters = 2
    sess = pb.Session("mix", t, r, s, pb.SolveOptions(rng_seed=SEED, max_iters=iters, bench_mode=True,
                                                      transform="dct", x_mutable=True, device=0))
    assert sess.fused, "C5 must run the persistent CPRAND-MIX kernel"
    snaps = snapshots(pb, sess, iters)
    print(f"C5: {sess.gram_fallbacks()} of {4 * iters} mode updates on the QR path")
    sess.close()
    tables = orc.sample_tables(dims, s, SEED, iters)
    init = orc.init_random(dims, r, SEED)
    worst = teacher_forced(orc, dims, r, SEED, tables, init, snaps, t.read_fibers, mix="dct")
    print(f"C5 MIX teacher-forced worst relative difference {worst:.3e}")
    t.close()
