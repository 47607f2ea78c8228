"""Shape / rank / sample-count sweep of the device execution paths.

The persistent kernels (CPRAND: fused_rand_kernel; CPRAND-MIX:
fused_iteration_kernel) against the multi-kernel chain on the same session
inputs, over the edges of their tilings: ranks 1 / 8 / 9 / 33 / 64 (one,
exactly one, just over one 8 x 8 Gram block; the RT = 64 maximum), more
tiles than CTAs (S far above a tile's Z capacity), orders 3-5, mode lengths
below, at and just over the 64-row tile, and the fixed-order vs atomic Gram.
The chain itself is checked against the oracle in test_gpu_parity.py.
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


CASES = [
    ((40, 30, 20), 1, 50),
    ((64, 65, 63), 8, 200),
    ((129, 70, 90), 9, 400),
    ((200, 150, 100), 33, 3000),
    ((300, 64, 64), 64, 4000),
    ((150, 140, 130), 64, 9000),
    ((20, 18, 16, 14), 5, 300),
    ((12, 11, 10, 9, 8), 4, 500),
]


def _run(pb, method, t, r, s, iters, **kw):
    base = dict(rng_seed=41, max_iters=iters, stall_limit=1000, bench_mode=True)
    if method == "mix":
        base["transform"] = "dct"
    base.update(kw)
    sess = pb.Session(method, t, r, s, pb.SolveOptions(**base))
    sess.run(iters)
    res = sess.result()
    sess.close()
    return res


@pytest.mark.parametrize("dims,r,s", CASES)
@pytest.mark.parametrize("method", ["rand", "mix"])
def test_persistent_kernel_matches_chain(pb, dims, r, s, method):
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.5, 0.01, 41)
    fused = _run(pb, method, t, r, s, 4)
    chain = _run(pb, method, t, r, s, 4, fused=0)
    variants = [fused]
    if method == "rand":
        variants.append(_run(pb, method, t, r, s, 4, atomic_gram=True))
    t.close()
    for res in variants:
        assert np.all(np.isfinite(res.lam))
        np.testing.assert_allclose(res.lam, chain.lam, rtol=1e-8)
        for a, b in zip(res.factors, chain.factors):
            assert rel(a, b) < 1e-8
