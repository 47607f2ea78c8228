"""cprand_solve with a pinned host tensor uploads it in parts along the last
mode while the session sets up (capi.cu, Tensor::chunk_ev; each part's share of
the mode-major replicas is built as it arrives). The result must be the one
the synchronous upload gives, bit for bit, on every path, and match the
oracle's trace (cprand, sampling.hpp:257-310)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

pytestmark = pytest.mark.gpu


def _solve_both(method, dims, r, s, **kw):
    import paper_1701_06600_b200 as pb
    n = int(np.prod(dims))
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.5, 0.01, 3)
    buf = pb.PinnedBuffer(n)
    t.download_into(buf.array)
    t.close()
    xh = buf.array.reshape(dims, order="F")
    out = []
    os.environ["CPRAND_UPLOAD_PARTS"] = "7"
    for sync in ("1", None):
        if sync:
            os.environ["CPRAND_SYNC_UPLOAD"] = sync
        else:
            os.environ.pop("CPRAND_SYNC_UPLOAD", None)
        out.append(pb.solve(method, xh, r, s, pb.SolveOptions(rng_seed=5, device=0, **kw)))
    os.environ.pop("CPRAND_UPLOAD_PARTS", None)
    return xh, buf, out


@pytest.mark.parametrize("dims", [(160, 230, 250), (96, 40, 50, 61)])
@pytest.mark.parametrize("bench_mode", [True, False])
def test_pipelined_upload_matches_synchronous_rand(dims, bench_mode):
    # 73.6 MB / 93.7 MB: above the 64 MB threshold, last modes that do not divide into the parts
    kw = dict(max_iters=6, bench_mode=bench_mode)
    if not bench_mode:
        kw.update(fit_sample_count=4096, stall_limit=1000)
    xh, buf, (a, b) = _solve_both("rand", dims, 6, 150, **kw)
    assert np.array_equal(a.lam, b.lam)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    if not bench_mode:
        assert [x[2] for x in a.trace] == [x[2] for x in b.trace]
        import oracle as orc
        ref = orc.cprand(xh, 6, 150, orc.SolveOptions(rng_seed=5, max_iters=6, fit_sample_count=4096, stall_limit=1000))
        assert max(abs(x[2] - y[2]) for x, y in zip(b.trace, ref.trace)) < 1e-8
    buf.close()


def test_pipelined_upload_matches_synchronous_mix():
    xh, buf, (a, b) = _solve_both("mix", (128, 256, 270), 5, 120, max_iters=5, bench_mode=True, transform="dct")
    assert np.array_equal(a.lam, b.lam)
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    buf.close()


def test_repeated_solves_are_bitwise_equal():
    """The default path is bitwise repeatable: four one-shot solves of one
    tensor in one process (sessions reuse each other's cached device and
    pinned blocks) return identical factors."""
    import paper_1701_06600_b200 as pb
    dims = (160, 230, 250)
    t = pb.DeviceTensor(dims)
    t.synth(6, 0.5, 0.01, 3)
    buf = pb.PinnedBuffer(int(np.prod(dims)))
    t.download_into(buf.array)
    t.close()
    xh = buf.array.reshape(dims, order="F")
    os.environ["CPRAND_SYNC_UPLOAD"] = "1"
    try:
        res = [pb.solve("rand", xh, 6, 150, pb.SolveOptions(rng_seed=5, device=0, max_iters=8, bench_mode=True))
               for _ in range(4)]
    finally:
        os.environ.pop("CPRAND_SYNC_UPLOAD", None)
    for r in res[1:]:
        assert np.array_equal(r.lam, res[0].lam)
        for fa, fb in zip(r.factors, res[0].factors):
            assert np.array_equal(fa, fb)
    buf.close()
