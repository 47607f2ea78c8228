"""Workload for the device-check build (libcprand_b200_check.so: bounds
asserts on the sampled reads and the apply rows, a 5 s time-out on the
persistent kernels' flag waits; a failed check traps with a message). Run by
tests/test_gpu_checked.py in a subprocess with CPRAND_LIB pointing at that
library. Every path is also compared with the oracle, as in the product
tests. Prints CHECKED OK at the end."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import oracle as orc  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402
from paper_1701_06600_b200 import shard  # noqa: E402

assert pb._lib.LIB_PATH.endswith("libcprand_b200_check.so"), pb._lib.LIB_PATH


def trace_diff(a, b):
    return max(abs(p[2] - q[2]) for p, q in zip(a.trace, b.trace))


def solve_both(method, x, r, s, **kw):
    base = dict(rng_seed=7, max_iters=6, stall_limit=1000)
    base.update(kw)
    fused = base.pop("fused", -1)
    got = pb.solve(method, x, r, s, pb.SolveOptions(fused=fused, **base))
    ref = orc.solve(method, x, r, s, orc.SolveOptions(**base))
    d = trace_diff(got, ref)
    assert d < 1e-8, (method, x.shape, r, s, d)
    print(f"{method:6s} {str(x.shape):20s} R={r:3d} S={s:4d} fused={fused:2d} trace diff {d:.1e}", flush=True)


# persistent CPRAND kernel: RT = 16 / 32 / 64, one and several row blocks and splits
for dims, r, s in (((40, 40, 40), 5, 100), ((200, 90, 61), 20, 500), ((64, 64, 64), 50, 900)):
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 3)
    solve_both("rand", x, r, s)
# persistent CPRAND-MIX kernel and the chain
x, _ = orc.gen_baseline((16, 12, 10, 8), 3, 0.9, 0.01, 5)
solve_both("mix", x, 3, 60, transform="dct")
x, _ = orc.gen_baseline((30, 28, 26), 6, 0.5, 0.01, 4)
solve_both("rand", x, 6, 120, fused=0)
# wide ranks (chain, RT = 128)
x, _ = orc.gen_baseline((90, 80, 70), 80, 0.0, 0.01, 31)
solve_both("rand", x, 80, 400)
# rank-deficient systems: the QR path in the persistent kernel (R above the data's rank)
x, _ = orc.gen_baseline((30, 28, 26), 2, 0.0, 0.0, 8)
res = pb.cprand(x, 4, 60, pb.SolveOptions(rng_seed=8, max_iters=4, stall_limit=1000))
assert np.all(np.isfinite(res.lam)) and all(np.all(np.isfinite(f)) for f in res.factors)
print("rank-deficient run finite", flush=True)


# the peer kernel: P rank groups of one launch exchanging through each other's buffers
def peer(x, r, s, nranks, method="rand", **kw):
    group = pb.LoopbackGroup(nranks)
    out = [None] * nranks
    total = x.shape[-1]

    def work(rank):
        comm = pb.Comm.loopback(group, rank, 0)
        off, ln = shard.slab(total, nranks, rank)
        t = pb.DeviceTensor(list(x.shape[:-1]) + [ln], device=0)
        if ln:
            t.upload(np.asfortranarray(x[..., off:off + ln]))
        sess = pb.Session(method, t, r, s, pb.SolveOptions(rng_seed=7, max_iters=6, stall_limit=1000, comm=comm,
                                                            shard_total=total, device=0, **kw))
        assert sess.fused
        sess.run(6)
        out[rank] = sess.result()
        sess.close()
        t.close()
        comm.close()

    ts = [threading.Thread(target=work, args=(q,)) for q in range(nranks)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    group.close()
    ref = orc.solve(method, x, r, s, orc.SolveOptions(rng_seed=7, max_iters=6, stall_limit=1000, **kw))
    d = trace_diff(out[0], ref)
    assert d < 1e-8, d
    print(f"peer {method} P={nranks} {x.shape} trace diff {d:.1e}", flush=True)


x, _ = orc.gen_baseline((24, 20, 23), 4, 0.5, 0.01, 11)
peer(x, 4, 60, 2)
peer(x, 4, 60, 3)
x, _ = orc.gen_baseline((130, 70, 90), 12, 0.5, 0.01, 21)
peer(x, 12, 400, 3)
x, _ = orc.gen_baseline((40, 36, 30, 33), 10, 0.5, 0.01, 13)
peer(x, 10, 300, 2, method="mix", transform="dct")
print("CHECKED OK", flush=True)
