"""Small runs of the persistent kernels (CPRAND, CPRAND-MIX DCT), the
multi-kernel chain and the peer kernel (2 loopback ranks) for
compute-sanitizer (not part of the product):
  compute-sanitizer --tool memcheck python tests/micro/sanitize_small.py"""
import os
import sys
import threading
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402
from paper_1701_06600_b200 import shard  # noqa: E402

rng = np.random.default_rng(3)
x = np.asfortranarray(rng.standard_normal((24, 20, 22)))
for method, kw in (("rand", {}), ("rand", {"fused": 0}), ("mix", {"transform": "dct"})):
    res = pb.solve(method, x, 4, 60, pb.SolveOptions(rng_seed=3, max_iters=4, stall_limit=100, **kw))
    print(method, kw, res.iterations, res.trace[-1][2], flush=True)

group = pb.LoopbackGroup(2)
out = [None, None]


def work(rank):
    comm = pb.Comm.loopback(group, rank, 0)
    off, ln = shard.slab(22, 2, rank)
    t = pb.DeviceTensor([24, 20, ln], device=0)
    t.upload(np.asfortranarray(x[..., off:off + ln]))
    s = pb.Session("rand", t, 4, 60, pb.SolveOptions(rng_seed=3, max_iters=4, stall_limit=100, comm=comm,
                                                      shard_total=22, device=0))
    s.run(4)
    out[rank] = (s.fused, s.result().trace[-1][2])
    s.close()
    t.close()
    comm.close()


ts = [threading.Thread(target=work, args=(q,)) for q in range(2)]
for th in ts:
    th.start()
for th in ts:
    th.join()
group.close()
print("peer", out, flush=True)
