import sys, os, faulthandler, numpy as np
faulthandler.enable()
H = os.path.dirname(os.path.abspath(__file__))
for p in (os.path.join(H, ".."), os.path.join(H, "..", ".."), os.path.join(H, "..", "..", "oracle")):
    sys.path.insert(0, p)
import oracle as orc, paper_1701_06600_b200 as pb
import test_gpu_loopback as T
nr, dims = int(sys.argv[1]), tuple(int(v) for v in sys.argv[2].split(","))
method = sys.argv[3] if len(sys.argv) > 3 else "rand"
tr = sys.argv[4] if len(sys.argv) > 4 else None
r, s = 4, 60
x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 11)
kw = dict(rng_seed=11, max_iters=10, stall_limit=1000, transform=tr)
print("start", nr, dims, method, flush=True)
res = T.sharded_solve(pb, x, method, r, s, nr, **kw)
print("sharded done", [q.iterations for q in res], flush=True)
T.check_against_unsharded(pb, x, method, r, s, res, **kw)
print("OK", flush=True)
