"""Bitwise repeatability of cprand_solve on one tensor: two synchronous and two
pipelined uploads, all pairs compared (not part of the product). Optional
argument: warm (run a C4-sized session first, as the config tests do)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1701_06600_b200 as pb
if len(sys.argv) > 1:
    t = pb.DeviceTensor((1000, 1000, 1000)); t.synth(50, 0.9, 0.01, 1)
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=20, bench_mode=True)); s.run(10); s.close(); t.close()
    t = pb.DeviceTensor((320, 320, 320, 320)); t.synth(20, 0.5, 0.001, 1)
    s = pb.Session("mix", t, 20, 1200, pb.SolveOptions(rng_seed=1, max_iters=5, bench_mode=True, transform="dct", x_mutable=True)); s.run(2); s.close(); t.close()
dims = (160, 230, 250)
n = int(np.prod(dims))
t = pb.DeviceTensor(dims); t.synth(6, 0.5, 0.01, 3)
buf = pb.PinnedBuffer(n); t.download_into(buf.array); t.close()
xh = buf.array.reshape(dims, order="F")
os.environ["CPRAND_UPLOAD_PARTS"] = "7"
res = []
for sync in ("1", "1", None, None, "1", None):
    if sync: os.environ["CPRAND_SYNC_UPLOAD"] = sync
    else: os.environ.pop("CPRAND_SYNC_UPLOAD", None)
    r = pb.solve("rand", xh, 6, 150, pb.SolveOptions(rng_seed=5, device=0, max_iters=6, bench_mode=True))
    res.append((sync, r))
for i in range(len(res)):
    print(i, "sync" if res[i][0] else "pipe", ["=" if all(np.array_equal(a, b) for a, b in zip(res[i][1].factors, res[j][1].factors)) else "x" for j in range(len(res))],
          "fallbacks", getattr(res[i][1], "gram_fallbacks", None))
