"""Where repeated one-shot solves of one tensor diverge (relative differences per factor by iteration count; not part of the product)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1701_06600_b200 as pb
dims = (160, 230, 250)
n = int(np.prod(dims))
t = pb.DeviceTensor(dims); t.synth(6, 0.5, 0.01, 3)
buf = pb.PinnedBuffer(n); t.download_into(buf.array); t.close()
xh = buf.array.reshape(dims, order="F")
os.environ["CPRAND_SYNC_UPLOAD"] = "1"
for iters in (1, 2, 3, 6):
    res = [pb.solve("rand", xh, 6, 150, pb.SolveOptions(rng_seed=5, device=0, max_iters=iters, bench_mode=True)) for _ in range(4)]
    for j in range(1, 4):
        d = [float(np.max(np.abs(a - b) / (np.abs(b) + 1e-300))) for a, b in zip(res[j].factors, res[0].factors)]
        print(f"iters {iters}: run {j} vs 0: max rel diff per factor {['%.1e' % v for v in d]}, lam {float(np.max(np.abs(res[j].lam - res[0].lam))):.1e}")
