"""cprand_solve from a pinned host tensor (C4): wall / setup / loop per call and, with
CPRAND_DEBUG_SETUP=2, the host-side setup timeline against the upload (not part of the product)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_1701_06600_b200 as pb
cfg = bench.CONFIGS["c4"]
dims = list(cfg["dims"]); p = int(np.prod(dims))
t = pb.DeviceTensor(dims, device=0); t.synth(cfg["r"], cfg["c"], cfg["eta"], 1)
buf = pb.PinnedBuffer(p); t.download_into(buf.array); t.close()
xh = buf.array.reshape(dims, order="F")
eo = pb.SolveOptions(rng_seed=1, max_iters=100, bench_mode=True, device=0)
for k in range(3):
    if k == 2: os.environ["CPRAND_DEBUG_SETUP"] = "2"
    t0 = time.perf_counter(); res = pb.solve("rand", xh, 50, 2000, eo); dt = time.perf_counter() - t0
    print(f"wall {dt:.4f} setup {res.setup_seconds:.4f} loop {res.loop_seconds_device:.4f}", flush=True)
