"""cprand_solve wall time on C1-C3 from a pinned host tensor (not part of the product)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_1701_06600_b200 as pb
for name in ("c1", "c2", "c3"):
    cfg = bench.CONFIGS[name]
    p = int(np.prod(cfg["dims"]))
    t = pb.DeviceTensor(cfg["dims"], device=0); t.synth(cfg["r"], cfg["c"], cfg["eta"], 1)
    buf = pb.PinnedBuffer(p); t.download_into(buf.array); t.close()
    xh = buf.array.reshape(cfg["dims"], order="F")
    eo = pb.SolveOptions(rng_seed=1, max_iters=100, bench_mode=True, transform=cfg["transform"], device=0)
    pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)
    out = []
    for k in range(4):
        t0 = time.perf_counter(); res = pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo); dt = time.perf_counter() - t0
        out.append(f"{1e3*dt:.2f} (setup {1e3*res.setup_seconds:.2f} loop {1e3*res.loop_seconds_device:.2f})")
    print(os.environ.get("CPRAND_LIB", "default"), name, "wall ms:", " | ".join(out), flush=True)
    buf.close()
