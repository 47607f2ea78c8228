"""Where the e2e time of cprand_solve goes (not part of the product): C4-sized
host tensor in pinned memory, one-shot solves with per-phase timings, with and
without another device tensor alive. python tests/micro/e2e_probe.py [c4]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
dims = list(cfg["dims"])
p = int(np.prod(dims))
t = pb.DeviceTensor(dims, device=0)
t.synth(cfg["r"], cfg["c"], cfg["eta"], 1)
buf = pb.PinnedBuffer(p)
t0 = time.perf_counter()
t.download_into(buf.array)
print(f"download_into: {time.perf_counter() - t0:.3f} s")
xh = buf.array.reshape(dims, order="F")
eo = pb.SolveOptions(rng_seed=1, max_iters=100, bench_mode=True, transform=cfg["transform"], device=0)


def solve(tag):
    t0 = time.perf_counter()
    res = pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)
    dt = time.perf_counter() - t0
    print(f"{tag}: wall {dt:.3f} s  setup {res.setup_seconds:.3f}  total {res.total_seconds:.3f}  "
          f"loop(dev) {res.loop_seconds_device:.4f}")


for k in range(3):
    solve(f"t alive #{k}")
t.close()
for k in range(3):
    solve(f"t closed #{k}")
t = pb.DeviceTensor(dims, device=0)
t.mix("dct", 1)
for k in range(2):
    solve(f"after mix pass #{k}")
