"""Session setup breakdown (CPRAND_DEBUG_SETUP=1) for the bench configs (not part of the product)."""
import os
import sys
import time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402

for name in sys.argv[1:] or ["c4"]:
    cfg = bench.CONFIGS[name]
    t = pb.DeviceTensor(cfg["dims"])
    t.synth(cfg["r"], cfg["c"], cfg["eta"], 1)
    for k in range(2):
        t0 = time.perf_counter()
        s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"],
                       pb.SolveOptions(rng_seed=1, fit_threshold=0.99, fit_sample_count=cfg["phat"],
                                       transform=cfg["transform"], x_mutable=name == "c5"))
        print(name, f"session ctor wall {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
        s.close()
        if name == "c5":
            t.synth(cfg["r"], cfg["c"], cfg["eta"], 1)
    t.close()
