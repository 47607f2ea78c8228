"""A/B rates of the persistent kernels (not part of the product): C4 CPRAND
bench mode and full loop, C3 / C5 CPRAND-MIX bench mode and full loop, all
event- or wall-timed on one box. Select a library variant with CPRAND_LIB
(tools/build_variant.sh). Arguments: any of c4 c3 c5 (default all)."""
import os
import sys
import time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

which = sys.argv[1:] or ["c4", "c3", "c5"]
out = []
if "c4" in which:
    t = pb.DeviceTensor((1000, 1000, 1000))
    t.synth(50, 0.9, 0.01, 1)
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=400, bench_mode=True))
    s.run(5)
    ms = min(s.timed_enqueue(100) for _ in range(3))
    out.append(f"c4 bench {100 / (ms * 1e-3):.0f}")
    s.close()
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=420, fit_sample_count=1 << 16,
                                                        stall_limit=1 << 30, fit_threshold=2.0))
    s.run(10)
    s.sync()
    t0 = time.perf_counter()
    n = s.run(300)
    dt = time.perf_counter() - t0
    out.append(f"c4 full {n / dt:.0f}")
    s.close()
    t.close()
for name, dims, r, sm, c, eta, phat in (("c3", (80, 80, 80, 80), 10, 300, 0.9, 0.01, 1 << 14),
                                        ("c5", (320, 320, 320, 320), 20, 1200, 0.5, 0.001, 1 << 18)):
    if name not in which:
        continue
    t = pb.DeviceTensor(dims)
    t.synth(r, c, eta, 1)
    s = pb.Session("mix", t, r, sm, pb.SolveOptions(rng_seed=1, max_iters=330, bench_mode=True, transform="dct",
                                                    x_mutable=True))
    s.run(5)
    ms = min(s.timed_enqueue(100) for _ in range(3))
    out.append(f"{name} bench {100 / (ms * 1e-3):.0f}")
    s.close()
    t.close()
    t = pb.DeviceTensor(dims)
    t.synth(r, c, eta, 1)
    s = pb.Session("mix", t, r, sm, pb.SolveOptions(rng_seed=1, max_iters=220, transform="dct", x_mutable=True,
                                                    fit_sample_count=phat, stall_limit=1 << 30, fit_threshold=2.0))
    s.run(10)
    s.sync()
    t0 = time.perf_counter()
    n = s.run(200)
    dt = time.perf_counter() - t0
    out.append(f"{name} full {n / dt:.0f}")
    s.close()
    t.close()
print(os.environ.get("CPRAND_LIB", "default"), " | ".join(out), flush=True)
