"""Per-launch time of the persistent CPRAND kernel with and without the
sampled fit (not part of the product): C4, bench mode vs full loop at
several fit sample counts."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

cfg = dict(dims=(1000, 1000, 1000), r=50, s=2000)
t = pb.DeviceTensor(cfg["dims"])
t.synth(50, 0.9, 0.01, 1)
for label, kw in [("bench", dict(bench_mode=True)), ("fit 65536", dict(fit_sample_count=65536)),
                  ("fit 4096", dict(fit_sample_count=4096)), ("fit 256", dict(fit_sample_count=256))]:
    s = pb.Session("rand", t, cfg["r"], cfg["s"], pb.SolveOptions(rng_seed=1, max_iters=80, stall_limit=1 << 30, **kw))
    s.run(10)
    s.set_kernel_timing(True)
    s.run(40) if not kw.get("bench_mode") else (s.enqueue(40), s.sync())
    n, ms, _ = s.kernel_stats(0, 7)
    print(f"{label:10s} launches {n} us/launch {1e3 * ms / max(n, 1):.1f}", flush=True)
    print("   phases", [round(v, 2) for v in s.phase_us()], flush=True)
    s.close()
