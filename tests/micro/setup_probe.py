"""Session setup timeline on a resident C4 tensor, full loop (fit + stop rule):
CPRAND_DEBUG_SETUP=2 prints host times, =1 times after a stream synchronize
(not part of the product)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1701_06600_b200 as pb
t = pb.DeviceTensor((1000, 1000, 1000), device=0); t.synth(50, 0.9, 0.01, 1)
for k in range(3):
    t0 = time.perf_counter()
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=200, fit_sample_count=1 << 16, fit_threshold=0.988, device=0))
    t1 = time.perf_counter()
    n = s.run(200)
    t2 = time.perf_counter()
    print(f"setup {1e3*(t1-t0):.2f} ms, run {n} iterations {1e3*(t2-t1):.2f} ms", flush=True)
    s.close()
