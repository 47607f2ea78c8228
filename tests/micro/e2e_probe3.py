"""Fresh-session per-iteration times with the tensor resident (not part of the product)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1701_06600_b200 as pb
t = pb.DeviceTensor((1000, 1000, 1000), device=0); t.synth(50, 0.9, 0.01, 1)
s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=300, bench_mode=True, device=0))
ms = [s.timed_enqueue(1) for _ in range(120)]
print("per-iteration us:", [round(1e3 * m) for m in ms], flush=True)
print("info", s.gram_fallbacks() if hasattr(s, "gram_fallbacks") else None)
