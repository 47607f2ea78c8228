"""C3 CPRAND-MIX bench-mode iterations on the persistent MIX kernel (for ncu; not part of the product)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

t = pb.DeviceTensor((80, 80, 80, 80))
t.synth(10, 0.9, 0.01, 1)
s = pb.Session("mix", t, 10, 300, pb.SolveOptions(rng_seed=1, max_iters=20, bench_mode=True, transform="dct"))
s.run(20)
s.sync()
print("ok")
