"""Full-loop C4 session on the multi-kernel chain (estimate_fit_kernel runs
standalone), for ncu (not part of the product)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

t = pb.DeviceTensor((1000, 1000, 1000))
t.synth(50, 0.9, 0.01, 1)
s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=8, stall_limit=1 << 30, fused=0,
                                                    fit_sample_count=65536))
s.run(8)
print("done", s.result().trace[-1])
