"""Launch targets for ncu captures (not part of the product).
  gather: C4 batched sampled-fiber gathers (gather_rows_kernel) from the
          tensor layout and from the mode-major replicas
  fit:    C4 multi-kernel chain with the sampled fit (estimate_fit_kernel)"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

what = sys.argv[1]
t = pb.DeviceTensor((1000, 1000, 1000))
t.synth(50, 0.9, 0.01, 1)
if what == "gather":
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=20, bench_mode=True))
    for rep in (False, True):
        ms, bu, bm = s.gather_bench(10, rep)
        print(f"replicas={rep}: {ms:.3f} ms, useful {bu / ms / 1e6:.0f} GB/s, B_min {bm / ms / 1e6:.0f} GB/s")
else:
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=20, fused=0, stall_limit=1 << 30,
                                                       fit_sample_count=1 << 16))
    s.run(6)
s.close()
