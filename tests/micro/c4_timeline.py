"""C4 persistent CPRAND kernel: event-timed rate and (CPRAND_DEBUG_CTA=1) the
per-CTA timeline of mode 1 (not part of the product)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

t = pb.DeviceTensor((1000, 1000, 1000))
t.synth(50, 0.9, 0.01, 1)
ga = len(sys.argv) > 1 and sys.argv[1] == "ga"
s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=400, bench_mode=True, atomic_gram=ga))
s.run(5)
ms = s.timed_enqueue(200)
print(f"rate {200 / (ms * 1e-3):.0f} it/s, {1e3 * ms / 200:.1f} us/it", flush=True)
s.set_kernel_timing(True)
s.enqueue(6)
s.sync()
print("phases", [round(v, 2) for v in s.phase_us()], flush=True)
s.close()
