"""Bench-mode iters/s of CPRAND-MIX with the FFT kind (cfft.cu chain) vs DCT
on the C3 and C2 shapes (not part of the product)."""
import os
import sys
import time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

for dims, r, s in [((80, 80, 80, 80), 10, 300), ((300, 300, 300), 10, 300)]:
    t = pb.DeviceTensor(dims)
    t.synth(r, 0.9, 0.01, 1)
    for tr in ("dct", "fft"):
        t0 = time.perf_counter()
        sess = pb.Session("mix", t, r, s, pb.SolveOptions(rng_seed=1, max_iters=400, bench_mode=True, transform=tr))
        setup = time.perf_counter() - t0
        sess.run(20)
        sess.sync()
        ms = sess.timed_enqueue(200)
        print(dims, tr, f"setup {setup:.3f} s  {200 / (ms * 1e-3):.0f} it/s", flush=True)
        sess.close()
    t.close()
