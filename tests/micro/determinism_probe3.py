"""Repeatability of a small bench-mode session after a C4-sized one in the
same process: QR-path count and a digest of the factors per run (not part of
the product)."""
import os, sys, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1701_06600_b200 as pb
t = pb.DeviceTensor((1000, 1000, 1000)); t.synth(50, 0.9, 0.01, 1)
s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=40, bench_mode=True)); s.run(30); s.close(); t.close()
dims = (160, 230, 250)
t = pb.DeviceTensor(dims); t.synth(6, 0.5, 0.01, 3)
for iters in (3, 4, 5, 8):
    out = []
    for k in range(5):
        s = pb.Session("rand", t, 6, 150, pb.SolveOptions(rng_seed=5, max_iters=iters, bench_mode=True))
        s.run(iters)
        r = s.result()
        h = hashlib.md5(b"".join(np.ascontiguousarray(f).tobytes() for f in r.factors)).hexdigest()[:6]
        out.append(f"{h}/{s.gram_fallbacks()}")
        s.close()
    print(f"iters {iters}: digest/QR-modes per run: {out}", flush=True)
