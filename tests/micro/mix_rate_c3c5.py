"""Bench-mode rate of the persistent CPRAND-MIX kernel on C3 (80^4, R = 10,
S = 300) and C5 (320^4, R = 20, S = 1200), event-timed (not part of the
product). CPRAND_LAZY_LAST=0 keeps the per-launch unmix for A/B."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

for dims, r, s, c, eta in (((80, 80, 80, 80), 10, 300, 0.9, 0.01), ((320, 320, 320, 320), 20, 1200, 0.5, 0.001)):
    t = pb.DeviceTensor(dims)
    t.synth(r, c, eta, 1)
    sess = pb.Session("mix", t, r, s, pb.SolveOptions(rng_seed=1, max_iters=230, bench_mode=True, transform="dct",
                                                      x_mutable=True))
    sess.run(5)
    ms = sess.timed_enqueue(200)
    res = sess.result()
    print(f"{dims} rate {200 / (ms * 1e-3):.0f} it/s ({1e3 * ms / 200:.1f} us/it), lambda[0] {res.lam[0]:.6e}", flush=True)
    sess.close()
    t.close()

# full loop (sampled fit + stop rule every iteration): the unmix runs in every launch
import time  # noqa: E402
for dims, r, s, c, eta, phat in (((80, 80, 80, 80), 10, 300, 0.9, 0.01, 1 << 14),
                                 ((320, 320, 320, 320), 20, 1200, 0.5, 0.001, 1 << 18)):
    t = pb.DeviceTensor(dims)
    t.synth(r, c, eta, 1)
    sess = pb.Session("mix", t, r, s, pb.SolveOptions(rng_seed=1, max_iters=220, transform="dct", x_mutable=True,
                                                      fit_sample_count=phat, stall_limit=1 << 30))
    sess.run(10)
    sess.sync()
    t0 = time.perf_counter()
    n = sess.run(200)
    dt = time.perf_counter() - t0
    print(f"{dims} full loop {n / dt:.0f} it/s, fit {sess.result().trace[-1][2]:.6f}", flush=True)
    sess.close()
    t.close()
