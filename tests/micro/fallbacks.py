import sys, json
sys.path.insert(0, '.')
import paper_1701_06600_b200 as pb
t = pb.DeviceTensor([1000,1000,1000], device=0)
t.synth(50, 0.9, 0.01, 1)
for fused in (1, 0):
    s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=200, bench_mode=True, device=0, fused=fused))
    out = []
    done = 0
    for k in (1, 2, 5, 10, 20, 50, 100, 200):
        s.run(k - done); done = k
        out.append((k, s.gram_fallbacks()))
    print("fused", fused, out, flush=True)
