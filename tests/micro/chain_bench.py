import sys; sys.path.insert(0, '.')
import paper_1701_06600_b200 as pb
t = pb.DeviceTensor((1000, 1000, 1000)); t.synth(50, 0.9, 0.01, 1)
s = pb.Session("rand", t, 50, 2000, pb.SolveOptions(rng_seed=1, max_iters=20, bench_mode=True, fused=int(sys.argv[1])))
s.run(3); print(s.timed_enqueue(10) / 10)
