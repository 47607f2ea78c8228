"""C4 bench-mode rate: persistent kernel vs multi-kernel chain vs single-rank
sharded (NCCL) path (not part of the product)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402

dims, r, s = (1000, 1000, 1000), 50, 2000
comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
t = pb.DeviceTensor(dims)
t.synth_slab(r, 0.9, 0.01, 1, dims[-1], comm)
for label, kw in [("fused", {}), ("chain", dict(fused=0)), ("sharded-1", dict(comm=comm, shard_total=dims[-1]))]:
    sess = pb.Session("rand", t, r, s, pb.SolveOptions(rng_seed=1, max_iters=400, bench_mode=True, **kw))
    sess.run(20)
    sess.sync()
    ms = sess.timed_enqueue(200)
    print(label, f"{200 / (ms * 1e-3):.0f} it/s", flush=True)
    if label != "fused":
        sess.set_kernel_timing(True)
        sess.enqueue(20)
        sess.sync()
        kinds = ["gather", "rhs_gemm", "z", "gram", "gram_inverse", "apply"]
        print("  us/launch by mode:", {k: [round(x[1] / x[0] * 1e3, 1) if x[0] else None for x in
                                              [sess.kernel_stats(m, i) for m in range(3)]] for i, k in enumerate(kinds)}, flush=True)
    sess.close()
comm.close()
