"""Rate of the slab-sharded CPRAND path on C4 (1000^3, R=50, S=2000, bench
mode) on one B200 (not part of the product):
  * one rank over NCCL (the peer kernel with np = 1, IPC mapping of itself),
  * the chain (fused=0) with one NCCL rank, for comparison,
  * P = 2 / 4 loopback ranks (rank groups of one cooperative launch on the one
    device: exercises the exchange at scale; it splits one GPU's SMs, so it is
    not a scaling measurement)."""
import sys
import os
import threading
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1701_06600_b200 as pb  # noqa: E402
from paper_1701_06600_b200 import shard  # noqa: E402

DIMS, R, S = (1000, 1000, 1000), 50, 2000
ITERS = 200


def one_rank(fused):
    comm = pb.Comm(pb.Comm.unique_id(), 0, 1, 0)
    t = pb.DeviceTensor(DIMS)
    t.synth(R, 0.9, 0.01, 1)
    s = pb.Session("rand", t, R, S, pb.SolveOptions(rng_seed=1, max_iters=ITERS + 10, bench_mode=True, comm=comm,
                                                      shard_total=DIMS[-1], fused=fused))
    s.run(5)
    ms = s.timed_enqueue(ITERS)
    print(f"1 rank NCCL, {'peer kernel' if s.fused else 'chain'}: {ITERS / (ms * 1e-3):.0f} it/s "
          f"({1e3 * ms / ITERS:.1f} us/it)", flush=True)
    s.close()
    t.close()
    comm.close()


def loopback(nranks):
    group = pb.LoopbackGroup(nranks)
    out = [None] * nranks

    def work(rank):
        comm = pb.Comm.loopback(group, rank, 0)
        off, ln = shard.slab(DIMS[-1], nranks, rank)
        t = pb.DeviceTensor(list(DIMS[:-1]) + [ln])
        t.synth_slab(R, 0.9, 0.01, 1, DIMS[-1], comm)
        s = pb.Session("rand", t, R, S, pb.SolveOptions(rng_seed=1, max_iters=ITERS + 10, bench_mode=True,
                                                          comm=comm, shard_total=DIMS[-1]))
        s.run(5)
        ms = s.timed_enqueue(ITERS)
        out[rank] = (ms, s.fused)
        s.close()
        t.close()
        comm.close()

    ts = [threading.Thread(target=work, args=(q,)) for q in range(nranks)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    group.close()
    ms = max(o[0] for o in out)
    print(f"{nranks} loopback ranks on one GPU (peer kernel: {out[0][1]}): {ITERS / (ms * 1e-3):.0f} it/s", flush=True)


if __name__ == "__main__":
    one_rank(-1)
    one_rank(0)
    for p in (2, 4):
        loopback(p)
