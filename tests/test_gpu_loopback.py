"""The product's slab-sharded path at P = 2, 3, 4 ranks on
one GPU, through loopback communicators (comm.hpp): every rank is a host
thread of this process with its own slab tensor and session; the
collectives (RHS allreduce, last-mode allgather, column sums of squares,
fit-value allreduce, the distributed mixing pass's block exchange) meet at
host barriers and sum in rank order. The same session code runs over NCCL
with one process per GPU (bench.py --gpus N).

Checked against the unsharded session (1e-10) and between ranks (bitwise:
every rank must hold the same replicated model), including last modes that
P does not divide and a rank whose slab is empty.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_1701_06600_b200 as pb
    assert pb.device_count() > 0, "GPU tests need a visible CUDA device"
    return pb


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def run_ranks(pb, nranks, body, timeout=600):
    """body(rank, comm) on nranks threads of a loopback group."""
    group = pb.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []

    def work(rank):
        comm = pb.Comm.loopback(group, rank, 0)
        try:
            out[rank] = body(rank, comm)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append((rank, e))
        finally:
            comm.close()

    ts = [threading.Thread(target=work, args=(q,), daemon=True) for q in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a rank did not finish (collective mismatch?)"
    if errs:
        raise errs[0][1]
    group.close()
    return out


def sharded_solve(pb, x, method, r, s, nranks, expect_fused=None, **kw):
    """expect_fused: assert that every rank's session runs (True) or does not
    run (False) the peer kernel (the persistent CPRAND kernel exchanging the
    RHS rows / last-mode slabs through peer memory)."""
    from paper_1701_06600_b200 import shard
    total = x.shape[-1]

    def body(rank, comm):
        off, ln = shard.slab(total, nranks, rank)
        t = pb.DeviceTensor(list(x.shape[:-1]) + [ln], device=0)
        if ln:
            t.upload(np.asfortranarray(x[..., off:off + ln]))
        sess = pb.Session(method, t, r, s, pb.SolveOptions(comm=comm, shard_total=total, device=0, **kw))
        if expect_fused is not None:
            assert sess.fused == expect_fused
        sess.run(kw["max_iters"])
        res = sess.result()
        sess.close()
        t.close()
        return res

    return run_ranks(pb, nranks, body)


def check_against_unsharded(pb, x, method, r, s, results, **kw):
    t = pb.DeviceTensor(x.shape, device=0)
    t.upload(x)
    kw = {k: v for k, v in kw.items() if k != "fused"}
    full = pb.Session(method, t, r, s, pb.SolveOptions(fused=0, device=0, **kw))
    full.run(kw["max_iters"])
    ref = full.result()
    full.close()
    t.close()
    first = results[0]
    for res in results:
        # replicated model: bit-identical on every rank
        assert np.array_equal(res.lam, first.lam)
        for a, b in zip(res.factors, first.factors):
            assert np.array_equal(a, b)
        assert res.iterations == ref.iterations and res.reason == ref.reason
        assert [tr[2] for tr in res.trace] == [tr[2] for tr in first.trace]
    for a, b in zip(first.factors, ref.factors):
        assert rel(a, b) < 1e-10
    assert rel(first.lam, ref.lam) < 1e-10
    if ref.trace:
        assert max(abs(a[2] - b[2]) for a, b in zip(first.trace, ref.trace)) < 1e-10
    return ref


@pytest.mark.parametrize("fused", [-1, 0])
@pytest.mark.parametrize("nranks,dims", [(2, (24, 20, 22)), (3, (24, 20, 23)), (4, (24, 20, 23)),
                                         (4, (24, 20, 5))])
def test_loopback_sharded_cprand(pb, orc, nranks, dims, fused):
    """Modes < N-1: local-sample RHS summed over the ranks; mode N-1: slab
    rows, column sums of squares over the ranks, slabs gathered (23 % 3,
    23 % 4 != 0; last dim 5 over 4 ranks leaves rank 3 with an empty slab).
    fused=-1: the peer kernel (every rank a group of one cooperative launch,
    exchanging through each other's buffers); fused=0: the multi-kernel
    chain with the loopback collectives."""
    r, s = 4, 60
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 11)
    kw = dict(rng_seed=11, max_iters=10, stall_limit=1000, fused=fused)
    res = sharded_solve(pb, x, "rand", r, s, nranks, expect_fused=(fused != 0), **kw)
    check_against_unsharded(pb, x, "rand", r, s, res, **kw)
    kw.pop("fused")
    o = orc.cprand(x, r, s, orc.SolveOptions(**kw))
    assert max(abs(a[2] - b[2]) for a, b in zip(res[0].trace, o.trace)) < 1e-8


@pytest.mark.parametrize("nranks,dims,r,s", [(2, (200, 90, 61), 20, 500), (3, (130, 70, 90), 12, 400),
                                             (4, (90, 300, 70), 36, 700), (2, (64, 64, 64), 50, 900)])
def test_loopback_peer_kernel_tiled(pb, orc, nranks, dims, r, s):
    """The peer kernel at sizes where a mode has several 64-row blocks and
    sample splits, every rank bucket (RT = 32 / 64), apply shares exchanged
    per counterpart CTA, 61 % 2 and 70 % 4 != 0."""
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 21)
    kw = dict(rng_seed=21, max_iters=6, stall_limit=1000)
    res = sharded_solve(pb, x, "rand", r, s, nranks, expect_fused=True, **kw)
    check_against_unsharded(pb, x, "rand", r, s, res, **kw)


@pytest.mark.parametrize("fused", [-1, 0])
@pytest.mark.parametrize("nranks,dims,transform", [(2, (16, 8, 32), "dct"), (3, (16, 8, 32), "dct"),
                                                   (4, (16, 8, 32), "wht"), (3, (16, 8, 32), "wht"),
                                                   (4, (12, 10, 5), "dct")])
def test_loopback_sharded_cprand_mix(pb, orc, nranks, dims, transform, fused):
    """Sharded CPRAND-MIX: the distributed mixing pass (row blocks of the
    slab exchanged so every rank transforms whole last-mode fibers, then
    exchanged back); then, for the DCT, the persistent MIX kernel's peer path
    (fused=-1: local-sample RHS sums exchanged per apply block, the last
    mode's mixed slab rows stored into every rank's factor), else the chain
    (local-sample RHS + allreduce + unmix, the last mode's RHS slabs
    allgathered and unmixed)."""
    r, s = 3, 60
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 12)
    kw = dict(rng_seed=12, max_iters=8, stall_limit=1000, transform=transform, fused=fused)
    res = sharded_solve(pb, x, "mix", r, s, nranks, expect_fused=(fused != 0 and transform == "dct"), **kw)
    check_against_unsharded(pb, x, "mix", r, s, res, **kw)
    kw.pop("fused")
    o = orc.solve("mix", x, r, s, orc.SolveOptions(**kw))
    assert max(abs(a[2] - b[2]) for a, b in zip(res[0].trace, o.trace)) < 1e-8


@pytest.mark.parametrize("nranks,dims,r,s", [(2, (40, 36, 30, 33), 10, 300), (3, (64, 50, 70), 20, 400),
                                             (4, (48, 40, 36, 30), 32, 500)])
def test_loopback_peer_mix_kernel(pb, orc, nranks, dims, r, s):
    """The MIX kernel's peer path at sizes with many apply blocks, strided
    modes read in place or from replicas, RT = 16 / 32 / 64 (R = 32), last
    dims P does not divide."""
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 13)
    kw = dict(rng_seed=13, max_iters=6, stall_limit=1000, transform="dct")
    res = sharded_solve(pb, x, "mix", r, s, nranks, expect_fused=True, **kw)
    check_against_unsharded(pb, x, "mix", r, s, res, **kw)


@pytest.mark.parametrize("extra", [dict(fit_threshold=0.97), dict(stall_limit=3)])
def test_loopback_sharded_stop_rule(pb, orc, extra):
    """Early stops: every rank enqueues the same iterations (and so the same
    collectives) and stops where the unsharded run stops."""
    dims, r, s = (24, 20, 22), 4, 60
    x, _ = orc.gen_baseline(dims, r, 0.5, 0.01, 9)
    kw = dict(rng_seed=9, max_iters=120, **extra)
    res = sharded_solve(pb, x, "rand", r, s, 3, **kw)
    ref = check_against_unsharded(pb, x, "rand", r, s, res, **kw)
    assert ref.iterations < 120


def test_loopback_synth_slab(pb):
    """The BASELINE.json generator per slab (noise scaled by the allreduced
    global norms) concatenates to the unsharded tensor."""
    dims, r, nranks = (20, 18, 13), 4, 3
    t = pb.DeviceTensor(dims, device=0)
    t.synth(r, 0.5, 0.01, 5)
    want = t.download()
    t.close()
    from paper_1701_06600_b200 import shard

    def body(rank, comm):
        off, ln = shard.slab(dims[-1], nranks, rank)
        ts = pb.DeviceTensor(list(dims[:-1]) + [ln], device=0)
        ts.synth_slab(r, 0.5, 0.01, 5, dims[-1], comm)
        out = ts.download()
        ts.close()
        return out

    parts = run_ranks(pb, nranks, body)
    got = np.concatenate(parts, axis=2)
    assert rel(got, want) < 1e-14
