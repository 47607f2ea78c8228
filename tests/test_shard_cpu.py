"""Slab sharding of the CPRAND loop, world_size 2 over gloo on CPU.

Each rank holds one slab of the last mode (paper_1701_06600_b200.shard, the
plan the C++ session implements with NCCL), contracts its own fibers with the
oracle's gather / skr, and the ranks combine partial right-hand sides
(allreduce) and factor slabs (allgather) exactly as enqueue_mode_sharded
does. The result must match the unsharded computation of the same
normal-equations iteration to round-off (the only difference is the
summation order of the partials), and both must track the oracle's
QR-based CPRAND at the LS-parity tolerance.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

DIMS = (9, 7, 11)
R, S, ITERS, SEED = 3, 60, 4, 5


def _problem():
    import oracle as orc
    g = orc.Engine(SEED, raw=True)
    fs = [g.matrix(d, R, 0.1, 1.0) for d in DIMS]
    x = np.einsum("ir,jr,kr->ijk", *fs)
    x = x + 0.01 * orc.random_tensor(DIMS, SEED + 1)
    return np.asfortranarray(x)


def _normal_eq_iterations(x_full_or_slab, rank, nranks, allreduce, allgather):
    """CPRAND iterations in the sharded normal-equations form (the GPU path's
    algebra): returns (lambda, factors)."""
    import oracle as orc
    from paper_1701_06600_b200 import shard
    N = len(DIMS)
    off, length = shard.slab(DIMS[-1], nranks, rank)
    lmax = shard.slab_max(DIMS[-1], nranks)
    tables = orc.sample_tables(DIMS, S, SEED, ITERS)
    lam, factors = orc.init_random(DIMS, R, SEED)
    factors = [np.array(f, order="F") for f in factors]
    lam = np.array(lam)
    for it in range(ITERS):
        for n in range(N):
            idxs = tables[it][n]
            z = orc.skr(idxs, factors, n)            # all samples, replicated
            g = z.T @ z
            mask = shard.local_samples(idxs, n, N, off, length)
            loc = shard.to_slab_indices(idxs[mask], n, N, off)
            xs = orc.gather_fibers(x_full_or_slab, n, loc) if mask.any() else np.zeros((0, 0))
            if n < N - 1:
                rhs = xs @ z[mask] if mask.any() else np.zeros((DIMS[n], R))
                rhs = allreduce(rhs)
                a = rhs @ np.linalg.inv(g)
            else:
                rows = xs @ z                          # slab rows of every fiber
                a_slab = rows @ np.linalg.inv(g)
                pad = np.zeros((lmax, R))
                pad[:length] = a_slab
                a = allgather(pad)[:DIMS[n]]
            nrm = np.sqrt((a * a).sum(axis=0))
            factors[n] = np.asfortranarray(a / nrm)
            lam = lam * nrm if n == 0 else nrm
    return lam, factors


def _worker(rank, nranks, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from paper_1701_06600_b200 import shard
    x = _problem()
    xs = shard.slab_of(x, nranks, rank)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        parts = [torch.empty_like(t) for _ in range(nranks)]
        dist.all_gather(parts, t)
        return torch.cat(parts).numpy()

    lam, fs = _normal_eq_iterations(xs, rank, nranks, allreduce, allgather)
    out[rank] = (lam, [np.array(f) for f in fs])
    dist.destroy_process_group()


def test_slab_plan_partitions_samples():
    import oracle as orc
    from paper_1701_06600_b200 import shard
    N = len(DIMS)
    for nranks in (1, 2, 3, 4):
        spans = [shard.slab(DIMS[-1], nranks, p) for p in range(nranks)]
        assert spans[0][0] == 0 and sum(s[1] for s in spans) == DIMS[-1]
        for (o0, l0), (o1, _) in zip(spans, spans[1:]):
            assert o0 + l0 == o1
        tables = orc.sample_tables(DIMS, S, SEED, 1)[0]
        for n in range(N - 1):
            masks = [shard.local_samples(tables[n], n, N, *spans[p]) for p in range(nranks)]
            assert np.array_equal(np.sum(masks, axis=0), np.ones(S))  # every fiber in exactly one slab
        assert all(shard.local_samples(tables[N - 1], N - 1, N, *spans[p]).all() for p in range(nranks))


def test_slab_gather_equals_full_gather():
    import oracle as orc
    from paper_1701_06600_b200 import shard
    x = _problem()
    N = len(DIMS)
    tables = orc.sample_tables(DIMS, S, SEED, 1)[0]
    for nranks in (2, 3):
        for p in range(nranks):
            off, length = shard.slab(DIMS[-1], nranks, p)
            xs = shard.slab_of(x, nranks, p)
            for n in range(N):
                mask = shard.local_samples(tables[n], n, N, off, length)
                if not mask.any():
                    continue
                loc = shard.to_slab_indices(tables[n][mask], n, N, off)
                got = orc.gather_fibers(xs, n, loc)
                want = orc.gather_fibers(x, n, tables[n][mask])
                if n == N - 1:
                    want = want[off:off + length]
                assert np.array_equal(got, want)  # bit-exact: pure copies


@pytest.mark.timeout(300)
def test_sharded_iterations_world2_gloo():
    nranks = 2
    port = 29500 + (os.getpid() % 2000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(nranks, port, out), nprocs=nranks, join=True)
    ident = lambda a: a  # noqa: E731
    lam1, fs1 = _normal_eq_iterations(_problem(), 0, 1, ident, ident)
    for p in range(nranks):
        lam, fs = out[p]
        np.testing.assert_allclose(lam, lam1, rtol=1e-12)
        for f, f1 in zip(fs, fs1):
            np.testing.assert_allclose(f, f1, rtol=1e-11, atol=1e-13)


def test_normal_equations_track_oracle_cprand():
    """The unsharded normal-equations loop vs the oracle's QR CPRAND (same
    samples, bench mode so the estimator's RNG use does not matter)."""
    import oracle as orc
    x = _problem()
    ident = lambda a: a  # noqa: E731
    lam1, fs1 = _normal_eq_iterations(x, 0, 1, ident, ident)
    res = orc.solve("rand", x, R, S, orc.SolveOptions(rng_seed=SEED, max_iters=ITERS, bench_mode=True))
    np.testing.assert_allclose(res.lam, lam1, rtol=1e-9)
    for f, f1 in zip(res.factors, fs1):
        np.testing.assert_allclose(f, f1, rtol=1e-8, atol=1e-10)


# ---------------------------------------------------------------------------
# Slab-sharded CPRAND-MIX (real transform): the distributed mixing pass
# (modes < N-1 inside the slab, mode N-1 through a block all-to-all, as
# Session::mix_last_mode_sharded) and the sharded MIX iteration (local-sample
# RHS + allreduce for modes < N-1, allgather of the last mode's slab rows;
# unmix, replicated solve, mix the new factor), against the unsharded
# computation and the oracle's cprand_mix.
MSEED, MKIND = SEED, "dct"  # cprand_mix seeds its operator with rng_seed


def _mix_mats(kind=MKIND, seed=MSEED):
    """F_n D_n as dense matrices (the oracle's mix_factor of the identity)."""
    import oracle as orc
    return [orc.mix_factor(np.eye(d), DIMS, kind, seed, n) for n, d in enumerate(DIMS)]


def _mode_apply(x, mat, n):
    """x x_n mat: transform every mode-n fiber by mat."""
    y = np.moveaxis(x, n, 0)
    y = np.tensordot(mat, y, axes=(1, 0))
    return np.asfortranarray(np.moveaxis(y, 0, n))


def _sharded_mix_pass(xs, rank, nranks, exchange):
    """mix_tensor of the slab: local modes, then mode N-1 across the ranks.
    exchange(send_blocks) -> recv_blocks (block q of send goes to rank q)."""
    from paper_1701_06600_b200 import shard
    mats = _mix_mats()
    N = len(DIMS)
    for n in range(N - 1):
        xs = _mode_apply(xs, mats[n], n)
    L = xs.shape[-1]
    M = int(np.prod(DIMS[:-1]))
    x2 = xs.reshape(M, L, order="F")
    mb = -(-M // nranks)
    blocks = [x2[q * mb:min(M, (q + 1) * mb)] for q in range(nranks)]
    got = exchange(blocks)                       # from rank p: my row block x p's slab columns
    w = np.concatenate(got, axis=1)              # [Mb][I_N]: whole last-mode fibers
    w = w @ mats[N - 1].T                        # transform along the last mode
    lmax = shard.slab_max(DIMS[-1], nranks)
    back = [w[:, p * lmax:p * lmax + shard.slab(DIMS[-1], nranks, p)[1]] for p in range(nranks)]
    ret = exchange(back)                         # from rank q: q's row block x my slab columns
    x2 = np.concatenate(ret, axis=0)
    return np.asfortranarray(x2.reshape(xs.shape, order="F"))


def _mix_iterations(xhat_slab, rank, nranks, allreduce, allgather):
    """Sharded CPRAND-MIX iterations in normal-equations form (bench mode)."""
    import oracle as orc
    from paper_1701_06600_b200 import shard
    N = len(DIMS)
    mats = _mix_mats()
    off, length = shard.slab(DIMS[-1], nranks, rank)
    lmax = shard.slab_max(DIMS[-1], nranks)
    tables = orc.sample_tables(DIMS, S, SEED, ITERS)
    lam, factors = orc.init_random(DIMS, R, SEED)
    factors = [np.array(f, order="F") for f in factors]
    mixed = [mats[n] @ factors[n] for n in range(N)]
    lam = np.array(lam)
    for it in range(ITERS):
        for n in range(N):
            idxs = tables[it][n]
            z = orc.skr(idxs, mixed, n)
            g = z.T @ z
            mask = shard.local_samples(idxs, n, N, off, length)
            loc = shard.to_slab_indices(idxs[mask], n, N, off)
            xs = orc.gather_fibers(xhat_slab, n, loc) if mask.any() else np.zeros((0, 0))
            if n < N - 1:
                rhs = xs @ z[mask] if mask.any() else np.zeros((DIMS[n], R))
                rhs = allreduce(rhs)
            else:
                pad = np.zeros((lmax, R))
                pad[:length] = xs @ z
                rhs = allgather(pad)[:DIMS[n]]
            a = (mats[n].T @ rhs) @ np.linalg.inv(g)  # unmix the RHS rows, solve
            nrm = np.sqrt((a * a).sum(axis=0))
            factors[n] = np.asfortranarray(a / nrm)
            lam = lam * nrm if n == 0 else nrm
            mixed[n] = mats[n] @ factors[n]
    return lam, factors


def _mix_worker(rank, nranks, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from paper_1701_06600_b200 import shard
    x = _problem()
    xs = shard.slab_of(x, nranks, rank)

    def exchange(blocks):  # point-to-point block exchange (ncclSend / ncclRecv group)
        recv = [None] * nranks
        reqs = []
        shapes = [None] * nranks
        for q in range(nranks):  # exchange shapes first
            sh = torch.tensor(blocks[q].shape, dtype=torch.int64)
            if q == rank:
                shapes[q] = tuple(blocks[q].shape)
                continue
            req = dist.isend(sh, q)
            buf = torch.empty(2, dtype=torch.int64)
            dist.recv(buf, q)
            req.wait()
            shapes[q] = tuple(buf.tolist())
        for q in range(nranks):
            if q == rank:
                recv[q] = blocks[q]
                continue
            t = torch.from_numpy(np.ascontiguousarray(blocks[q]))
            reqs.append(dist.isend(t, q))
            buf = torch.empty(shapes[q], dtype=torch.float64)
            dist.recv(buf, q)
            recv[q] = buf.numpy()
        for r_ in reqs:
            r_.wait()
        return recv

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        parts = [torch.empty_like(t) for _ in range(nranks)]
        dist.all_gather(parts, t)
        return torch.cat(parts).numpy()

    xh = _sharded_mix_pass(xs, rank, nranks, exchange)
    lam, fs = _mix_iterations(xh, rank, nranks, allreduce, allgather)
    out[rank] = (xh, lam, [np.array(f) for f in fs])
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_mix_world2_gloo():
    import oracle as orc
    from paper_1701_06600_b200 import shard
    nranks = 2
    port = 29500 + ((os.getpid() + 777) % 2000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_mix_worker, args=(nranks, port, out), nprocs=nranks, join=True)
    x = _problem()
    want = orc.mix_tensor(x, MKIND, MSEED)      # the unsharded mixing pass
    ident = lambda a: a  # noqa: E731
    lam1, fs1 = _mix_iterations(want, 0, 1, ident, ident)
    for p in range(nranks):
        xh, lam, fs = out[p]
        np.testing.assert_allclose(xh, shard.slab_of(want, nranks, p), rtol=0, atol=1e-13 * np.abs(want).max())
        np.testing.assert_allclose(lam, lam1, rtol=1e-11)
        for f, f1 in zip(fs, fs1):
            np.testing.assert_allclose(f, f1, rtol=1e-10, atol=1e-12)
    # the normal-equations MIX loop tracks the oracle's QR cprand_mix
    res = orc.solve("mix", x, R, S, orc.SolveOptions(rng_seed=SEED, max_iters=ITERS, bench_mode=True,
                                                        transform=MKIND))
    np.testing.assert_allclose(res.lam, lam1, rtol=1e-8)
    for f, f1 in zip(res.factors, fs1):
        np.testing.assert_allclose(f, f1, rtol=1e-7, atol=1e-9)
