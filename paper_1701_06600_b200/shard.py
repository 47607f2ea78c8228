"""Slab plan of the sharded CPRAND loop (host logic, mirrors session.cu).

The tensor is split along its last mode: rank p of P holds rows
[p * ceil(I/P), min(I, (p + 1) * ceil(I/P))). The sample tables are drawn for
the global shape on every rank (sampling is data independent), so every rank
knows which sampled fibers lie in its slab:

* modes n < N-1: a sampled fiber lies wholly in the slab that owns its
  last-mode index (the last column of the sample table); each rank contracts
  its own fibers and the R x I_n right-hand sides are summed over the ranks;
* mode N-1: every fiber crosses all slabs; each rank contracts the slab rows
  of every fiber, forms its factor rows, and the slabs are gathered.

The C++ session (csrc/session.cu, enqueue_mode_sharded) implements the same
plan with NCCL; tests/test_shard_cpu.py checks the decomposition against the
unsharded computation with the gloo backend.
"""
from __future__ import annotations

import numpy as np


def slab(total: int, nranks: int, rank: int) -> tuple[int, int]:
    """(offset, length) of rank's slab of a last mode of length total."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / nranks")
    lmax = -(-total // nranks)
    off = rank * lmax
    return off, max(0, min(total, off + lmax) - off)


def slab_max(total: int, nranks: int) -> int:
    """Rows per slab in the allgather layout (the last slab is padded)."""
    return -(-total // nranks)


def local_samples(idxs: np.ndarray, mode: int, order: int, off: int, length: int) -> np.ndarray:
    """Boolean mask of the samples whose fiber lies in the slab. idxs is the
    S x (N-1) table of mode `mode` (kept modes ascending): the last column is
    the last mode's index for every mode but the last."""
    if mode == order - 1:
        return np.ones(idxs.shape[0], dtype=bool)
    last = np.asarray(idxs)[:, order - 2]
    return (last >= off) & (last < off + length)


def slab_of(x: np.ndarray, nranks: int, rank: int) -> np.ndarray:
    """Rank's slab of a host tensor (generalized column-major storage)."""
    off, length = slab(x.shape[-1], nranks, rank)
    return np.asfortranarray(x[..., off:off + length])


def to_slab_indices(idxs: np.ndarray, mode: int, order: int, off: int) -> np.ndarray:
    """Sample table with the last mode's index taken relative to the slab."""
    out = np.array(idxs, dtype=np.int64, order="F", copy=True)
    if mode < order - 1:
        out[:, order - 2] -= off
    return out
