"""Multi-GPU partitioning of the hot path, one process per
GPU over torch.distributed (NCCL on the GPU box, gloo in the CPU tests).

* configs 1/2/3: independent units (points, RVE instances) — contiguous
  shards, no collective on the data path; only the bench's max-over-ranks
  timing reduction.
* config 4 Gram: dof rows of S sharded; local S_k^T S_k then one SUM
  all-reduce of the n_snap x n_snap Gram.
* config 4 ECM greedy: candidates (quadrature points) sharded; each
  iteration a local argmax, then an all-gather of (score, index) pairs and
  the reference's tie rule (larger score, then smaller index) — identical
  selection to the single-GPU greedy.  ecm_comm() hands these exchanges to
  the device greedy (podecm_ecm_select_sharded) as host callbacks.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous [lo, hi) of n_total units for `rank`."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_seed(base: int, rank: int) -> int:
    return base + 7919 * rank


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(x: float, device=None) -> float:
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_gram(local_gram: torch.Tensor) -> torch.Tensor:
    """Sum of the per-shard S_k^T S_k (in place)."""
    dist = _dist()
    if dist is not None and dist.get_world_size() > 1:
        dist.all_reduce(local_gram, op=dist.ReduceOp.SUM)
    return local_gram


def argmax_over_ranks(score: float, index: int, device=None) -> tuple[float, int]:
    """Global (score, index) of the ECM greedy step from per-rank candidates
    (index = global candidate id, -1 if the rank has none): larger score wins,
    ties go to the smaller index (ecm.cpp:164-173 scans ascending with '>')."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return score, index
    w = dist.get_world_size()
    mine = torch.tensor([score, float(index)], dtype=torch.float64, device=device)
    allv = [torch.empty_like(mine) for _ in range(w)]
    dist.all_gather(allv, mine)
    best_s, best_i = 0.0, -1
    for v in allv:
        s, i = float(v[0]), int(v[1])
        if i >= 0 and (best_i < 0 or s > best_s or (s == best_s and i < best_i)):
            best_s, best_i = s, i
    return best_s, best_i


def _host_group():
    """The group host (CPU) tensors reduce over: the default group when it has
    a CPU backend (gloo, or "cuda:nccl,cpu:gloo"), else a gloo group."""
    dist = _dist()
    be = str(dist.get_backend())
    if "gloo" in be:
        return None
    global _GLOO
    try:
        return _GLOO
    except NameError:
        _GLOO = dist.new_group(backend="gloo")
        return _GLOO


def allreduce_host(a: np.ndarray) -> None:
    """In-place SUM over ranks of a host float64 array."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return
    dist.all_reduce(torch.from_numpy(a), op=dist.ReduceOp.SUM, group=_host_group())


def bcast_host(a: np.ndarray, root: int) -> None:
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return
    dist.broadcast(torch.from_numpy(a), src=root, group=_host_group())


def argmax_owner(score: float, index: int) -> tuple[float, int, int]:
    """argmax_over_ranks plus the rank that owns the winning candidate."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return score, index, 0
    w, me = dist.get_world_size(), dist.get_rank()
    mine = torch.tensor([score, float(index), float(me)], dtype=torch.float64)
    allv = [torch.empty_like(mine) for _ in range(w)]
    dist.all_gather(allv, mine, group=_host_group())
    best_s, best_i, owner = 0.0, -1, 0
    for v in allv:
        s, i, r = float(v[0]), int(v[1]), int(v[2])
        if i >= 0 and (best_i < 0 or s > best_s or (s == best_s and i < best_i)):
            best_s, best_i, owner = s, i, r
    return best_s, best_i, owner


def ecm_comm(q0: int, nq_local: int):
    """podecm_ecm_comm for this rank's candidate shard [q0, q0 + nq_local):
    host callbacks over torch.distributed (returns the struct; the callback
    objects are kept alive on it)."""
    from . import _lib

    def _ar(user, ptr, n):
        try:
            allreduce_host(np.ctypeslib.as_array(ptr, shape=(n,)))
            return 0
        except Exception:
            return -1

    def _am(user, score, index, owner):
        try:
            s, i, r = argmax_owner(float(score[0]), int(index[0]))
            score[0], index[0], owner[0] = s, i, r
            return 0
        except Exception:
            return -1

    def _bc(user, ptr, n, root):
        try:
            bcast_host(np.ctypeslib.as_array(ptr, shape=(n,)), root)
            return 0
        except Exception:
            return -1

    cbs = (_lib.ECM_ALLREDUCE(_ar), _lib.ECM_ARGMAX(_am), _lib.ECM_BCAST(_bc))
    comm = _lib.podecm_ecm_comm(None, int(q0), int(nq_local), *cbs)
    comm._keep = cbs
    return comm
