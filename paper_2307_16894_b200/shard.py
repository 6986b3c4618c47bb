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
  selection to the single-GPU greedy.
"""
from __future__ import annotations

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
