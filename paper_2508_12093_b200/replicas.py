"""Multi-GPU as replicas: one process per GPU, each
owning a contiguous shard of independent work units (columns, Pearson pairs, C5
batch elements); no collective on the data path.  The only exchanges are the
host-side gather of decrypted scalars and the max-over-ranks of timings, both
through torch.distributed (NCCL on the GPU box, gloo in the CPU tests)."""
from __future__ import annotations

from typing import Any, List, Sequence


def shard(n_units: int, world: int, rank: int) -> range:
    """Contiguous, balanced split of n_units over world ranks (first ranks take one extra)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def c4_pairs(n_columns: int = 8) -> List[tuple]:
    """The 28 (i, j) Pearson pairs of C4, in the order a single process visits them."""
    return [(i, j) for i in range(n_columns) for j in range(i + 1, n_columns)]


def gather_results(local: Sequence[Any], world: int, rank: int) -> List[Any]:
    """Concatenate every rank's results in rank order (on all ranks)."""
    if world == 1:
        return list(local)
    import torch.distributed as dist
    parts: List[Any] = [None] * world
    dist.all_gather_object(parts, list(local))
    return [v for p in parts for v in p]


def max_over_ranks(x: float, world: int, device=None) -> float:
    """The job's time is the slowest rank's (bench.py contract)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
