"""Multi-rank host logic for the fine-propagator batch.

The N fine propagators of one PP-PC iteration are independent units
(proj/src/engine.cpp:226-227), so they shard by subinterval with no data-path
collective.  bench.py runs one independent batch per rank (weak scaling); a
sharded PP-PC iteration additionally all-gathers the N end states so every rank
can run assemble_rhs and the multiharmonic solve.  Both are plain
torch.distributed calls (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np


def shard(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced split of subintervals 1..n_total: (n_first, count)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    n_first = 1 + rank * base + min(rank, extra)
    return n_first, count


def sharded_fine_phase(propagate: Callable[[int, np.ndarray], np.ndarray], U: np.ndarray, rank: int,
                       world: int, group=None) -> np.ndarray:
    """F_n(U_{n-1}) for all n, each rank computing its shard, then an all-gather.

    propagate(n_first, U_shard) -> F_shard  (e.g. Propagator.fine_propagate_batch)."""
    import torch
    import torch.distributed as dist
    n_total = U.shape[0]
    n_first, count = shard(n_total, rank, world)
    local = propagate(n_first, U[n_first - 1:n_first - 1 + count]) if count else np.zeros((0, U.shape[1]))
    if world == 1:
        return local
    sizes = [shard(n_total, r, world)[1] for r in range(world)]
    width = max(sizes)
    buf = torch.zeros((width, U.shape[1]), dtype=torch.float64)
    buf[:count] = torch.from_numpy(np.ascontiguousarray(local))
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return np.concatenate([out[r][:sizes[r]].numpy() for r in range(world)], axis=0)
