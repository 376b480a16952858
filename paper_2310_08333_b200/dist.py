"""Row sharding of the data matrix across GPUs.

GPU g of p holds rows [g N/p, (g+1) N/p) of A and of every N-length vector;
every n-length vector (x, z, u, CG vectors, Omega, Y, U) is replicated.  The
exchange steps are sums of A^T partials: one n-vector all-reduce per HVP, one
packed (k n + scalars) all-reduce per ADMM iteration, one n x s all-reduce per
sketch.  ``torch.distributed`` (NCCL over NVLink on B200, gloo in the CPU
tests) is the transport; with one process nothing is communicated.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class Shard:
    rank: int = 0
    world: int = 1
    row_start: int = 0
    row_stop: int = 0
    rows_global: int = 0
    # run the exchange steps even on one rank (a world-size-1 process group: the
    # NCCL path of the tests on a one-GPU box)
    collectives: bool = False

    @property
    def sharded(self) -> bool:
        return self.world > 1 or self.collectives

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        """Sum ``t`` in place over all ranks (no-op on one rank)."""
        if self.sharded:
            torch.distributed.all_reduce(t)
        return t


def row_range(N: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row block of rank ``rank``."""
    base, extra = divmod(N, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


# harness hook (bench.py --collectives, tests): a world-size-1 process group still runs the
# exchange steps, so the NCCL path can be exercised on a one-GPU box
FORCE_COLLECTIVES = False


def current_shard(N: int) -> Shard:
    """Shard of an N-row matrix for this process (whole matrix without a
    process group)."""
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        rank = torch.distributed.get_rank()
        world = torch.distributed.get_world_size()
    else:
        rank, world = 0, 1
    a, b = row_range(N, rank, world)
    return Shard(rank, world, a, b, N, collectives=bool(FORCE_COLLECTIVES and world == 1
                                                       and torch.distributed.is_initialized()))
