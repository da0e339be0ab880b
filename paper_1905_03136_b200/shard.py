"""K-sharding of the tall dimension across ranks.

Rank r of p holds the contiguous row block [start, start + count) of A and B
(row-distributed block vectors, as in the distributed solvers the paper's
kernels serve).  TSMTTSM then needs one sum of the small C
over ranks; TSMM needs C on every rank (a broadcast) and no other exchange.
"""
from __future__ import annotations


def shard_range(K: int, world: int, rank: int) -> tuple[int, int]:
    """Rows of rank `rank`: the first K % world ranks get one extra row."""
    if world < 1 or not 0 <= rank < world or K < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(K, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def rank_order_sum(parts):
    """The deterministic combine of TSM_COMM_DETERMINISTIC: partial C's summed
    in rank order 0, 1, ..., p-1 (mirrors rank_sum_kernel in csrc/tsm_comm.cu)."""
    total = parts[0].copy()
    for p in parts[1:]:
        total = total + p
    return total
