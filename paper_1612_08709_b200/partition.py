"""Row partitioning of the tall matrix over ranks (host-side bookkeeping only).

The paper's data layout is a row-partitioned IndexedRowMatrix (P:294-295,
P:884); here each rank (GPU) owns one contiguous block of rows, ranks in order.
"""
from __future__ import annotations


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) rows of `rank` when m rows are split as evenly as possible over `world` ranks."""
    if world < 1 or not (0 <= rank < world) or m < 0:
        raise ValueError("bad partition arguments")
    base, extra = divmod(m, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)
