"""Work partitioning across ranks (one process per GPU).

BASELINE config C5 (a batch of independent images): images are split into contiguous,
balanced ranges; each rank deblurs its own range with a replica of the operator — no
collective on the data path (weak scaling). Used by bench.py and tests/test_batch.py.
"""
from __future__ import annotations


def shard(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank `rank` when n_items are split over `world` ranks as evenly as
    possible (the first n_items % world ranks take one extra)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per, extra = divmod(n_items, world)
    lo = rank * per + min(rank, extra)
    return lo, lo + per + (1 if rank < extra else 0)
