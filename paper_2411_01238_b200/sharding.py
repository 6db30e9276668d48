"""Row sharding of the SparseDrop layer across data-parallel ranks.

Large-M workloads split M into contiguous runs of whole mask block rows, one per
rank. Each rank generates its own mask rows from their GLOBAL block-row index
(the reference's draw depends only on (seed, r, c), block_mask.cpp:70), so the
shard masks are bit-identical to the global mask with no communication; Y and
dX are row-local; the only exchange is the sum of the partial dW over ranks
(one all-reduce of K x N fp32 per step).
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class RowShard:
    rank: int
    world: int
    row0: int              # first global row
    rows: int              # rows owned
    row_block_offset: int  # first global mask block row (row0 / m_blk)


def shard_rows(m: int, m_blk: int, world: int, rank: int) -> RowShard:
    """Contiguous split of the M/m_blk block rows; the first (R mod world) ranks
    get one extra block row."""
    if m_blk <= 0 or m % m_blk:
        raise ValueError(f"mask block size m_blk={m_blk} does not divide rows={m}")
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    R = m // m_blk
    if R < world:
        raise ValueError(f"cannot split {R} block rows over {world} ranks")
    base, extra = divmod(R, world)
    r0 = rank * base + min(rank, extra)
    nr = base + (1 if rank < extra else 0)
    return RowShard(rank, world, r0 * m_blk, nr * m_blk, r0)


def all_shards(m: int, m_blk: int, world: int):
    return [shard_rows(m, m_blk, world, r) for r in range(world)]
