"""Row sharding of a fit across ranks.

Each class block (signal, background; reference sample.py:112-116) is split
contiguously across ``world`` ranks, so the global subsample mask — defined
in class-block order by the reference's RNG (sample.py:128-132) — slices
directly: rank g owns signal rows [g*nS/G, (g+1)*nS/G) and the same share of
the background block.  Every rank accumulates integer fixed-point partial
histograms over its rows; an int64 SUM all-reduce per layer makes them
identical on every rank, and integer sums are exact and order-free, so cuts
are identical for any world size.
"""

from __future__ import annotations

import numpy as np

__all__ = ["class_block_shard", "shard_rows", "slice_mask"]


def class_block_shard(n_sig: int, n_bkg: int, rank: int, world: int):
    """((s0, s1), (b0, b1)): this rank's row ranges inside each class block."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    s0, s1 = n_sig * rank // world, n_sig * (rank + 1) // world
    b0, b1 = n_bkg * rank // world, n_bkg * (rank + 1) // world
    return (s0, s1), (b0, b1)


def shard_rows(y01: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Input-row indices owned by ``rank`` (signal shard first, then
    background shard, each in input order = class-block order)."""
    y01 = np.asarray(y01)
    sig = np.flatnonzero(y01 > 0)
    bkg = np.flatnonzero(y01 <= 0)
    (s0, s1), (b0, b1) = class_block_shard(sig.size, bkg.size, rank, world)
    return np.concatenate([sig[s0:s1], bkg[b0:b1]])


def slice_mask(mask_sig: np.ndarray, mask_bkg: np.ndarray, rank: int, world: int) -> np.ndarray:
    """This rank's active flags (its signal shard then background shard)."""
    (s0, s1), (b0, b1) = class_block_shard(mask_sig.size, mask_bkg.size, rank, world)
    return np.concatenate([mask_sig[s0:s1], mask_bkg[b0:b1]])
