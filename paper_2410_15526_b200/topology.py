"""Host-side topology and layout logic of the path (no arithmetic of the method).

P = M * N workers, M groups ("nodes") of N, rank r = m*N + l (sec. 2.3).  On one
8xB200 NVSwitch box the paper's node split is emulated as groups of GPUs.
"""
from __future__ import annotations

from typing import Optional, Tuple


def default_split(world: int, groups: Optional[int] = None) -> Tuple[int, int]:
    """(M, N) for `world` ranks: `groups` groups if given, else 2 groups when world is even
    (the 2 x 4 split of BASELINE.json config 2 at world 8), else 1."""
    if groups is None:
        groups = 2 if world % 2 == 0 else 1
    if groups < 1 or world % groups:
        raise ValueError(f"groups={groups} does not divide world={world}")
    return groups, world // groups


def coords(rank: int, N: int) -> Tuple[int, int]:
    """(m, l) of a rank."""
    return divmod(rank, N)


def intra_block_shards(lp: int, M: int, N: int):
    """Shards carried by intra block lp, in unit order m' = 0..M-1 (R9)."""
    return [mp * N + lp for mp in range(M)]


def pad_numel(numel: int, world: int, group: int) -> int:
    """Smallest padded numel satisfying the ABI rule numel % (P * lcm(G, 64)) == 0 (R1)."""
    a = world * max(group, 64)
    return (numel + a - 1) // a * a
