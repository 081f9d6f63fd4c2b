"""Oracle: HRCS statistic (Fig.1c; SPEC hrcs_stats S:158-166).

TEST INFRASTRUCTURE ONLY: imported by tests/ and tools/ reports, never by the product
path (paper_2603_25260_b200).  Shares no code with csrc/ (no Morton keys, no hashing):
the plain definition written out with numpy set membership.

P:60-61: "For the octree of each sample, we collected two key statistics: (i) the total
number of nodes at each level, and (ii) the average number of occupied neighbors within
a 3x3x3 neighborhood."  Reading: a depth-d node is an occupied coordinate
of the voxel grid at d bits, i.e. the distinct values of xyz >> (L - d); its neighbour
count is how many of the 26 coordinates c + delta (delta in {-1,0,1}^3 \\ {0}) are
occupied nodes of the same depth.  Pinned by tests/test_oracle_hrcs.py (closed form
for full cubes, brute force on tiny clouds, single point).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def level_nodes(xyz: np.ndarray, L: int, d: int) -> np.ndarray:
    """Occupied depth-d coordinates (unique rows of xyz >> (L - d)), int64 [N_d][3]."""
    return np.unique(np.asarray(xyz, np.int64) >> (L - d), axis=0)


def hrcs_stats(xyz: np.ndarray, L: int) -> Tuple[np.ndarray, np.ndarray]:
    """(nodes[d], neighbour_sum[d]) for d = 0..L; the paper's mean is their ratio."""
    nodes = np.zeros(L + 1, np.uint64)
    nsum = np.zeros(L + 1, np.uint64)
    for d in range(L + 1):
        c = level_nodes(xyz, L, d)
        side = np.int64(1) << d
        # a coordinate in [-1, 2^d] per axis -> one integer id (no wrap-around: shift by 1)
        w = side + 2

        def ident(p):
            return ((p[:, 0] + 1) * w + (p[:, 1] + 1)) * w + (p[:, 2] + 1)

        occ = ident(c)
        total = 0
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    if dx == dy == dz == 0:
                        continue
                    total += int(np.isin(ident(c + np.array([dx, dy, dz], np.int64)), occ).sum())
        nodes[d] = len(c)
        nsum[d] = total
    return nodes, nsum
