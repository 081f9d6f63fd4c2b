"""Oracle pins: HRCS statistic (Fig.1c; SPEC hrcs_stats S:158-166).

* full n^3 cube: ordered neighbour pairs = (3n - 2)^3 - n^3 (per axis, offset 0 keeps n
  positions, offsets +-1 keep n - 1 each), so at n = 2 the mean is exactly 7;
* single point: 0 neighbours at every depth, one node per depth;
* brute force over python tuples on tiny random clouds;
* the synthetic 16-beam scan: mean neighbours fall below one at the deepest levels
  ("At certain levels, the average number of neighbors even falls below one").
"""
import itertools

import numpy as np
import pytest

from oracle import hrcs as H
from paper_2603_25260_b200 import inputs as I


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_full_cube_closed_form(n):
    g = np.arange(n)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    L = 4
    nodes, nsum = H.hrcs_stats(pts, L)
    assert nodes[L] == n ** 3
    assert nsum[L] == (3 * n - 2) ** 3 - n ** 3
    if n == 2:
        assert nsum[L] / nodes[L] == 7.0


def test_single_point():
    nodes, nsum = H.hrcs_stats(np.array([[5, 9, 1]]), 6)
    assert nodes.tolist() == [1] * 7 and nsum.tolist() == [0] * 7


def _brute(pts, L):
    out = []
    for d in range(L + 1):
        s = {tuple(int(v) >> (L - d) for v in p) for p in pts}
        tot = 0
        for c in s:
            for o in itertools.product((-1, 0, 1), repeat=3):
                if o != (0, 0, 0) and (c[0] + o[0], c[1] + o[1], c[2] + o[2]) in s:
                    tot += 1
        out.append((len(s), tot))
    return out


@pytest.mark.parametrize("seed,n,L", [(1, 40, 5), (2, 300, 6), (3, 200, 9)])
def test_brute_force(seed, n, L):
    pts = I.random_cloud(n, L, seed)
    nodes, nsum = H.hrcs_stats(pts, L)
    assert list(zip(nodes.tolist(), nsum.tolist())) == _brute(pts, L)


def test_synthetic_scan_falls_below_one():
    pts = I.make_frame(I.CFG1)
    nodes, nsum = H.hrcs_stats(pts, 12)
    mean = nsum / np.maximum(nodes, 1)
    assert nodes[0] == 1 and mean[0] == 0
    assert mean[12] < 1.5 and mean.max() > 4 * mean[12]
