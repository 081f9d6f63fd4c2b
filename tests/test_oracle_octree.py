"""Oracle pins: octree construction / expansion.

Independent of the oracle's own code: brute-force Python sets over coordinates,
SPEC worked examples (tests/golden/octree_examples.json), and the inverse identities.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "octree_examples.json")


def _coords_of(keys, bits):
    """Decode Morton keys by explicit bit extraction (x is the MSB of each triple)."""
    out = []
    for k in keys:
        k = int(k)
        x = y = z = 0
        for b in range(bits):
            t = (k >> (3 * b)) & 7
            x |= ((t >> 2) & 1) << b
            y |= ((t >> 1) & 1) << b
            z |= (t & 1) << b
        out.append((x, y, z))
    return out


def _brute_levels(points, L):
    """Per depth: sorted-by-Morton coordinate list and the child-occupancy bytes,
    from set arithmetic (floor division by 2) and the child bit c = 4bx+2by+bz."""
    pts = {tuple(int(v) for v in p) for p in points}
    levels = {L: pts}
    for d in range(L - 1, -1, -1):
        levels[d] = {(x >> 1, y >> 1, z >> 1) for (x, y, z) in levels[d + 1]}

    def mkey(p, bits):
        # ordering key for Morton order without building the interleave: compare
        # coordinates bit-plane by bit-plane from the top, x before y before z
        return tuple(((p[0] >> b) & 1, (p[1] >> b) & 1, (p[2] >> b) & 1) for b in range(bits - 1, -1, -1))

    coords = {d: sorted(levels[d], key=lambda p, d=d: mkey(p, d)) for d in range(L + 1)}
    codes = {}
    for d in range(L):
        occ = {}
        for (x, y, z) in levels[d + 1]:
            par = (x >> 1, y >> 1, z >> 1)
            occ[par] = occ.get(par, 0) | (1 << (4 * (x & 1) + 2 * (y & 1) + (z & 1)))
        codes[d] = [occ[p] for p in coords[d]]
    return coords, codes


def test_spec_build_examples():
    g = json.load(open(GOLD))
    for ex in g["build"]:
        keys, codes = O.build_octree(np.array(ex["points"], np.int32), ex["L"])
        assert [list(map(int, c)) for c in codes] == ex["codes"], ex["cite"]


def test_spec_expand_examples():
    g = json.load(open(GOLD))
    for ex in g["expand"]:
        px, py, pz = ex["parent"]
        bits = 3  # enough for the example coordinates
        k = O.morton(px, py, pz, bits)
        ch = O.expand(np.array([k], np.uint64), np.array([ex["code"]], np.uint8))
        assert _coords_of(ch, bits + 1) == [tuple(c) for c in ex["children"]], ex["cite"]


@pytest.mark.parametrize("seed,n,L", [(1, 1, 9), (2, 50, 4), (3, 500, 6), (4, 3000, 12), (5, 200, 21)])
def test_build_matches_brute_force(seed, n, L):
    pts = I.random_cloud(n, L, seed, spread=0.01 if L > 12 else 1.0)
    keys, codes = O.build_octree(pts, L)
    coords, bcodes = _brute_levels(pts, L)
    for d in range(L + 1):
        assert _coords_of(keys[d], d) == coords[d], f"depth {d}"
    for d in range(L):
        assert list(map(int, codes[d])) == bcodes[d], f"codes depth {d}"


def test_invariants_and_inverse_on_lidar_frame():
    pts = I.make_frame(I.CFG1)
    L = I.CFG1.bit_depth
    keys, codes = O.build_octree(pts, L)
    assert len(keys[0]) == 1
    for d in range(L):
        # sum popcount X_d = N_{d+1}; X_d in [1, 255]; expand(key_d, X_d) = key_{d+1}
        assert int(np.unpackbits(codes[d]).sum()) == len(keys[d + 1])
        assert codes[d].min() >= 1
        assert np.array_equal(O.expand(keys[d], codes[d]), keys[d + 1])
        assert np.all(np.diff(keys[d + 1].astype(np.uint64)) > 0)  # strictly increasing
    # reconstruct(build(C)) = dedup(C)
    rec = set(_coords_of(keys[L], L))
    assert rec == {tuple(p) for p in pts.tolist()}


def test_duplicates_and_order_do_not_matter():
    pts = I.random_cloud(400, 10, 7)
    rng = np.random.default_rng(0)
    dup = np.concatenate([pts, pts[rng.integers(0, 400, 300)]])[rng.permutation(700)]
    k1, c1 = O.build_octree(pts, 10)
    k2, c2 = O.build_octree(dup, 10)
    for d in range(10):
        assert np.array_equal(c1[d], c2[d])


def test_errors():
    with pytest.raises(O.OracleError) as e:
        O.build_octree(np.zeros((0, 3), np.int32), 9)
    assert e.value.name == "EMPTY"
    with pytest.raises(O.OracleError) as e:
        O.build_octree(np.array([[0, 0, 512]], np.int32), 9)
    assert e.value.name == "RANGE"
    with pytest.raises(O.OracleError) as e:
        O.build_octree(np.array([[0, -1, 0]], np.int32), 9)
    assert e.value.name == "RANGE"
