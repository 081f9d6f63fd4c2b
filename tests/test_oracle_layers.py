"""Oracle pins: kernel map, integer sparse conv, K2S2 down, requant, up/prune, wiring.

Pins (DESIGN.md §"Oracle pins"):
* kernel map == brute-force neighbour search over a Python dict;
* K3S1 sparse conv == dense 3-D correlation on a zero-padded numpy grid;
* K2S2 down == dense stride-2 conv on the grid (Eq.4 reading Q4);
* rq / prq == exact-rational round-half-up of acc*m/2^r (Eq.14, reading Q15) and
  the SPEC values (tests/golden/requant_examples.json);
* up/prune: code 255 -> 8 blocks in child order, code 1 -> block 0, and
  the naive Concat+Linear definition of Eq.6/9 evaluated with numpy int64 matmul;
* wiring special cases: zero ResBlock convs with k_s = 1 and identity requant give
  S = F (Eq.8 skip); an XFP ResBlock with zero convs and P = [I|0] / [0|I] gives
  H = F_D / H = G_D (Eq.10).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "requant_examples.json")


def _coords(keys, bits):
    k = keys.astype(np.uint64)
    x = np.zeros(k.size, np.int64); y = np.zeros_like(x); z = np.zeros_like(x)
    for b in range(bits):
        t = (k >> np.uint64(3 * b)) & np.uint64(7)
        x |= ((t >> np.uint64(2)) & np.uint64(1)).astype(np.int64) << b
        y |= ((t >> np.uint64(1)) & np.uint64(1)).astype(np.int64) << b
        z |= (t & np.uint64(1)).astype(np.int64) << b
    return np.stack([x, y, z], 1)


def _sparse_grid(seed, side, frac):
    rng = np.random.default_rng(seed)
    occ = rng.random((side, side, side)) < frac
    pts = np.argwhere(occ).astype(np.int32)
    return pts


@pytest.mark.parametrize("seed", range(6))
def test_kernel_map_brute_force(seed):
    bits = 4
    pts = _sparse_grid(seed, 16, 0.15)
    keys, _ = O.build_octree(pts, bits)
    k = keys[bits]
    nbr = O.kernel_map(k, bits)
    cs = _coords(k, bits)
    index = {tuple(c): i for i, c in enumerate(cs.tolist())}
    for i, c in enumerate(cs.tolist()):
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    want = index.get((c[0] + dx, c[1] + dy, c[2] + dz), -1)
                    assert nbr[i, (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1)] == want


def test_kernel_map_single_coord():
    k = np.array([O.morton(0, 0, 0, 3)], np.uint64)
    nbr = O.kernel_map(k, 3)
    assert (nbr[0] >= 0).sum() == 1 and nbr[0, 13] == 0


@pytest.mark.parametrize("seed,side,cin,cout", [(0, 4, 8, 8), (1, 6, 16, 8), (2, 6, 8, 32), (3, 8, 64, 32)])
def test_conv3_equals_dense_conv(seed, side, cin, cout):
    rng = np.random.default_rng(100 + seed)
    bits = int(np.ceil(np.log2(side)))
    pts = _sparse_grid(seed, side, 0.4)
    keys, _ = O.build_octree(pts, bits)
    k = keys[bits]
    cs = _coords(k, bits)
    f = rng.integers(-128, 128, size=(k.size, cin)).astype(np.int8)
    W = rng.integers(-127, 128, size=(27, cout, cin)).astype(np.int8)
    acc = O.conv3_acc(k, bits, f, W)
    # dense zero-padded grid, out(p) = sum_delta W_delta in(p + delta)
    G = np.zeros((side + 2, side + 2, side + 2, cin), np.int64)
    G[cs[:, 0] + 1, cs[:, 1] + 1, cs[:, 2] + 1] = f
    out = np.zeros((side, side, side, cout), np.int64)
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                sl = G[1 + dx:1 + dx + side, 1 + dy:1 + dy + side, 1 + dz:1 + dz + side]
                out += sl @ W[(dx + 1) * 9 + (dy + 1) * 3 + (dz + 1)].astype(np.int64).T
    assert np.array_equal(acc, out[cs[:, 0], cs[:, 1], cs[:, 2]])


def test_conv3_identity_and_zero():
    pts = _sparse_grid(9, 8, 0.3)
    keys, _ = O.build_octree(pts, 3)
    k = keys[3]
    f = np.random.default_rng(1).integers(-128, 128, size=(k.size, 8)).astype(np.int8)
    W = np.zeros((27, 8, 8), np.int8)
    W[13] = np.eye(8, dtype=np.int8)     # W_0 = I
    assert np.array_equal(O.conv3_acc(k, 3, f, W), f.astype(np.int64))
    assert not O.conv3_acc(k, 3, f, np.zeros_like(W)).any()


@pytest.mark.parametrize("seed", range(4))
def test_down_equals_dense_stride2_conv(seed):
    rng = np.random.default_rng(200 + seed)
    side, C = 8, 16
    pts = _sparse_grid(seed, side, 0.3)
    keys, _ = O.build_octree(pts, 3)
    ck, pk = keys[3], keys[2]
    g = rng.integers(-128, 128, size=(ck.size, C)).astype(np.int8)
    W = rng.integers(-127, 128, size=(8, C, C)).astype(np.int8)
    acc = O.down_acc(ck, pk, g, W)
    cc, pc = _coords(ck, 3), _coords(pk, 2)
    G = np.zeros((side, side, side, C), np.int64)
    G[cc[:, 0], cc[:, 1], cc[:, 2]] = g
    out = np.zeros((side // 2,) * 3 + (C,), np.int64)
    for c in range(8):
        ox, oy, oz = c >> 2, (c >> 1) & 1, c & 1
        out += G[ox::2, oy::2, oz::2] @ W[c].astype(np.int64).T
    assert np.array_equal(acc, out[pc[:, 0], pc[:, 1], pc[:, 2]])


def _exact_rq(acc, m, r):
    v = Fraction(acc * m, 2 ** r)
    q = (v + Fraction(1, 2)).__floor__()     # round half up
    return max(-128, min(127, q))


def test_rq_golden_values():
    g = json.load(open(GOLD))
    for ex in g["requant"]:
        assert O.rq(ex["acc"], ex["m"], ex["r"]) == ex["q"], ex["cite"]
    for ex in g["linear"]:
        x = np.array(ex["x"]); w = np.array(ex["w"])
        assert int(x @ w) + ex["b"] == ex["y"]


def test_rq_prq_exact_rational():
    rng = np.random.default_rng(5)
    for _ in range(20000):
        acc = int(rng.integers(-2 ** 31, 2 ** 31))
        m = int(rng.integers(0, 2 ** 31))
        r = int(rng.integers(0, 63))
        assert O.rq(acc, m, r) == _exact_rq(acc, m, r)
        mn = int(rng.integers(0, 2 ** 31))
        assert O.prq(acc, m, mn, r) == _exact_rq(acc, m if acc >= 0 else mn, r)
    # ties round up
    assert O.rq(1, 1, 1) == 1 and O.rq(-1, 1, 1) == 0 and O.rq(3, 1, 1) == 2 and O.rq(-3, 1, 1) == -1


def test_rq_monotone():
    accs = np.sort(np.random.default_rng(6).integers(-2 ** 24, 2 ** 24, 3000))
    q = [O.rq(int(a), 12345, 17) for a in accs]
    assert all(b >= a for a, b in zip(q, q[1:]))


def _naive_up(S, X, W, b, mp, mn, r, q_one):
    C = S.shape[1]
    onehot = np.zeros((X.size, 255), np.int64)
    onehot[np.arange(X.size), X.astype(np.int64) - 1] = q_one
    x = np.concatenate([S.astype(np.int64), onehot], 1)          # Concat(S, X)
    acc = x @ W.astype(np.int64).T + b                            # Linear
    U = np.vectorize(lambda a: _exact_rq(int(a), mp if a >= 0 else mn, r))(acc)  # PReLU-requant
    rows = []
    for p in range(X.size):                                       # Pruning
        for c in range(8):
            if (int(X[p]) >> c) & 1:
                rows.append(U[p, c * C:(c + 1) * C])
    return np.array(rows, np.int64).reshape(-1, C)


@pytest.mark.parametrize("seed", range(3))
def test_up_prune(seed):
    rng = np.random.default_rng(300 + seed)
    C, n = 8, 40
    S = rng.integers(-128, 128, size=(n, C)).astype(np.int8)
    X = rng.integers(1, 256, size=n).astype(np.uint8)
    X[0], X[1] = 255, 1
    W = rng.integers(-63, 64, size=(8 * C, C + 255)).astype(np.int8)
    b = rng.integers(-2000, 2000, size=8 * C).astype(np.int32)
    out = O.up_prune(S, X, W, b, 9000, 2250, 20, 127)
    assert out.shape[0] == int(np.unpackbits(X).sum())
    assert np.array_equal(out.astype(np.int64), _naive_up(S, X, W, b, 9000, 2250, 20, 127))
    # code 255 -> 8 rows, block c to child c; code 1 -> only block 0
    one = O.up_prune(S[:1], X[:1], W, b, 1, 1, 0, 127)
    full = _naive_up(S[:1], np.array([255], np.uint8), W, b, 1, 1, 0, 127)
    assert one.shape == (8, C) and np.array_equal(one.astype(np.int64), full)
    z = O.up_prune(S[1:2], X[1:2], W, b, 1, 1, 0, 127)
    assert z.shape == (1, C) and np.array_equal(z.astype(np.int64), _naive_up(S[1:2], X[1:2], W, b, 1, 1, 0, 127))


def _wired_model(**kw):
    m = I.make_model(C=8, H=8, seed=3, min_depth=9, max_depth=12)
    return m


def test_resblock_identity_skip_wiring():
    """Eq.8: S = ResBlock(F); with zero convs, zero bias, k_s = 1, rq = identity -> S = F."""
    m = _wired_model()
    for d, s in m.shallow.items():
        s.Wa[:] = 0; s.Wb[:] = 0; s.ba[:] = 0; s.bb[:] = 0
        s.k_s = 1; s.rqb = I.RQ(1, 1, 0)
    om = O.Model(m.to_bytes())
    pts = I.make_frame(I.CFG1)
    D = O.Dump()
    O.encode(om, pts, 12, D)
    for d in range(m.R, 12 - 1 - m.n_deep + 1):
        assert np.array_equal(D.get(f"S/{d}", np.int8), D.get(f"F/{d - 1}", np.int8)), d


@pytest.mark.parametrize("which", ["F", "G"])
def test_xfp_concat_wiring(which):
    """Eq.10: H = ResBlock(Concat(F^k, G^k)); zero convs + identity requant and the 1x1
    projection P = [I|0] selects F_D, P = [0|I] selects G_D (the channel order of the concat)."""
    m = _wired_model()
    C = m.C
    for dp in m.deep:
        dp.Wa[:] = 0; dp.Wb[:] = 0; dp.ba[:] = 0; dp.bb[:] = 0
        dp.P[:] = 0
        off = 0 if which == "F" else C
        dp.P[np.arange(C), off + np.arange(C)] = 1
        dp.rqb = I.RQ(1, 1, 0)
    om = O.Model(m.to_bytes())
    pts = I.make_frame(I.CFG1)
    D = O.Dump()
    O.encode(om, pts, 12, D)
    Dd = 12 - 1 - m.n_deep
    for j in range(1, m.n_deep + 1):
        d = Dd + j
        want = D.get(f"F/{Dd}", np.int8) if which == "F" else D.get(f"G/{d}/{Dd}", np.int8)
        assert np.array_equal(D.get(f"H/{d}", np.int8), want), d
    # j = 1: no down steps, G_D is the plain embedding E_1[X_D] (Eq.4 with k = l-1)
    codes = D.get(f"code/{Dd}", np.uint8)
    assert np.array_equal(D.get(f"G/{Dd + 1}/{Dd}", np.int8).reshape(-1, C), m.deep[0].E[codes.astype(int) - 1])
