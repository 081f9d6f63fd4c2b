"""Oracle pins of the functions the codec itself runs (round 2).

* K2S2 down (Eq.4, reading Q4): the codec's `down_step` accumulator (`oracle_down_acc`
  now calls the same `down_acc`) against a dense stride-2 numpy conv, and every G/d/k
  dump of a real encode against a numpy int64 stride-2 conv + PReLU-requant of the
  dump one depth below (so a transposed W index in the codec fails here);
* Eq.7 predictor (reading Q9): `head_logits` on random W1, b1, W2, b2
  against numpy int64 matmuls, and the a/d, z/d dumps of a real encode against the
  same numpy Eq.7 evaluated on the dumped predictor input;
* model-file validation: exp tables outside (65281, 2^24] or increasing, and R > 6,
  are rejected (INVALID_ARG) — reading Q20/Q21 need S in (65281, 255 * 2^24];
* Table 4 ablations: XFP off (H = ResBlock(G_D)) and GRED off (n_deep = 0)
  round-trip, and their wiring special cases (zero convs + k_s = 1 + identity requant
  give H = G_D);
* the symbol-frequency raw-prefix coder (reading Q13'): round trip, the first
  symbol's closed-form Q16 mass (257 / 258), and the coded length against the ideal
  adaptive code length sum log2(T_i / n_i) of the textbook frequency-count model.
"""
import math
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I


def _coords(keys, bits):
    k = np.asarray(keys, np.uint64)
    x = np.zeros(k.size, np.int64); y = np.zeros_like(x); z = np.zeros_like(x)
    for b in range(bits):
        t = (k >> np.uint64(3 * b)) & np.uint64(7)
        x |= ((t >> np.uint64(2)) & np.uint64(1)).astype(np.int64) << b
        y |= ((t >> np.uint64(1)) & np.uint64(1)).astype(np.int64) << b
        z |= (t & np.uint64(1)).astype(np.int64) << b
    return np.stack([x, y, z], 1)


def _prq(acc, rq):
    """Eq.14 round half up with PReLU slope (m_neg for acc < 0), int64 floor division."""
    acc = np.asarray(acc, np.int64)
    m = np.where(acc >= 0, rq.m_pos, rq.m_neg).astype(np.int64)
    v = acc * m
    if rq.r > 0:
        v = (v + (1 << (rq.r - 1))) // (1 << rq.r)
    return np.clip(v, -128, 127)


def _dense_down(child_keys, parent_keys, depth_c, g, W):
    """Dense stride-2 conv on the depth-depth_c grid: out(p) = sum_c W_c g(2p + c)."""
    cc, pc = _coords(child_keys, depth_c), _coords(parent_keys, depth_c - 1)
    lo = pc.min(0)
    side = int((pc.max(0) - lo).max()) + 1
    C = g.shape[1]
    G = np.zeros((2 * side, 2 * side, 2 * side, C), np.int64)
    rel = cc - 2 * lo
    G[rel[:, 0], rel[:, 1], rel[:, 2]] = g
    out = np.zeros((side, side, side, C), np.int64)
    for c in range(8):
        ox, oy, oz = c >> 2, (c >> 1) & 1, c & 1
        out += G[ox::2, oy::2, oz::2] @ W[c].astype(np.int64).T
    q = pc - lo
    return out[q[:, 0], q[:, 1], q[:, 2]]


@pytest.fixture(scope="module")
def encoded():
    m = I.make_model(C=8, H=8, seed=11, min_depth=9, max_depth=12)
    om = O.Model(m.to_bytes())
    pts = I.make_frame(I.CFG1, 4)
    D = O.Dump()
    bs = O.encode(om, pts, 12, D)
    return m, om, pts, D, bs


def test_down_step_codec_dumps_equal_dense_stride2(encoded):
    """Every K2S2 step the codec ran (G/d/k -> G/d/k-1) equals a dense stride-2 conv."""
    m, _, _, D, _ = encoded
    L, C = 12, m.C
    Dd = L - 1 - m.n_deep
    keys = {d: D.get(f"key/{d}", np.uint64) for d in range(L + 1)}
    steps = 0
    for j in range(2, m.n_deep + 1):
        d = Dd + j
        for s in range(j - 1):
            k = d - 1 - s
            g = D.get(f"G/{d}/{k}", np.int8).reshape(-1, C)
            want = D.get(f"G/{d}/{k - 1}", np.int8).reshape(-1, C)
            dn = m.deep[j - 1].downs[s]
            acc = _dense_down(keys[k], keys[k - 1], k, g, dn.W) + dn.b.astype(np.int64)
            assert np.array_equal(_prq(acc, dn.rq), want.astype(np.int64)), (d, k)
            steps += 1
    assert steps == 6


@pytest.mark.parametrize("seed", range(3))
def test_down_acc_is_the_codec_accumulator(seed):
    rng = np.random.default_rng(400 + seed)
    pts = np.argwhere(rng.random((16, 16, 16)) < 0.2).astype(np.int32)
    keys, _ = O.build_octree(pts, 4)
    C = 16
    g = rng.integers(-128, 128, size=(keys[4].size, C)).astype(np.int8)
    W = rng.integers(-127, 128, size=(8, C, C)).astype(np.int8)
    assert np.array_equal(O.down_acc(keys[4], keys[3], g, W), _dense_down(keys[4], keys[3], 4, g, W))
    with pytest.raises(O.OracleError):  # a child without its parent is an argument error
        O.down_acc(keys[4], keys[3][1:], g, W)


@pytest.mark.parametrize("C,H", [(8, 8), (32, 32), (16, 24)])
def test_head_logits_eq7_random_weights(C, H):
    rng = np.random.default_rng(C * 100 + H)
    n = 300
    F = rng.integers(-128, 128, size=(n, C)).astype(np.int8)
    W1 = rng.integers(-127, 128, size=(H, C)).astype(np.int8)
    b1 = rng.integers(-5000, 5000, size=H).astype(np.int32)
    W2 = rng.integers(-127, 128, size=(255, H)).astype(np.int8)
    b2 = rng.integers(-10 ** 6, 10 ** 6, size=255).astype(np.int32)
    rq1 = I.RQ(700, 180, 16)
    a, z = O.head_logits(F, W1, b1, (rq1.m_pos, rq1.m_neg, rq1.r), W2, b2)
    want_a = _prq(F.astype(np.int64) @ W1.astype(np.int64).T + b1, rq1)   # a = PReLU-rq(W1 F + b1)
    assert np.array_equal(a.astype(np.int64), want_a)
    want_z = want_a @ W2.astype(np.int64).T + b2                           # z = W2 a + b2
    assert np.array_equal(z.astype(np.int64), want_z)


def test_head_logits_codec_dumps_eq7(encoded):
    """The a/d and z/d tensors of a real encode equal numpy Eq.7 on the dumped head input."""
    m, _, _, D, _ = encoded
    L, C, H = 12, m.C, m.H
    Dd = L - 1 - m.n_deep
    for d in range(m.R, L):
        if d <= Dd:
            F, hd = D.get(f"F/{d}", np.int8), m.shallow[d].head
        else:
            F, hd = D.get(f"Fp/{d}/{d}", np.int8), m.deep[d - Dd - 1].head
        F = F.reshape(-1, C).astype(np.int64)
        a = _prq(F @ hd.W1.astype(np.int64).T + hd.b1, hd.rq1)
        assert np.array_equal(D.get(f"a/{d}", np.int8).reshape(-1, H).astype(np.int64), a), d
        z = a @ hd.W2.astype(np.int64).T + hd.b2
        assert np.array_equal(D.get(f"z/{d}", np.int32).reshape(-1, 255).astype(np.int64), z), d


# ---------------------------------------------------------------------------------------
# model-file validation (exp table, raw_bytes width)
# ---------------------------------------------------------------------------------------

def _with_lut(mb, lut):
    body = bytearray(mb[:-8])
    body[64:64 + 4096] = np.asarray(lut, "<u4").tobytes()
    return bytes(body) + struct.pack("<Q", I.fnv1a64(bytes(body)))


@pytest.mark.parametrize("bad", ["zero", "small", "big", "increasing"])
def test_bad_exp_table_rejected(bad):
    mb = I.make_model(C=8, H=8, seed=1, max_depth=12).to_bytes()
    lut = I.exp_lut().astype(np.int64)
    if bad == "zero":
        lut[:] = 0
    elif bad == "small":   # a scaled table, non-increasing, with LUT[0] = 65281
        lut = lut * 65281 // (1 << 24)
    elif bad == "big":
        lut[0] = (1 << 24) + 1
    else:
        lut[500] = lut[499] + 1
    with pytest.raises(O.OracleError) as e:
        O.Model(_with_lut(mb, lut))
    assert e.value.name == "INVALID_ARG"
    O.Model(_with_lut(mb, I.exp_lut()))  # the table itself is accepted


def test_raw_levels_cap():
    m = I.make_model(C=8, H=8, seed=1, R=6, n_deep=2, min_depth=9, max_depth=12)
    O.Model(m.to_bytes())
    m.R = 7
    m.shallow = {d: m.shallow.get(d, m.shallow[6]) for d in range(7, 12 - 2)}
    with pytest.raises(O.OracleError) as e:
        O.Model(m.to_bytes())
    assert e.value.name == "INVALID_ARG"


# ---------------------------------------------------------------------------------------
# Table 4 ablation variants (NEXT-1)
# ---------------------------------------------------------------------------------------

def _dedup_sorted(pts, L):
    keys, _ = O.build_octree(pts, L)
    return _coords(keys[L], L).astype(np.int32)


@pytest.mark.parametrize("variant", ["xfp_off", "gred_off", "xfp_off_raw_freq"])
@pytest.mark.parametrize("L", [10, 12])
def test_ablation_variants_round_trip(variant, L):
    kw = {"xfp_off": dict(xfp=False), "gred_off": dict(n_deep=0),
          "xfp_off_raw_freq": dict(xfp=False, raw_freq=True)}[variant]
    m = I.make_model(C=8, H=8, seed=9, min_depth=9, max_depth=13, **kw)
    om = O.Model(m.to_bytes())
    pts = I.make_frame(I.CFG1, 2) >> (12 - L)
    bs = O.encode(om, pts, L)
    assert bs[8] == m.n_deep and bs[9] == m.flags
    xyz, LL = O.decode(om, bs)
    assert LL == L and np.array_equal(xyz, _dedup_sorted(pts, L))
    full = O.Model(I.make_model(C=8, H=8, seed=9, min_depth=9, max_depth=13).to_bytes())
    with pytest.raises(O.OracleError) as e:
        O.decode(full, bs)
    assert e.value.name == "MODEL_MISMATCH"


def test_xfp_off_wiring_is_resblock_of_g():
    """XFP off: zero convs, k_s = 1 and an identity requant give H = G_D exactly."""
    m = I.make_model(C=8, H=8, seed=3, min_depth=9, max_depth=12, xfp=False)
    for dp in m.deep:
        dp.Wa[:] = 0; dp.Wb[:] = 0; dp.ba[:] = 0; dp.bb[:] = 0
        dp.k_s = 1; dp.rqb = I.RQ(1, 1, 0)
    om = O.Model(m.to_bytes())
    D = O.Dump()
    O.encode(om, I.make_frame(I.CFG1), 12, D)
    Dd = 12 - 1 - m.n_deep
    for j in range(1, m.n_deep + 1):
        d = Dd + j
        assert np.array_equal(D.get(f"H/{d}", np.int8), D.get(f"G/{d}/{Dd}", np.int8)), d


def test_gred_off_every_level_is_shallow():
    """n_deep = 0: every coded level runs the Eq.8-9 shallow step; no G/H tensors exist."""
    m = I.make_model(C=8, H=8, seed=3, n_deep=0, min_depth=9, max_depth=12)
    om = O.Model(m.to_bytes())
    D = O.Dump()
    O.encode(om, I.make_frame(I.CFG1), 12, D)
    names = D.names()
    assert all(f"S/{d}" in names and f"F/{d}" in names for d in range(4, 12))
    assert not any(n.startswith(("G/", "H/", "hx/", "Fp/")) for n in names)


# ---------------------------------------------------------------------------------------
# symbol-frequency raw-prefix coder (NEXT-4)
# ---------------------------------------------------------------------------------------

def _raw_region(bs):
    L, Rr = bs[6], bs[7]
    raw = struct.unpack_from("<H", bs, 10)[0]
    p = 24 + 4 * (L - Rr)
    return bs[p:p + raw]


def _raw_symbols(pts, L, R=4):
    _, codes = O.build_octree(pts, L)
    return np.concatenate(codes[:R]).astype(np.int64)


def _ideal_adaptive_bits(sym, inc=32, limit=1 << 15):
    """Ideal code length of the frequency-count model: sum_i log2(T_i / n_{s_i})."""
    n = np.ones(255, np.int64)
    bits = 0.0
    for s in sym:
        bits += math.log2(n.sum() / n[s - 1])
        n[s - 1] += inc
        if n.sum() > limit:
            n = (n + 1) // 2
    return bits


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "single", "cube", "random"])
def test_raw_freq_round_trip_and_length(case):
    m = I.make_model(C=8, H=8, seed=4, min_depth=9, max_depth=12, raw_freq=True)
    om = O.Model(m.to_bytes())
    plain = O.Model(I.make_model(C=8, H=8, seed=4, min_depth=9, max_depth=12).to_bytes())
    g = np.arange(2, dtype=np.int32)
    pts = {"cfg1": I.make_frame(I.CFG1), "cfg2": I.make_frame(I.CFG2, 7),
           "single": np.array([[5, 600, 7]], np.int32),
           "cube": np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) * 512,
           "random": I.random_cloud(3000, 12, 8)}[case]
    bs = O.encode(om, pts, 12)
    xyz, _ = O.decode(om, bs)
    assert np.array_equal(xyz, _dedup_sorted(pts, 12))
    reg = _raw_region(bs)
    W = struct.unpack_from("<I", reg, 0)[0]
    assert len(reg) == 8 + 4 * ((W + 1) // 2)
    sym = _raw_symbols(pts, 12)
    ideal = _ideal_adaptive_bits(sym)
    # one rANS lane: the words carry the information up to the Q16 mass quantisation
    # (each p within one count of 65281 n / T, under 0.05 bit for n/T >= 2^-8 here) and
    # the final state's up to 32 bits
    assert 16 * W <= ideal * 1.01 + 1 + 0.05 * sym.size
    assert 16 * W + 32 >= ideal * 0.98 - 16
    # the neural payload is untouched by the raw coder: only the raw region differs
    bp = O.encode(plain, pts, 12)
    assert _raw_region(bp) == bytes(sym.astype(np.uint8))


@pytest.mark.parametrize("pt,v", [((0, 0, 0), 1), ((4095, 4095, 4095), 128), ((0, 4095, 4095), 8)])
def test_raw_freq_first_symbol_closed_form(pt, v):
    """All counts 1, T = 255: C_i = i + floor(i * 65281 / 255) = 257 i, so every symbol but
    the last has mass 257.  With R = 1 the raw prefix is the single root code X_0 = v of a
    one-point cloud; one rANS step from x = 2^16 (no word emitted since x < 257 * 2^16)
    leaves x = ((2^16 // 257) << 16) + 2^16 % 257 + 257 (v - 1)."""
    m = I.make_model(C=8, H=8, seed=4, R=1, min_depth=9, max_depth=12, raw_freq=True)
    om = O.Model(m.to_bytes())
    pts = np.array([pt], np.int32)
    bs = O.encode(om, pts, 12)
    reg = _raw_region(bs)
    assert _raw_symbols(pts, 12, R=1).tolist() == [v]
    W, x = struct.unpack_from("<II", reg, 0)
    assert len(reg) == 8 and W == 0
    assert x == ((65536 // 257) << 16) + 65536 % 257 + 257 * (v - 1)
    assert np.array_equal(O.decode(om, bs)[0], pts)
