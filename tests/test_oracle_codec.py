"""Oracle pins: end-to-end codec (encode/decode, container, errors).

Pins (DESIGN.md §"Oracle pins"):
* decode(encode(x)) == dedup(x) in Morton order (north_star);
* zero model: every pmf is [257 x 254, 258] (closed form), so the payload length is
  fixed by the code histogram alone, within the rANS bound (words <= 1.002*ideal
  + 16K bits; >= 0.98*ideal - 32: the integer state update x' = (x//f)*M + x%f + c
  has a zero-mean deviation from x*M/f whose Jensen gap makes the words ~0.5 %
  SHORTER than sum -log2 p, the rest of the information sits in the K final states);
* bias-only head: every node of a level shares one pmf, so the length is
  sum_v count_v * log2(65536 / p_v) within the rANS bound;
* any model: payload == sum -log2(p_sym) over the oracle's own pmf dumps within
  the rANS bound (north_star: "code length within a few bytes of the sum of -log2 p");
* determinism, input-order and duplicate invariance; error statuses
   for bad magic/version/model/truncation/corruption/empty/range/depth.
"""
import math
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

R = 4


def _small_model(kind="random", max_depth=12, C=8):
    return I.make_model(C=C, H=C, seed=5, min_depth=9, max_depth=max_depth, kind=kind)


def _sets_equal(a, b):
    return {tuple(p) for p in np.asarray(a).tolist()} == {tuple(p) for p in np.asarray(b).tolist()}


def _morton_sorted(xyz, L):
    def key(p):
        k = 0
        for b in range(L):
            k |= (((p[0] >> b) & 1) << 2 | ((p[1] >> b) & 1) << 1 | ((p[2] >> b) & 1)) << (3 * b)
        return k
    return sorted(set(map(tuple, np.asarray(xyz).tolist())), key=key)


def _parse(bs):
    L, Rr, nd = bs[6], bs[7], bs[8]
    raw = struct.unpack_from("<H", bs, 10)[0]
    lb = struct.unpack_from(f"<{L - Rr}I", bs, 24)
    pos = 24 + 4 * (L - Rr) + (raw + 3) // 4 * 4
    levels = {}
    for i, n in enumerate(lb):
        levels[Rr + i] = bs[pos:pos + n]
        pos += n
    assert pos == len(bs)
    return L, levels


def _payload_bits(level_bytes, N):
    """Bits of rANS words in a level payload (segment headers/states excluded) and lane count."""
    bits, lanes, pos, left = 0, 0, 0, N
    while left > 0:
        n = min(4096, left)
        K = min(8, max(1, -(-n // 512)))
        W = struct.unpack_from("<I", level_bytes, pos)[0]
        bits += 16 * W
        lanes += K
        pos += 4 + 4 * K + 4 * ((W + 1) // 2)
        left -= n
    assert pos == len(level_bytes)
    return bits, lanes


@pytest.fixture(scope="module")
def model():
    return O.Model(_small_model().to_bytes())


@pytest.mark.parametrize("L,cloud", [(12, "cfg1"), (9, "single"), (10, "random"), (12, "cube")])
def test_round_trip(model, L, cloud):
    if cloud == "cfg1":
        pts = I.make_frame(I.CFG1)
    elif cloud == "single":
        pts = np.array([[3, 400, 511]], np.int32)
    elif cloud == "random":
        pts = I.random_cloud(3000, L, 1)
    else:
        g = np.arange(4, dtype=np.int32)
        pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 1000
    bs = O.encode(model, pts, L)
    out, Lo = O.decode(model, bs)
    assert Lo == L
    assert _sets_equal(out, pts)
    assert [tuple(p) for p in out.tolist()] == _morton_sorted(pts, L)


def test_max_depth_21_round_trip():
    m = O.Model(_small_model(max_depth=21).to_bytes())
    pts = I.random_cloud(500, 21, 3)
    bs = O.encode(m, pts, 21)
    out, L = O.decode(m, bs)
    assert L == 21 and _sets_equal(out, pts)


@pytest.mark.parametrize("n_deep,L", [(1, 9), (2, 11), (3, 12), (3, 14)])
def test_deep_level_variants_round_trip(n_deep, L):
    """NEXT-1 variants: t = L - n_deep + 1 (paper t = L-4 is n_deep = 4; the t = L-3
    ablation of P:681-710 is n_deep = 3).  The deep/shallow split moves, the container
    records n_deep, and decode(encode(x)) is still dedup(x) in Morton order."""
    m = O.Model(I.make_model(C=8, H=8, seed=11, n_deep=n_deep, min_depth=max(R + 1 + n_deep, 9),
                             max_depth=16).to_bytes())
    pts = I.random_cloud(2500, L, 4)
    bs = O.encode(m, pts, L)
    assert bs[8] == n_deep
    out, Lo = O.decode(m, bs)
    assert Lo == L and [tuple(p) for p in out.tolist()] == _morton_sorted(pts, L)
    # a stream coded with another n_deep is refused before any entropy decoding
    other = O.Model(I.make_model(C=8, H=8, seed=11, n_deep=4 if n_deep != 4 else 3, min_depth=9,
                                 max_depth=16).to_bytes())
    with pytest.raises(O.OracleError):
        O.decode(other, bs)


def test_zero_model_closed_form_length():
    m = O.Model(_small_model("zero").to_bytes())
    pts = I.make_frame(I.CFG1)
    keys, codes = O.build_octree(pts, 12)
    L, levels = _parse(O.encode(m, pts, 12))
    for d in range(R, L):
        n255 = int((codes[d] == 255).sum())  # symbol 255 = index 254 gets 258 (reading Q21)
        ideal = n255 * math.log2(65536 / 258) + (codes[d].size - n255) * math.log2(65536 / 257)
        bits, K = _payload_bits(levels[d], codes[d].size)
        assert ideal * 0.98 - 16 * K - 16 <= bits <= ideal * 1.002 + 16 * K, d


def test_bias_only_head_length():
    mm = _small_model("bias_head")
    m = O.Model(mm.to_bytes())
    pts = I.make_frame(I.CFG1)
    keys, codes = O.build_octree(pts, 12)
    L, levels = _parse(O.encode(m, pts, 12))
    D = L - 1 - mm.n_deep
    for d in range(R, L):
        head = mm.shallow[d].head if d <= D else mm.deep[d - D - 1].head
        p = O.cdf(head.b2[None, :].astype(np.int32), head.rq_logit.m_pos, head.rq_logit.r, mm.lut)[0]
        hist = np.bincount(codes[d], minlength=256)[1:]
        ideal = float(np.sum(hist * np.log2(65536.0 / p)))
        bits, K = _payload_bits(levels[d], codes[d].size)
        assert ideal * 0.98 - 16 * K - 16 <= bits <= ideal * 1.002 + 16 * K, d


def test_length_matches_pmf_dumps(model):
    pts = I.make_frame(I.CFG1)
    D = O.Dump()
    L, levels = _parse(O.encode(model, pts, 12, D))
    for d in range(R, L):
        p = D.get(f"p/{d}", np.uint16).reshape(-1, 255).astype(np.float64)
        x = D.get(f"code/{d}", np.uint8).astype(np.int64)
        ideal = float(np.sum(np.log2(65536.0 / p[np.arange(x.size), x - 1])))
        bits, K = _payload_bits(levels[d], x.size)
        assert ideal * 0.98 - 16 * K - 16 <= bits <= ideal * 1.002 + 16 * K, d
        # pmf rows are valid Q16 distributions
        assert np.all(p.sum(1) == 65536) and p.min() >= 1


def test_decoder_reproduces_encoder_pmfs(model):
    pts = I.make_frame(I.CFG1)
    De, Dd = O.Dump(), O.Dump()
    bs = O.encode(model, pts, 12, De)
    O.decode(model, bs, Dd)
    for d in range(R, 12):
        assert np.array_equal(De.get(f"p/{d}", np.uint16), Dd.get(f"p/{d}", np.uint16)), d


def test_determinism_order_duplicates(model):
    pts = I.random_cloud(2000, 11, 8)
    rng = np.random.default_rng(1)
    a = O.encode(model, pts, 11)
    assert O.encode(model, pts, 11) == a
    assert O.encode(model, pts[rng.permutation(len(pts))], 11) == a
    assert O.encode(model, np.concatenate([pts, pts[:500]]), 11) == a


def test_errors(model):
    pts = I.random_cloud(300, 10, 2)
    bs = O.encode(model, pts, 10)

    def st(f):
        with pytest.raises(O.OracleError) as e:
            f()
        return e.value.name

    assert st(lambda: O.encode(model, np.zeros((0, 3), np.int32), 10)) == "EMPTY"
    assert st(lambda: O.encode(model, np.array([[0, 0, 1024]], np.int32), 10)) == "RANGE"
    assert st(lambda: O.encode(model, pts, 8)) == "UNSUPPORTED_DEPTH"
    assert st(lambda: O.encode(model, pts, 13)) == "UNSUPPORTED_DEPTH"
    assert st(lambda: O.decode(model, b"XCC1" + bs[4:])) == "BAD_MAGIC"
    assert st(lambda: O.decode(model, bs[:4] + b"\x01\x00" + bs[6:])) == "VERSION"
    other = O.Model(I.make_model(C=8, H=8, seed=6, min_depth=9, max_depth=12).to_bytes())
    assert st(lambda: O.decode(other, bs)) == "MODEL_MISMATCH"
    assert st(lambda: O.decode(model, bs[:len(bs) - 7])) in ("TRUNCATED", "CORRUPT")
    assert st(lambda: O.decode(model, bs[:20])) == "TRUNCATED"


def test_bitflips_never_crash(model):
    pts = I.random_cloud(800, 10, 4)
    bs = O.encode(model, pts, 10)
    rng = np.random.default_rng(3)
    for _ in range(60):
        d = bytearray(bs)
        pos = int(rng.integers(24, len(d)))
        d[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            out, _ = O.decode(model, bytes(d))
        except O.OracleError as e:
            assert e.name in ("CORRUPT", "TRUNCATED")
