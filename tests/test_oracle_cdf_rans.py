"""Oracle pins: exp LUT, integer softmax -> Q16 pmf (Eq.15), rANS segments.

Pins (DESIGN.md §"Oracle pins"):
* LUT entries vs math.exp (the LUT is data written by the model generator);
* closed forms (tests/golden/cdf_closed_forms.json): all-equal logits, a logit >= 16
  nats above the rest, two equal maxima >= 16 nats above the rest;
* invariants on random rows: sum p = 65536, min p >= 1, invariant to a common shift;
  each p_i is 1 + floor or 1 + ceil of e_i 65281 / S (a difference of two floors,
  reading Q21), hence monotone in the logit up to one count;
* the derived approximation bound |p_i/2^16 - softmax_i| <= 0.012*softmax_i + 0.0040
  (LUT step e^{3/256}-1 < 0.0118 relative; normalisation <= 256/65536 absolute);
* rANS: decode(encode(s)) = s; code length within the entropy bound of the
  (cum, freq) it was given (north_star: "code length within a few bytes of the sum
  of -log2 p").
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cdf_closed_forms.json")
LUT = I.exp_lut()


def test_lut_against_math_exp():
    assert LUT[0] == 2 ** 24
    for j in range(1024):
        assert abs(int(LUT[j]) - 2 ** 24 * math.exp(-j / 64.0)) <= 0.5 + 1e-6
    assert np.all(np.diff(LUT.astype(np.int64)) <= 0)
    assert LUT[1023] >= 1


def test_closed_forms():
    g = {c["name"]: c for c in json.load(open(GOLD))["cases"]}
    p = O.cdf(np.full((1, 255), 12345, np.int32), 1, 0, LUT)[0]
    assert p[254] == g["all_equal"]["p_last"] and np.all(p[:254] == g["all_equal"]["p_rest"])
    for pos in (0, 17, 254):
        z = np.zeros((1, 255), np.int32)
        z[0, pos] = g["dominant"]["gap_q8"]
        p = O.cdf(z, 1, 0, LUT)[0]
        assert p[pos] == g["dominant"]["p_max"] and np.all(np.delete(p, pos) == g["dominant"]["p_rest"])
    t = g["two_maxima"]
    for a, b in ((0, 1), (3, 200), (100, 254)):
        z = np.zeros((1, 255), np.int32)
        z[0, a] = z[0, b] = t["gap_q8"]
        p = O.cdf(z, 1, 0, LUT)[0]
        assert p[a] == t["p_first_max"] and p[b] == t["p_second_max"]
        assert np.all(np.delete(p, [a, b]) == t["p_rest"])


def _softmax_q8(z):
    l = z.astype(np.float64) / 256.0
    e = np.exp(l - l.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def test_invariants_and_bound():
    rng = np.random.default_rng(11)
    for scale in (64, 512, 2048, 8192):
        z = rng.normal(0, scale, size=(2000, 255)).astype(np.int32)
        p = O.cdf(z, 1, 0, LUT).astype(np.int64)
        assert np.all(p.sum(1) == 65536) and p.min() >= 1
        q = _softmax_q8(z)
        err = np.abs(p / 65536.0 - q)
        assert np.all(err <= 0.012 * q + 0.0040), err.max()
        # p_i - 1 is floor(E_{i+1} K/S) - floor(E_i K/S), i.e. floor or ceil of e_i K/S:
        # checked against exact rationals from the model's LUT exponentials
        l = z.astype(np.int64)  # m = 1, r = 0: Q8 logits are z itself (|z| < 2^24)
        d = l.max(1, keepdims=True) - l
        e = np.where(d < 4096, LUT[np.minimum(d, 4095) >> 2].astype(np.int64), 0)
        S = e.sum(1, keepdims=True)
        lo, hi = 1 + (e * 65281) // S, 1 + -((-e * 65281) // S)
        assert np.all((p == lo) | (p == hi))
        # hence monotone in the logit up to one count: l_i >= l_j -> p_i >= p_j - 1
        for r in range(0, 2000, 97):
            o = np.argsort(z[r], kind="stable")
            assert np.all(np.diff(p[r][o]) >= -1)


def test_shift_and_cumulative_structure():
    rng = np.random.default_rng(12)
    z = rng.normal(0, 1000, size=(200, 255)).astype(np.int32)
    p = O.cdf(z, 1, 0, LUT)
    assert np.array_equal(O.cdf(z + 77777, 1, 0, LUT), p)
    # splitting the row at any symbol: the cumulative count before it is the floor of its
    # exact share of the prefix mass, i.e. within one count of 65536 * (prefix softmax mass)
    cum = np.concatenate([np.zeros((200, 1), np.int64), np.cumsum(p.astype(np.int64), 1)], 1)
    q = _softmax_q8(z)
    qc = np.concatenate([np.zeros((200, 1)), np.cumsum(q, 1)], 1)
    i = np.arange(256)[None, :]
    assert np.all(np.abs(cum - i - 65281 * qc) <= 1 + 0.012 * 65281 * qc + 1e-6)


def test_logit_requant_clamp():
    # l = clamp(round(z*m/2^r), +-2^24): huge z saturate but stay exact
    z = np.zeros((1, 255), np.int32)
    z[0, 3] = 2 ** 31 - 1
    p = O.cdf(z, 2 ** 20, 0, LUT)[0]
    assert p[3] == 65282


def _random_stream(rng, n, peaky):
    pmf = []
    sym = rng.integers(1, 256, size=n)
    z = rng.normal(0, 256 * peaky, size=(n, 255)).astype(np.int32)
    pmf = O.cdf(z, 1, 0, LUT)
    cum = np.concatenate([np.zeros((n, 1), np.int64), np.cumsum(pmf, 1)[:, :-1]], 1)
    c = cum[np.arange(n), sym - 1]
    f = pmf[np.arange(n), sym - 1]
    return sym.astype(np.uint8), pmf, c.astype(np.uint32), f.astype(np.uint32)


@pytest.mark.parametrize("n,peaky", [(1, 1.0), (7, 0.5), (511, 2.0), (513, 1.0), (16384, 3.0), (40000, 0.1)])
def test_rans_round_trip_and_length(n, peaky):
    rng = np.random.default_rng(n)
    sym, pmf, c, f = _random_stream(rng, n, peaky)
    data = O.rans_encode(c, f)
    out, used = O.rans_decode(data, pmf)
    assert used == len(data) and np.array_equal(out, sym)
    K = min(8, max(1, -(-n // 512)))
    ideal_bits = float(np.sum(np.log2(65536.0 / f)))
    payload_bits = 8 * (len(data) - 4 - 4 * K)       # words (+pad), excluding W and states
    # upper: each lane's flush costs its 32-bit final state (counted separately) and
    # rANS loses < 0.2 % to integer division; lower: the integer state update has a
    # zero-mean deviation from x*M/f, whose Jensen gap makes the words slightly shorter
    # than sum -log2 p (the final states carry the rest).
    assert payload_bits <= ideal_bits * 1.002 + 16 * K
    assert payload_bits >= ideal_bits * 0.98 - 16 * K - 16


def test_rans_corrupt_streams_fail_cleanly():
    rng = np.random.default_rng(99)
    sym, pmf, c, f = _random_stream(rng, 5000, 1.0)
    data = bytearray(O.rans_encode(c, f))
    with pytest.raises(O.OracleError):
        O.rans_decode(bytes(data[:len(data) // 2]), pmf)
    bad = 0
    for i in range(40):
        d = bytearray(data)
        pos = int(rng.integers(4, len(d)))
        d[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            out, _ = O.rans_decode(bytes(d), pmf)
            bad += not np.array_equal(out, sym)
        except O.OracleError as e:
            assert e.name in ("CORRUPT", "TRUNCATED")
    assert bad == 0  # a flipped bit is always caught (final-state check) or harmless
