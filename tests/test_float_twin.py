"""NEXT-2: float twin of the occupancy head and the decode-collapse demo.

The paper's motivation (Fig.2b/c): a floating-point entropy model is
not bit-reproducible across devices / evaluation orders, and an arithmetic decoder fed a
CDF that differs from the encoder's in a single entry decodes garbage from there on; the
integer-only model is exact everywhere (our GPU path reproduces the oracle's CDFs and
bitstreams bit for bit: tests/test_gpu_parity.py).

Float twin (same weights, dequantised): a = PReLU(W1 F + b1) with slopes m_pos / 2^r and
m_neg / 2^r (the requant multipliers without rounding or clipping); z = W2 a + b2; logits
in nats l = z m_l / 2^r_l / 256 (Q8 -> nats, reading Q20); pmf p = softmax(l) quantised
like reading Q21: 1 + floor(p * 65281), leftover to the first argmax.  Two evaluation
orders stand in for two devices: float32 BLAS matmul vs float32 accumulation in reversed
order (and, on a GPU box, torch fp32 on cuda:0).  The rANS coder here is the single-lane
form of reading O9 (32-bit state, 16-bit words, M = 2^16).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

M = 1 << 16


def _head_inputs(model_obj, D, d, Dcut):
    F = D.get(f"F/{d}" if d <= Dcut else f"Fp/{d}/{d}", np.int8)
    hd = model_obj.shallow[d].head if d <= Dcut else model_obj.deep[d - Dcut - 1].head
    return F.reshape(-1, model_obj.C), hd


def float_logits(F, hd, order):
    """Float twin of Eq.7's predictor: nats, float32, evaluated in `order`."""
    f32 = np.float32
    W1, b1, W2, b2 = hd.W1.astype(f32), hd.b1.astype(f32), hd.W2.astype(f32), hd.b2.astype(f32)
    Fx = F.astype(f32)
    if order == "blas":
        h = Fx @ W1.T + b1
    else:  # reversed accumulation order, one float32 add at a time
        h = np.zeros((F.shape[0], W1.shape[0]), f32)
        for c in reversed(range(W1.shape[1])):
            h = (h + Fx[:, c:c + 1] * W1[None, :, c]).astype(f32)
        h = (h + b1).astype(f32)
    sp, sn = f32(hd.rq1.m_pos / 2.0 ** hd.rq1.r), f32(hd.rq1.m_neg / 2.0 ** hd.rq1.r)
    a = np.where(h >= 0, h * sp, h * sn).astype(f32)
    if order == "blas":
        z = a @ W2.T + b2
    else:
        z = np.zeros((F.shape[0], W2.shape[0]), f32)
        for k in reversed(range(W2.shape[1])):
            z = (z + a[:, k:k + 1] * W2[None, :, k]).astype(f32)
        z = (z + b2).astype(f32)
    return (z * f32(hd.rq_logit.m_pos / 2.0 ** hd.rq_logit.r / 256.0)).astype(f32)


def quantise_pmf(logits):
    """softmax in float32, then reading Q21's quantiser (every p >= 1, sum 2^16)."""
    l = logits.astype(np.float32)
    e = np.exp(l - l.max(1, keepdims=True)).astype(np.float32)
    pr = (e / e.sum(1, keepdims=True)).astype(np.float32)
    p = 1 + np.floor(pr * np.float32(65281)).astype(np.int64)
    p[np.arange(len(p)), np.argmax(p, 1)] += M - p.sum(1)
    return p


def rans_encode(sym, pmfs):
    """Reading O9, one lane: returns (words, final state); sym in 0..254."""
    cum = np.concatenate([np.zeros((len(pmfs), 1), np.int64), np.cumsum(pmfs, 1)], 1)
    x, words = 1 << 16, []
    for i in reversed(range(len(sym))):
        s = int(sym[i])
        f, c = int(pmfs[i, s]), int(cum[i, s])
        if x >= f << 16:
            words.append(x & 0xFFFF)
            x >>= 16
        x = ((x // f) << 16) + (x % f) + c
    return words[::-1], x


def rans_decode(words, x, pmfs):
    cum = np.concatenate([np.zeros((len(pmfs), 1), np.int64), np.cumsum(pmfs, 1)], 1)
    out, w = [], 0
    for i in range(len(pmfs)):
        slot = x & 0xFFFF
        s = int(np.searchsorted(cum[i], slot, side="right") - 1)
        s = min(max(s, 0), 254)
        out.append(s)
        x = int(pmfs[i, s]) * (x >> 16) + slot - int(cum[i, s])
        if x < (1 << 16) and w < len(words):
            x = (x << 16) | words[w]
            w += 1
    return np.array(out)


@pytest.fixture(scope="module")
def level_data():
    mobj = I.make_model(C=8, H=8, seed=1, min_depth=9, max_depth=12)
    om = O.Model(mobj.to_bytes())
    D = O.Dump()
    O.encode(om, I.make_frame(I.CFG1), 12, D)
    Dcut = 12 - 1 - mobj.n_deep
    out = []
    for d in range(mobj.R, 12):
        F, hd = _head_inputs(mobj, D, d, Dcut)
        sym = D.get(f"code/{d}", np.uint8).astype(np.int64) - 1
        p_int = D.get(f"p/{d}", np.uint16).reshape(-1, 255).astype(np.int64)
        out.append((d, F, hd, sym, p_int))
    return out


def test_integer_pmfs_round_trip(level_data):
    """The integer model's pmfs (identical on CPU oracle and GPU) always decode."""
    for d, F, hd, sym, p_int in level_data:
        assert (p_int >= 1).all() and (p_int.sum(1) == M).all()
        words, x = rans_encode(sym, p_int)
        assert np.array_equal(rans_decode(words, x, p_int), sym), d


def test_float_twin_orders_disagree_and_decode_collapses(level_data):
    """Two float32 evaluation orders of the same network give different quantised CDFs on
    some nodes; decoding a stream encoded with one using the other derails."""
    differing, total, collapsed = 0, 0, 0
    for d, F, hd, sym, p_int in level_data:
        pa = quantise_pmf(float_logits(F, hd, "blas"))
        pb = quantise_pmf(float_logits(F, hd, "reversed"))
        rows = np.any(pa != pb, 1)
        differing += int(rows.sum())
        total += len(rows)
        words, x = rans_encode(sym, pa)
        assert np.array_equal(rans_decode(words, x, pa), sym), d  # same order: fine
        if rows.any():
            dec = rans_decode(words, x, pb)
            first = int(np.argmax(rows))
            assert np.array_equal(dec[:first], sym[:first])
            if not np.array_equal(dec, sym):
                collapsed += 1
    print(f"float twin: {differing} of {total} node CDFs differ between evaluation orders; "
          f"{collapsed} level streams fail to decode")
    assert differing > 0 and collapsed > 0


@pytest.mark.gpu
def test_float_twin_cross_device(level_data):
    """Cross-device form: the float twin on cuda:0 (torch fp32, cuBLAS order) against the
    CPU float32 twin; the integer path has no such split (GPU CDFs == oracle CDFs)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    differing = 0
    for d, F, hd, sym, p_int in level_data:
        Ft = torch.from_numpy(F.astype(np.float32)).cuda()
        W1 = torch.from_numpy(hd.W1.astype(np.float32)).cuda()
        W2 = torch.from_numpy(hd.W2.astype(np.float32)).cuda()
        h = Ft @ W1.T + torch.from_numpy(hd.b1.astype(np.float32)).cuda()
        a = torch.where(h >= 0, h * (hd.rq1.m_pos / 2.0 ** hd.rq1.r), h * (hd.rq1.m_neg / 2.0 ** hd.rq1.r))
        z = a @ W2.T + torch.from_numpy(hd.b2.astype(np.float32)).cuda()
        lg = (z * (hd.rq_logit.m_pos / 2.0 ** hd.rq_logit.r / 256.0)).cpu().numpy()
        differing += int(np.any(quantise_pmf(lg) != quantise_pmf(float_logits(F, hd, "blas")), 1).sum())
    print(f"float twin GPU vs CPU: {differing} node CDFs differ")
