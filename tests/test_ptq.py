"""NEXT-4 PTQ tooling (paper_2603_25260_b200/ptq.py; Eq.12-14).

* derive_mr: m < 2^31, |m / 2^r - M| <= 2^-(r+1), r maximal (m >= 2^30 unless r = 62);
* Eq.12 quantiser: half-up rounding and clipping on hand-checked values;
* quantize_linear: the integer layer (int32 accumulate + fixed-point requant, Eq.13-14)
  tracks the float layer within the quantisation error bound on random data;
* quantize_head: a float predictor calibrated and quantised end to end gives Q8 logits
  within a small fraction of a nat of the float logits, and the resulting model file
  codes and decodes (oracle round trip; GPU bit-exact on a GPU box).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I
from paper_2603_25260_b200 import ptq


def _rq(acc, t):
    """Eq.14 with PReLU folded (reading Q15/Q18), numpy int64."""
    acc = np.asarray(acc, np.int64)
    m = np.where(acc >= 0, t.m_pos, t.m_neg).astype(np.int64)
    half = (1 << (t.r - 1)) if t.r > 0 else 0
    return np.clip((acc * m + half) >> t.r, -128, 127)


def test_derive_mr_precision():
    rng = np.random.default_rng(0)
    for M in np.exp2(rng.uniform(-30, 20, 2000)):
        m, r = ptq.derive_mr(float(M))
        assert 0 <= m < 2 ** 31 and 0 <= r <= 62
        assert abs(m / 2.0 ** r - M) <= 2.0 ** -(r + 1) * (1 + 1e-12)
        assert m >= 2 ** 30 or r == 62
    assert ptq.derive_mr(0.5) == (2 ** 30, 31)
    assert ptq.derive_mr(0.0) == (0, 0)
    with pytest.raises(ValueError):
        ptq.derive_mr(2.0 ** 40)


def test_eq12_quantiser():
    x = np.array([-1000.0, -2.5, -0.5, 0.49, 0.5, 1.5, 2.5, 126.6, 1000.0])
    assert ptq.quantize(x, 1.0).tolist() == [-128, -2, 0, 0, 1, 2, 3, 127, 127]
    assert ptq.quantize(np.array([3.0]), 2.0, z=5).tolist() == [7]


@pytest.mark.parametrize("alpha", [1.0, 0.25])
def test_quantize_linear_tracks_float(alpha):
    rng = np.random.default_rng(1)
    C, N, K = 32, 2000, 16
    W = rng.normal(0, 0.2, (K, C))
    b = rng.normal(0, 0.3, K)
    x = rng.normal(0, 1.0, (N, C))
    s_x = ptq.activation_scale(x)
    pre = x @ W.T + b
    y = np.where(pre >= 0, pre, alpha * pre)
    s_y = ptq.activation_scale(y)
    Wq, bq, t, s_w = ptq.quantize_linear(W, b, s_x, s_y, alpha)
    xq = ptq.quantize(x, s_x)
    yq = _rq(xq @ Wq.astype(np.int64).T + bq, t)
    # error in output LSBs: input/weight rounding propagated + one requant rounding
    bound = (0.5 * s_x * np.abs(W).sum(1).max() + 0.5 * s_w * np.abs(x).sum(1).max()) / s_y + 1.5
    err = np.abs(yq - y / s_y)
    assert err.max() <= bound
    assert err.mean() < 1.5


def test_quantize_head_end_to_end():
    rng = np.random.default_rng(2)
    C = H = 8
    fh = ptq.FloatHead(rng.normal(0, 0.3, (H, C)), rng.normal(0, 0.2, H), 0.1,
                       rng.normal(0, 0.4, (255, H)), rng.normal(0, 0.5, 255))
    F = rng.normal(0, 1.0, (3000, C))
    s_F = ptq.activation_scale(F)
    hd = ptq.quantize_head(fh, s_F, F[:500])  # calibrate on a small subset
    Fq = ptq.quantize(F, s_F)
    a = _rq(Fq @ hd.W1.astype(np.int64).T + hd.b1, hd.rq1)
    z = a @ hd.W2.astype(np.int64).T + hd.b2
    lq8 = (z * hd.rq_logit.m_pos + (1 << (hd.rq_logit.r - 1))) >> hd.rq_logit.r
    _, lf = ptq.float_head_forward(fh, F)
    err = np.abs(lq8 / 256.0 - lf)
    assert err.mean() < 0.1, err.mean()
    agree = np.mean(np.argmax(lq8, 1) == np.argmax(lf, 1))
    assert agree > 0.9, agree
    # the quantised head drops into a model file that codes losslessly
    m = I.make_model(C=C, H=H, seed=3, min_depth=9, max_depth=12)
    for d in m.shallow:
        m.shallow[d].head = hd
    for dp in m.deep:
        dp.head = hd
    om = O.Model(m.to_bytes())
    pts = I.random_cloud(2000, 12, 5)
    out, L = O.decode(om, O.encode(om, pts, 12))
    assert L == 12 and len(out) == len(np.unique(pts, axis=0))


@pytest.mark.gpu
def test_ptq_model_gpu_bit_exact():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_25260_b200 import pcc
    rng = np.random.default_rng(4)
    C = H = 32
    fh = ptq.FloatHead(rng.normal(0, 0.2, (H, C)), rng.normal(0, 0.2, H), 0.1,
                       rng.normal(0, 0.3, (255, H)), rng.normal(0, 0.5, 255))
    F = rng.normal(0, 1.0, (500, C))
    hd = ptq.quantize_head(fh, ptq.activation_scale(F), F)
    m = I.make_model(C=C, H=H, seed=3, min_depth=9, max_depth=12)
    for d in m.shallow:
        m.shallow[d].head = hd
    for dp in m.deep:
        dp.head = hd
    mb = m.to_bytes()
    codec = pcc.Codec(mb, 0)
    pts = I.make_frame(I.CFG1)
    out, oo = codec.encode_frames(torch.from_numpy(pts).cuda(), [0, len(pts)], 12)
    assert out[:oo[1]].cpu().numpy().tobytes() == O.encode(O.Model(mb), pts, 12)
    codec.close()
