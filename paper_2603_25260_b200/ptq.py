"""Post-training quantisation tooling (NEXT-4): float weights -> the integer
model the hot path runs (host-side; produces model files, never runs on the coding path).

Follows the paper's quantisation paragraph:
* Eq.12  q_x = clip(round(x / s) + z, q_min, q_max); rounding is half up (reading Q15),
  zero-points are 0 (reading Q16: z = 0 for activations, symmetric weights z_w = 0);
* 8-bit weights and activations for linear layers / sparse convolutions, int32 bias
  b_int32 = round(b / (s_x s_w)) (Eq.13);
* Eq.14  q_y = clip(round(y_int32 m / 2^r) + z_y): the real multiplier M = s_x s_w / s_y
  becomes an integer m < 2^31 and a shift r (`derive_mr`); PReLU folds into the same
  requant with the negative-side multiplier M * alpha (reading Q18/Q19);
* activation scales come from a "lightweight calibration on a small subset":
  symmetric max-abs over calibration samples (`activation_scale`).

`quantize_head` turns a float predictor (Eq.7: C -> H PReLU -> 255 logits in nats) into the
model file's `Head`: the logit requant maps z_int32 to Q8 logits (1/256 nat, reading Q20).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Tuple

import numpy as np

from . import inputs as I


def quantize(x: np.ndarray, s: float, z: int = 0, qmin: int = -128, qmax: int = 127) -> np.ndarray:
    """Eq.12 with round-half-up (reading Q15)."""
    return np.clip(np.floor(np.asarray(x, np.float64) / s + 0.5) + z, qmin, qmax).astype(np.int64)


def symmetric_weight_scale(W: np.ndarray, qmax: int = 127) -> float:
    """z_w = 0; the largest |w| maps to qmax."""
    m = float(np.max(np.abs(W))) if np.size(W) else 0.0
    return m / qmax if m > 0 else 1.0


def activation_scale(samples: np.ndarray, qmax: int = 127) -> float:
    """Calibration: symmetric max-abs over the calibration samples (z = 0)."""
    return symmetric_weight_scale(samples, qmax)


def derive_mr(M: float, m_bits: int = 31, r_max: int = 62) -> Tuple[int, int]:
    """Integer multiplier m < 2^m_bits and shift r <= r_max with m / 2^r ~= M (Eq.14).

    The largest admissible r is taken (most precision): |m / 2^r - M| <= 2^-(r+1)."""
    if not (M >= 0.0) or math.isinf(M):
        raise ValueError("multiplier must be finite and >= 0")
    if M == 0.0:
        return 0, 0
    r = r_max
    while r > 0 and math.floor(M * 2.0 ** r + 0.5) >= (1 << m_bits):
        r -= 1
    m = int(math.floor(M * 2.0 ** r + 0.5))
    if m >= (1 << m_bits):
        raise ValueError("multiplier too large for the integer requant")
    return m, r


def rq_pair(M: float, alpha: float = 1.0) -> I.RQ:
    """Requant triple for the real multiplier M, PReLU slope alpha on the negative side
    (alpha = 1: plain requant), sharing one shift r (reading Q18/Q19)."""
    big = max(M, M * alpha)
    _, r = derive_mr(big)
    mp = int(math.floor(M * 2.0 ** r + 0.5))
    mn = int(math.floor(M * alpha * 2.0 ** r + 0.5))
    return I.RQ(mp, mn, r)


def quantize_linear(W: np.ndarray, b: np.ndarray, s_x: float, s_y: float, alpha: float = 1.0):
    """Float y = act(W x + b) -> (int8 W, int32 b, RQ) for int8 input scale s_x and int8
    output scale s_y (Eq.12-14)."""
    s_w = symmetric_weight_scale(W)
    Wq = quantize(W, s_w, qmin=-127, qmax=127).astype(np.int8)
    bq = np.clip(np.floor(np.asarray(b, np.float64) / (s_x * s_w) + 0.5), -(2 ** 31), 2 ** 31 - 1).astype(np.int32)
    return Wq, bq, rq_pair(s_x * s_w / s_y, alpha), s_w


@dataclasses.dataclass
class FloatHead:
    """Float predictor of Eq.7: a = PReLU(W1 F + b1; alpha), logits = W2 a + b2 (nats)."""
    W1: np.ndarray   # [H, C]
    b1: np.ndarray   # [H]
    alpha: float     # PReLU negative slope
    W2: np.ndarray   # [255, H]
    b2: np.ndarray   # [255]


def float_head_forward(h: FloatHead, F: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """(hidden activations, logits in nats), float64."""
    pre = F @ h.W1.T + h.b1
    a = np.where(pre >= 0, pre, h.alpha * pre)
    return a, a @ h.W2.T + h.b2


def quantize_head(h: FloatHead, s_F: float, calib_F: np.ndarray) -> I.Head:
    """Float head + the int8 scale of its input features + float calibration inputs ->
    the integer Head of the model file (W1/b1/rq1, W2/b2, logit requant to Q8)."""
    a_cal, _ = float_head_forward(h, calib_F)
    s_a = activation_scale(a_cal)
    W1, b1, rq1, _ = quantize_linear(h.W1, h.b1, s_F, s_a, h.alpha)
    s_w2 = symmetric_weight_scale(h.W2)
    W2 = quantize(h.W2, s_w2, qmin=-127, qmax=127).astype(np.int8)
    b2 = np.clip(np.floor(np.asarray(h.b2, np.float64) / (s_a * s_w2) + 0.5), -(2 ** 31), 2 ** 31 - 1).astype(np.int32)
    # z_int32 * (s_a s_w2) nats = z_int32 * (s_a s_w2 * 256) Q8 logits
    m, r = derive_mr(s_a * s_w2 * 256.0)
    return I.Head(W1, b1, rq1, W2, b2, I.RQ(m, m, r))
