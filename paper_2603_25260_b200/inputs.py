"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the coding method (no Morton keys, no octree,
no convolution, no requantisation, no softmax, no entropy coding).  It produces
exactly two kinds of input, both plain data:

1. LiDAR frames: a seeded ray-caster over a procedural ground + boxes + facade
   scene (SURVEY.md §8(d) "Generator"), quantised to integer voxel coordinates
   with the KITTI bounding-box scheme of PAPER.md P:636 ("normalizes the point
   clouds within a bounding box of size 400x400x400 centered at the origin")
   under DESIGN.md reading Q26: q = clip(floor((p + 200) * 2^L / 400), 0, 2^L-1).
   Quantisation is a harness step, outside the coded hot path.

2. A seeded random integer model (int8 weights, int32 biases, fixed-point
   requant triples, the exp LUT) serialised to the model-file format of
   DESIGN.md §"Model file".  No trained checkpoint exists offline
   (BASELINE.json north_star), so weights are random; the LUT is the one
   piece of transcendental arithmetic and it is evaluated here, once, and
   stored in the file ("precomputed lookup table").
"""
from __future__ import annotations

import dataclasses
import struct
from typing import Dict, List, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# LiDAR frames
# ---------------------------------------------------------------------------

GROUND_Z = -1.73          # sensor height above ground (KITTI HDL-64E mount), SURVEY §8(d)
MAX_RANGE = 120.0
RING_RADIUS = 60.0
RING_TOP = 30.0 + GROUND_Z
SCENE_PERIOD = 160.0      # box layout period along the road (x), metres


@dataclasses.dataclass(frozen=True)
class ScanConfig:
    name: str
    beams: int
    azimuths: int
    elev_top_deg: float
    elev_bot_deg: float
    bit_depth: int
    channels: int          # C of the model used with this config
    head_hidden: int       # H


# BASELINE.json configs[0..2]; cfg4 is the decode of cfg2, cfg5 a cfg2 sequence.
CFG1 = ScanConfig("cfg1_16x512_L12_C8", 16, 512, 15.0, -15.0, 12, 8, 8)
CFG2 = ScanConfig("cfg2_64x2048_L12_C32", 64, 2048, 2.0, -24.8, 12, 32, 32)
CFG3 = ScanConfig("cfg3_64x1400_L18_C32", 64, 1400, 2.0, -24.8, 18, 32, 32)
CONFIGS = {"cfg1": CFG1, "cfg2": CFG2, "cfg3": CFG3}


def _scene_boxes(scene_seed: int, n_boxes: int = 60) -> np.ndarray:
    """Axis-aligned boxes [n, 6] = (xmin, ymin, zmin, xmax, ymax, zmax) in world coords.

    Footprint 1.5-12 m, height 1.2-10 m, centres within +-80 m, kept off the
    |y| < 4 m road corridor the sensor drives along (x axis).
    """
    rng = np.random.default_rng(np.uint64(scene_seed) ^ np.uint64(0x5CE7E))
    boxes = []
    while len(boxes) < n_boxes:
        cx, cy = rng.uniform(-80.0, 80.0, size=2)
        w, l = rng.uniform(1.5, 12.0, size=2)
        h = rng.uniform(1.2, 10.0)
        if abs(cy) - l / 2.0 < 4.0:
            continue
        boxes.append((cx - w / 2, cy - l / 2, GROUND_Z, cx + w / 2, cy + l / 2, GROUND_Z + h))
    return np.asarray(boxes, dtype=np.float64)


def raycast_frame(cfg: ScanConfig, frame_index: int = 0, scene_seed: int = 1,
                  noise_seed: int | None = None) -> np.ndarray:
    """Float points [n, 3] (sensor frame) of one spinning-LiDAR sweep.

    The sensor sits at x = frame_index metres along the road (SURVEY §8(d) cfg5:
    "sensor advances 1 m/frame along x"), at the origin of its own frame.
    """
    if noise_seed is None:
        noise_seed = (scene_seed * 1_000_003 + frame_index) & 0xFFFFFFFF
    el = np.deg2rad(np.linspace(cfg.elev_top_deg, cfg.elev_bot_deg, cfg.beams))
    az = 2.0 * np.pi * np.arange(cfg.azimuths) / cfg.azimuths
    ce, se = np.cos(el)[:, None], np.sin(el)[:, None]
    d = np.stack([np.broadcast_to(ce * np.cos(az)[None, :], (cfg.beams, cfg.azimuths)),
                  np.broadcast_to(ce * np.sin(az)[None, :], (cfg.beams, cfg.azimuths)),
                  np.broadcast_to(se, (cfg.beams, cfg.azimuths))], axis=-1).reshape(-1, 3)
    n = d.shape[0]
    t = np.full(n, np.inf)
    # ground plane z = GROUND_Z
    down = d[:, 2] < -1e-9
    t[down] = GROUND_Z / d[down, 2]
    # facade ring x^2 + y^2 = R^2 (sensor-centred), hit only below its top
    rxy = np.hypot(d[:, 0], d[:, 1])
    tr = RING_RADIUS / np.maximum(rxy, 1e-12)
    zr = tr * d[:, 2]
    ok = (zr >= GROUND_Z) & (zr <= RING_TOP)
    t = np.where(ok & (tr < t), tr, t)
    # boxes (slab test), translated into the sensor frame.  The street scene tiles along
    # the road with period SCENE_PERIOD: every box copy is placed within +-80 m of the
    # sensor along x, so every frame of a long sequence (cfg5: 1000 frames, 1 m apart)
    # sees a full scene of objects, not the empty road beyond the first tile
    boxes = _scene_boxes(scene_seed).copy()
    cx = 0.5 * (boxes[:, 0] + boxes[:, 3]) - float(frame_index)
    shift = np.floor((cx + SCENE_PERIOD / 2.0) / SCENE_PERIOD) * SCENE_PERIOD + float(frame_index)
    boxes[:, 0] -= shift
    boxes[:, 3] -= shift
    inv = 1.0 / np.where(np.abs(d) < 1e-12, 1e-12, d)
    inv3 = inv.reshape(cfg.beams, cfg.azimuths, 3)
    t2d = t.reshape(cfg.beams, cfg.azimuths)
    for b in boxes:
        # cull to the azimuth columns the box subtends (boxes never contain the sensor)
        cx = np.array([b[0], b[3], b[0], b[3]])
        cy = np.array([b[1], b[1], b[4], b[4]])
        ang = np.mod(np.arctan2(cy, cx), 2.0 * np.pi)
        ang.sort()
        gaps = np.diff(np.concatenate([ang, ang[:1] + 2.0 * np.pi]))
        k = int(np.argmax(gaps))           # the box spans the complement of the largest gap
        a0, a1 = ang[(k + 1) % 4], ang[k]
        i0 = int(np.floor(a0 / (2.0 * np.pi) * cfg.azimuths)) - 1
        i1 = int(np.ceil(a1 / (2.0 * np.pi) * cfg.azimuths)) + 1
        if i1 < i0:
            i1 += cfg.azimuths
        cols = np.arange(i0, i1 + 1) % cfg.azimuths
        iv = inv3[:, cols, :]
        t1 = b[None, None, 0:3] * iv
        t2 = b[None, None, 3:6] * iv
        tmin = np.minimum(t1, t2).max(axis=-1)
        tmax = np.maximum(t1, t2).min(axis=-1)
        hit = (tmax >= tmin) & (tmin > 0.0)
        th = np.where(hit, tmin, np.inf)
        t2d[:, cols] = np.minimum(t2d[:, cols], th)
    t = t2d.reshape(-1)
    keep = np.isfinite(t) & (t < MAX_RANGE)
    rng = np.random.default_rng(noise_seed)
    noise = rng.normal(0.0, 0.01, size=n)
    t = t + noise
    pts = d[keep] * t[keep, None]
    return pts


def quantize(points: np.ndarray, bit_depth: int) -> np.ndarray:
    """DESIGN.md reading Q26 of PAPER.md P:636: 400 m box at the origin, 2^L cells per axis."""
    q = np.floor((points + 200.0) * (2.0 ** bit_depth) / 400.0)
    q = np.clip(q, 0, 2 ** bit_depth - 1)
    return np.ascontiguousarray(q.astype(np.int32))


def make_frame(cfg: ScanConfig, frame_index: int = 0, scene_seed: int = 1) -> np.ndarray:
    """int32 [n, 3] quantised coordinates of one frame (duplicates kept, scan order)."""
    return quantize(raycast_frame(cfg, frame_index, scene_seed), cfg.bit_depth)


def make_frames(cfg: ScanConfig, count: int, first: int = 0, scene_seed: int = 1) -> List[np.ndarray]:
    return [make_frame(cfg, first + i, scene_seed) for i in range(count)]


def random_cloud(n: int, bit_depth: int, seed: int, spread: float = 1.0) -> np.ndarray:
    """Uniform random integer coordinates (edge-case and property tests)."""
    rng = np.random.default_rng(seed)
    hi = max(1, int((2 ** bit_depth) * spread))
    return rng.integers(0, min(hi, 2 ** bit_depth), size=(n, 3), dtype=np.int64).astype(np.int32)


# ---------------------------------------------------------------------------
# Integer model
# ---------------------------------------------------------------------------

MODEL_MAGIC = b"PCCM"
# model-file flags (header word at byte 44): the Table 4 ablation without
# cross-scale propagation and the symbol-frequency raw-prefix coder
FLAG_XFP_OFF = 1
FLAG_RAW_FREQ = 2
MODEL_VERSION = 1
LUT_LEN = 1024
N_CODES = 255
NOMINAL_ACT_STD = 40.0
W_MAX = 63


def exp_lut() -> np.ndarray:
    """LUT[j] = floor(2^24 * exp(-j/64) + 1/2), j = 0..1023 (reading Q20).

    PAPER.md P:350: "a precomputed lookup table that only covers the
    non-positive domain".  Evaluated once at model creation; stored in the file.
    """
    j = np.arange(LUT_LEN, dtype=np.float64)
    return np.floor(np.ldexp(np.exp(-j / 64.0), 24) + 0.5).astype(np.uint32)


@dataclasses.dataclass
class RQ:
    """Requant triple (m_pos, m_neg, r); m_neg == m_pos means no PReLU."""
    m_pos: int
    m_neg: int
    r: int


@dataclasses.dataclass
class Head:
    W1: np.ndarray   # int8 [H, C]
    b1: np.ndarray   # int32 [H]
    rq1: RQ
    W2: np.ndarray   # int8 [255, H]
    b2: np.ndarray   # int32 [255]
    rq_logit: RQ     # (m_l, m_l, r_l) -> Q8 logits


@dataclasses.dataclass
class Up:
    W: np.ndarray        # int8 [8C, C + 255]: linear over Concat(S, q_one * onehot(X))
    b: np.ndarray        # int32 [8C]
    rq: RQ
    q_one: int           # int8 value of the one-hot "1"


@dataclasses.dataclass
class Shallow:
    Wa: np.ndarray; ba: np.ndarray; rqa: RQ             # conv3 C->C, PReLU
    Wb: np.ndarray; bb: np.ndarray; k_s: int; rqb: RQ   # conv3 C->C + k_s*F skip
    up: Up
    head: Head


@dataclasses.dataclass
class Down:
    W: np.ndarray   # int8 [8, C, C]  (child index c, out, in)
    b: np.ndarray
    rq: RQ


@dataclasses.dataclass
class Deep:
    E: np.ndarray                          # int8 [255, C]
    downs: List[Down]                      # j-1 steps, depth d-1 -> D
    Wa: np.ndarray; ba: np.ndarray; rqa: RQ                  # conv3 2C->C (C->C with XFP off)
    Wb: np.ndarray; P: np.ndarray; bb: np.ndarray; rqb: RQ   # conv3 C->C + 1x1 2C->C (P None: XFP off)
    ups: List[Up]                          # j steps, depth D -> d
    head: Head
    k_s: int = 0                           # XFP off: identity skip k_s * G_D


@dataclasses.dataclass
class Model:
    C: int
    H: int
    R: int
    n_deep: int
    min_depth: int
    max_depth: int
    seed: int
    lut: np.ndarray
    E0: np.ndarray                      # int8 [255, C]
    shallow: Dict[int, Shallow]         # absolute depth d in [R, max_depth - 1 - n_deep]
    deep: List[Deep]                    # j = 1..n_deep (index j-1)
    flags: int = 0                      # FLAG_XFP_OFF | FLAG_RAW_FREQ

    # -- serialisation (DESIGN.md §"Model file") --------------------------
    def to_bytes(self) -> bytes:
        out = bytearray()
        out += MODEL_MAGIC
        out += struct.pack("<7I", MODEL_VERSION, self.C, self.H, self.R, self.n_deep,
                           self.min_depth, self.max_depth)
        out += struct.pack("<QII", self.seed, LUT_LEN, self.flags)
        out += bytes(64 - len(out))
        assert len(out) == 64
        out += self.lut.astype("<u4").tobytes()

        def i8(a, shape):
            a = np.asarray(a)
            assert a.shape == shape, (a.shape, shape)
            assert a.dtype == np.int8
            return a.tobytes()

        def i32(a, shape):
            a = np.asarray(a)
            assert a.shape == shape, (a.shape, shape)
            return a.astype("<i4").tobytes()

        def rq(t: RQ):
            return struct.pack("<3i", t.m_pos, t.m_neg, t.r)

        C, H = self.C, self.H

        def head(h: Head):
            return (i8(h.W1, (H, C)) + i32(h.b1, (H,)) + rq(h.rq1)
                    + i8(h.W2, (N_CODES, H)) + i32(h.b2, (N_CODES,)) + rq(h.rq_logit))

        def up(u: Up):
            return (i8(u.W, (8 * C, C + N_CODES)) + i32(u.b, (8 * C,)) + rq(u.rq)
                    + struct.pack("<i", u.q_one))

        out += i8(self.E0, (N_CODES, C))
        for d in range(self.R, self.max_depth - self.n_deep):
            s = self.shallow[d]
            out += i8(s.Wa, (27, C, C)) + i32(s.ba, (C,)) + rq(s.rqa)
            out += i8(s.Wb, (27, C, C)) + i32(s.bb, (C,)) + struct.pack("<i", s.k_s) + rq(s.rqb)
            out += up(s.up)
            out += head(s.head)
        for j in range(1, self.n_deep + 1):
            dp = self.deep[j - 1]
            out += i8(dp.E, (N_CODES, C))
            assert len(dp.downs) == j - 1 and len(dp.ups) == j
            for dn in dp.downs:
                out += i8(dn.W, (8, C, C)) + i32(dn.b, (C,)) + rq(dn.rq)
            if self.flags & FLAG_XFP_OFF:   # ResBlock(G_D): the shallow ResBlock layout
                out += i8(dp.Wa, (27, C, C)) + i32(dp.ba, (C,)) + rq(dp.rqa)
                out += i8(dp.Wb, (27, C, C)) + i32(dp.bb, (C,)) + struct.pack("<i", dp.k_s) + rq(dp.rqb)
            else:
                out += i8(dp.Wa, (27, C, 2 * C)) + i32(dp.ba, (C,)) + rq(dp.rqa)
                out += i8(dp.Wb, (27, C, C)) + i8(dp.P, (C, 2 * C)) + i32(dp.bb, (C,)) + rq(dp.rqb)
            for u in dp.ups:
                out += up(u)
            out += head(dp.head)
        out += struct.pack("<Q", fnv1a64(bytes(out)))
        return bytes(out)


def fnv1a64(data: bytes) -> int:
    """64-bit FNV-1a content hash of the model file body (stamped into bitstreams)."""
    h = 0xCBF29CE484222325
    arr = np.frombuffer(data, dtype=np.uint8)
    # chunked pure-python loop is slow for MBs; use numpy-free fast path via bytes iteration
    for b in arr.tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def model_hash(model_bytes: bytes) -> int:
    return struct.unpack("<Q", model_bytes[-8:])[0]


def _rq_for(acc_std: float, prelu: bool, target_std: float = NOMINAL_ACT_STD, r: int = 24) -> RQ:
    scale = target_std / max(acc_std, 1e-9)
    m = int(round(scale * (1 << r)))
    while m >= (1 << 31):
        r -= 1
        m = int(round(scale * (1 << r)))
    m = max(m, 1)
    return RQ(m, max(1, int(round(m / 4))) if prelu else m, r)


def make_model(C: int = 32, H: int = 32, seed: int = 1, R: int = 4, n_deep: int = 4,
               min_depth: int = 9, max_depth: int = 18, kind: str = "random", xfp: bool = True,
               raw_freq: bool = False) -> Model:
    """Seeded random integer model (DESIGN.md §"Model generator").

    kind = "random" | "zero" (all weights/biases/tables 0) | "bias_head"
    (random network, W2 = 0 so every node's logits are b2).
    Table 4 ablations: xfp=False is "Baseline + GRED" (deep levels code
    from H = ResBlock(G_D) alone); n_deep=0 is the GRED-off "Baseline" (every level a
    shallow level).  raw_freq=True codes the raw prefix with the adaptive
    symbol-frequency coder instead of plain bytes.
    Magnitudes follow a nominal activation std of 40 with requant multipliers
    set from each layer's nominal fan-in, so activations neither saturate nor
    collapse (SURVEY §7 hard part (f)).
    """
    assert C % 8 == 0 and H % 8 == 0 and 8 <= C <= 64 and 8 <= H <= 64
    assert R + 1 + n_deep <= min_depth <= max_depth <= 21 and 0 <= n_deep <= 4 and 1 <= R <= 6
    rng = np.random.default_rng(seed)
    sa = NOMINAL_ACT_STD
    sw = W_MAX / np.sqrt(3.0)
    zero = kind == "zero"

    def w(*shape):
        if zero:
            return np.zeros(shape, np.int8)
        return rng.integers(-W_MAX, W_MAX + 1, size=shape).astype(np.int8)

    def emb(*shape):
        if zero:
            return np.zeros(shape, np.int8)
        return rng.integers(-100, 101, size=shape).astype(np.int8)

    def bias(n, acc_std):
        if zero:
            return np.zeros(n, np.int32)
        lim = int(acc_std / 4)
        return rng.integers(-lim, lim + 1, size=n).astype(np.int32)

    def head() -> Head:
        s1 = sa * sw * np.sqrt(C)
        sz = sa * sw * np.sqrt(H)
        W1 = w(H, C); b1 = bias(H, s1); rq1 = _rq_for(s1, True)
        W2 = w(N_CODES, H)
        b2 = bias(N_CODES, sz) if not zero else np.zeros(N_CODES, np.int32)
        if kind == "bias_head":
            W2 = np.zeros((N_CODES, H), np.int8)
            b2 = rng.integers(-int(sz), int(sz) + 1, size=N_CODES).astype(np.int32)
        rql = _rq_for(sz, False, target_std=1.5 * 256.0, r=20)
        return Head(W1, b1, rq1, W2, b2, rql)

    def up() -> Up:
        q_one = 127
        s = np.sqrt(C * (sa * sw) ** 2 + (q_one * sw) ** 2)
        return Up(w(8 * C, C + N_CODES), bias(8 * C, s), _rq_for(s, True), q_one)

    E0 = emb(N_CODES, C)
    shallow = {}
    for d in range(R, max_depth - n_deep):
        sc = sa * sw * np.sqrt(7 * C)
        k_s = 0 if zero else int(round(sc / sa))
        shallow[d] = Shallow(w(27, C, C), bias(C, sc), _rq_for(sc, True),
                             w(27, C, C), bias(C, sc), k_s, _rq_for(np.sqrt(2) * sc, False),
                             up(), head())
    deep = []
    for j in range(1, n_deep + 1):
        E = emb(N_CODES, C)
        downs = []
        for _ in range(j - 1):
            s = sa * sw * np.sqrt(3 * C)
            downs.append(Down(w(8, C, C), bias(C, s), _rq_for(s, True)))
        if not xfp:   # ResBlock(G_D) in the shallow form (C -> C, identity skip k_s)
            sc = sa * sw * np.sqrt(7 * C)
            k_s = 0 if zero else int(round(sc / sa))
            deep.append(Deep(E, downs, w(27, C, C), bias(C, sc), _rq_for(sc, True),
                             w(27, C, C), None, bias(C, sc), _rq_for(np.sqrt(2) * sc, False),
                             [up() for _ in range(j)], head(), k_s))
            continue
        sa2 = sa * sw * np.sqrt(7 * 2 * C)
        sb = sa * sw * np.sqrt(7 * C)
        sp = sa * sw * np.sqrt(2 * C)
        deep.append(Deep(E, downs, w(27, C, 2 * C), bias(C, sa2), _rq_for(sa2, True),
                         w(27, C, C), w(C, 2 * C), bias(C, sb), _rq_for(np.hypot(sb, sp), False),
                         [up() for _ in range(j)], head()))
    flags = (0 if xfp else FLAG_XFP_OFF) | (FLAG_RAW_FREQ if raw_freq else 0)
    return Model(C, H, R, n_deep, min_depth, max_depth, seed, exp_lut(), E0, shallow, deep, flags)


def model_bytes(C: int = 32, H: int = 32, seed: int = 1, **kw) -> bytes:
    return make_model(C=C, H=H, seed=seed, **kw).to_bytes()
