"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, tolerance 0.

The pipeline is integer-only, so every intermediate tensor, every CDF and every
bitstream must be bit-identical (BASELINE.json north_star).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2603_25260_b200 import inputs as I  # noqa: E402


@pytest.fixture(scope="module")
def pcc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_25260_b200 import pcc as P
    return P


_models = {}


def model_pair(C, max_depth=18, kind="random", seed=1):
    key = (C, max_depth, kind, seed)
    if key not in _models:
        mb = I.make_model(C=C, H=C, seed=seed, min_depth=9, max_depth=max_depth, kind=kind).to_bytes()
        _models[key] = (mb, O.Model(mb))
    return _models[key]


@pytest.fixture(scope="module")
def ctx(pcc):
    c = pcc.pcc_ctx_create(0, torch.cuda.current_stream().cuda_stream)
    yield c
    pcc.pcc_ctx_destroy(c)


_gpu_models = {}


def gpu_model(pcc, mb):
    h = hash(mb)
    if h not in _gpu_models:
        _gpu_models[h] = pcc.pcc_model_load(mb, 0)
    return _gpu_models[h]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_encode(pcc, ctx, m, frames, L):
    offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
    x = dev(np.concatenate(frames).astype(np.int32))
    cap = sum(pcc.pcc_encode_bound(len(f), L) + 4 for f in frames)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    oo = pcc.pcc_encode_batch(ctx, m, x, offs, L, out, cap)
    host = out[:oo[-1]].cpu().numpy().tobytes()
    return [host[oo[i]:oo[i + 1]] for i in range(len(frames))], oo


def gpu_decode(pcc, ctx, m, streams, cap_points):
    offs = [0]
    blob = b""
    for s in streams:
        blob += s + bytes((-len(s)) % 4)
        offs.append(len(blob))
    d = dev(np.frombuffer(blob, np.uint8))
    out = torch.empty((cap_points, 3), dtype=torch.int32, device="cuda")
    oo = pcc.pcc_decode_batch(ctx, m, d, offs, out, cap_points)
    xyz = out[:oo[-1]].cpu().numpy()
    return [xyz[oo[i]:oo[i + 1]] for i in range(len(streams))]


def morton_sorted_unique(pts, L):
    keys, _ = O.build_octree(pts, L)
    k = keys[L].astype(np.uint64)
    out = np.zeros((k.size, 3), np.int64)
    for b in range(L):
        t = (k >> np.uint64(3 * b)) & np.uint64(7)
        out[:, 0] |= ((t >> np.uint64(2)) & np.uint64(1)).astype(np.int64) << b
        out[:, 1] |= ((t >> np.uint64(1)) & np.uint64(1)).astype(np.int64) << b
        out[:, 2] |= (t & np.uint64(1)).astype(np.int64) << b
    return out.astype(np.int32)


# ---------------------------------------------------------------------------------------
# tensor-core primitive (tcgen05.mma kind::i8, TMEM int32 accumulators)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("N", [32, 64, 256])
def test_tcgen05_int8_gemm(pcc, ctx, N):
    rng = np.random.default_rng(N)
    a = rng.integers(-128, 128, size=(128, 32)).astype(np.int8)
    b = rng.integers(-128, 128, size=(N, 32)).astype(np.int8)
    a[0] = -128
    b[0] = -128   # extreme corner: 32 * 2^14 = 2^19
    d = pcc.pcc_debug_gemm_i8(ctx, a, b)
    assert np.array_equal(d, a.astype(np.int64) @ b.astype(np.int64).T)


# ---------------------------------------------------------------------------------------
# octree (a1, a2)
# ---------------------------------------------------------------------------------------

def _octree_cases():
    g = np.arange(2, dtype=np.int32)
    cube = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    rng = np.random.default_rng(0)
    dup = I.random_cloud(1000, 10, 3)
    dup = np.concatenate([dup, dup[rng.integers(0, 1000, 2000)]])[rng.permutation(3000)]
    return [("single", np.array([[5, 6, 7]], np.int32), 9), ("cube", cube, 1), ("dups", dup, 10),
            ("cfg1", I.make_frame(I.CFG1), 12), ("cfg2", I.make_frame(I.CFG2), 12),
            ("cfg3", I.make_frame(I.CFG3), 18), ("L21", I.random_cloud(5000, 21, 4), 21),
            ("ragged", I.random_cloud(4097, 12, 5), 12)]


@pytest.mark.parametrize("name,pts,L", _octree_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_build_octree(pcc, ctx, name, pts, L):
    keys, codes = O.build_octree(pts, L)
    tot = sum(len(c) for c in codes)
    d_codes = torch.empty(tot + 16, dtype=torch.uint8, device="cuda")
    counts = pcc.pcc_build_octree(ctx, dev(pts.astype(np.int32)), len(pts), L, d_codes, tot + 16)
    assert counts == [len(k) for k in keys]
    assert np.array_equal(d_codes[:tot].cpu().numpy(), np.concatenate(codes))


def test_build_octree_errors(pcc, ctx):
    with pytest.raises(pcc.PCCError) as e:
        pcc.pcc_build_octree(ctx, dev(np.array([[0, 0, 4096]], np.int32)), 1, 12)
    assert e.value.name == "RANGE"


# ---------------------------------------------------------------------------------------
# per-tensor parity of the encoder (a3-a9)
# ---------------------------------------------------------------------------------------

def _compare_dumps(pcc, ctx, D, L, R=4):
    names = D.names()
    checked = 0
    for name in names:
        kind = name.split("/")[0]
        if kind in ("p", "seg", "z"):
            continue
        want = D.get(name, np.uint8)
        got = pcc.pcc_debug_tensor(ctx, name)
        assert got is not None, name
        got = np.frombuffer(got, np.uint8)
        if kind == "nbr":
            g = got.view(np.int32).copy()
            n = g.size // 27
            g[g == n] = -1
            got = g.view(np.uint8)
        assert got.size == want.size, (name, got.size, want.size)
        if not np.array_equal(got, want):
            bad = np.flatnonzero(got != want)
            raise AssertionError(f"{name}: {bad.size} bytes differ, first at {bad[:8]}")
        checked += 1
    return checked


@pytest.mark.parametrize("C,cfg", [(8, "cfg1"), (32, "cfg1"), (32, "random10")])
def test_encoder_per_tensor_parity(pcc, ctx, C, cfg):
    mb, om = model_pair(C)
    m = gpu_model(pcc, mb)
    if cfg == "cfg1":
        pts, L = I.make_frame(I.CFG1), 12
    else:
        pts, L = I.random_cloud(4000, 10, 11, spread=0.3), 10
    D = O.Dump()
    want = O.encode(om, pts, L, D)
    pcc.pcc_ctx_set_debug(ctx, True)
    try:
        got, _ = gpu_encode(pcc, ctx, m, [pts], L)
        n = _compare_dumps(pcc, ctx, D, L)
    finally:
        pcc.pcc_ctx_set_debug(ctx, False)
    assert n > 40
    assert got[0] == want


def check_decoder_rows(pcc, ctx, D, d, model, L=12):
    """The decoder rows of level d (pcc_internal.cuh DROW_*: S, floor(65281 2^32 / S), mu,
    E_{16k}, a) hold exactly the oracle's hidden activations (a/d), and rebuild exactly
    the oracle's cumulative bounds C_i = i + floor(E_i 65281 / S) (reading Q21) from the
    Eq.7 logits z = b2 + a W2 and the Eq.15 exponentials; the decoded codes are the
    oracle's."""
    Dd = L - 1 - model.n_deep
    hd = model.shallow[d].head if d <= Dd else model.deep[d - Dd - 1].head
    H = model.H
    p = D.get(f"p/{d}", np.uint16).reshape(-1, 255).astype(np.int64)
    cum = np.concatenate([np.zeros((p.shape[0], 1), np.int64), np.cumsum(p, 1)[:, :254]], 1)
    raw = np.frombuffer(pcc.pcc_debug_tensor(ctx, f"cdf/{d}"), np.uint8).reshape(-1, 112)
    hdr = raw[:, :72].copy().view(np.uint32).astype(np.int64)
    a = raw[:, 80:80 + H].copy().view(np.int8).astype(np.int64)
    assert np.array_equal(a, D.get(f"a/{d}", np.int8).reshape(-1, H).astype(np.int64)), d
    assert not raw[:, 72:80].any() and not raw[:, 80 + H:].any(), d
    z = a @ hd.W2.astype(np.int64).T + hd.b2.astype(np.int64)
    assert np.array_equal(z, D.get(f"z/{d}", np.int32).reshape(-1, 255).astype(np.int64)), d
    m_l, r_l = hd.rq_logit.m_pos, hd.rq_logit.r
    l = np.clip((z * m_l + ((1 << (r_l - 1)) if r_l else 0)) >> r_l, -(1 << 24), 1 << 24)
    mu = l.max(1)
    assert np.array_equal(hdr[:, 2].astype(np.uint32).view(np.int32).astype(np.int64), mu), d
    dl = mu[:, None] - l
    lut = I.exp_lut().astype(np.int64)
    e = np.where(dl < 4096, lut[np.minimum(dl, 4095) >> 2], 0)
    E = np.concatenate([np.zeros((e.shape[0], 1), np.int64), np.cumsum(e, 1)], 1)
    S = hdr[:, 0]
    assert np.array_equal(E[:, 255], S), d
    assert np.array_equal(hdr[:, 1], (65281 << 32) // S), d
    assert np.array_equal(hdr[:, 3:18], E[:, 16:241:16]), d
    C = np.arange(255)[None, :] + (E[:, :255] * 65281) // S[:, None]
    assert np.array_equal(C, cum), d
    assert np.array_equal(np.frombuffer(pcc.pcc_debug_tensor(ctx, f"code/{d}"), np.uint8),
                          D.get(f"code/{d}", np.uint8)), d


def test_decoder_cdf_parity(pcc, ctx):
    mb, om = model_pair(8)
    m = gpu_model(pcc, mb)
    pts = I.make_frame(I.CFG1)
    D = O.Dump()
    bs = O.encode(om, pts, 12, D)
    pcc.pcc_ctx_set_debug(ctx, True)
    try:
        out = gpu_decode(pcc, ctx, m, [bs], len(pts))
        mobj = I.make_model(C=8, H=8, seed=1, min_depth=9, max_depth=18)
        for d in range(4, 12):
            check_decoder_rows(pcc, ctx, D, d, mobj)
    finally:
        pcc.pcc_ctx_set_debug(ctx, False)
    assert np.array_equal(out[0], morton_sorted_unique(pts, 12))


# ---------------------------------------------------------------------------------------
# end-to-end bitstreams (a10-a12) at the benchmark's sizes and launch configuration
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg,C,B", [("cfg1", 8, 7), ("cfg2", 32, 4), ("cfg3", 32, 1)])
def test_batch_bitstreams_match_oracle(pcc, ctx, cfg, C, B):
    sc = I.CONFIGS[cfg]
    mb, om = model_pair(C)
    m = gpu_model(pcc, mb)
    frames = I.make_frames(sc, B, first=3)
    got, _ = gpu_encode(pcc, ctx, m, frames, sc.bit_depth)
    for f, g in zip(frames, got):
        assert g == O.encode(om, f, sc.bit_depth)
    dec = gpu_decode(pcc, ctx, m, got, sum(len(f) for f in frames))
    for f, x in zip(frames, dec):
        assert np.array_equal(x, morton_sorted_unique(f, sc.bit_depth))


@pytest.mark.parametrize("L", [11, 12, 13, 14, 15, 16])
def test_precision_sweep_matches_oracle(pcc, ctx, L):
    """NEXT-1 precision sweep (Table 3 averages over 11-16 bit): the 16-beam
    sensor quantised at L bits, C = 32 GRED+XFP model, bit-identical to the oracle."""
    import dataclasses
    sc = dataclasses.replace(I.CFG1, bit_depth=L)
    mb, om = model_pair(32)
    m = gpu_model(pcc, mb)
    frames = I.make_frames(sc, 2, first=5)
    got, _ = gpu_encode(pcc, ctx, m, frames, L)
    for f, g in zip(frames, got):
        assert g == O.encode(om, f, L)
    dec = gpu_decode(pcc, ctx, m, got, sum(len(f) for f in frames))
    for f, x in zip(frames, dec):
        assert np.array_equal(x, morton_sorted_unique(f, L))


@pytest.mark.parametrize("n_deep,C", [(3, 32), (3, 8), (2, 32), (1, 16)])
def test_deep_level_variants_match_oracle(pcc, ctx, n_deep, C):
    """NEXT-1 t = L-3 variant (n_deep = 3) and shallower splits: the level partition
    moves, every kernel is reused, the bitstream stays bit-identical."""
    mb = I.make_model(C=C, H=C, seed=7, n_deep=n_deep, min_depth=9, max_depth=16).to_bytes()
    om = O.Model(mb)
    m = gpu_model(pcc, mb)
    frames = I.make_frames(I.CFG1, 2, first=2)
    got, _ = gpu_encode(pcc, ctx, m, frames, 12)
    for f, g in zip(frames, got):
        assert g[8] == n_deep and g == O.encode(om, f, 12)
    dec = gpu_decode(pcc, ctx, m, got, sum(len(f) for f in frames))
    for f, x in zip(frames, dec):
        assert np.array_equal(x, morton_sorted_unique(f, 12))


@pytest.mark.parametrize("case", ["cfg1x3", "cfg2", "cube", "single_L21", "cfg3"])
def test_hrcs_stats_match_oracle(pcc, ctx, case):
    """NEXT-3 HRCS statistic: per frame and depth, node count and summed
    occupied 26-neighbours, exact (integer) against the numpy set-membership oracle."""
    from oracle import hrcs as OH
    if case == "cfg1x3":
        frames, L = I.make_frames(I.CFG1, 3, first=1), 12
    elif case == "cfg2":
        frames, L = [I.make_frame(I.CFG2, 2)], 12
    elif case == "cfg3":
        frames, L = [I.make_frame(I.CFG3, 1)], 18
    elif case == "cube":
        g = np.arange(6, dtype=np.int32)
        frames, L = [np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 17], 9
    else:
        frames, L = [np.array([[7, (1 << 21) - 1, 0]], np.int32), I.random_cloud(800, 21, 3, spread=0.01)], 21
    offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
    nodes, nsum = pcc.pcc_hrcs_stats(ctx, dev(np.concatenate(frames).astype(np.int32)), offs, L)
    for i, f in enumerate(frames):
        wn, ws = OH.hrcs_stats(f, L)
        assert nodes[i].tolist() == wn.tolist(), i
        assert nsum[i].tolist() == ws.tolist(), i


def test_batch_equals_single_and_deterministic(pcc, ctx):
    mb, om = model_pair(8)
    m = gpu_model(pcc, mb)
    frames = [I.random_cloud(n, 11, s) for s, n in [(1, 1), (2, 700), (3, 5000), (4, 64)]]
    batch, _ = gpu_encode(pcc, ctx, m, frames, 11)
    again, _ = gpu_encode(pcc, ctx, m, frames, 11)
    assert batch == again
    for f, b in zip(frames, batch):
        single, _ = gpu_encode(pcc, ctx, m, [f], 11)
        assert single[0] == b == O.encode(om, f, 11)


def test_zero_model_and_max_depth(pcc, ctx):
    mb, om = model_pair(8, max_depth=21, kind="zero")
    m = gpu_model(pcc, mb)
    pts = I.random_cloud(3000, 21, 9, spread=0.001)
    got, _ = gpu_encode(pcc, ctx, m, [pts], 21)
    assert got[0] == O.encode(om, pts, 21)
    dec = gpu_decode(pcc, ctx, m, got, len(pts))
    assert np.array_equal(dec[0], morton_sorted_unique(pts, 21))


def test_large_level_multi_segment(pcc, ctx):
    """A level with > 4096 nodes spans several rANS segments (reading Q24')."""
    mb, om = model_pair(8, max_depth=12)
    m = gpu_model(pcc, mb)
    pts = I.random_cloud(150000, 12, 21)
    got, _ = gpu_encode(pcc, ctx, m, [pts], 12)
    assert got[0] == O.encode(om, pts, 12)
    dec = gpu_decode(pcc, ctx, m, got, len(pts))
    assert np.array_equal(dec[0], morton_sorted_unique(pts, 12))


def _map_rqs(obj, fn):
    """Apply fn to every activation requant of a Model (the logit requant is separate)."""
    import dataclasses
    seen = set()

    def walk(o):
        if isinstance(o, list):
            for v in o:
                walk(v)
        elif isinstance(o, dict):
            for v in o.values():
                walk(v)
        elif dataclasses.is_dataclass(o) and not isinstance(o, I.RQ):
            for fl in dataclasses.fields(o):
                v = getattr(o, fl.name)
                if isinstance(v, I.RQ):
                    if fl.name != "rq_logit" and id(v) not in seen:
                        seen.add(id(v))
                        fn(v)
                else:
                    walk(v)
    walk(obj)
    return len(seen)


@pytest.mark.parametrize("form", ["generic", "abs"])
@pytest.mark.parametrize("C,cfg", [(32, "cfg2"), (8, "cfg1")])
def test_requant_forms(pcc, ctx, form, C, cfg):
    """The three device forms of Eq.14's requant (rq.cuh) against the oracle: the default
    model takes the signed one-multiply form; r > 32 forces the generic 64-bit form
    (same real multipliers as the default model), m >= 2^(r-1) the
    |x| form (saturating layers)."""
    model = I.make_model(C=C, H=C, seed=3, min_depth=9, max_depth=18)

    def generic(q):  # r' = 33 > 32, m' = m * 2^(33 - r): the same real multiplier
        k = 33 - q.r
        assert k >= 0 and (q.m_pos << k) < 2**31 and (q.m_neg << k) < 2**31
        q.m_pos, q.m_neg, q.r = q.m_pos << k, q.m_neg << k, 33

    def absform(q):
        q.m_pos, q.m_neg, q.r = int(0.6 * (1 << 24)), int(0.15 * (1 << 24)), 24

    assert _map_rqs(model, generic if form == "generic" else absform) > 10
    mb = model.to_bytes()
    om = O.Model(mb)
    m = pcc.pcc_model_load(mb, 0)
    try:
        sc = I.CONFIGS[cfg]
        frames = I.make_frames(sc, 2, first=5)
        got, _ = gpu_encode(pcc, ctx, m, frames, sc.bit_depth)
        for f, g in zip(frames, got):
            assert g == O.encode(om, f, sc.bit_depth)
        dec = gpu_decode(pcc, ctx, m, got, sum(len(f) for f in frames))
        for f, x in zip(frames, dec):
            assert np.array_equal(x, morton_sorted_unique(f, sc.bit_depth))
    finally:
        pcc.pcc_model_destroy(m)


# ---------------------------------------------------------------------------------------
# errors and robustness
# ---------------------------------------------------------------------------------------

def test_errors(pcc, ctx):
    mb, om = model_pair(8, max_depth=12)
    m = gpu_model(pcc, mb)
    pts = I.random_cloud(500, 10, 2)
    bs = O.encode(om, pts, 10)

    def st(fn):
        with pytest.raises(pcc.PCCError) as e:
            fn()
        return e.value.name

    assert st(lambda: gpu_encode(pcc, ctx, m, [np.zeros((0, 3), np.int32)], 10)) == "EMPTY"
    assert st(lambda: gpu_encode(pcc, ctx, m, [np.array([[0, 2000, 0]], np.int32)], 10)) == "RANGE"
    assert st(lambda: gpu_encode(pcc, ctx, m, [pts], 13)) == "UNSUPPORTED_DEPTH"
    assert st(lambda: gpu_decode(pcc, ctx, m, [b"XCC1" + bs[4:]], 600)) == "BAD_MAGIC"
    assert st(lambda: gpu_decode(pcc, ctx, m, [bs[:4] + b"\x07\x00" + bs[6:]], 600)) == "VERSION"
    other = gpu_model(pcc, model_pair(8, max_depth=12, seed=2)[0])
    assert st(lambda: gpu_decode(pcc, ctx, other, [bs], 600)) == "MODEL_MISMATCH"
    assert st(lambda: gpu_decode(pcc, ctx, m, [bs[:len(bs) - 8]], 600)) in ("TRUNCATED", "CORRUPT")
    assert st(lambda: gpu_decode(pcc, ctx, m, [bs], 10)) == "CAPACITY"
    rng = np.random.default_rng(7)
    for _ in range(40):
        d = bytearray(bs)
        pos = int(rng.integers(24, len(d)))
        d[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            want = O.decode(om, bytes(d))[0]
        except O.OracleError as e:
            want = e.name
        try:
            got = gpu_decode(pcc, ctx, m, [bytes(d)], 4096)[0]
        except pcc.PCCError as e:
            got = e.name
        if isinstance(want, str):
            assert got in ("CORRUPT", "TRUNCATED"), (want, got)
        else:
            assert not isinstance(got, str) and np.array_equal(got, want)
    # the context is still usable after errors
    good, _ = gpu_encode(pcc, ctx, m, [pts], 10)
    assert good[0] == bs


# ---------------------------------------------------------------------------------------
# alternate kernel variants (A/B baselines selected by environment) stay bit-exact
# ---------------------------------------------------------------------------------------

_ALT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I, pcc
mb = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18).to_bytes()
om = O.Model(mb)
codec = pcc.Codec(mb, 0)
for pts, L in [(I.make_frame(I.CFG1), 12), (I.random_cloud(3000, 10, 5, spread=0.3), 10)]:
    x = torch.from_numpy(pts).cuda()
    out, oo = codec.encode_frames(x, [0, len(pts)], L)
    assert out[:oo[1]].cpu().numpy().tobytes() == O.encode(om, pts, L)
    xyz, no = codec.decode_frames(out, oo, len(pts))
    assert np.array_equal(xyz[:no[1]].cpu().numpy(), O.decode(om, O.encode(om, pts, L))[0])
print("ALT-OK")
"""


@pytest.mark.parametrize("env", [{"PCC_UP": "simt", "PCC_DOWN": "simt"}, {"PCC_HEAD": "simt", "PCC_CONV": "simt"},
                                 {"PCC_HEAD": "t2"}, {"PCC_HEAD": "q4"}, {"PCC_KMAP": "hash"},
                                 {"PCC_CONV": "tc1"}, {"PCC_HEAD": "t3g3"}, {"PCC_HEAD": "t1"},
                                 {"PCC_KMAP": "derive27"}, {"PCC_HEAD": "t3"}, {"PCC_RDEC": "t2"}, {"PCC_RDEC": "t4"},
                                 {"PCC_RDEC": "old"}])
def test_alternate_kernels_bit_exact(pcc, env):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ALT.format(root=root)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert "ALT-OK" in r.stdout, r.stdout + r.stderr


def test_bench_launch_configuration_sampled(pcc):
    """BASELINE.json full size in the launch configuration bench.py times (cfg2, 512 frames
    per codec launch = one of its 4 lanes at the default batch of 2048, C = H = 32): sampled
    bitstreams byte-identical to the oracle, and every frame of the batch decodes to its
    unique voxels in Morton order."""
    from paper_2603_25260_b200.pcc import Codec
    mb, om = model_pair(32)
    nf = 512
    frames = I.make_frames(I.CFG2, nf, first=0, scene_seed=1)
    offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
    codec = Codec(mb, 0)
    out, oo = codec.encode_frames(dev(np.concatenate(frames)), offs, 12)
    xyz, no = codec.decode_frames(out, oo, offs[-1])
    host = out[:oo[-1]].cpu().numpy().tobytes()
    for i in (0, 137, 300, nf - 1):
        assert host[oo[i]:oo[i + 1]] == O.encode(om, frames[i], 12), i
    dec = xyz[:no[-1]].cpu().numpy()
    for i in range(nf):
        assert np.array_equal(dec[no[i]:no[i + 1]], morton_sorted_unique(frames[i], 12)), i
