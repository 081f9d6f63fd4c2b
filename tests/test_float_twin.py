"""NEXT-2: whole-network float twin and the cross-platform decode collapse.

P:85-99 (Fig. 2b): encoding on one GPU and decoding on another with floating-point
inference "collapses into an approximately uniform distribution"; Fig. 2c / P:287-290:
integer-only inference decodes bit-exactly.  tests/float_twin.py builds the float32 twin
of the ENTIRE integer network (every layer, not only the predictor) and codes with it.

* the twin is the same network: its logits track the integer model's (correlation);
* same backend and order: float encode -> float decode is lossless;
* another evaluation order (CPU) or another device (GPU fp32 vs CPU fp32): some node
  CDFs differ, the decoder derails at the first differing node of a level, and the
  decoded cloud is not the input (asserted);
* the integer path is identical across devices: GPU encode -> oracle (CPU) decode and
  oracle encode -> GPU decode are both exact (asserted on a GPU box).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_25260_b200 import inputs as I

from float_twin import FloatTwin, float_decode, float_encode, quantise_pmf, rans_decode, rans_encode

L = 12


@pytest.fixture(scope="module")
def setup():
    model = I.make_model(C=8, H=8, seed=1, min_depth=9, max_depth=12)
    pts = I.make_frame(I.CFG1, 3)
    keys, _ = O.build_octree(pts, L)
    return model, pts, keys[L]


@pytest.fixture(scope="module")
def cpu_stream(setup):
    model, pts, _ = setup
    return float_encode(FloatTwin(model, "cpu", "fused"), pts, L)


def test_quantiser_and_coder():
    rng = np.random.default_rng(0)
    lg = rng.normal(0, 2, size=(500, 255)).astype(np.float32)
    p = quantise_pmf(lg)
    assert (p >= 1).all() and (p.sum(1) == 1 << 16).all()
    sym = rng.integers(0, 255, size=500)
    w, x = rans_encode(sym, p)
    assert np.array_equal(rans_decode(w, x, p)[0], sym)


def test_twin_is_the_same_network(setup):
    """The twin's logits track the integer model's on the same (integer) octree: the
    integer z/d dumps (Eq.7) and the twin's float logits correlate strongly per level."""
    model, pts, _ = setup
    om = O.Model(model.to_bytes())
    D = O.Dump()
    O.encode(om, pts, L, D)
    keys, codes = O.build_octree(pts, L)
    tw = FloatTwin(model, "cpu", "fused")
    tw.reset()
    for d in range(model.R, L):
        p_f = tw.level_pmf(keys, codes, d, L)
        p_i = D.get(f"p/{d}", np.uint16).reshape(-1, 255).astype(np.float64)
        lf, li = np.log(p_f.astype(np.float64)), np.log(p_i)
        r = np.corrcoef(lf.ravel(), li.ravel())[0, 1]
        assert r > 0.9, (d, r)


def test_float_same_order_round_trip(setup, cpu_stream):
    model, _, leaf = setup
    stream, _ = cpu_stream
    got, depth, _ = float_decode(FloatTwin(model, "cpu", "fused"), stream, L)
    assert depth == L and np.array_equal(np.sort(got), leaf)


def _collapse_report(enc_pmfs, dec_pmfs, got, depth, leaf):
    differ = sum(int(np.any(a != b, 1).sum()) for a, b in zip(enc_pmfs, dec_pmfs) if a.shape == b.shape)
    kept = np.intersect1d(got, leaf).size if depth == L else 0
    return differ, kept


def test_float_other_order_collapses(setup, cpu_stream):
    """Decoding the fused-order float stream with the per-offset order (the same network,
    float32, summed in another order) derails: CDFs differ and the cloud is wrong."""
    model, _, leaf = setup
    stream, enc_pmfs = cpu_stream
    got, depth, dec_pmfs = float_decode(FloatTwin(model, "cpu", "per_offset"), stream, L)
    differ, kept = _collapse_report(enc_pmfs, dec_pmfs, got, depth, leaf)
    print(f"float twin, CPU fused vs CPU per-offset: {differ} node CDFs differ; decode reached depth {depth}, "
          f"{kept} of {leaf.size} voxels recovered")
    assert differ > 0
    assert depth < L or not np.array_equal(np.sort(got), leaf)


@pytest.mark.gpu
def test_float_cross_device_collapses_integer_does_not(setup, cpu_stream):
    """Encode with the CPU float twin, decode with the same twin on cuda:0 (torch fp32,
    TF32 off): the decode derails (Fig. 2b).  The integer pipeline on the same frame:
    GPU encode -> CPU oracle decode and CPU oracle encode -> GPU decode are exact (Fig. 2c)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    model, pts, leaf = setup
    stream, enc_pmfs = cpu_stream
    got, depth, dec_pmfs = float_decode(FloatTwin(model, "cuda", "fused"), stream, L)
    differ, kept = _collapse_report(enc_pmfs, dec_pmfs, got, depth, leaf)
    print(f"float twin, CPU encode -> GPU decode: {differ} node CDFs differ; decode reached depth {depth}, "
          f"{kept} of {leaf.size} voxels recovered")
    assert differ > 0
    assert depth < L or not np.array_equal(np.sort(got), leaf)
    # integer-only: bit-exact across the two platforms, both directions
    from paper_2603_25260_b200.pcc import Codec
    mb = model.to_bytes()
    om = O.Model(mb)
    codec = Codec(mb, 0)
    out, oo = codec.encode_frames(torch.from_numpy(pts).cuda(), [0, len(pts)], L)
    gpu_bs = out[:oo[1]].cpu().numpy().tobytes()
    xyz_cpu, _ = O.decode(om, gpu_bs)
    cpu_bs = O.encode(om, pts, L)
    d_bs = torch.from_numpy(np.frombuffer(cpu_bs, np.uint8).copy()).cuda()
    xyz, no = codec.decode_frames(d_bs, [0, len(cpu_bs)], len(pts))
    codec.close()
    keys, _ = O.build_octree(xyz_cpu, L)
    assert gpu_bs == cpu_bs
    assert np.array_equal(np.sort(keys[L]), leaf)
    assert np.array_equal(xyz[:no[1]].cpu().numpy(), xyz_cpu)
