"""GPU parity, round 2: the CUDA path (C ABI) against the CPU oracle, tolerance 0.

* models created by the library itself (pcc_model_create_random / pcc_model_save, §8(b));
* the Table 4 ablation variants (XFP off, GRED off) and the P:601
  symbol-frequency raw-prefix coder, per tensor and end to end;
* a logit requant that saturates (Eq.15 clamp, reading Q20), so the SAT=true predictor
  kernels run in both encode and decode;
* the decoder rows at C = 32 (not only C = 8);
* model-file validation on the GPU loader (bad exp tables, R > 6) and the per-device
  kernel attributes (a second context after errors);
* ALL 256 frames of the bench launch configuration against a threaded oracle.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2603_25260_b200 import inputs as I  # noqa: E402
from test_gpu_parity import (_compare_dumps, check_decoder_rows, dev, gpu_decode, gpu_encode,  # noqa: E402
                             morton_sorted_unique)


@pytest.fixture(scope="module")
def pcc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_25260_b200 import pcc as P
    return P


@pytest.fixture(scope="module")
def ctx(pcc):
    c = pcc.pcc_ctx_create(0, torch.cuda.current_stream().cuda_stream)
    yield c
    pcc.pcc_ctx_destroy(c)


def _check_frames(pcc, ctx, m, om, frames, L):
    got, _ = gpu_encode(pcc, ctx, m, frames, L)
    for i, (f, g) in enumerate(zip(frames, got)):
        assert g == O.encode(om, f, L), i
    dec = gpu_decode(pcc, ctx, m, got, sum(len(f) for f in frames))
    for i, (f, x) in enumerate(zip(frames, dec)):
        assert np.array_equal(x, morton_sorted_unique(f, L)), i
    return got


# ---------------------------------------------------------------------------------------
# §8(b): the library's own model creation and serialisation
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("C,nd,flags", [(8, 4, 0), (32, 4, 0), (16, 3, 2), (32, 0, 0), (32, 4, 1)])
def test_create_random_save_matches_oracle(pcc, ctx, C, nd, flags):
    cfg = pcc.model_config(C, deep_levels=nd, max_depth=14, seed=21 + C, flags=flags)
    m = pcc.pcc_model_create_random(cfg, 0)
    try:
        saved = pcc.pcc_model_save(m)
        assert saved == pcc.pcc_model_random_file(cfg)
        assert pcc.pcc_model_hash(m) == I.model_hash(saved) and pcc.pcc_model_flags(m) == flags
        om = O.Model(saved)
        _check_frames(pcc, ctx, m, om, I.make_frames(I.CFG1, 2, first=9), 12)
    finally:
        pcc.pcc_model_destroy(m)


def test_gpu_loader_validates_model_files(pcc):
    import struct
    mb = I.make_model(C=8, H=8, seed=1, max_depth=12).to_bytes()

    def with_lut(lut):
        body = bytearray(mb[:-8])
        body[64:64 + 4096] = np.asarray(lut, "<u4").tobytes()
        return bytes(body) + struct.pack("<Q", I.fnv1a64(bytes(body)))

    lut = I.exp_lut().astype(np.int64)
    bad = [np.zeros(1024, np.int64), lut * 65281 // (1 << 24), np.concatenate([[(1 << 24) + 1], lut[1:]]),
           np.concatenate([lut[:500], [lut[499] + 1], lut[501:]])]
    for b in bad:
        with pytest.raises(pcc.PCCError) as e:
            pcc.pcc_model_load(with_lut(b), 0)
        assert e.value.name == "INVALID_ARG"
    m = pcc.pcc_model_load(with_lut(lut), 0)
    pcc.pcc_model_destroy(m)
    with pytest.raises(pcc.PCCError) as e:
        pcc.pcc_model_create_random(pcc.model_config(8, raw_levels=7, deep_levels=0, min_depth=9, max_depth=12), 0)
    assert e.value.name == "INVALID_ARG"


# ---------------------------------------------------------------------------------------
# NEXT-1: Table 4 ablation variants; NEXT-4: the frequency-coded raw prefix
# ---------------------------------------------------------------------------------------

_VARIANTS = {"xfp_off": dict(xfp=False), "gred_off": dict(n_deep=0), "raw_freq": dict(raw_freq=True),
             "xfp_off_raw_freq": dict(xfp=False, raw_freq=True)}


@pytest.mark.parametrize("variant", sorted(_VARIANTS))
@pytest.mark.parametrize("C", [8, 32])
def test_variant_per_tensor_parity(pcc, ctx, variant, C):
    mb = I.make_model(C=C, H=C, seed=13, min_depth=9, max_depth=14, **_VARIANTS[variant]).to_bytes()
    om = O.Model(mb)
    m = pcc.pcc_model_load(mb, 0)
    try:
        pts = I.make_frame(I.CFG1, 6)
        D = O.Dump()
        want = O.encode(om, pts, 12, D)
        pcc.pcc_ctx_set_debug(ctx, True)
        try:
            got, _ = gpu_encode(pcc, ctx, m, [pts], 12)
            n = _compare_dumps(pcc, ctx, D, 12)
        finally:
            pcc.pcc_ctx_set_debug(ctx, False)
        assert n > 30 and got[0] == want
        _check_frames(pcc, ctx, m, om, I.make_frames(I.CFG1, 3, first=1) + [I.make_frame(I.CFG2, 2)], 12)
    finally:
        pcc.pcc_model_destroy(m)


@pytest.mark.parametrize("variant", sorted(_VARIANTS))
def test_variant_cfg2_batch(pcc, ctx, variant):
    mb = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18, **_VARIANTS[variant]).to_bytes()
    om = O.Model(mb)
    m = pcc.pcc_model_load(mb, 0)
    try:
        _check_frames(pcc, ctx, m, om, I.make_frames(I.CFG2, 3, first=40), 12)
    finally:
        pcc.pcc_model_destroy(m)


def test_raw_freq_large_prefix(pcc, ctx):
    """R = 6 (up to 37449 raw symbols, the count rescale of the frequency model triggers)
    on a dense random cloud, frequency-coded raw prefix vs the oracle."""
    mb = I.make_model(C=8, H=8, seed=2, R=6, n_deep=2, min_depth=9, max_depth=12, raw_freq=True).to_bytes()
    om = O.Model(mb)
    m = pcc.pcc_model_load(mb, 0)
    try:
        _check_frames(pcc, ctx, m, om, [I.random_cloud(60000, 12, 3), I.random_cloud(500, 12, 4)], 12)
    finally:
        pcc.pcc_model_destroy(m)


# ---------------------------------------------------------------------------------------
# Eq.15 clamp: a logit requant that saturates at +-2^24 (SAT=true predictor kernels)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("sat_frac", [0.02, 0.4])
@pytest.mark.parametrize("C", [8, 32])
def test_saturating_logit_requant(pcc, ctx, sat_frac, C):
    """m_l / 2^r_l set so that a fraction sat_frac of the logits clamp at +-2^24 (Eq.15,
    reading Q20); z itself does not depend on the logit requant, so m_l is derived from
    the unclamped model's z dumps."""
    model = I.make_model(C=C, H=C, seed=5, min_depth=9, max_depth=14)
    pts = I.make_frame(I.CFG1, 3)
    D0 = O.Dump()
    O.encode(O.Model(model.to_bytes()), pts, 12, D0)
    z = np.concatenate([D0.get(f"z/{d}", np.int32) for d in range(4, 12)]).astype(np.int64)
    m_l = int(np.ceil((1 << 24) / np.quantile(np.abs(z), 1.0 - sat_frac)))
    for h in [s.head for s in model.shallow.values()] + [dp.head for dp in model.deep]:
        h.rq_logit = I.RQ(m_l, m_l, 0)
    mb = model.to_bytes()
    om = O.Model(mb)
    D = O.Dump()
    O.encode(om, pts, 12, D)
    frac = (np.abs(z * m_l) >= 1 << 24).mean()
    assert 0.5 * sat_frac < frac < 2 * sat_frac   # the clamp is exercised
    m = pcc.pcc_model_load(mb, 0)
    try:
        pcc.pcc_ctx_set_debug(ctx, True)
        try:
            gpu_encode(pcc, ctx, m, [pts], 12)
            assert _compare_dumps(pcc, ctx, D, 12) > 30
            gpu_decode(pcc, ctx, m, [O.encode(om, pts, 12)], len(pts))
            for d in range(4, 12):
                check_decoder_rows(pcc, ctx, D, d, model)
        finally:
            pcc.pcc_ctx_set_debug(ctx, False)
        _check_frames(pcc, ctx, m, om, [pts, I.make_frame(I.CFG2, 1)], 12)
    finally:
        pcc.pcc_model_destroy(m)


@pytest.mark.parametrize("bmax", [500_000, 3_000_000])
@pytest.mark.parametrize("C", [8, 32])
def test_bias_fold_boundary(pcc, ctx, bmax, C):
    """head4_tc.cu carries b1 / b2 as a second MMA slab of base-127 digits, exact for |b| <=
    500000 (31 * 127 * 127 + 126); beyond it the library runs head3 (TMEM-seeded bias).
    Biases drawn up to bmax, with the extremes +-bmax present, on both sides of the bound."""
    model = I.make_model(C=C, H=C, seed=11, min_depth=9, max_depth=14)
    rng = np.random.default_rng(bmax + C)
    for h in [s.head for s in model.shallow.values()] + [dp.head for dp in model.deep]:
        h.b1 = rng.integers(-bmax, bmax + 1, size=h.b1.shape).astype(np.int32)
        h.b2 = rng.integers(-bmax, bmax + 1, size=h.b2.shape).astype(np.int32)
        h.b1.flat[0], h.b2.flat[0], h.b2.flat[-1] = bmax, -bmax, bmax
    mb = model.to_bytes()
    om = O.Model(mb)
    pts = I.make_frame(I.CFG1, 2)
    D = O.Dump()
    O.encode(om, pts, 12, D)
    m = pcc.pcc_model_load(mb, 0)
    try:
        pcc.pcc_ctx_set_debug(ctx, True)
        try:
            gpu_encode(pcc, ctx, m, [pts], 12)
            assert _compare_dumps(pcc, ctx, D, 12) > 30
            gpu_decode(pcc, ctx, m, [O.encode(om, pts, 12)], len(pts))
            for d in range(4, 12):
                check_decoder_rows(pcc, ctx, D, d, model)
        finally:
            pcc.pcc_ctx_set_debug(ctx, False)
        _check_frames(pcc, ctx, m, om, [pts, I.make_frame(I.CFG2, 1)], 12)
    finally:
        pcc.pcc_model_destroy(m)


# ---------------------------------------------------------------------------------------
# decoder rows at C = 32 (the bench's model width)
# ---------------------------------------------------------------------------------------

def test_decoder_rows_c32(pcc, ctx):
    mobj = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18)
    mb = mobj.to_bytes()
    om = O.Model(mb)
    m = pcc.pcc_model_load(mb, 0)
    try:
        pts = I.make_frame(I.CFG2, 5)
        D = O.Dump()
        bs = O.encode(om, pts, 12, D)
        pcc.pcc_ctx_set_debug(ctx, True)
        try:
            out = gpu_decode(pcc, ctx, m, [bs], len(pts))
            for d in range(4, 12):
                check_decoder_rows(pcc, ctx, D, d, mobj)
        finally:
            pcc.pcc_ctx_set_debug(ctx, False)
        assert np.array_equal(out[0], morton_sorted_unique(pts, 12))
    finally:
        pcc.pcc_model_destroy(m)


# ---------------------------------------------------------------------------------------
# the bench's launch configuration, every frame against the oracle
# ---------------------------------------------------------------------------------------

def test_bench_launch_configuration_all_frames(pcc):
    """cfg2 at full size, 512 frames per codec launch (one of bench.py's 4 lanes at its
    default batch of 2048), C = H = 32: EVERY frame's bitstream byte-identical to the
    oracle (oracle encodes on all host cores), every frame decodes to its voxels."""
    from paper_2603_25260_b200.pcc import Codec
    mb = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18).to_bytes()
    om = O.Model(mb)
    nf = 512
    frames = I.make_frames(I.CFG2, nf, first=0, scene_seed=1)
    offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
    codec = Codec(mb, 0)
    out, oo = codec.encode_frames(dev(np.concatenate(frames)), offs, 12)
    xyz, no = codec.decode_frames(out, oo, offs[-1])
    host = out[:oo[-1]].cpu().numpy().tobytes()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        want = list(ex.map(lambda f: O.encode(om, f, 12), frames))
    bad = [i for i in range(nf) if host[oo[i]:oo[i + 1]] != want[i]]
    assert not bad, bad[:10]
    dec = xyz[:no[-1]].cpu().numpy()
    for i in range(nf):
        assert np.array_equal(dec[no[i]:no[i + 1]], morton_sorted_unique(frames[i], 12)), i
    codec.close()


# ---------------------------------------------------------------------------------------
# host-buffer calls (the e2e path)
# ---------------------------------------------------------------------------------------

def test_host_buffer_api(pcc, ctx):
    """pcc_encode_batch_host / pcc_decode_batch_host on 70 cfg2 frames, pinned and pageable
    host buffers: the device-buffer batch call's bytes and decodes; sampled frames equal the
    oracle."""
    mobj = I.make_model(C=32, H=32, seed=1, min_depth=9, max_depth=18)
    mb = mobj.to_bytes()
    om = O.Model(mb)
    frames = I.make_frames(I.CFG2, 70, 0)
    L = I.CFG2.bit_depth
    m = pcc.pcc_model_load(mb, 0)
    try:
        want, oo_dev = gpu_encode(pcc, ctx, m, frames, L)
        offs = np.cumsum([0] + [len(f) for f in frames]).tolist()
        h_xyz = torch.from_numpy(np.concatenate(frames).astype(np.int32)).pin_memory()
        cap = sum(pcc.pcc_encode_bound(len(f), L) + 4 for f in frames)
        h_bs = torch.empty(cap, dtype=torch.uint8).pin_memory()
        oo = pcc.pcc_encode_batch_host(ctx, m, h_xyz, offs, L, h_bs, cap)
        blob = h_bs[:oo[-1]].numpy().tobytes()
        got = [blob[oo[i]:oo[i + 1]] for i in range(len(frames))]
        assert got == want
        for i in (0, 63, 64, 69):
            assert got[i] == O.encode(om, frames[i], L), i
        n = offs[-1]
        h_out = torch.empty((n, 3), dtype=torch.int32).pin_memory()
        no = pcc.pcc_decode_batch_host(ctx, m, h_bs, list(oo), h_out, n)
        dec = gpu_decode(pcc, ctx, m, want, n)
        xyz = h_out[:no[-1]].numpy()
        for i in range(len(frames)):
            assert np.array_equal(xyz[no[i]:no[i + 1]], dec[i]), i
        for i in (0, 64, 69):
            assert np.array_equal(dec[i], morton_sorted_unique(frames[i], L)), i
        # pageable host buffers (numpy)
        sub = frames[:5]
        soffs = np.cumsum([0] + [len(f) for f in sub]).tolist()
        p_xyz = np.ascontiguousarray(np.concatenate(sub).astype(np.int32))
        p_bs = np.zeros(sum(pcc.pcc_encode_bound(len(f), L) + 4 for f in sub), np.uint8)
        poo = pcc.pcc_encode_batch_host(ctx, m, p_xyz, soffs, L, p_bs, p_bs.size)
        assert [p_bs[poo[i]:poo[i + 1]].tobytes() for i in range(5)] == want[:5]
        p_out = np.zeros((soffs[-1], 3), np.int32)
        pno = pcc.pcc_decode_batch_host(ctx, m, p_bs, list(poo), p_out, soffs[-1])
        for i in range(5):
            assert np.array_equal(p_out[pno[i]:pno[i + 1]], dec[i]), i
    finally:
        pcc.pcc_model_destroy(m)
