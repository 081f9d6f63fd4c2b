"""CPU checks of the boundary: libpcc.so builds, loads, and exports every function that
include/pcc.h declares; without a GPU every compute entry point fails loudly with
PCC_ERR_CUDA (no CPU fallback exists)."""
import ctypes as ct
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcc.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pcc_[a-z_0-9]+)\s*\(", txt)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2603_25260_b200 import build
    path = build.build()
    lib = ct.CDLL(path)
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_binding_exposes_same_names():
    from paper_2603_25260_b200 import pcc
    for n in _declared():
        assert hasattr(pcc, n), n


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_25260_b200 import pcc
    with pytest.raises(pcc.PCCError) as e:
        pcc.pcc_ctx_create(0)
    assert e.value.name == "CUDA"
    from paper_2603_25260_b200 import inputs as I
    with pytest.raises(pcc.PCCError) as e:
        pcc.pcc_model_load(I.model_bytes(8, 8, 1, max_depth=12), 0)
    assert e.value.name == "CUDA"


def test_status_strings():
    from paper_2603_25260_b200 import pcc
    assert pcc.pcc_status_string(0) == "OK"
    assert pcc.pcc_status_string(10) == "CORRUPT"
    assert pcc.pcc_encode_bound(131072, 12) > 2 * 131072


SURVEY_8B = ("pcc_model_create_random", "pcc_model_load", "pcc_model_save", "pcc_model_hash", "pcc_model_destroy",
             "pcc_ctx_create", "pcc_ctx_destroy", "pcc_encode_bound", "pcc_build_octree", "pcc_encode", "pcc_decode",
             "pcc_encode_batch", "pcc_decode_batch", "pcc_status_string")


def test_survey_8b_boundary_is_declared():
    """Every call SURVEY.md §8(b) lists is declared in include/pcc.h (and so exported)."""
    names = set(_declared())
    assert not [n for n in SURVEY_8B if n not in names]


@pytest.mark.parametrize("C,nd,flags", [(8, 4, 0), (32, 4, 0), (16, 0, 0), (8, 2, 1), (8, 4, 2), (8, 3, 3)])
def test_random_model_file_without_gpu(C, nd, flags):
    """pcc_model_random_file builds the model file on the host (no GPU): same layout and
    size as the Python generator's file for the same architecture, valid FNV trailer,
    and the oracle codes a frame losslessly with it."""
    import numpy as np
    from oracle import oracle as O
    from paper_2603_25260_b200 import inputs as I
    from paper_2603_25260_b200 import pcc
    cfg = pcc.model_config(C, deep_levels=nd, min_depth=9, max_depth=12, seed=77, flags=flags)
    mb = pcc.pcc_model_random_file(cfg)
    assert mb == pcc.pcc_model_random_file(cfg)            # deterministic in the seed
    assert mb != pcc.pcc_model_random_file(pcc.model_config(C, deep_levels=nd, min_depth=9, max_depth=12, seed=78,
                                                            flags=flags))
    py = I.make_model(C=C, H=C, seed=77, n_deep=nd, min_depth=9, max_depth=12, xfp=not (flags & 1),
                      raw_freq=bool(flags & 2)).to_bytes()
    assert len(mb) == len(py) and mb[:64] == py[:64]       # same header and layout
    assert I.model_hash(mb) == I.fnv1a64(mb[:-8])
    om = O.Model(mb)
    pts = I.make_frame(I.CFG1, 1)
    xyz, L = O.decode(om, O.encode(om, pts, 12))
    keys, _ = O.build_octree(pts, 12)
    assert L == 12 and xyz.shape[0] == keys[12].size


def test_random_model_file_rejects_bad_configs():
    from paper_2603_25260_b200 import pcc
    for kw in (dict(channels=24), dict(channels=8, head_hidden=16), dict(raw_levels=7), dict(deep_levels=5),
               dict(min_depth=5), dict(max_depth=22), dict(flags=4)):
        base = dict(channels=8, deep_levels=4, min_depth=9, max_depth=12)
        base.update(kw)
        with pytest.raises(pcc.PCCError) as e:
            pcc.pcc_model_random_file(pcc.model_config(**base))
        assert e.value.name == "INVALID_ARG", kw
