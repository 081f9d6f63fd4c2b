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
