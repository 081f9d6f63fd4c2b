"""Thin ctypes binding of libpcc.so (include/pcc.h).  Argument marshalling only.

Every compute step runs in the CUDA library; this module never computes any part
of the coder and has no CPU fallback: importing it on a machine where the library
cannot be loaded raises, and every call without an sm_100 device returns
PCC_ERR_CUDA (raised as PCCError).

Functions keep the C names (pcc_encode, pcc_decode, ...).  Device buffers are
passed as torch CUDA tensors (their data_ptr()) or raw integer addresses; host
offset arrays as Python sequences.
"""
from __future__ import annotations

import ctypes as ct
import os
from typing import Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCC_LIB") or os.path.join(HERE, "libpcc.so")  # PCC_LIB: dev builds only

STATUS = ["OK", "INVALID_ARG", "EMPTY", "RANGE", "UNSUPPORTED_DEPTH", "CAPACITY", "BAD_MAGIC", "VERSION",
          "MODEL_MISMATCH", "TRUNCATED", "CORRUPT", "CUDA", "OOM"]


MODEL_XFP_OFF = 1   # PCC_MODEL_XFP_OFF
MODEL_RAW_FREQ = 2  # PCC_MODEL_RAW_FREQ


class ModelConfig(ct.Structure):
    """pcc_model_config (include/pcc.h)."""
    _fields_ = [("channels", ct.c_int), ("head_hidden", ct.c_int), ("raw_levels", ct.c_int), ("deep_levels", ct.c_int),
                ("min_depth", ct.c_int), ("max_depth", ct.c_int), ("seed", ct.c_uint64), ("flags", ct.c_uint32)]


def model_config(channels=32, head_hidden=None, raw_levels=4, deep_levels=4, min_depth=9, max_depth=18, seed=1,
                 flags=0) -> ModelConfig:
    return ModelConfig(channels, channels if head_hidden is None else head_hidden, raw_levels, deep_levels, min_depth,
                       max_depth, seed, flags)


class PCCError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: PCC_ERR_{self.name}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run paper_2603_25260_b200/build.py (no CPU fallback exists)")
    L = ct.CDLL(LIB_PATH)
    P, S, I, U64 = ct.c_void_p, ct.c_size_t, ct.c_int, ct.c_uint64
    SP = ct.POINTER(ct.c_size_t)
    L.pcc_model_load.argtypes = [P, S, I, ct.POINTER(P)]
    L.pcc_model_hash.argtypes = [P, ct.POINTER(U64)]
    L.pcc_model_flags.argtypes = [P, ct.POINTER(ct.c_uint32)]
    L.pcc_model_create_random.argtypes = [ct.POINTER(ModelConfig), I, ct.POINTER(P)]
    L.pcc_model_random_file.argtypes = [ct.POINTER(ModelConfig), P, S, SP]
    L.pcc_model_save.argtypes = [P, P, S, SP]
    L.pcc_model_info.argtypes = [P] + [ct.POINTER(I)] * 6
    L.pcc_model_destroy.argtypes = [P]
    L.pcc_ctx_create.argtypes = [I, P, ct.POINTER(P)]
    L.pcc_ctx_destroy.argtypes = [P]
    L.pcc_encode_bound.argtypes = [S, I]
    L.pcc_encode_bound.restype = S
    L.pcc_build_octree.argtypes = [P, P, S, I, P, S, ct.POINTER(ct.c_uint32)]
    L.pcc_hrcs_stats.argtypes = [P, P, SP, I, I, ct.POINTER(U64), ct.POINTER(U64)]
    L.pcc_encode.argtypes = [P, P, P, S, I, P, S, SP]
    L.pcc_decode.argtypes = [P, P, P, S, P, S, SP, ct.POINTER(I)]
    L.pcc_encode_batch.argtypes = [P, P, P, SP, I, I, P, S, SP]
    L.pcc_decode_batch.argtypes = [P, P, P, SP, I, P, S, SP]
    L.pcc_encode_batch_host.argtypes = [P, P, P, SP, I, I, P, S, SP]
    L.pcc_decode_batch_host.argtypes = [P, P, P, SP, I, P, S, SP]
    L.pcc_debug_tensor.argtypes = [P, ct.c_char_p, P, S, SP]
    L.pcc_ctx_set_debug.argtypes = [P, I]
    L.pcc_ctx_launch_count.argtypes = [P]
    L.pcc_ctx_launch_count.restype = U64
    L.pcc_ctx_set_profile.argtypes = [P, I]
    L.pcc_ctx_set_profile.restype = I
    L.pcc_ctx_profile_get.argtypes = [P, ct.c_char_p, ct.POINTER(ct.c_double), ct.POINTER(U64), ct.POINTER(U64)]
    L.pcc_ctx_profile_get.restype = I
    L.pcc_ctx_profile_categories.argtypes = [P]
    L.pcc_ctx_profile_categories.restype = ct.c_char_p
    L.pcc_debug_gemm_i8.argtypes = [P, P, P, I, P]
    L.pcc_debug_gemm_i8.restype = I
    L.pcc_status_string.argtypes = [I]
    L.pcc_status_string.restype = ct.c_char_p
    for f in ("pcc_model_load", "pcc_model_hash", "pcc_model_info", "pcc_model_flags", "pcc_model_create_random",
              "pcc_model_random_file", "pcc_model_save", "pcc_ctx_create", "pcc_build_octree", "pcc_hrcs_stats",
              "pcc_encode", "pcc_decode", "pcc_encode_batch", "pcc_decode_batch", "pcc_encode_batch_host",
              "pcc_decode_batch_host", "pcc_debug_tensor", "pcc_ctx_set_debug"):
        getattr(L, f).restype = I
    return L


lib = _load()

EXPORTS = ("pcc_model_load", "pcc_model_create_random", "pcc_model_random_file", "pcc_model_save", "pcc_model_hash",
           "pcc_model_flags", "pcc_model_info", "pcc_model_destroy", "pcc_ctx_create",
           "pcc_ctx_destroy", "pcc_encode_bound", "pcc_build_octree", "pcc_hrcs_stats", "pcc_encode", "pcc_decode",
           "pcc_encode_batch", "pcc_decode_batch", "pcc_encode_batch_host", "pcc_decode_batch_host",
           "pcc_debug_tensor", "pcc_ctx_set_debug", "pcc_ctx_launch_count", "pcc_ctx_set_profile",
           "pcc_ctx_profile_get", "pcc_ctx_profile_categories", "pcc_debug_gemm_i8", "pcc_status_string")


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(type(x))


def _chk(st: int, where: str, ok=(0,)):
    if st not in ok:
        raise PCCError(st, where)
    return st


def _sizes(seq: Sequence[int]):
    return (ct.c_size_t * len(seq))(*[int(v) for v in seq])


# ---- handles -----------------------------------------------------------------------

def pcc_model_load(model_bytes: bytes, device: int = 0) -> ct.c_void_p:
    h = ct.c_void_p()
    buf = ct.create_string_buffer(model_bytes, len(model_bytes))
    _chk(lib.pcc_model_load(buf, len(model_bytes), device, ct.byref(h)), "pcc_model_load")
    return h


def pcc_model_create_random(cfg: ModelConfig, device: int = 0) -> ct.c_void_p:
    h = ct.c_void_p()
    _chk(lib.pcc_model_create_random(ct.byref(cfg), device, ct.byref(h)), "pcc_model_create_random")
    return h


def pcc_model_random_file(cfg: ModelConfig) -> bytes:
    n = ct.c_size_t()
    _chk(lib.pcc_model_random_file(ct.byref(cfg), None, 0, ct.byref(n)), "pcc_model_random_file", ok=(0, 5))
    buf = ct.create_string_buffer(n.value)
    _chk(lib.pcc_model_random_file(ct.byref(cfg), buf, n.value, ct.byref(n)), "pcc_model_random_file")
    return buf.raw[:n.value]


def pcc_model_save(m) -> bytes:
    n = ct.c_size_t()
    _chk(lib.pcc_model_save(m, None, 0, ct.byref(n)), "pcc_model_save", ok=(0, 5))
    buf = ct.create_string_buffer(n.value)
    _chk(lib.pcc_model_save(m, buf, n.value, ct.byref(n)), "pcc_model_save")
    return buf.raw[:n.value]


def pcc_model_flags(m) -> int:
    v = ct.c_uint32()
    _chk(lib.pcc_model_flags(m, ct.byref(v)), "pcc_model_flags")
    return v.value


def pcc_model_hash(m) -> int:
    v = ct.c_uint64()
    _chk(lib.pcc_model_hash(m, ct.byref(v)), "pcc_model_hash")
    return v.value


def pcc_model_info(m) -> dict:
    vals = [ct.c_int() for _ in range(6)]
    _chk(lib.pcc_model_info(m, *[ct.byref(v) for v in vals]), "pcc_model_info")
    return dict(zip(("C", "H", "R", "n_deep", "min_depth", "max_depth"), [v.value for v in vals]))


def pcc_model_destroy(m) -> None:
    lib.pcc_model_destroy(m)


def pcc_ctx_create(device: int = 0, stream: int = 0) -> ct.c_void_p:
    h = ct.c_void_p()
    _chk(lib.pcc_ctx_create(device, stream or None, ct.byref(h)), "pcc_ctx_create")
    return h


def pcc_ctx_destroy(c) -> None:
    lib.pcc_ctx_destroy(c)


def pcc_encode_bound(n: int, bit_depth: int) -> int:
    return int(lib.pcc_encode_bound(n, bit_depth))


# ---- compute entry points (same names as the C ABI) ----------------------------------

def pcc_build_octree(ctx, d_xyz, n: int, bit_depth: int, d_codes=None, codes_cap: int = 0):
    counts = (ct.c_uint32 * (bit_depth + 1))()
    _chk(lib.pcc_build_octree(ctx, _ptr(d_xyz), n, bit_depth, _ptr(d_codes), codes_cap, counts), "pcc_build_octree")
    return list(counts)


def pcc_hrcs_stats(ctx, d_xyz, offs: Sequence[int], bit_depth: int):
    """Per frame and depth: (node counts, summed occupied 26-neighbours), numpy u64 [frames][L+1]."""
    frames = len(offs) - 1
    nodes = (ct.c_uint64 * (frames * (bit_depth + 1)))()
    nbr = (ct.c_uint64 * (frames * (bit_depth + 1)))()
    _chk(lib.pcc_hrcs_stats(ctx, _ptr(d_xyz), _sizes(offs), frames, bit_depth, nodes, nbr), "pcc_hrcs_stats")
    import numpy as np
    shape = (frames, bit_depth + 1)
    return (np.frombuffer(nodes, np.uint64).reshape(shape).copy(), np.frombuffer(nbr, np.uint64).reshape(shape).copy())


def pcc_encode(ctx, model, d_xyz, n: int, bit_depth: int, d_out, out_cap: int) -> int:
    ln = ct.c_size_t()
    _chk(lib.pcc_encode(ctx, model, _ptr(d_xyz), n, bit_depth, _ptr(d_out), out_cap, ct.byref(ln)), "pcc_encode")
    return ln.value


def pcc_decode(ctx, model, d_bs, length: int, d_xyz_out, cap_points: int) -> Tuple[int, int]:
    n, L = ct.c_size_t(), ct.c_int()
    _chk(lib.pcc_decode(ctx, model, _ptr(d_bs), length, _ptr(d_xyz_out), cap_points, ct.byref(n), ct.byref(L)),
         "pcc_decode")
    return n.value, L.value


def pcc_encode_batch(ctx, model, d_xyz, offs: Sequence[int], bit_depth: int, d_out, out_cap: int):
    frames = len(offs) - 1
    oo = (ct.c_size_t * (frames + 1))()
    _chk(lib.pcc_encode_batch(ctx, model, _ptr(d_xyz), _sizes(offs), frames, bit_depth, _ptr(d_out), out_cap, oo),
         "pcc_encode_batch")
    return list(oo)


def pcc_decode_batch(ctx, model, d_bs, bs_offs: Sequence[int], d_xyz_out, cap_points: int):
    frames = len(bs_offs) - 1
    oo = (ct.c_size_t * (frames + 1))()
    _chk(lib.pcc_decode_batch(ctx, model, _ptr(d_bs), _sizes(bs_offs), frames, _ptr(d_xyz_out), cap_points, oo),
         "pcc_decode_batch")
    return list(oo)


def pcc_encode_batch_host(ctx, model, h_xyz, offs: Sequence[int], bit_depth: int, h_out, out_cap: int):
    frames = len(offs) - 1
    oo = (ct.c_size_t * (frames + 1))()
    _chk(lib.pcc_encode_batch_host(ctx, model, _ptr(h_xyz), _sizes(offs), frames, bit_depth, _ptr(h_out), out_cap, oo),
         "pcc_encode_batch_host")
    return list(oo)


def pcc_decode_batch_host(ctx, model, h_bs, bs_offs: Sequence[int], h_xyz_out, cap_points: int):
    frames = len(bs_offs) - 1
    oo = (ct.c_size_t * (frames + 1))()
    _chk(lib.pcc_decode_batch_host(ctx, model, _ptr(h_bs), _sizes(bs_offs), frames, _ptr(h_xyz_out), cap_points, oo),
         "pcc_decode_batch_host")
    return list(oo)


def pcc_ctx_set_debug(ctx, on: bool) -> None:
    _chk(lib.pcc_ctx_set_debug(ctx, 1 if on else 0), "pcc_ctx_set_debug")


def pcc_debug_tensor(ctx, name: str) -> Optional[bytes]:
    ln = ct.c_size_t()
    if lib.pcc_debug_tensor(ctx, name.encode(), None, 0, ct.byref(ln)) != 0:
        return None
    buf = ct.create_string_buffer(max(ln.value, 1))
    _chk(lib.pcc_debug_tensor(ctx, name.encode(), buf, ln.value, ct.byref(ln)), "pcc_debug_tensor")
    return buf.raw[:ln.value]


def pcc_ctx_launch_count(ctx) -> int:
    return int(lib.pcc_ctx_launch_count(ctx))


def pcc_ctx_set_profile(ctx, on: bool) -> None:
    _chk(lib.pcc_ctx_set_profile(ctx, 1 if on else 0), "pcc_ctx_set_profile")


def pcc_ctx_profile_get(ctx, category: Optional[str] = None) -> Tuple[float, int, int]:
    ms, nl, nb = ct.c_double(), ct.c_uint64(), ct.c_uint64()
    _chk(lib.pcc_ctx_profile_get(ctx, category.encode() if category else None, ct.byref(ms), ct.byref(nl),
                                 ct.byref(nb)), "pcc_ctx_profile_get")
    return ms.value, nl.value, nb.value


def pcc_ctx_profile_categories(ctx) -> list:
    return lib.pcc_ctx_profile_categories(ctx).decode().split()


def pcc_debug_gemm_i8(ctx, a, b):
    """a: int8 numpy [128, 32], b: int8 numpy [N, 32] -> int32 numpy [128, N] via tcgen05."""
    import numpy as np
    a = np.ascontiguousarray(a, np.int8)
    b = np.ascontiguousarray(b, np.int8)
    d = np.zeros((128, b.shape[0]), np.int32)
    _chk(lib.pcc_debug_gemm_i8(ctx, a.ctypes.data, b.ctypes.data, b.shape[0], d.ctypes.data), "pcc_debug_gemm_i8")
    return d


def pcc_status_string(st: int) -> str:
    return lib.pcc_status_string(st).decode()


# ---- convenience wrapper (torch for device memory only) -----------------------------

class Codec:
    """Model + context on one device; buffers are torch CUDA tensors."""

    def __init__(self, model_bytes: bytes, device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.model = pcc_model_load(model_bytes, device)
        self.ctx = pcc_ctx_create(device, self.stream.cuda_stream)
        self.info = pcc_model_info(self.model)

    def close(self):
        if self.ctx:
            pcc_ctx_destroy(self.ctx)
            self.ctx = None
        if self.model:
            pcc_model_destroy(self.model)
            self.model = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode_frames(self, d_xyz, offs: Sequence[int], bit_depth: int, out=None):
        """d_xyz: int32 CUDA tensor [n, 3] of concatenated frames; returns (uint8 CUDA tensor, offsets)."""
        t = self.torch
        if out is None:
            cap = sum(pcc_encode_bound(offs[i + 1] - offs[i], bit_depth) + 4 for i in range(len(offs) - 1))
            out = t.empty(cap, dtype=t.uint8, device=d_xyz.device)
        oo = pcc_encode_batch(self.ctx, self.model, d_xyz, offs, bit_depth, out, out.numel())
        return out, oo

    def decode_frames(self, d_bs, bs_offs: Sequence[int], cap_points: int, out=None):
        t = self.torch
        if out is None:
            out = t.empty((cap_points, 3), dtype=t.int32, device=d_bs.device)
        oo = pcc_decode_batch(self.ctx, self.model, d_bs, bs_offs, out, cap_points)
        return out, oo
