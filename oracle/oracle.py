"""ctypes wrapper of the CPU oracle (oracle/pcc_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product path
(paper_2603_25260_b200.pcc) never imports this module.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from typing import Dict, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "pcc_oracle.cpp")
# PCC_ORACLE_LIB: a mutated build for tools/oracle_mutation.py only (never the product path)
LIB = os.environ.get("PCC_ORACLE_LIB") or os.path.join(HERE, "liboracle.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "EMPTY", 3: "RANGE", 4: "UNSUPPORTED_DEPTH", 5: "CAPACITY",
          6: "BAD_MAGIC", 7: "VERSION", 8: "MODEL_MISMATCH", 9: "TRUNCATED", 10: "CORRUPT",
          100: "EXCEPTION"}


class OracleError(RuntimeError):
    def __init__(self, status: int):
        super().__init__(f"oracle status {status} ({STATUS.get(status, '?')})")
        self.status = status
        self.name = STATUS.get(status, "?")


def build(force: bool = False) -> str:
    """Compile the oracle with plain g++ (no SIMD intrinsics, no OpenMP)."""
    if os.environ.get("PCC_ORACLE_LIB"):
        return LIB
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ct.CDLL(build())
        P, S, I = ct.c_void_p, ct.c_size_t, ct.c_int
        L.oracle_model_load.argtypes = [P, S, ct.POINTER(P)]
        L.oracle_model_free.argtypes = [P]
        L.oracle_model_hash.argtypes = [P]
        L.oracle_model_hash.restype = ct.c_uint64
        L.oracle_dump_new.restype = P
        L.oracle_dump_free.argtypes = [P]
        L.oracle_dump_get.argtypes = [P, ct.c_char_p, ct.POINTER(P)]
        L.oracle_dump_get.restype = S
        L.oracle_dump_has.argtypes = [P, ct.c_char_p]
        L.oracle_dump_names.argtypes = [P]
        L.oracle_dump_names.restype = ct.c_char_p
        L.oracle_free.argtypes = [P]
        L.oracle_build_octree.argtypes = [P, S, I, ct.POINTER(P), ct.POINTER(P), P]
        L.oracle_expand.argtypes = [P, P, S, ct.POINTER(P), ct.POINTER(S)]
        L.oracle_morton.argtypes = [ct.c_uint32, ct.c_uint32, ct.c_uint32, I]
        L.oracle_morton.restype = ct.c_uint64
        L.oracle_kernel_map.argtypes = [P, S, I, P]
        L.oracle_conv3_acc.argtypes = [P, S, I, P, I, P, I, P]
        L.oracle_down_acc.argtypes = [P, S, P, S, P, I, P, P]
        L.oracle_head_logits.argtypes = [P, S, I, I, P, P, ct.c_int32, ct.c_int32, ct.c_int32, P, P, P, P]
        L.oracle_rq.argtypes = [ct.c_int32, ct.c_int32, ct.c_int32]
        L.oracle_rq.restype = ct.c_int32
        L.oracle_prq.argtypes = [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32]
        L.oracle_prq.restype = ct.c_int32
        L.oracle_up_prune.argtypes = [P, P, S, I, P, P, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32,
                                      ct.POINTER(P), ct.POINTER(S)]
        L.oracle_cdf.argtypes = [P, S, ct.c_int32, ct.c_int32, P, P]
        L.oracle_rans_encode.argtypes = [P, P, S, ct.POINTER(P), ct.POINTER(S)]
        L.oracle_rans_decode.argtypes = [P, S, P, S, P, ct.POINTER(S)]
        L.oracle_encode.argtypes = [P, P, S, I, P, ct.POINTER(P), ct.POINTER(S)]
        L.oracle_decode.argtypes = [P, P, S, P, ct.POINTER(P), ct.POINTER(S), ct.POINTER(I)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p)


def _check(st: int):
    if st != 0:
        raise OracleError(st)


def _take(p: ct.c_void_p, nbytes: int, dtype) -> np.ndarray:
    buf = (ct.c_uint8 * max(nbytes, 1)).from_address(p.value) if nbytes else None
    arr = np.frombuffer(bytes(buf)[:nbytes], dtype=dtype).copy() if nbytes else np.zeros(0, dtype)
    lib().oracle_free(p)
    return arr


class Model:
    def __init__(self, model_bytes: bytes):
        self._buf = np.frombuffer(model_bytes, dtype=np.uint8).copy()
        h = ct.c_void_p()
        _check(lib().oracle_model_load(_ptr(self._buf), self._buf.size, ct.byref(h)))
        self.h = h

    @property
    def hash(self) -> int:
        return int(lib().oracle_model_hash(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().oracle_model_free(self.h)
                self.h = None
        except Exception:  # interpreter shutdown: the library may already be gone
            pass


class Dump:
    def __init__(self):
        self.h = ct.c_void_p(lib().oracle_dump_new())

    def names(self):
        return lib().oracle_dump_names(self.h).decode().split()

    def get(self, name: str, dtype=np.uint8) -> Optional[np.ndarray]:
        p = ct.c_void_p()
        n = lib().oracle_dump_get(self.h, name.encode(), ct.byref(p))
        if not lib().oracle_dump_has(self.h, name.encode()):
            return None
        if n == 0:
            return np.zeros(0, dtype)
        return np.frombuffer(ct.string_at(p.value, n), dtype=dtype).copy()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().oracle_dump_free(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass


def build_octree(xyz: np.ndarray, L: int) -> Tuple[list, list]:
    """Returns (keys[d] for d=0..L, codes[d] for d=0..L-1)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.int32)
    kp, cp = ct.c_void_p(), ct.c_void_p()
    counts = np.zeros(L + 1, np.uint32)
    _check(lib().oracle_build_octree(_ptr(xyz), xyz.shape[0], L, ct.byref(kp), ct.byref(cp), _ptr(counts)))
    nk = int(counts.sum())
    nc = int(counts[:L].sum())
    keys = _take(kp, nk * 8, np.uint64)
    codes = _take(cp, nc, np.uint8)
    ks, cs, o, oc = [], [], 0, 0
    for d in range(L + 1):
        ks.append(keys[o:o + counts[d]]); o += int(counts[d])
        if d < L:
            cs.append(codes[oc:oc + counts[d]]); oc += int(counts[d])
    return ks, cs


def expand(keys: np.ndarray, codes: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint64)
    codes = np.ascontiguousarray(codes, np.uint8)
    p, n = ct.c_void_p(), ct.c_size_t()
    _check(lib().oracle_expand(_ptr(keys), _ptr(codes), keys.size, ct.byref(p), ct.byref(n)))
    return _take(p, n.value * 8, np.uint64)


def morton(x: int, y: int, z: int, bits: int) -> int:
    return int(lib().oracle_morton(x, y, z, bits))


def kernel_map(keys: np.ndarray, depth: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint64)
    nbr = np.zeros((keys.size, 27), np.int32)
    _check(lib().oracle_kernel_map(_ptr(keys), keys.size, depth, _ptr(nbr)))
    return nbr


def conv3_acc(keys, depth, f, W) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint64)
    f = np.ascontiguousarray(f, np.int8)
    W = np.ascontiguousarray(W, np.int8)
    cin, cout = f.shape[1], W.shape[1]
    acc = np.zeros((keys.size, cout), np.int64)
    _check(lib().oracle_conv3_acc(_ptr(keys), keys.size, depth, _ptr(f), cin, _ptr(W), cout, _ptr(acc)))
    return acc


def down_acc(child_keys, parent_keys, g, W) -> np.ndarray:
    ck = np.ascontiguousarray(child_keys, np.uint64)
    pk = np.ascontiguousarray(parent_keys, np.uint64)
    g = np.ascontiguousarray(g, np.int8)
    W = np.ascontiguousarray(W, np.int8)
    C = g.shape[1]
    acc = np.zeros((pk.size, C), np.int64)
    _check(lib().oracle_down_acc(_ptr(ck), ck.size, _ptr(pk), pk.size, _ptr(g), C, _ptr(W), _ptr(acc)))
    return acc


def head_logits(F, W1, b1, rq1, W2, b2):
    """The codec's own Eq.7 predictor: (a int8 [n, H], z int32 [n, 255])."""
    F = np.ascontiguousarray(F, np.int8)
    W1 = np.ascontiguousarray(W1, np.int8)
    W2 = np.ascontiguousarray(W2, np.int8)
    b1 = np.ascontiguousarray(b1, np.int32)
    b2 = np.ascontiguousarray(b2, np.int32)
    n, C = F.shape
    H = W1.shape[0]
    a = np.zeros((n, H), np.int8)
    z = np.zeros((n, 255), np.int32)
    _check(lib().oracle_head_logits(_ptr(F), n, C, H, _ptr(W1), _ptr(b1), rq1[0], rq1[1], rq1[2], _ptr(W2), _ptr(b2),
                                    _ptr(a), _ptr(z)))
    return a, z


def rq(acc: int, m: int, r: int) -> int:
    return int(lib().oracle_rq(acc, m, r))


def prq(acc: int, mp: int, mn: int, r: int) -> int:
    return int(lib().oracle_prq(acc, mp, mn, r))


def up_prune(S, X, W, b, mp, mn, r, q_one) -> np.ndarray:
    S = np.ascontiguousarray(S, np.int8)
    X = np.ascontiguousarray(X, np.uint8)
    W = np.ascontiguousarray(W, np.int8)
    b = np.ascontiguousarray(b, np.int32)
    C = S.shape[1]
    p, rows = ct.c_void_p(), ct.c_size_t()
    _check(lib().oracle_up_prune(_ptr(S), _ptr(X), X.size, C, _ptr(W), _ptr(b), mp, mn, r, q_one,
                                 ct.byref(p), ct.byref(rows)))
    return _take(p, rows.value * C, np.int8).reshape(rows.value, C)


def cdf(z: np.ndarray, m_l: int, r_l: int, lut: np.ndarray) -> np.ndarray:
    z = np.ascontiguousarray(z, np.int32).reshape(-1, 255)
    lut = np.ascontiguousarray(lut, np.uint32)
    p = np.zeros(z.shape, np.uint32)
    _check(lib().oracle_cdf(_ptr(z), z.shape[0], m_l, r_l, _ptr(lut), _ptr(p)))
    return p


def rans_encode(cum: np.ndarray, freq: np.ndarray) -> bytes:
    cum = np.ascontiguousarray(cum, np.uint32)
    freq = np.ascontiguousarray(freq, np.uint32)
    p, n = ct.c_void_p(), ct.c_size_t()
    _check(lib().oracle_rans_encode(_ptr(cum), _ptr(freq), cum.size, ct.byref(p), ct.byref(n)))
    return _take(p, n.value, np.uint8).tobytes()


def rans_decode(data: bytes, pmf: np.ndarray) -> Tuple[np.ndarray, int]:
    buf = np.frombuffer(data, np.uint8).copy()
    pmf = np.ascontiguousarray(pmf, np.uint32).reshape(-1, 255)
    sym = np.zeros(pmf.shape[0], np.uint8)
    used = ct.c_size_t()
    _check(lib().oracle_rans_decode(_ptr(buf), buf.size, _ptr(pmf), pmf.shape[0], _ptr(sym), ct.byref(used)))
    return sym, used.value


def encode(model: Model, xyz: np.ndarray, L: int, dump: Optional[Dump] = None) -> bytes:
    xyz = np.ascontiguousarray(xyz, np.int32)
    p, n = ct.c_void_p(), ct.c_size_t()
    _check(lib().oracle_encode(model.h, _ptr(xyz), xyz.shape[0], L, dump.h if dump else None,
                               ct.byref(p), ct.byref(n)))
    return _take(p, n.value, np.uint8).tobytes()


def decode(model: Model, bs: bytes, dump: Optional[Dump] = None) -> Tuple[np.ndarray, int]:
    buf = np.frombuffer(bs, np.uint8).copy()
    p, n, L = ct.c_void_p(), ct.c_size_t(), ct.c_int()
    _check(lib().oracle_decode(model.h, _ptr(buf), buf.size, dump.h if dump else None,
                               ct.byref(p), ct.byref(n), ct.byref(L)))
    return _take(p, n.value * 12, np.int32).reshape(-1, 3), L.value
