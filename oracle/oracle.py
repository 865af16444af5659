"""ctypes binding of oracle/oracle.c plus plain numpy bookkeeping helpers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  P:n = PAPER.md line n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_I64 = ctypes.c_int64
_I32 = ctypes.c_int


def build_oracle(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        lib.orc_dot.restype = ctypes.c_double
        lib.orc_dot.argtypes = [_f32p, _f32p, _I32]
        lib.orc_norms.argtypes = [_f32p, _I64, _I32, _f64p]
        lib.orc_sort_by_norm_desc.argtypes = [_f64p, _I64, _i64p]
        lib.orc_topk.argtypes = [_f32p, _I64, _f32p, _I64, _I32, _I32, _f64p, _i32p, _I32]
        lib.orc_rkmips_naive.argtypes = [_f32p, _I64, _f32p, _I64, _I32, _f32p, _I64, _I32, _u8p, _I32]
        lib.orc_rkmips_twophase.argtypes = [_f32p, _I64, _I32, _f64p, _I32, _f32p, _I64, _I32, _u8p, _I32]
        lib.orc_linear_scan.restype = ctypes.c_int
        lib.orc_linear_scan.argtypes = [_f32p, ctypes.c_double, _f32p, _f32p, _f64p, _I64, _I32, _I32,
                                        ctypes.POINTER(ctypes.c_int64)]
        lib.orc_block_bounds.argtypes = [_f64p, _I64, _I32, _I64, _f64p]
        lib.orc_margin.argtypes = [_f32p, _I64, _f32p, _I64, _I32, _f32p, _i64p, _I64, _I32, _f64p, _I32]
        lib.orc_margin_lists.argtypes = [_f32p, _I64, _f32p, _I64, _I32, _f32p, _f64p, _i32p, _I32, _i64p, _I64,
                                         _I32, _f64p, _I32]
        _lib = lib
    return _lib


def _c32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if a.ndim == 2 else a.reshape(1, -1)


def dot(a, b) -> float:
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    assert a.shape == b.shape
    return _load().orc_dot(a, b, a.size)


def norms(X) -> np.ndarray:
    X = _c32(X)
    out = np.empty(X.shape[0], np.float64)
    _load().orc_norms(X, X.shape[0], X.shape[1], out)
    return out


def sort_by_norm_desc(nrm) -> np.ndarray:
    nrm = np.ascontiguousarray(nrm, np.float64)
    perm = np.empty(nrm.size, np.int64)
    _load().orc_sort_by_norm_desc(nrm, nrm.size, perm)
    return perm


def topk(U, P, kk: int, threads: int = 0):
    """Exact top-kk (values desc, ties by ascending item id) of u.p over all of P."""
    U, P = _c32(U), _c32(P)
    n, d = U.shape
    vals = np.empty((n, kk), np.float64)
    ids = np.empty((n, kk), np.int32)
    if n:
        _load().orc_topk(U, n, P, P.shape[0], d, kk, vals, ids, threads)
    return vals, ids


def rkmips_naive(U, P, Qy, k: int, threads: int = 0) -> np.ndarray:
    """member[q, u] (bool) = c(u, q) < k by full enumeration (Def. 2)."""
    U, P, Qy = _c32(U), _c32(P), _c32(Qy)
    n, d = U.shape
    out = np.zeros((Qy.shape[0], n), np.uint8)
    if n and Qy.shape[0]:
        _load().orc_rkmips_naive(U, n, P, P.shape[0], d, Qy, Qy.shape[0], k, out, threads)
    return out.astype(bool)


def rkmips_twophase(U, topvals, Qy, k: int, threads: int = 0) -> np.ndarray:
    U, Qy = _c32(U), _c32(Qy)
    topvals = np.ascontiguousarray(topvals, np.float64)
    n, d = U.shape
    kk = topvals.shape[1]
    assert k <= kk
    out = np.zeros((Qy.shape[0], n), np.uint8)
    if n and Qy.shape[0]:
        _load().orc_rkmips_twophase(U, n, d, topvals, kk, Qy, Qy.shape[0], k, out, threads)
    return out.astype(bool)


def linear_scan(u, unorm, q, P_sorted, pnorm_sorted, k: int):
    """Alg. 2, readings R3/R4.  Returns (decision, items scanned)."""
    u = np.ascontiguousarray(u, np.float32).ravel()
    q = np.ascontiguousarray(q, np.float32).ravel()
    P_sorted = _c32(P_sorted)
    pnorm_sorted = np.ascontiguousarray(pnorm_sorted, np.float64)
    sc = ctypes.c_int64(0)
    r = _load().orc_linear_scan(u, float(unorm), q, P_sorted, pnorm_sorted, P_sorted.shape[0], u.size, k,
                                ctypes.byref(sc))
    return bool(r), int(sc.value)


def block_bounds(L, b: int) -> np.ndarray:
    """Eq. (1): per block of b consecutive rows, elementwise min of L."""
    L = np.ascontiguousarray(L, np.float64)
    n, kk = L.shape
    nb = (n + b - 1) // b
    out = np.empty((nb, kk), np.float64)
    if n:
        _load().orc_block_bounds(L, n, kk, b, out)
    return out


def margins(U, P, Qy, pairs, k: int, threads: int = 0) -> np.ndarray:
    """Relative margin (q.u - tau'_k(u)) / (|q||u|) for (query, user) pairs; reading R9."""
    U, P, Qy = _c32(U), _c32(P), _c32(Qy)
    pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
    mu = np.empty(pairs.shape[0], np.float64)
    if pairs.shape[0]:
        _load().orc_margin(U, U.shape[0], P, P.shape[0], U.shape[1], Qy, pairs, pairs.shape[0], k, mu, threads)
    return mu


def margins_from_lists(U, P, Qy, topvals, topids, pairs, k: int, threads: int = 0) -> np.ndarray:
    """Same margins as margins(), from exact top-kk lists (topk(U, P, kk) output, kk > k so that a
    copy of q in the list still leaves k competitors); O(d + kk) per pair (reading R9)."""
    U, P, Qy = _c32(U), _c32(P), _c32(Qy)
    topvals = np.ascontiguousarray(topvals, np.float64)
    topids = np.ascontiguousarray(topids, np.int32)
    assert topvals.shape == topids.shape and topvals.shape[0] == U.shape[0]
    pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
    mu = np.empty(pairs.shape[0], np.float64)
    if pairs.shape[0]:
        _load().orc_margin_lists(U, U.shape[0], P, P.shape[0], U.shape[1], Qy, topvals, topids, topvals.shape[1],
                                 pairs, pairs.shape[0], k, mu, threads)
    return mu


def sets_from_member(member: np.ndarray):
    """member[q, u] -> list of ascending user-id arrays, one per query."""
    return [np.flatnonzero(row).astype(np.int32) for row in member]


def to_csr(member: np.ndarray):
    sets = sets_from_member(member)
    offsets = np.zeros(len(sets) + 1, np.int64)
    offsets[1:] = np.cumsum([s.size for s in sets])
    ids = np.concatenate(sets) if sets else np.zeros(0, np.int32)
    return offsets, ids.astype(np.int32)
