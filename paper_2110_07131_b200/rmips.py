"""Thin ctypes binding of the C ABI in include/rmips.h (argument marshalling only).

Every step of the path runs in librmips.so's CUDA kernels; PyTorch is used here only for
device memory and streams.  There is NO CPU fallback: if librmips.so is missing or cannot be
loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMIPS_LIB") or os.path.join(_HERE, "librmips.so")  # RMIPS_LIB: dev-only profiling build

RMIPS_OK, RMIPS_ERR_INVALID, RMIPS_ERR_NONFINITE, RMIPS_ERR_K_RANGE, RMIPS_ERR_CAPACITY, RMIPS_ERR_CUDA, \
    RMIPS_ERR_OOM = range(7)
RMIPS_FLAG_NONE = 0
RMIPS_FLAG_NO_BLOCKS = 1
RMIPS_FLAG_VERIFY_SCAN = 2
RMIPS_FLAG_FORCE_VERIFY = 4
RMIPS_FLAG_SIMT = 8
RMIPS_FLAG_TIMING = 16
RMIPS_FLAG_NO_EXTEND = 32
RMIPS_FLAG_KEY_SORT = 64
RMIPS_BUILD_DEFAULT = 0
RMIPS_BUILD_SIMT = 1
RMIPS_BUILD_TIMING = 2

EXPORTED = ["rmips_build_index", "rmips_build_index_ex", "rmips_build_index_pprime", "rmips_build_index_host", "rmips_query", "rmips_query_ex",
            "rmips_query_host", "rmips_query_batches", "rmips_query_batches_host", "rmips_query_stats", "rmips_phase_times", "rmips_index_info", "rmips_index_export", "rmips_free_index",
            "rmips_status_string", "rmips_last_error", "rmips_version"]


class RmipsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (status, msg))
        self.status = status


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "queries", "block_query_pairs", "block_query_pruned", "pairs_scored", "pairs_rejected",
        "pairs_accepted_fast", "pairs_undecided", "pairs_exact_accepted", "scans", "items_scanned",
        "result_total", "filter_kernel", "tiles_scored", "scan_exact")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError("librmips.so not built (run `python -c 'import __graft_entry__ as g; g.build()'`); "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, VP = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    pidx = ctypes.POINTER(ctypes.c_void_p)
    lib.rmips_build_index.argtypes = [P, I64, P, I64, I32, I32, VP, pidx]
    lib.rmips_build_index_ex.argtypes = [P, I64, P, I64, I32, I32, I32, VP, pidx]
    lib.rmips_build_index_pprime.argtypes = [P, I64, P, I64, I32, I32, I64, I32, VP, pidx]
    lib.rmips_build_index_host.argtypes = [P, I64, P, I64, I32, I32, VP, pidx]
    lib.rmips_query.argtypes = [VP, P, I32, I32, P, P, I64, ctypes.POINTER(I64), VP]
    lib.rmips_query_ex.argtypes = [VP, P, I32, I32, I32, P, P, I64, ctypes.POINTER(I64), VP]
    lib.rmips_query_host.argtypes = [VP, P, I32, I32, P, P, I64, ctypes.POINTER(I64), VP]
    lib.rmips_query_batches.argtypes = [VP, P, I64, I32, I32, I32, P, P, I64, ctypes.POINTER(I64), VP]
    lib.rmips_query_batches_host.argtypes = [VP, P, I64, I32, I32, P, P, I64, ctypes.POINTER(I64), VP]
    lib.rmips_query_stats.argtypes = [VP, ctypes.POINTER(Stats)]
    lib.rmips_index_info.argtypes = [VP, ctypes.POINTER(I64)]
    lib.rmips_phase_times.argtypes = [VP, ctypes.POINTER(ctypes.c_double)]
    lib.rmips_index_export.argtypes = [VP, P, P, P, P]
    lib.rmips_free_index.argtypes = [VP]
    lib.rmips_free_index.restype = None
    for f in ("rmips_status_string", "rmips_last_error", "rmips_version"):
        getattr(lib, f).restype = ctypes.c_char_p
    lib.rmips_status_string.argtypes = [ctypes.c_int]
    for f in ("rmips_build_index", "rmips_build_index_ex", "rmips_build_index_pprime", "rmips_build_index_host",
              "rmips_query",
              "rmips_query_ex", "rmips_query_host", "rmips_query_batches", "rmips_query_batches_host", "rmips_query_stats",
              "rmips_phase_times", "rmips_index_info", "rmips_index_export"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


lib = _load()


def _check(status: int):
    if status != RMIPS_OK:
        raise RmipsError(status, "%s (%s)" % (lib.rmips_status_string(status).decode(),
                                              lib.rmips_last_error().decode()))


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev_f32(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError("expected a CUDA tensor")
    if t.dtype != torch.float32 or not t.is_contiguous() or t.dim() != 2:
        raise TypeError("expected a contiguous 2-D float32 tensor")
    return t


class Index:
    """Owning handle of an rmips index (freed on close() / garbage collection)."""

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)
        info = (ctypes.c_int64 * 16)()
        _check(lib.rmips_index_info(self.handle, info))
        self.n, self.m, self.d, self.k_max, self.d_pad, self.block_size, self.overflow_rows, self.build_flags, \
            self.cand_total, self.tiles_done, self.m_prime, self.build_kernel, self.cand_slots = \
            [int(v) for v in info[:13]]

    def close(self):
        if self.handle:
            lib.rmips_free_index(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def refresh_info(self):
        """Re-read the index header (k_max grows when a query with k > k_max extended the index)."""
        info = (ctypes.c_int64 * 16)()
        _check(lib.rmips_index_info(self.handle, info))
        self.k_max = int(info[3])

    def export(self):
        """(perm_u, perm_p, tau [k_max, n] fp64, ids [k_max, n] int32), users in ORIGINAL order."""
        self.refresh_info()
        pu = np.empty(self.n, np.int64)
        pp = np.empty(self.m, np.int64)
        tau = np.empty((self.k_max, self.n), np.float64)
        ids = np.empty((self.k_max, self.n), np.int32)
        _check(lib.rmips_index_export(self.handle, pu.ctypes.data if self.n else None, pp.ctypes.data,
                                      tau.ctypes.data if self.n else None, ids.ctypes.data if self.n else None))
        return pu, pp, tau, ids

    def phase_times(self):
        """Per-phase CUDA-event times (ms) of the last timed build / query, see rmips_phase_times."""
        ms = (ctypes.c_double * 16)()
        _check(lib.rmips_phase_times(self.handle, ms))
        return list(ms)

    def stats(self) -> dict:
        s = Stats()
        _check(lib.rmips_query_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()


def rmips_build_index(Q, P, k_max: int, build_flags: int = RMIPS_BUILD_DEFAULT, stream=None) -> Index:
    """Build an index from device tensors Q [n, d] and P [m, d] (float32, contiguous)."""
    P = _dev_f32(P)
    n = int(Q.shape[0]) if Q is not None else 0
    qptr = _dev_f32(Q).data_ptr() if n else None
    h = ctypes.c_void_p()
    _check(lib.rmips_build_index_ex(qptr, n, P.data_ptr(), int(P.shape[0]), int(P.shape[1]), int(k_max),
                                    int(build_flags), _stream_ptr(stream), ctypes.byref(h)))
    return Index(h.value)


def rmips_build_index_pprime(Q, P, k_max: int, m_prime: int, build_flags: int = RMIPS_BUILD_DEFAULT,
                             stream=None) -> Index:
    """Alg. 1 as printed: lists over the first m_prime norm-sorted items (P'); queries then
    decide by Lemmas 1-2 and the scan after P' (include/rmips.h)."""
    P = _dev_f32(P)
    n = int(Q.shape[0]) if Q is not None else 0
    qptr = _dev_f32(Q).data_ptr() if n else None
    h = ctypes.c_void_p()
    _check(lib.rmips_build_index_pprime(qptr, n, P.data_ptr(), int(P.shape[0]), int(P.shape[1]), int(k_max),
                                        int(m_prime), int(build_flags), _stream_ptr(stream), ctypes.byref(h)))
    return Index(h.value)


def rmips_build_index_host(Q: np.ndarray, P: np.ndarray, k_max: int, stream=None) -> Index:
    """Same as rmips_build_index with host (numpy, or pinned CPU torch) inputs."""
    Q = _host_f32(Q)
    P = _host_f32(P)
    n = Q.shape[0]
    h = ctypes.c_void_p()
    _check(lib.rmips_build_index_host(_hptr(Q) if n else None, n, _hptr(P), P.shape[0], P.shape[1], int(k_max),
                                      _stream_ptr(stream), ctypes.byref(h)))
    return Index(h.value)


def _host_f32(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            assert not a.is_cuda and a.dtype == torch.float32 and a.is_contiguous()
            return a
    except ImportError:
        pass
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim != 2:
        raise TypeError("expected a 2-D array")
    return a


def _hptr(a):
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def rmips_query(index: Index, q_batch, k: int, flags: int = RMIPS_FLAG_NONE, capacity: Optional[int] = None,
                stream=None) -> Tuple["object", "object"]:
    """Reverse k-MIPS for a device batch q_batch [b, d].  Returns (offsets int64 [b+1], user_ids int32 [total])
    as CUDA tensors; query i's users (original ids, ascending) are user_ids[offsets[i]:offsets[i+1]]."""
    import torch
    q_batch = _dev_f32(q_batch)
    b = int(q_batch.shape[0])
    dev = q_batch.device
    offsets = torch.empty(b + 1, dtype=torch.int64, device=dev)
    cap = int(capacity) if capacity is not None else max(1 << 16, 64 * b)
    total = ctypes.c_int64(0)
    for _ in range(2):
        ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        st = lib.rmips_query_ex(index.handle, q_batch.data_ptr() if b else None, b, int(k), int(flags),
                                offsets.data_ptr(), ids.data_ptr(), cap, ctypes.byref(total), _stream_ptr(stream))
        if st == RMIPS_ERR_CAPACITY and capacity is None:
            cap = int(total.value)
            continue
        _check(st)
        break
    return offsets, ids[: total.value]


def rmips_query_batches(index: Index, q_all, batch: int, k: int, flags: int = RMIPS_FLAG_NONE,
                        capacity: Optional[int] = None, stream=None) -> Tuple["object", "object"]:
    """q_all [nq, d] (device) answered in consecutive batches of `batch`, one host sync in total.
    Returns (offsets int64 [nq+1], user_ids int32 [total]) as CUDA tensors, as rmips_query."""
    import torch
    q_all = _dev_f32(q_all)
    nq = int(q_all.shape[0])
    dev = q_all.device
    offsets = torch.empty(nq + 1, dtype=torch.int64, device=dev)
    cap = int(capacity) if capacity is not None else max(1 << 16, 64 * nq)
    total = ctypes.c_int64(0)
    for _ in range(2):
        ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        st = lib.rmips_query_batches(index.handle, q_all.data_ptr() if nq else None, nq, int(batch), int(k),
                                     int(flags), offsets.data_ptr(), ids.data_ptr(), cap, ctypes.byref(total),
                                     _stream_ptr(stream))
        if st == RMIPS_ERR_CAPACITY and capacity is None:
            cap = int(total.value)
            continue
        _check(st)
        break
    return offsets, ids[: total.value]


def rmips_query_batches_host(index: Index, q_all, batch: int, k: int, capacity: Optional[int] = None,
                             out_offsets=None, out_ids=None, stream=None):
    """Host-buffer variant of rmips_query_batches (one copy each way inside the call)."""
    q_all = _host_f32(q_all)
    nq = q_all.shape[0]
    offsets = out_offsets if out_offsets is not None else np.empty(nq + 1, np.int64)
    cap = int(capacity) if capacity is not None else max(1 << 16, 64 * nq)
    total = ctypes.c_int64(0)
    for _ in range(2):
        ids = out_ids if (out_ids is not None and _numel(out_ids) >= cap) else np.empty(max(cap, 1), np.int32)
        st = lib.rmips_query_batches_host(index.handle, _hptr(q_all) if nq else None, nq, int(batch), int(k),
                                          _hptr(offsets), _hptr(ids), cap, ctypes.byref(total), _stream_ptr(stream))
        if st == RMIPS_ERR_CAPACITY and capacity is None:
            cap = int(total.value)
            continue
        _check(st)
        break
    return offsets, ids[: total.value]


def rmips_query_host(index: Index, q_batch, k: int, capacity: Optional[int] = None, out_offsets=None,
                     out_ids=None, stream=None):
    """Host-buffer variant: q_batch, offsets and ids live in host memory (copies inside the call)."""
    q_batch = _host_f32(q_batch)
    b = q_batch.shape[0]
    offsets = out_offsets if out_offsets is not None else np.empty(b + 1, np.int64)
    cap = int(capacity) if capacity is not None else max(1 << 16, 64 * b)
    total = ctypes.c_int64(0)
    for _ in range(2):
        ids = out_ids if (out_ids is not None and _numel(out_ids) >= cap) else np.empty(max(cap, 1), np.int32)
        st = lib.rmips_query_host(index.handle, _hptr(q_batch) if b else None, b, int(k), _hptr(offsets),
                                  _hptr(ids), cap, ctypes.byref(total), _stream_ptr(stream))
        if st == RMIPS_ERR_CAPACITY and capacity is None:
            cap = int(total.value)
            continue
        _check(st)
        break
    return offsets, ids[: total.value]


def _numel(a):
    return a.numel() if hasattr(a, "numel") else a.size


def split_sets(offsets, ids):
    """(offsets, ids) -> list of numpy arrays, one ascending user-id array per query."""
    if hasattr(offsets, "cpu"):
        offsets = offsets.cpu().numpy()
        ids = ids.cpu().numpy()
    return [ids[offsets[i]:offsets[i + 1]] for i in range(len(offsets) - 1)]
