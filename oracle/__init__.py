"""CPU oracle for the IVF-PQ hot-partition search -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package. The product path never does.
It shares no code with paper_2504_08930_b200/.

The arithmetic lives in oracle.c (plain C, fp64, sequential sums,
-ffp-contract=off); this module only compiles and marshals (ctypes).
Pins: tests/test_oracle_pins.py. Every function here is pinned (no
"parity unpinned" entries); see DESIGN.md §Oracle pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]

_lib = None


def build(force: bool = False, extra_flags=()) -> str:
    """Compile oracle.c -> liboracle.so (gcc). Returns the path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *CFLAGS, *extra_flags, "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int32
        L.oracle_coarse.argtypes = [P, ctypes.c_int64, P, I, I, I, P, P, I, I]
        L.oracle_search.argtypes = [P, ctypes.c_int64, I, P, I, P, I, I, P, P, P, P, I, I, P, P, P, P, P, P, I, I, I]
        L.oracle_dist_many.argtypes = [P, I, P, P, I, I, P, P, P, P, ctypes.c_int64, P, I, I, I]
        L.oracle_coarse_dist.argtypes = [P, P, ctypes.c_int32]
        L.oracle_coarse_dist.restype = ctypes.c_double
        L.oracle_adc_dist.argtypes = [P, P, P, P, ctypes.c_int32, ctypes.c_int32]
        L.oracle_adc_dist.restype = ctypes.c_double
        L.oracle_coarse_ip.argtypes = [P, P, ctypes.c_int32]
        L.oracle_coarse_ip.restype = ctypes.c_double
        L.oracle_adc_dist_v.argtypes = [P, P, P, P, I, I, I, I, I]
        L.oracle_adc_dist_v.restype = ctypes.c_double
        for f in (L.oracle_coarse, L.oracle_search, L.oracle_dist_many):
            f.restype = ctypes.c_int
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def _variant(index, metric, by_residual):
    """metric 0 = squared L2, 1 = inner product (reported as -<q, x>);
    by_residual 1 = codes encode x - c_l. Defaults: the index's own."""
    if metric is None:
        metric = int(getattr(index, "metric", 0)) if index is not None else 0
    if by_residual is None:
        by_residual = int(getattr(index, "by_residual", 1)) if index is not None else 1
    return int(metric), int(by_residual)


def _nbits(index) -> int:
    """bits per sub-code (8, or 4 for the packed 4-bit PQ of NEXT-3)."""
    nb = int(getattr(index, "nbits", 8))
    if nb not in (4, 8):
        raise ValueError("nbits must be 4 or 8")
    return nb


def coarse(Q, centroids, nprobe, nthreads=0, metric=0):
    """O2/O3: (probes int32 [nq,nprobe'], fp64 keys [nq,nprobe']): squared L2
    distances (metric 0) or negated inner products (metric 1)."""
    Q = _c(Q, np.float32); C = _c(centroids, np.float32)
    nq, d = Q.shape
    L = C.shape[0]
    npr = min(nprobe, L)
    probes = np.empty((nq, npr), np.int32)
    dist = np.empty((nq, npr), np.float64)
    rc = lib().oracle_coarse(_p(Q), nq, _p(C), L, d, nprobe, _p(probes), _p(dist), int(metric),
                             nthreads or default_threads())
    if rc:
        raise ValueError("oracle_coarse: invalid arguments")
    return probes, dist


def hot_mask(nlist, hot) -> np.ndarray:
    m = np.zeros(nlist, np.uint8)
    if hot is not None and len(hot):
        m[np.asarray(hot, dtype=np.int64)] = 1
    return m


def search(index, Q, nprobe, k, hot=None, nthreads=0, metric=None, by_residual=None):
    """O2-O7. index: datagen.IndexArrays-like. hot=None means all lists hot.
    metric / by_residual default to the index's attributes (0 / 1).
    Returns dict(ids int64 [nq,k], dist f64 [nq,k], miss u8, probes i32,
    kth1 f64 [nq], ncand i64 [nq])."""
    Q = _c(Q, np.float32)
    nq, d = Q.shape
    L = index.nlist
    isht = np.ones(L, np.uint8) if hot is None else hot_mask(L, hot)
    npr = min(nprobe, L)
    C = _c(index.centroids, np.float32)
    Y = _c(index.codebooks, np.float32)
    offs = _c(index.list_offsets, np.int64)
    ids = _c(index.ids, np.int64)
    codes = _c(index.codes, np.uint8)
    out = dict(ids=np.empty((nq, k), np.int64), dist=np.empty((nq, k), np.float64),
               miss=np.empty((nq, npr), np.uint8), probes=np.empty((nq, npr), np.int32),
               kth1=np.empty(nq, np.float64), ncand=np.empty(nq, np.int64))
    rc = lib().oracle_search(_p(Q), nq, d, _p(C), L, _p(Y), index.m, _nbits(index), _p(offs), _p(ids), _p(codes),
                             _p(isht),
                             nprobe, k, _p(out["ids"]), _p(out["dist"]), _p(out["miss"]), _p(out["probes"]),
                             _p(out["kth1"]), _p(out["ncand"]), *_variant(index, metric, by_residual),
                             nthreads or default_threads())
    if rc:
        raise ValueError("oracle_search: invalid arguments")
    return out


class IdMap:
    """id -> (list, position) lookup for dist_ref (host-side bookkeeping)."""

    def __init__(self, index):
        self.order = np.argsort(index.ids, kind="stable")
        self.sorted_ids = index.ids[self.order]
        self.list_of_pos = (np.searchsorted(index.list_offsets, np.arange(index.N), side="right") - 1).astype(np.int32)

    def locate(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        j = np.searchsorted(self.sorted_ids, ids)
        j = np.clip(j, 0, len(self.sorted_ids) - 1)
        ok = self.sorted_ids[j] == ids
        pos = self.order[j]
        return ok, self.list_of_pos[pos], pos


def dist_ref(index, Q, qidx, ids, idmap: IdMap | None = None, nthreads=0, metric=None, by_residual=None):
    """O6 distance of each (query row qidx[i], vector id ids[i]); NaN for unknown ids."""
    idmap = idmap or IdMap(index)
    qidx = _c(qidx, np.int64).reshape(-1)
    ok, lst, pos = idmap.locate(ids)
    out = np.full(len(qidx), np.nan, np.float64)
    sel = np.nonzero(ok)[0]
    if len(sel):
        Q = _c(Q, np.float32)
        tmp = np.empty(len(sel), np.float64)
        lib().oracle_dist_many(_p(Q), index.d, _p(_c(index.centroids, np.float32)), _p(_c(index.codebooks, np.float32)),
                               index.m, _nbits(index), _p(_c(index.codes, np.uint8)), _p(_c(qidx[sel], np.int64)),
                               _p(_c(lst[sel], np.int32)), _p(_c(pos[sel], np.int64)), len(sel), _p(tmp),
                               *_variant(index, metric, by_residual), nthreads or default_threads())
        out[sel] = tmp
    return out


def num_threads() -> int:
    return int(lib().oracle_num_threads())
