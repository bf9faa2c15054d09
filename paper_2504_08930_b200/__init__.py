"""paper_2504_08930_b200 -- B200-native IVF-PQ hot-partition search.

Thin Python binding (ctypes, argument marshalling only) over libvlr.so, whose
C ABI is declared in include/vlr.h. Every step of search runs in the
library's sm_100a kernels; there is no CPU or PyTorch fallback: if libvlr.so
is missing or the device is unusable, these calls raise.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvlr.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "DIM_MISMATCH", 3: "NONFINITE", 4: "UNKNOWN_CLUSTER",
          5: "DUPLICATE_ID", 6: "OOM", 7: "CUDA", 8: "NCCL", 9: "UNSUPPORTED"}

# every symbol include/vlr.h declares (checked by tests/test_abi.py)
EXPORTS = ["vlr_load_index", "vlr_search_async", "vlr_search", "vlr_search_host", "vlr_search_host_async",
           "vlr_search_release_async", "vlr_coarse_stage1", "vlr_coarse_stage2", "vlr_search_stage3",
           "vlr_poll_ready", "vlr_wait_ready", "vlr_merge_ready", "vlr_p2p_export", "vlr_p2p_connect",
           "vlr_p2p_setup", "vlr_reserve", "vlr_set_pipeline", "vlr_deal_owners", "vlr_update_hot",
           "vlr_merge_partials", "vlr_access_counts", "vlr_index_info", "vlr_index_owners", "vlr_set_profiling", "vlr_stage_times",
           "vlr_last_launch_count", "vlr_nccl_unique_id", "vlr_index_free", "vlr_last_error", "vlr_version"]


class VlrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"vlr {self.name}: {msg}")


class _Desc(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("nlist", ctypes.c_int32), ("m", ctypes.c_int32), ("nbits", ctypes.c_int32),
                ("metric", ctypes.c_int32), ("by_residual", ctypes.c_int32),
                ("centroids", ctypes.c_void_p), ("codebooks", ctypes.c_void_p), ("list_offsets", ctypes.c_void_p),
                ("ids", ctypes.c_void_p), ("codes", ctypes.c_void_p), ("hot", ctypes.c_void_p),
                ("n_hot", ctypes.c_int32), ("hot_owner", ctypes.c_void_p)]


class _Comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libvlr.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2504_08930_b200.build` "
                              "(there is no CPU fallback for the search path)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        sig = {
            "vlr_load_index": [P, P, P],
            "vlr_search_async": [P, P, I32, I32, I32, P, P, P, P, P],
            "vlr_search": [P, P, I32, I32, I32, P, P, P, P, P],
            "vlr_search_host": [P, P, I32, I32, I32, P, P, P, P, P],
            "vlr_search_host_async": [P, P, I32, I32, I32, P, P, P, P, P],
            "vlr_search_release_async": [P, P, I32, I32, I32, P, P, P, P, P, ctypes.c_uint32, P],
            "vlr_coarse_stage1": [P, P, I32, I32, P, P],
            "vlr_p2p_export": [P, P],
            "vlr_p2p_connect": [P, P],
            "vlr_p2p_setup": [P],
            "vlr_coarse_stage2": [P, P, I32, I32, P, P, P],
            "vlr_search_stage3": [P, P, I32, I32, I32, P, P, P, P, P, P],
            "vlr_reserve": [P, I32, I32, I32],
            "vlr_set_pipeline": [P, I32, I32],
            "vlr_deal_owners": [P, I32, P, P, I32, I32, P],
            "vlr_update_hot": [P, P],
            "vlr_merge_partials": [P, P, I32, I32, I32, P, P, P],
            "vlr_index_info": [P, P, P, P],
            "vlr_access_counts": [P, P, I64, P, P],
            "vlr_index_owners": [P, P],
            "vlr_set_profiling": [P, I32],
            "vlr_stage_times": [P, I32, P, I32],
            "vlr_nccl_unique_id": [P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.vlr_poll_ready.argtypes = [P, I32, ctypes.c_uint32, P, P, P, I32, I64]
        L.vlr_poll_ready.restype = I32
        L.vlr_wait_ready.argtypes = [P, I32, ctypes.c_uint32, P, I64]
        L.vlr_wait_ready.restype = I32
        L.vlr_merge_ready.argtypes = [I32, P, ctypes.c_uint32, I32, I32, P, P, P, P, P, I64]
        L.vlr_merge_ready.restype = I32
        L.vlr_last_launch_count.argtypes = [P]
        L.vlr_last_launch_count.restype = I32
        L.vlr_index_free.argtypes = [P]
        L.vlr_index_free.restype = None
        L.vlr_last_error.restype = ctypes.c_char_p
        L.vlr_version.restype = I32
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise VlrError(st, lib().vlr_last_error().decode(errors="replace"))


def _host(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().vlr_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class Index:
    """A device-resident hot shard (vlr_index*)."""

    def __init__(self, handle, d, nlist, rank, world, device):
        self._h = handle
        self.d, self.nlist, self.rank, self.world, self.device = d, nlist, rank, world, device

    @classmethod
    def load(cls, centroids, codebooks, list_offsets, ids, codes, hot=None, hot_owner=None, *, rank=0, world=1,
             device=None, nccl_id: bytes | None = None, nbits=8, metric=0, by_residual=1):
        """vlr_load_index. hot=None means every cluster is resident."""
        C = _host(centroids, np.float32)
        Y = _host(codebooks, np.float32)
        offs = _host(list_offsets, np.int64)
        idv = _host(ids, np.int64)
        cd = _host(codes, np.uint8)
        nlist, d = C.shape
        m = Y.shape[0] if Y.ndim == 3 else int(cd.shape[1])
        hotv = np.arange(nlist, dtype=np.int32) if hot is None else _host(hot, np.int32).reshape(-1)
        own = None if hot_owner is None else _host(hot_owner, np.int32).reshape(-1)
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        desc = _Desc(d, nlist, m, nbits, metric, by_residual, _ptr(C), _ptr(Y), _ptr(offs), _ptr(idv), _ptr(cd),
                     _ptr(hotv), int(hotv.size), _ptr(own))
        uid = None
        if nccl_id is not None:
            uid = ctypes.create_string_buffer(bytes(nccl_id), 128)
        comm = _Comm(rank, world, device, ctypes.cast(uid, ctypes.c_void_p) if uid is not None else None)
        h = ctypes.c_void_p()
        _check(lib().vlr_load_index(ctypes.byref(desc), ctypes.byref(comm), ctypes.byref(h)))
        return cls(h, d, nlist, rank, world, device)

    def update_hot(self, centroids, codebooks, list_offsets, ids, codes, hot=None, hot_owner=None, *, nbits=8,
                   metric=0, by_residual=1):
        """vlr_update_hot (NEXT-2 shard refresh): rebuild the resident lists for
        a new hot set while the current residency keeps serving."""
        C = _host(centroids, np.float32)
        Y = _host(codebooks, np.float32)
        offs = _host(list_offsets, np.int64)
        idv = _host(ids, np.int64)
        cd = _host(codes, np.uint8)
        nlist, d = C.shape
        m = Y.shape[0] if Y.ndim == 3 else int(cd.shape[1])
        hotv = np.arange(nlist, dtype=np.int32) if hot is None else _host(hot, np.int32).reshape(-1)
        own = None if hot_owner is None else _host(hot_owner, np.int32).reshape(-1)
        desc = _Desc(d, nlist, m, nbits, metric, by_residual, _ptr(C), _ptr(Y), _ptr(offs), _ptr(idv), _ptr(cd),
                     _ptr(hotv), int(hotv.size), _ptr(own))
        _check(lib().vlr_update_hot(self._h, ctypes.byref(desc)))

    def update_hot_arrays(self, ix, hot=None, hot_owner=None):
        self.update_hot(ix.centroids, ix.codebooks, ix.list_offsets, ix.ids, ix.codes, hot=hot, hot_owner=hot_owner,
                        nbits=int(getattr(ix, "nbits", 8)), metric=int(getattr(ix, "metric", 0)),
                        by_residual=int(getattr(ix, "by_residual", 1)))

    @classmethod
    def from_arrays(cls, ix, hot=None, **kw):
        """Load from a datagen.IndexArrays-like object (its metric / by_residual
        attributes, when present, select the variant)."""
        kw.setdefault("metric", int(getattr(ix, "metric", 0)))
        kw.setdefault("by_residual", int(getattr(ix, "by_residual", 1)))
        kw.setdefault("nbits", int(getattr(ix, "nbits", 8)))
        return cls.load(ix.centroids, ix.codebooks, ix.list_offsets, ix.ids, ix.codes, hot=hot, **kw)

    # ------------------------------------------------------------------ search
    def search(self, Q, nprobe: int, k: int, out=None, stream=None, sync=False, probes=True):
        """Q: torch float32 CUDA tensor [nq, d]. Returns (ids, dist, miss, probes)
        torch CUDA tensors; stream-ordered on `stream` (default: current)."""
        import torch
        assert Q.is_cuda and Q.dtype == torch.float32 and Q.is_contiguous()
        nq = int(Q.shape[0])
        npr = min(nprobe, self.nlist)
        if out is None:
            dev = Q.device
            out = (torch.empty(nq, k, dtype=torch.int64, device=dev), torch.empty(nq, k, dtype=torch.float32, device=dev),
                   torch.empty(nq, npr, dtype=torch.uint8, device=dev),
                   torch.empty(nq, npr, dtype=torch.int32, device=dev) if probes else None)
        ids, dist, miss, prb = out
        fn = lib().vlr_search if sync else lib().vlr_search_async
        _check(fn(self._h, Q.data_ptr(), nq, nprobe, k, ids.data_ptr(), dist.data_ptr(), miss.data_ptr(),
                  prb.data_ptr() if prb is not None else None, _stream_handle(stream)))
        return out

    # ------------------------------------------------------------------ staged (caller-exchanged) search
    def coarse_stage1(self, Q, nprobe: int, stream=None):
        """vlr_coarse_stage1 -> x1: float32 CUDA [nq, nprobe'] (this rank's
        nprobe' smallest filter group minima)."""
        import torch
        assert Q.is_cuda and Q.dtype == torch.float32 and Q.is_contiguous()
        nq, npr = int(Q.shape[0]), min(nprobe, self.nlist)
        x1 = torch.empty(nq, npr, dtype=torch.float32, device=Q.device)
        _check(lib().vlr_coarse_stage1(self._h, Q.data_ptr(), nq, nprobe, x1.data_ptr(), _stream_handle(stream)))
        return x1

    def coarse_stage2(self, Q, nprobe: int, x1_all, stream=None):
        """vlr_coarse_stage2(x1_all [world, nq, nprobe'] float32 CUDA) -> x2:
        int64 CUDA [nq, nprobe', 2] (16-byte {double D; int32 l; int32 pad}
        entries: this rank's sorted exact top-nprobe')."""
        import torch
        nq, npr = int(Q.shape[0]), min(nprobe, self.nlist)
        x1_all = x1_all.contiguous()
        x2 = torch.empty(nq, npr, 2, dtype=torch.int64, device=Q.device)
        _check(lib().vlr_coarse_stage2(self._h, Q.data_ptr(), nq, nprobe, x1_all.data_ptr(), x2.data_ptr(),
                                       _stream_handle(stream)))
        return x2

    def search_stage3(self, Q, nprobe: int, k: int, x2_all, out=None, stream=None):
        """vlr_search_stage3(x2_all [world, nq, nprobe', 2] int64 CUDA) ->
        (ids, dist, miss, probes): global probes / mask, THIS shard's partial top-k."""
        import torch
        nq, npr = int(Q.shape[0]), min(nprobe, self.nlist)
        if out is None:
            dev = Q.device
            out = (torch.empty(nq, k, dtype=torch.int64, device=dev), torch.empty(nq, k, dtype=torch.float32, device=dev),
                   torch.empty(nq, npr, dtype=torch.uint8, device=dev), torch.empty(nq, npr, dtype=torch.int32, device=dev))
        ids, dist, miss, prb = out
        x2_all = x2_all.contiguous()
        _check(lib().vlr_search_stage3(self._h, Q.data_ptr(), nq, nprobe, k, x2_all.data_ptr(), ids.data_ptr(),
                                       dist.data_ptr(), miss.data_ptr(), prb.data_ptr() if prb is not None else None,
                                       _stream_handle(stream)))
        return out

    def search_staged(self, Q, nprobe: int, k: int, allgather, stream=None, out=None):
        """The sharded collective search with a caller-supplied transport:
        allgather(t) must return the rank-ordered stack [world, *t.shape] of
        every rank's t (a CUDA tensor), e.g. over torch.distributed. Returns
        (ids, dist, miss, probes) with this shard's PARTIAL top-k (merge the
        gathered partials with merge_partials)."""
        x1 = self.coarse_stage1(Q, nprobe, stream=stream)
        x2 = self.coarse_stage2(Q, nprobe, allgather(x1), stream=stream)
        return self.search_stage3(Q, nprobe, k, allgather(x2), out=out, stream=stream)

    def search_release(self, Q, nprobe: int, k: int, stream=None, on_ready=None, timeout_s: float = 30.0,
                       out=None):
        """NEXT-4 early per-query release (vlr_search_release_async +
        vlr_poll_ready): rows are written to pinned host memory and released
        one query at a time while the batch is still being scanned.
        on_ready(qs: np.ndarray) is called for each group of newly released
        queries (their rows of the returned ids/dist are final by then).
        Returns (ids, dist, miss, probes, t_ready_ns) with ids/dist pinned CPU
        tensors, miss/probes CUDA tensors, and t_ready_ns[q] the host
        CLOCK_MONOTONIC time (ns) at which query q was seen released; t0
        (time.monotonic_ns() just before the launch) is t_ready_ns.t0."""
        import time
        import torch
        assert Q.is_cuda and Q.dtype == torch.float32 and Q.is_contiguous()
        nq = int(Q.shape[0])
        npr = min(nprobe, self.nlist)
        if out is None:
            out = (torch.empty(nq, k, dtype=torch.int64, pin_memory=True),
                   torch.empty(nq, k, dtype=torch.float32, pin_memory=True),
                   torch.empty(nq, npr, dtype=torch.uint8, device=Q.device),
                   torch.empty(nq, npr, dtype=torch.int32, device=Q.device),
                   torch.zeros(nq, dtype=torch.int32, pin_memory=True))
        ids, dist, miss, prb, ready = out
        self._epoch = (getattr(self, "_epoch", 0) % 0x7FFFFFFF) + 1
        seen = np.zeros(nq, np.uint8)
        qs = np.empty(nq, np.int32)
        ts = np.empty(nq, np.int64)
        t_ready = np.zeros(nq, np.int64)
        t0 = time.monotonic_ns()
        _check(lib().vlr_search_release_async(self._h, Q.data_ptr(), nq, nprobe, k, ids.data_ptr(), dist.data_ptr(),
                                              miss.data_ptr(), prb.data_ptr(), ready.data_ptr(), self._epoch,
                                              _stream_handle(stream)))
        got = 0
        deadline = t0 + int(timeout_s * 1e9)
        if on_ready is None:  # native dispatcher loop (no per-query Python work while the batch runs)
            got = lib().vlr_wait_ready(ready.data_ptr(), nq, self._epoch, t_ready.ctypes.data, int(timeout_s * 1e6))
            if got < nq:
                raise VlrError(7, f"search_release: {nq - max(got, 0)} queries not released within {timeout_s} s")
        while got < nq:
            n = lib().vlr_poll_ready(ready.data_ptr(), nq, self._epoch, seen.ctypes.data, qs.ctypes.data,
                                     ts.ctypes.data, nq, 100_000)
            if n < 0:
                raise VlrError(1, "vlr_poll_ready: bad arguments")
            if n:
                t_ready[qs[:n]] = ts[:n]
                got += n
                if on_ready is not None:
                    on_ready(qs[:n].copy())
            elif time.monotonic_ns() > deadline:
                raise VlrError(7, f"search_release: {nq - got} queries not released within {timeout_s} s")
        t_ready = _Stamps(t_ready)
        t_ready.t0 = t0
        return ids, dist, miss, prb, t_ready

    def search_release_launch(self, Q, nprobe: int, k: int, stream=None):
        """vlr_search_release_async without waiting: returns (ids, dist, miss,
        probes, ready, epoch) with ids/dist/ready pinned CPU tensors (the rows
        and flags the dispatcher reads; on a sharded handle: THIS shard's
        partial rows, merged across shards with merge_ready)."""
        import torch
        assert Q.is_cuda and Q.dtype == torch.float32 and Q.is_contiguous()
        nq, npr = int(Q.shape[0]), min(nprobe, self.nlist)
        ids = torch.empty(nq, k, dtype=torch.int64, pin_memory=True)
        dist = torch.empty(nq, k, dtype=torch.float32, pin_memory=True)
        miss = torch.empty(nq, npr, dtype=torch.uint8, device=Q.device)
        prb = torch.empty(nq, npr, dtype=torch.int32, device=Q.device)
        ready = torch.zeros(nq, dtype=torch.int32, pin_memory=True)
        self._epoch = (getattr(self, "_epoch", 0) % 0x7FFFFFFF) + 1
        _check(lib().vlr_search_release_async(self._h, Q.data_ptr(), nq, nprobe, k, ids.data_ptr(), dist.data_ptr(),
                                              miss.data_ptr(), prb.data_ptr(), ready.data_ptr(), self._epoch,
                                              _stream_handle(stream)))
        return ids, dist, miss, prb, ready, self._epoch

    def search_host(self, Q: np.ndarray, nprobe: int, k: int, out=None, stream=None):
        """vlr_search_host: host buffers in and out (copies inside the call)."""
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        nq = Q.shape[0]
        npr = min(nprobe, self.nlist)
        if out is None:
            out = (np.empty((nq, k), np.int64), np.empty((nq, k), np.float32), np.empty((nq, npr), np.uint8),
                   np.empty((nq, npr), np.int32))
        ids, dist, miss, prb = out
        _check(lib().vlr_search_host(self._h, Q.ctypes.data, nq, nprobe, k, ids.ctypes.data, dist.ctypes.data,
                                     miss.ctypes.data, prb.ctypes.data if prb is not None else None,
                                     _stream_handle(stream)))
        return out

    def search_host_ptr(self, q_ptr: int, nq: int, nprobe: int, k: int, ids_ptr: int, dist_ptr: int, miss_ptr: int,
                        probes_ptr: int | None, stream=None):
        """vlr_search_host on raw (e.g. pinned torch) host pointers."""
        _check(lib().vlr_search_host(self._h, q_ptr, nq, nprobe, k, ids_ptr, dist_ptr, miss_ptr, probes_ptr,
                                     _stream_handle(stream)))

    def search_host_ptr_async(self, q_ptr: int, nq: int, nprobe: int, k: int, ids_ptr: int, dist_ptr: int,
                              miss_ptr: int, probes_ptr: int | None, stream=None):
        """vlr_search_host_async on raw pinned host pointers (no synchronisation)."""
        _check(lib().vlr_search_host_async(self._h, q_ptr, nq, nprobe, k, ids_ptr, dist_ptr, miss_ptr, probes_ptr,
                                           _stream_handle(stream)))

    def p2p_export(self) -> bytes:
        """vlr_p2p_export: allocate this rank's inbox (after reserve) -> its 64-byte IPC handle."""
        buf = ctypes.create_string_buffer(64)
        _check(lib().vlr_p2p_export(self._h, ctypes.cast(buf, ctypes.c_void_p)))
        return buf.raw

    def p2p_connect(self, handles):
        """vlr_p2p_connect: every rank's handle in rank order; searches become collective."""
        blob = b"".join(bytes(hh) for hh in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib().vlr_p2p_connect(self._h, ctypes.cast(buf, ctypes.c_void_p)))

    def p2p_setup(self):
        """vlr_p2p_setup: export + NCCL all-gather of the handles + connect (collective)."""
        _check(lib().vlr_p2p_setup(self._h))

    def reserve(self, max_nq: int, max_nprobe: int, max_k: int):
        _check(lib().vlr_reserve(self._h, max_nq, max_nprobe, max_k))

    def set_pipeline(self, slots: int = 2, scan_reserve_sms: int = 0):
        """vlr_set_pipeline: workspace slots for searches in flight on different streams, and the SMs
        the scan leaves to the other stream's coarse stage."""
        _check(lib().vlr_set_pipeline(self._h, slots, scan_reserve_sms))

    def access_counts(self, probes, counts=None, stream=None):
        """vlr_access_counts: accumulate per-cluster probe counts (torch int32
        CUDA probes of any shape) into an int64 [nlist] CUDA tensor."""
        import torch
        if counts is None:
            counts = torch.zeros(self.nlist, dtype=torch.int64, device=probes.device)
        _check(lib().vlr_access_counts(self._h, probes.data_ptr(), probes.numel(), counts.data_ptr(),
                                       _stream_handle(stream)))
        return counts

    # ------------------------------------------------------------------ info
    def info(self):
        b, n, v = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
        _check(lib().vlr_index_info(self._h, ctypes.byref(b), ctypes.byref(n), ctypes.byref(v)))
        return dict(bytes_on_device=b.value, n_owned_lists=n.value, n_owned_vectors=v.value)

    def owners(self) -> np.ndarray:
        out = np.empty(self.nlist, np.int32)
        _check(lib().vlr_index_owners(self._h, out.ctypes.data))
        return out

    def set_profiling(self, enable=True):
        """True/1: events at every stage boundary; 2: only around the scan; False/0: off."""
        mode = int(enable) if not isinstance(enable, bool) else (1 if enable else 0)
        _check(lib().vlr_set_profiling(self._h, mode))

    STAGES = ["coarse_filter", "select", "refine", "route", "lut", "scan", "rank_merge", "exchange_merge"]

    def stage_times(self, back: int = 0) -> dict:
        """Per-stage ms of the search `back` searches ago (0 = last)."""
        ms = np.zeros(8, np.float32)
        _check(lib().vlr_stage_times(self._h, back, ms.ctypes.data, 8))
        return dict(zip(self.STAGES, ms.tolist()))

    @property
    def last_launch_count(self) -> int:
        return int(lib().vlr_last_launch_count(self._h))

    def close(self):
        if self._h:
            lib().vlr_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Stamps(np.ndarray):
    """int64 ndarray of release times with the launch time as .t0"""

    def __new__(cls, a):
        return np.asarray(a).view(cls)

    def __array_finalize__(self, obj):
        self.t0 = getattr(obj, "t0", 0)


def deal_owners(list_offsets, hot, world: int, counts=None) -> np.ndarray:
    """vlr_deal_owners: owner rank per hot list -- the paper's size-descending
    round-robin (counts=None) or the traffic-aware LPT deal (counts =
    per-cluster access counts, NEXT-2)."""
    offs = _host(list_offsets, np.int64)
    hotv = _host(hot, np.int32).reshape(-1)
    cnt = None if counts is None else _host(counts, np.int64).reshape(-1)
    out = np.empty(hotv.size, np.int32)
    _check(lib().vlr_deal_owners(offs.ctypes.data, int(offs.size - 1), cnt.ctypes.data if cnt is not None else None,
                                 _ptr(hotv), int(hotv.size), int(world), _ptr(out)))
    return out


def merge_ready(readys, epochs, part_ids, part_dist, timeout_s: float = 30.0):
    """vlr_merge_ready: the cross-shard dispatcher merge of released partial
    rows (pinned CPU tensors from search_release_launch on each shard; every
    shard's flags must use one epoch). Returns (ids, dist, t_merged_ns)."""
    import torch
    S = len(readys)
    assert len(set(int(e) for e in epochs)) == 1, "one epoch for every shard"
    nq, k = part_ids[0].shape
    P = ctypes.c_void_p
    rr = (P * S)(*[r.data_ptr() for r in readys])
    pi = (P * S)(*[t.data_ptr() for t in part_ids])
    pd = (P * S)(*[t.data_ptr() for t in part_dist])
    ids = np.empty((nq, k), np.int64)
    dist = np.empty((nq, k), np.float32)
    t = np.zeros(nq, np.int64)
    n = lib().vlr_merge_ready(S, ctypes.cast(rr, P), int(epochs[0]), nq, k, ctypes.cast(pi, P), ctypes.cast(pd, P),
                              ids.ctypes.data, dist.ctypes.data, t.ctypes.data, int(timeout_s * 1e6))
    if n < 0:
        raise VlrError(1, "vlr_merge_ready: bad arguments")
    if n < nq:
        raise VlrError(7, f"merge_ready: {nq - n} queries not released by every shard within {timeout_s} s")
    return torch.from_numpy(ids), torch.from_numpy(dist), t


def merge_partials(part_ids, part_dist, stream=None):
    """vlr_merge_partials: [S, nq, k] device partials -> final (ids, dist)."""
    import torch
    S, nq, k = part_ids.shape
    ids = torch.empty(nq, k, dtype=torch.int64, device=part_ids.device)
    dist = torch.empty(nq, k, dtype=torch.float32, device=part_ids.device)
    _check(lib().vlr_merge_partials(part_ids.data_ptr(), part_dist.data_ptr(), S, nq, k, ids.data_ptr(),
                                    dist.data_ptr(), _stream_handle(stream)))
    return ids, dist


def version() -> tuple:
    v = int(lib().vlr_version())
    return v >> 16, v & 0xFFFF
