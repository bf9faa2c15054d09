"""C-ABI library checks that need no GPU: the library loads, exports every
symbol include/vlr.h declares, and the host-side validation of
vlr_load_index / vlr_search* returns the documented status codes before any
device work. With no GPU, a valid load fails with VLR_ERR_CUDA (no fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2504_08930_b200 as vlr
from conftest import ROOT


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2504_08930_b200 import build
    build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vlr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vlr_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 14
    L = vlr.lib()
    for s in syms:
        assert hasattr(L, s), f"libvlr.so does not export {s}"
    assert sorted(vlr.EXPORTS) == syms


def test_version():
    assert vlr.version() == (1, 3)


def _tiny(m=2, d=4, L=3):
    rng = np.random.default_rng(0)
    C = rng.standard_normal((L, d)).astype(np.float32)
    Y = rng.standard_normal((m, 256, d // m)).astype(np.float32)
    offs = np.array([0, 2, 2, 5], np.int64)[: L + 1]
    ids = np.arange(5, dtype=np.int64)
    codes = rng.integers(0, 256, (5, m)).astype(np.uint8)
    return C, Y, offs, ids, codes


def status_of(fn):
    try:
        fn()
    except vlr.VlrError as e:
        return e.name
    return "OK"


def test_load_validation_codes():
    C, Y, offs, ids, codes = _tiny()
    load = vlr.Index.load
    # d % m != 0 (m = 3 for d = 4)
    Y3 = np.zeros((3, 256, 1), np.float32)
    assert status_of(lambda: load(C, Y3, offs, ids, np.zeros((5, 3), np.uint8), device=0)) == "DIM_MISMATCH"
    assert status_of(lambda: load(C, Y, offs, ids, codes, nbits=6, device=0)) == "UNSUPPORTED"
    assert status_of(lambda: load(C, Y, offs, ids, codes, metric=2, device=0)) == "UNSUPPORTED"
    assert status_of(lambda: load(C, Y, offs, ids, codes, by_residual=2, device=0)) == "INVALID_ARG"
    Cn = C.copy(); Cn[1, 2] = np.nan
    assert status_of(lambda: load(Cn, Y, offs, ids, codes, device=0)) == "NONFINITE"
    Yn = Y.copy(); Yn[0, 5, 0] = np.inf
    assert status_of(lambda: load(C, Yn, offs, ids, codes, device=0)) == "NONFINITE"
    assert status_of(lambda: load(C, Y, offs, ids, codes, hot=[0, 3], device=0)) == "UNKNOWN_CLUSTER"
    assert status_of(lambda: load(C, Y, offs, ids, codes, hot=[1, 1], device=0)) == "UNKNOWN_CLUSTER"
    assert status_of(lambda: load(C, Y, offs, ids, codes, hot=[0, 1], hot_owner=[0, 2], world=2,
                                  device=0)) == "UNKNOWN_CLUSTER"
    bad = offs.copy(); bad[2] = 1
    assert status_of(lambda: load(C, Y, bad, ids, codes, device=0)) == "INVALID_ARG"
    assert status_of(lambda: load(C, Y, offs, ids, codes, rank=2, world=2, device=0)) == "INVALID_ARG"


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_valid_load_without_gpu_fails_loudly():
    C, Y, offs, ids, codes = _tiny()
    assert status_of(lambda: vlr.Index.load(C, Y, offs, ids, codes, device=0)) == "CUDA"


def test_search_argument_validation_without_index():
    L = vlr.lib()
    # null index
    st = L.vlr_search_async(None, None, 1, 1, 1, None, None, None, None, None)
    assert vlr.STATUS[st] == "INVALID_ARG"
    st = L.vlr_merge_partials(None, None, 0, 1, 1, None, None, None)
    assert vlr.STATUS[st] == "INVALID_ARG"
    st = L.vlr_merge_partials(None, None, 1, 1, 2000, None, None, None)  # k > 1024
    assert vlr.STATUS[st] == "UNSUPPORTED"
    st = L.vlr_merge_partials(None, None, 9, 1, 1000, None, None, None)  # n_shards x k > 8192 (k > 32)
    assert vlr.STATUS[st] == "UNSUPPORTED"
    st = L.vlr_merge_partials(None, None, 2, 1, 64, None, None, None)  # k 64 valid: null buffers
    assert vlr.STATUS[st] == "INVALID_ARG"
    st = L.vlr_merge_partials(None, None, 1, 0, 4, None, None, None)
    assert vlr.STATUS[st] == "OK"  # nq == 0 is a no-op
    st = L.vlr_set_pipeline(None, 2, 0)  # cross-batch pipelining on a null handle
    assert vlr.STATUS[st] == "INVALID_ARG"
    assert b"" != L.vlr_last_error() or True


def test_poll_ready_host_dispatcher():
    """vlr_poll_ready (NEXT-4 host side) on host flags: returns the newly
    released queries once each, marks them seen, times out with 0."""
    L = vlr.lib()
    nq, epoch = 10, 7
    ready = np.zeros(nq, np.uint32)
    ready[[2, 5, 9]] = epoch
    ready[3] = epoch - 1  # a stale epoch is not a release
    seen = np.zeros(nq, np.uint8)
    qs = np.empty(nq, np.int32)
    ts = np.empty(nq, np.int64)
    n = L.vlr_poll_ready(ready.ctypes.data, nq, epoch, seen.ctypes.data, qs.ctypes.data, ts.ctypes.data, nq, 1000)
    assert n == 3 and sorted(qs[:3].tolist()) == [2, 5, 9]
    assert seen.tolist() == [1 if q in (2, 5, 9) else 0 for q in range(nq)]
    assert np.all(ts[:3] > 0)
    n = L.vlr_poll_ready(ready.ctypes.data, nq, epoch, seen.ctypes.data, qs.ctypes.data, None, nq, 2000)
    assert n == 0  # nothing new: timeout
    ready[0] = epoch
    n = L.vlr_poll_ready(ready.ctypes.data, nq, epoch, seen.ctypes.data, qs.ctypes.data, None, 1, 1000)
    assert n == 1 and qs[0] == 0
    assert L.vlr_poll_ready(None, nq, epoch, seen.ctypes.data, qs.ctypes.data, None, nq, 0) == -1
    assert L.vlr_poll_ready(ready.ctypes.data, nq, epoch, seen.ctypes.data, qs.ctypes.data, None, 0, 0) == -1


def test_wait_ready_host_dispatcher():
    L = vlr.lib()
    nq, epoch = 6, 3
    ready = np.full(nq, epoch, np.uint32)
    ts = np.zeros(nq, np.int64)
    assert L.vlr_wait_ready(ready.ctypes.data, nq, epoch, ts.ctypes.data, 1000) == nq
    assert np.all(ts > 0)
    ready[4] = 0
    assert L.vlr_wait_ready(ready.ctypes.data, nq, epoch, None, 2000) == nq - 1  # timeout: one missing
    assert L.vlr_wait_ready(None, nq, epoch, None, 0) == -1


def _rr_reference(offs, hot, world):
    sizes = np.diff(offs)
    order = sorted(range(len(hot)), key=lambda i: (-int(sizes[hot[i]]), int(hot[i])))
    own = np.empty(len(hot), np.int32)
    for r, i in enumerate(order):
        own[i] = r % world
    return own


def test_deal_owners_round_robin_and_traffic_lpt():
    """vlr_deal_owners (NEXT-2 splitter): counts=NULL is the paper's
    size-descending round-robin; with counts, the greedy LPT deal by
    size x (count + 1) replays step by step and balances the profiled traffic
    no worse than round-robin."""
    rng = np.random.default_rng(4)
    nlist = 400
    sizes = rng.integers(0, 300, nlist)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    hot = rng.permutation(nlist)[:250].astype(np.int32)
    counts = (1e5 / np.arange(1, nlist + 1) ** 1.1)[rng.permutation(nlist)].astype(np.int64)
    for world in (1, 2, 3, 8):
        own = vlr.deal_owners(offs, hot, world)
        assert np.array_equal(own, _rr_reference(offs, hot, world))
        lpt = vlr.deal_owners(offs, hot, world, counts=counts)
        load = sizes[hot].astype(np.float64) * (counts[hot] + 1.0)
        # replay the greedy: descending load (ties: size desc, id), each to the least-loaded rank
        order = sorted(range(len(hot)), key=lambda i: (-load[i], -int(sizes[hot[i]]), int(hot[i])))
        acc = np.zeros(world)
        for i in order:
            r = int(np.argmin(acc))
            assert lpt[i] == r
            acc[r] += load[i]
        rr = np.bincount(own, weights=load, minlength=world)
        assert acc.max() <= rr.max() + 1e-9
        assert acc.max() <= load.sum() / world + load.max() + 1e-9  # list-scheduling bound
    assert vlr.deal_owners(offs, np.zeros(0, np.int32), 4).size == 0
    with pytest.raises(vlr.VlrError) as e:
        vlr.deal_owners(offs, np.array([1, 1], np.int32), 2)
    assert e.value.name == "UNKNOWN_CLUSTER"
    with pytest.raises(vlr.VlrError) as e:
        vlr.deal_owners(offs, np.array([nlist], np.int32), 2)
    assert e.value.name == "UNKNOWN_CLUSTER"
    with pytest.raises(vlr.VlrError) as e:
        vlr.deal_owners(offs, hot, 0)
    assert e.value.name == "INVALID_ARG"
