"""NEXT-4: early per-query release (vlr_search_release_async + vlr_poll_ready),
the GPU analog of the paper's dynamic dispatcher (P:408-414 [§IV.C], Fig. 14).

The released rows must be bit-identical to vlr_search_async (same scan, same
merge code) and pass the oracle parity rules; every query (including those
with no resident probe) must be released exactly once per epoch.
"""
import ctypes

import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2504_08930_b200 as vlr
from parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2504_08930_b200 import build
    build.build()
    assert torch.cuda.is_available()


def release(h, Q, nprobe, k):
    Qd = torch.from_numpy(np.ascontiguousarray(Q, np.float32)).cuda()
    order = []
    ids, dist, miss, probes, t = h.search_release(Qd, nprobe, k, on_ready=lambda qs: order.extend(qs.tolist()))
    torch.cuda.synchronize()
    assert sorted(order) == list(range(len(Q)))  # each query released exactly once
    assert np.all(t >= t.t0)
    return dict(ids=ids.numpy().copy(), dist=dist.numpy().copy(), miss=miss.cpu().numpy(),
                probes=probes.cpu().numpy()), t


def plain(h, Q, nprobe, k):
    Qd = torch.from_numpy(np.ascontiguousarray(Q, np.float32)).cuda()
    ids, dist, miss, probes = h.search(Qd, nprobe, k, sync=True)
    return dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())


@pytest.mark.parametrize("hot_mass", [1.0, 0.5, 0.02])
def test_release_equals_search_and_oracle(c1_index, c1_queries, hot_mass):
    c = datagen.CONFIGS["C1"]
    hot = None
    if hot_mass < 1.0:
        Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 2000, stream=1, alpha=c["alpha"])
        hot = datagen.hot_from_mass(datagen.access_counts(c1_index.centroids, Qc, c["nprobe"]), hot_mass)
    h = vlr.Index.from_arrays(c1_index, hot=hot)
    r, _ = release(h, c1_queries, c["nprobe"], c["k"])
    p = plain(h, c1_queries, c["nprobe"], c["k"])
    for key in p:
        assert np.array_equal(r[key], p[key]), key
    o = oracle.search(c1_index, c1_queries, c["nprobe"], c["k"], hot=hot)
    errs = check(c1_index, c1_queries, r, o, hot=hot, idmap=oracle.IdMap(c1_index))
    assert not errs, errs
    if hot_mass == 0.02:  # queries with no resident probe are released as padding
        empty = r["miss"].all(axis=1)
        assert empty.any()
        assert np.all(r["ids"][empty] == -1) and np.all(np.isinf(r["dist"][empty]))
    h.close()


def test_release_batch_sizes_and_repeats(c1_index):
    """nq = 1 (one query spans every scan CTA), nq > scan CTAs (several queries
    per CTA), k = 32 and 1; repeated calls on the same handle (new epochs)."""
    h = vlr.Index.from_arrays(c1_index)
    big = datagen.make_queries(100_000, 128, 1024, 400, stream=3)
    for nq, nprobe, k in ((1, 16, 10), (1, 64, 32), (7, 16, 1), (400, 16, 10), (400, 32, 32)):
        Q = big[:nq]
        for _ in range(2):
            r, _ = release(h, Q, nprobe, k)
            p = plain(h, Q, nprobe, k)
            for key in p:
                assert np.array_equal(r[key], p[key]), (nq, nprobe, k, key)
    h.close()


def test_release_long_lists_small_batch():
    """Long lists, batch 1-8: queries span many CTAs, so the completing CTA's
    merge sees hundreds of partial lists (the multi-warp merge path)."""
    ix = datagen.make_index(2_000_000, 128, 1024, 16, device="cuda")
    h = vlr.Index.from_arrays(ix)
    Qa = datagen.make_queries(2_000_000, 128, 1024, 8, stream=2)
    for nq, k in ((1, 10), (3, 32), (8, 10)):
        r, _ = release(h, Qa[:nq], 64, k)
        o = oracle.search(ix, Qa[:nq], 64, k)
        assert not check(ix, Qa[:nq], r, o), (nq, k)
    h.close()


def test_release_pq4(c1_queries):
    ix = datagen.make_index(100_000, 128, 1024, 32, seed=5, nbits=4)
    h = vlr.Index.from_arrays(ix)
    r, _ = release(h, c1_queries, 16, 10)
    p = plain(h, c1_queries, 16, 10)
    for key in p:
        assert np.array_equal(r[key], p[key]), key
    h.close()


def test_release_errors(c1_index, c1_queries):
    L = vlr.lib()
    h = vlr.Index.from_arrays(c1_index)
    Qd = torch.from_numpy(c1_queries[:4]).cuda()
    ids = torch.empty(4, 10, dtype=torch.int64, pin_memory=True)
    dist = torch.empty(4, 10, dtype=torch.float32, pin_memory=True)
    miss = torch.empty(4, 16, dtype=torch.uint8, device="cuda")
    ready = torch.zeros(4, dtype=torch.int32, pin_memory=True)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (h._h, Qd.data_ptr(), 4, 16, 10, ids.data_ptr(), dist.data_ptr(), miss.data_ptr(), None)
    assert L.vlr_search_release_async(*args, ready.data_ptr(), 0, s) == 1  # epoch 0
    pageable = np.zeros(4, np.uint32)
    assert L.vlr_search_release_async(*args, pageable.ctypes.data, 5, s) == 1  # not device-accessible
    assert L.vlr_search_release_async(*args, None, 5, s) == 1
    h.close()
    torch.cuda.synchronize()
    args = (h._h, Qd.data_ptr(), 4, 16, 40, ids.data_ptr(), dist.data_ptr(), miss.data_ptr(), None)
    h = vlr.Index.from_arrays(c1_index)
    args = (h._h,) + args[1:]
    assert L.vlr_search_release_async(*args, ready.data_ptr(), 5, s) == 9  # UNSUPPORTED: k > 32
    h.close()


def test_release_sharded_dispatcher_merge(c1_index, c1_queries):
    """NEXT-4 at world > 1: G shard-only handles each release their
    partial rows (own probes only) with completion flags; the host dispatcher
    (vlr_merge_ready) merges a query as soon as every shard released it. The
    merged rows equal the single-GPU search bitwise; shards launched on their
    own streams run concurrently."""
    c = datagen.CONFIGS["C1"]
    Qd = torch.from_numpy(c1_queries).cuda()
    h1 = vlr.Index.from_arrays(c1_index)
    ref = h1.search(Qd, c["nprobe"], c["k"], sync=True)
    h1.close()
    for G in (2, 3):
        hs = [vlr.Index.from_arrays(c1_index, rank=r, world=G) for r in range(G)]
        for h in hs:  # identical epochs across shards (first release on each handle)
            h._epoch = 100
        streams = [torch.cuda.Stream() for _ in range(G)]
        outs = [h.search_release_launch(Qd, c["nprobe"], c["k"], stream=s) for h, s in zip(hs, streams)]
        ids, dist, t = vlr.merge_ready([o[4] for o in outs], [o[5] for o in outs], [o[0] for o in outs],
                                       [o[1] for o in outs])
        torch.cuda.synchronize()
        assert torch.equal(ids, ref[0].cpu()) and torch.equal(dist, ref[1].cpu()), G
        for o in outs[1:]:
            assert torch.equal(o[2], outs[0][2]) and torch.equal(o[3], outs[0][3])
        assert (t > 0).all()
        for h in hs:
            h.close()
