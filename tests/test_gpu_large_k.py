"""k > 32 (up to 1024): the DUMP scan + per-query radix select
path (k_select_large) and the large-k merges (K8 / vlr_merge_partials),
against the oracle (rules R1-R4) and bitwise across shards (R5).
"""
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


@pytest.fixture(scope="module")
def big_nlist():
    ix = datagen.make_index(60_000, 32, 4096, 8, seed=23)
    Q = datagen.make_queries(60_000, 32, 4096, 24, seed=23, stream=2)
    return ix, Q


def run(ix, Q, nprobe, k, **kw):
    h = vlr.Index.from_arrays(ix, **kw)
    ids, dist, miss, probes = h.search(torch.from_numpy(Q).cuda(), nprobe, k, sync=True)
    h.close()
    return dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())


@pytest.mark.parametrize("nprobe,k", [(2048, 25), (2048, 100), (300, 1024), (16, 64), (2048, 1024)])
def test_large_k_parity(big_nlist, nprobe, k):
    """the paper's operating point nprobe 2048 with k 25 (warp path) and k 100 (large path), and k up to
    1024 incl. queries with fewer than k candidates (padding)"""
    ix, Q = big_nlist
    g = run(ix, Q, nprobe, k)
    o = oracle.search(ix, Q, nprobe, k)
    errs = check(ix, Q, g, o, idmap=oracle.IdMap(ix))
    assert not errs, errs


def test_large_k_prefix_of_larger_k(big_nlist):
    """the top-k by (dist, id) is unique: the k = 33 rows are the first 33 entries of the k = 700 rows"""
    ix, Q = big_nlist
    a = run(ix, Q, 512, 33)
    b = run(ix, Q, 512, 700)
    assert np.array_equal(a["ids"], b["ids"][:, :33]) and np.array_equal(a["dist"], b["dist"][:, :33])
    c = run(ix, Q, 512, 32)  # warp path vs large path: the same unique rows
    assert np.array_equal(c["ids"], b["ids"][:, :32]) and np.array_equal(c["dist"], b["dist"][:, :32])


def test_large_k_hot_subset_and_shards(big_nlist):
    ix, Q = big_nlist
    Qc = datagen.make_queries(60_000, 32, 4096, 3000, seed=23, stream=1)
    hot = datagen.hot_from_mass(datagen.access_counts(ix.centroids, Qc, 256), 0.6)
    a = run(ix, Q, 256, 200, hot=hot)
    o = oracle.search(ix, Q, 256, 200, hot=hot)
    assert not check(ix, Q, a, o, hot=hot, idmap=oracle.IdMap(ix))
    Qd = torch.from_numpy(Q).cuda()
    for G in (2, 3):
        pi, pd = [], []
        for r in range(G):
            h = vlr.Index.from_arrays(ix, hot=hot, rank=r, world=G)
            ids, dist, miss, probes = h.search(Qd, 256, 200, sync=True)
            assert np.array_equal(miss.cpu().numpy(), a["miss"])
            pi.append(ids)
            pd.append(dist)
            h.close()
        mi, md = vlr.merge_partials(torch.stack(pi), torch.stack(pd))
        torch.cuda.synchronize()
        assert np.array_equal(mi.cpu().numpy(), a["ids"]) and np.array_equal(md.cpu().numpy(), a["dist"]), G


def test_large_k_nccl_single_rank(big_nlist, monkeypatch):
    """k > 32 through the collective path (packed large-k rows -> ncclAllGather -> large K8 merge)"""
    ix, Q = big_nlist
    a = run(ix, Q, 128, 300)
    monkeypatch.setenv("VLR_FORCE_EXCHANGE", "1")
    b = run(ix, Q, 128, 300, nccl_id=vlr.nccl_unique_id())
    for key in a:
        assert np.array_equal(a[key], b[key]), key


def test_large_k_limits(big_nlist):
    ix, Q = big_nlist
    h = vlr.Index.from_arrays(ix)
    Qd = torch.from_numpy(Q).cuda()
    with pytest.raises(vlr.VlrError) as e:
        h.search(Qd, 16, 1025, sync=True)
    assert e.value.name == "UNSUPPORTED"
    with pytest.raises(vlr.VlrError) as e:
        h.search_release(Qd, 16, 64)
    assert e.value.name == "UNSUPPORTED"
    h.close()


@pytest.mark.parametrize("d,m,nbits", [(768, 384, 4), (640, 320, 4), (384, 192, 8), (320, 160, 8)])
def test_wide_pq_parity(d, m, nbits):
    """the paper's inferred index format PQ384x4 at 768-d (~205 B/vector, SURVEY reading A4; pair
    slots: 192 bytes) and the other widened scan instantiations (160 / 192 byte slots)"""
    ix = datagen.make_index(12_000, d, 64, m, seed=29, nbits=nbits)
    Q = datagen.make_queries(12_000, d, 64, 20, seed=29, stream=2)
    for npb, k in ((8, 10), (64, 50)):
        g = run(ix, Q, npb, k)
        o = oracle.search(ix, Q, npb, k)
        errs = check(ix, Q, g, o, idmap=oracle.IdMap(ix))
        assert not errs, (d, m, nbits, npb, k, errs)
