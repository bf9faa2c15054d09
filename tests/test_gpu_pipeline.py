"""Cross-batch pipelining (vlr_set_pipeline): searches on two
streams with two workspace slots overlap on the device; every row must equal
the serial single-stream search bitwise and pass the oracle rules R1-R4."""
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


def _batches(c, n):
    Q = datagen.make_queries(c["N"], c["d"], c["nlist"], n * c["batch"], stream=2, alpha=c["alpha"])
    return Q.reshape(n, c["batch"], c["d"])


@pytest.mark.parametrize("reserve", [0, 8, 32])
def test_two_streams_two_slots_bitwise_and_oracle(c1_index, reserve):
    c = datagen.CONFIGS["C1"]
    n = 6
    Q = _batches(c, n)
    Qd = torch.from_numpy(Q).cuda()
    h = vlr.Index.from_arrays(c1_index)
    ref = [h.search(Qd[i], c["nprobe"], c["k"], sync=True) for i in range(n)]
    h.set_pipeline(2, reserve)
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(2):  # twice: the slots' done events are waited for on the second round
        got = [h.search(Qd[i], c["nprobe"], c["k"], stream=ss[i % 2]) for i in range(n)]
        torch.cuda.synchronize()
        for i in range(n):
            for a, b in zip(got[i], ref[i]):
                assert torch.equal(a, b), (rep, i)
    h.close()
    o = oracle.search(c1_index, Q[n - 1], c["nprobe"], c["k"])
    g = dict(ids=got[-1][0].cpu().numpy(), dist=got[-1][1].cpu().numpy(), miss=got[-1][2].cpu().numpy(),
             probes=got[-1][3].cpu().numpy())
    errs = check(c1_index, Q[n - 1], g, o, idmap=oracle.IdMap(c1_index))
    assert not errs, errs


def test_pipelined_host_async_and_hot_subset(c1_index):
    """vlr_search_host_async on two streams (each slot stages its own queries), hot subset (miss mask)."""
    c = datagen.CONFIGS["C1"]
    n = 4
    Q = _batches(c, n)
    counts = datagen.access_counts(c1_index.centroids, datagen.make_queries(c["N"], c["d"], c["nlist"], 2000,
                                                                             stream=1, alpha=c["alpha"]), c["nprobe"])
    hot = datagen.hot_from_mass(counts, 0.5)
    h = vlr.Index.from_arrays(c1_index, hot=hot)
    ref = [h.search_host(Q[i], c["nprobe"], c["k"]) for i in range(n)]
    h.set_pipeline(2, 16)
    B, K, NP = c["batch"], c["k"], min(c["nprobe"], c["nlist"])
    hq = [torch.from_numpy(Q[i].copy()).pin_memory() for i in range(n)]
    outs = [(torch.empty(B, K, dtype=torch.int64).pin_memory(), torch.empty(B, K).pin_memory(),
             torch.empty(B, NP, dtype=torch.uint8).pin_memory()) for _ in range(n)]
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    for i in range(n):
        h.search_host_ptr_async(hq[i].data_ptr(), B, c["nprobe"], K, outs[i][0].data_ptr(), outs[i][1].data_ptr(),
                                outs[i][2].data_ptr(), None, stream=ss[i % 2])
    torch.cuda.synchronize()
    for i in range(n):
        assert np.array_equal(outs[i][0].numpy(), ref[i][0])
        assert np.array_equal(outs[i][1].numpy(), ref[i][1])
        assert np.array_equal(outs[i][2].numpy(), ref[i][2])
    h.close()


def test_pipelined_release_and_large_k(c1_index):
    """The release mode and the k > 32 path run on their slot's workspace too."""
    c = datagen.CONFIGS["C1"]
    Q = _batches(c, 2)
    Qd = torch.from_numpy(Q).cuda()
    h = vlr.Index.from_arrays(c1_index)
    ref_big = [h.search(Qd[i], c["nprobe"], 100, sync=True) for i in range(2)]
    ref = [h.search(Qd[i], c["nprobe"], c["k"], sync=True) for i in range(2)]
    h.set_pipeline(2, 8)
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    big = [h.search(Qd[i], c["nprobe"], 100, stream=ss[i]) for i in range(2)]
    torch.cuda.synchronize()
    for a, b in zip(big, ref_big):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    for i in range(2):
        rows = h.search_release(Qd[i], c["nprobe"], c["k"], stream=ss[i])
        assert torch.equal(torch.as_tensor(rows[0]).cpu(), ref[i][0].cpu())
    h.close()
