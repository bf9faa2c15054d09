"""The centroid-sharded coarse stage on one GPU.

Rank r of G filters only its 128-centroid tiles; the ranks exchange their
nprobe' smallest group minima (x1), refine their own candidates exactly and
exchange their sorted exact top-nprobe' lists (x2); every rank then routes the
exact global probes. Here the G ranks are G shard-only handles on one GPU and
the exchanges are torch.stack (the staged C-ABI calls vlr_coarse_stage1/2,
vlr_search_stage3), so the same kernels as the NCCL path run. Results must be
BITWISE those of the single-GPU search (R5) and pass the oracle rules R1-R4.
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2504_08930_b200 as vlr
from parity import check

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2504_08930_b200 import build
    build.build()
    assert torch.cuda.is_available()


def plain(ix, Q, nprobe, k, hot=None):
    h = vlr.Index.from_arrays(ix, hot=hot)
    ids, dist, miss, probes = h.search(torch.from_numpy(Q).cuda(), nprobe, k, sync=True)
    out = dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())
    h.close()
    return out


def staged(ix, Q, nprobe, k, G, hot=None):
    """G shard-only handles; the exchanges are stacks of the ranks' buffers."""
    hs = [vlr.Index.from_arrays(ix, hot=hot, rank=r, world=G) for r in range(G)]
    Qd = torch.from_numpy(np.ascontiguousarray(Q, np.float32)).cuda()
    x1_all = torch.stack([h.coarse_stage1(Qd, nprobe) for h in hs])
    x2_all = torch.stack([h.coarse_stage2(Qd, nprobe, x1_all) for h in hs])
    outs = [h.search_stage3(Qd, nprobe, k, x2_all) for h in hs]
    torch.cuda.synchronize()
    for o in outs[1:]:  # every rank holds the same global probes and mask
        assert torch.equal(o[2], outs[0][2]) and torch.equal(o[3], outs[0][3])
    mi, md = vlr.merge_partials(torch.stack([o[0] for o in outs]), torch.stack([o[1] for o in outs]))
    torch.cuda.synchronize()
    res = dict(ids=mi.cpu().numpy(), dist=md.cpu().numpy(), miss=outs[0][2].cpu().numpy(),
               probes=outs[0][3].cpu().numpy())
    x1 = x1_all.cpu().numpy()
    for h in hs:
        h.close()
    return res, x1


def assert_bitwise(a, b, what=""):
    for key in ("probes", "miss", "ids", "dist"):
        assert np.array_equal(a[key], b[key]), f"{what}: {key} differs"


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_coarse_bitwise_c1(c1_index, c1_queries, G):
    c = datagen.CONFIGS["C1"]
    a = plain(c1_index, c1_queries, c["nprobe"], c["k"])
    b, x1 = staged(c1_index, c1_queries, c["nprobe"], c["k"], G)
    assert_bitwise(a, b, f"G={G}")
    # x1 rows hold each rank's nprobe' smallest group minima (+inf padding when a rank has fewer groups):
    # sorted, they are non-decreasing with at least nprobe' finite values in the union
    assert (np.isfinite(x1).sum(axis=(0, 2)) >= c["nprobe"]).all()
    o = oracle.search(c1_index, c1_queries, c["nprobe"], c["k"])
    assert not check(c1_index, c1_queries, b, o, idmap=oracle.IdMap(c1_index))


@pytest.mark.parametrize("nprobe,k", [(1, 1), (64, 32), (1024, 10)])
def test_sharded_coarse_nprobe_k(c1_index, c1_queries, nprobe, k):
    Q = c1_queries[:20]
    a = plain(c1_index, Q, nprobe, k)
    b, _ = staged(c1_index, Q, nprobe, k, 4)
    assert_bitwise(a, b, f"nprobe={nprobe}")


def test_sharded_coarse_empty_ranges():
    # nlist 200 = 2 filter tiles over 4 ranks: ranks 0 and 2 own no centroid (their x1 rows are +inf)
    ix = datagen.make_index(8000, 32, 200, 8, seed=5)
    Q = datagen.make_queries(8000, 32, 200, 17, seed=5, stream=2)
    for npb in (3, 40, 200):
        a = plain(ix, Q, npb, 10)
        b, x1 = staged(ix, Q, npb, 10, 4)
        assert_bitwise(a, b, f"nprobe={npb}")
        assert np.isinf(x1[0]).all() and np.isinf(x1[2]).all()


def test_sharded_coarse_hot_subset_and_variants(c1_index, c1_queries):
    c = datagen.CONFIGS["C1"]
    Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 2000, stream=1, alpha=c["alpha"])
    hot = datagen.hot_from_mass(datagen.access_counts(c1_index.centroids, Qc, c["nprobe"]), 0.5)
    a = plain(c1_index, c1_queries, c["nprobe"], c["k"], hot=hot)
    b, _ = staged(c1_index, c1_queries, c["nprobe"], c["k"], 3, hot=hot)
    assert_bitwise(a, b, "hot 50%")
    assert 0 < b["miss"].mean() < 1
    small = dict(N=6000, d=32, nlist=300, m=8)
    for kw in (dict(metric=1), dict(by_residual=0), dict(nbits=4), dict(metric=1, by_residual=0)):
        ix = datagen.make_index(small["N"], small["d"], small["nlist"], small["m"], seed=11, **kw)
        Q = datagen.make_queries(small["N"], small["d"], small["nlist"], 19, seed=11, stream=2)
        a = plain(ix, Q, 24, 10)
        b, _ = staged(ix, Q, 24, 10, 3)
        assert_bitwise(a, b, str(kw))
        o = oracle.search(ix, Q, 24, 10)
        assert not check(ix, Q, b, o, idmap=oracle.IdMap(ix)), kw


def test_sharded_coarse_overflow_rescan():
    # 20000 identical centroids: each of 2 ranks holds 10000 band candidates > the 8192 list
    # capacity, so stage 2 takes the rescan path on its own filter columns
    rng = np.random.default_rng(9)
    L, d = 20000, 8
    cvec = rng.standard_normal(d).astype(np.float32)
    C = np.repeat(cvec[None], L, 0)
    C[19990:] += np.float32(2.0)
    Y = (0.2 * rng.standard_normal((2, 256, 4))).astype(np.float32)
    lists = [(np.arange(i * 2, i * 2 + 2), rng.integers(0, 256, (2, 2)).astype(np.uint8)) for i in range(L)]
    ix = datagen.index_from_parts(C, Y, lists)
    Q = (cvec + 0.01 * rng.standard_normal((3, d))).astype(np.float32)
    for npb in (8, 2048):
        a = plain(ix, Q, npb, 10)
        b, _ = staged(ix, Q, npb, 10, 2)
        assert_bitwise(a, b, f"nprobe={npb}")
        assert b["probes"][0].tolist() == list(range(npb))  # equal distances -> ascending id


def test_staged_calls_validate_order(c1_index, c1_queries):
    h = vlr.Index.from_arrays(c1_index, rank=0, world=2)
    Qd = torch.from_numpy(c1_queries).cuda()
    x2_all = torch.zeros(2, len(c1_queries), 16, 2, dtype=torch.int64, device="cuda")
    with pytest.raises(vlr.VlrError) as e:  # stage 3 without stages 1-2
        h.search_stage3(Qd, 16, 10, x2_all)
    assert e.value.name == "INVALID_ARG"
    h.close()
    h1 = vlr.Index.from_arrays(c1_index)  # a single-GPU handle has no staged search
    with pytest.raises(vlr.VlrError):
        h1.coarse_stage1(Qd, 16)
    h1.close()


def test_nccl_sharded_path_single_rank(c1_index, c1_queries, monkeypatch):
    """The collective search with the sharded coarse stage (three ncclAllGathers
    on the search stream) through a 1-rank communicator: bitwise the plain
    search, and the oracle rules R1-R4."""
    c = datagen.CONFIGS["C1"]
    a = plain(c1_index, c1_queries, c["nprobe"], c["k"])
    monkeypatch.setenv("VLR_FORCE_EXCHANGE", "1")
    hx = vlr.Index.from_arrays(c1_index, nccl_id=vlr.nccl_unique_id())
    ids, dist, miss, probes = hx.search(torch.from_numpy(c1_queries).cuda(), c["nprobe"], c["k"], sync=True)
    b = dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())
    hx.close()
    assert_bitwise(a, b, "nccl sharded")
    o = oracle.search(c1_index, c1_queries, c["nprobe"], c["k"])
    assert not check(c1_index, c1_queries, b, o, idmap=oracle.IdMap(c1_index))


def _run_py(code, env_extra, timeout=240):
    env = dict(os.environ)
    env.update(env_extra)
    env["PYTHONPATH"] = ROOT + os.pathsep + os.path.join(ROOT, "tests")
    return subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env, capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_nccl_init_timeout_is_an_error_not_a_hang():
    """A peer that never joins: vlr_load_index of rank 0 of a 2-rank communicator
    returns VLR_ERR_NCCL after VLR_NCCL_TIMEOUT_MS instead of blocking forever."""
    code = """
        import time, torch, datagen, paper_2504_08930_b200 as vlr
        ix = datagen.make_index(4000, 16, 64, 4, seed=1)
        t = time.time()
        try:
            vlr.Index.from_arrays(ix, rank=0, world=2, device=0, nccl_id=vlr.nccl_unique_id())
            print("NO ERROR")
        except vlr.VlrError as e:
            print("ERR", e.name, round(time.time() - t, 1), str(e)[:200])
    """
    r = _run_py(code, {"VLR_NCCL_TIMEOUT_MS": "4000"})
    assert "ERR NCCL" in r.stdout, (r.stdout, r.stderr[-2000:])
    secs = float(r.stdout.split("ERR NCCL")[1].split()[0])
    assert secs < 60


def test_nccl_search_stall_times_out_with_error():
    """A collective that does not complete (injected: a bounded device stall
    before the first all-gather of every search, VLR_FAULT_STALL_US) makes
    vlr_search return VLR_ERR_NCCL after VLR_NCCL_TIMEOUT_MS; the handle is
    then dead. The first search on a fresh communicator is a warm-up: NCCL's
    lazy connection setup of its first collective waits for the stream (the
    whole stall) inside the enqueue, so the timeout is armed after it."""
    code = """
        import os, time, torch, datagen, paper_2504_08930_b200 as vlr
        ix = datagen.make_index(4000, 16, 64, 4, seed=1)
        Q = torch.from_numpy(datagen.make_queries(4000, 16, 64, 8, seed=1, stream=2)).cuda()
        h = vlr.Index.from_arrays(ix, device=0, nccl_id=vlr.nccl_unique_id())
        for i in range(3):
            if i == 1:
                os.environ["VLR_NCCL_TIMEOUT_MS"] = "500"
            t = time.time()
            try:
                h.search(Q, 4, 5, sync=True)
                print("CALL", i, "OK", round(time.time() - t, 2))
            except vlr.VlrError as e:
                print("CALL", i, e.name, round(time.time() - t, 2))
        torch.cuda.synchronize()
    """
    r = _run_py(code, {"VLR_FORCE_EXCHANGE": "1", "VLR_FAULT_STALL_US": "3000000"})
    lines = {ln.split()[1]: ln.split()[2:] for ln in r.stdout.splitlines() if ln.startswith("CALL")}
    assert lines.get("0", [None])[0] == "OK", (r.stdout, r.stderr[-2000:])
    assert lines.get("1", [None])[0] == "NCCL", (r.stdout, r.stderr[-2000:])
    # detected at the 0.5 s timeout; ncclCommAbort may then wait for the bounded stall to drain
    assert 0.4 < float(lines["1"][1]) < 20
    assert lines.get("2", [None])[0] == "NCCL"  # the handle is dead after an NCCL failure
