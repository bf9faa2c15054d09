"""World-size-2 CPU (gloo) tests of the N > 1 host path.

What runs here is the host logic of the sharded search, not the kernels:
the size-descending round-robin deal, per-rank shard generation,
SPMD exchange of rank-partial top-k (all-gather) and the (dist, id) merge
(P:412-414). The rank-partial results are produced by the oracle restricted
to each rank's resident lists, so the test checks that the sharding
arithmetic reproduces the monolithic search exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle
        N, d, L, m = 5000, 32, 48, 8
        full = datagen.make_index(N, d, L, m, seed=21)
        Q = datagen.make_queries(N, d, L, 24, seed=21, stream=2)
        rng = np.random.default_rng(0)
        hot = np.sort(rng.choice(L, 36, replace=False)).astype(np.int32)
        own = datagen.deal_owners(full.list_sizes, hot, world)
        mine = np.nonzero(own == rank)[0]
        # per-rank generation of the owned shard equals the full generation there
        shard = datagen.make_index(N, d, L, m, seed=21, owned=own == rank)
        for l in mine:
            a, b = full.list_offsets[l], full.list_offsets[l + 1]
            assert np.array_equal(shard.codes[a:b], full.codes[a:b])
        # rank-partial top-k over the resident lists this rank owns
        k, npb = 10, 12
        part = oracle.search(full, Q, npb, k, hot=mine, nthreads=2)
        ids = torch.from_numpy(part["ids"].copy())
        dd = torch.from_numpy(part["dist"].copy())
        gi = [torch.empty_like(ids) for _ in range(world)]
        gd = [torch.empty_like(dd) for _ in range(world)]
        dist.all_gather(gi, ids)
        dist.all_gather(gd, dd)
        # every rank merges (SPMD) and must hold the same result
        ai = torch.stack(gi).numpy()
        ad = torch.stack(gd).numpy()
        merged_i = np.empty_like(part["ids"])
        merged_d = np.empty_like(part["dist"])
        for q in range(len(Q)):
            i = ai[:, q].reshape(-1)
            dv = ad[:, q].reshape(-1)
            o = np.lexsort((np.where(i < 0, np.iinfo(np.int64).max, i), dv))[:k]
            merged_i[q], merged_d[q] = i[o], dv[o]
        ref = oracle.search(full, Q, npb, k, hot=hot, nthreads=2)
        ok = np.array_equal(merged_i, ref["ids"]) and np.array_equal(merged_d, ref["dist"])
        # disjoint shards covering the hot set, sizes balanced by the deal
        cnt = torch.tensor([len(mine)])
        tot = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(tot, cnt)
        # the library's deal (vlr_deal_owners, host only) is the same round-robin deal
        import paper_2504_08930_b200 as vlr
        ok = ok and np.array_equal(vlr.deal_owners(full.list_offsets, hot, world), own[hot])
        # NEXT-2 distributed profiling: each rank counts the probes of its half of a calibration
        # stream, the counts are summed across ranks, and every rank derives the same
        # traffic-aware deal; the merged partials over that deal still equal the monolithic search
        Qc = datagen.make_queries(N, d, L, 200, seed=21, stream=1)
        half = Qc[rank::world]
        pr, _ = oracle.coarse(half, full.centroids, npb)
        cnt_l = torch.from_numpy(np.bincount(pr.reshape(-1), minlength=L).astype(np.int64))
        dist.all_reduce(cnt_l, op=dist.ReduceOp.SUM)
        own_t = torch.from_numpy(vlr.deal_owners(full.list_offsets, hot, world, counts=cnt_l.numpy()).astype(np.int64))
        go = [torch.empty_like(own_t) for _ in range(world)]
        dist.all_gather(go, own_t)
        ok = ok and all(torch.equal(g, own_t) for g in go)
        mine_t = hot[own_t.numpy() == rank]
        part = oracle.search(full, Q, npb, k, hot=mine_t, nthreads=2)
        ids = torch.from_numpy(part["ids"].copy())
        dd = torch.from_numpy(part["dist"].copy())
        dist.all_gather(gi, ids)
        dist.all_gather(gd, dd)
        ai = torch.stack(gi).numpy()
        ad = torch.stack(gd).numpy()
        for q in range(len(Q)):
            i = ai[:, q].reshape(-1)
            dv = ad[:, q].reshape(-1)
            o = np.lexsort((np.where(i < 0, np.iinfo(np.int64).max, i), dv))[:k]
            ok = ok and np.array_equal(i[o], ref["ids"][q]) and np.array_equal(dv[o], ref["dist"][q])
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out_q.put((rank, ok, int(sum(int(x) for x in tot)), float(t.item()), sorted(mine.tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_matches_monolithic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res), "merged shard partials differ from the monolithic oracle"
    assert res[0][2] == 36 and res[0][3] == float(world)
    owned = [set(r[4]) for r in res]
    assert not (owned[0] & owned[1])
