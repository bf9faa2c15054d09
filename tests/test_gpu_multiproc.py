"""Two processes, one GPU: the N > 1 search path with a real process group.

Two ranks (torch.distributed, gloo) share cuda:0. Each loads its shard-only
handle (its hot lists dealt by size, and its centroid tiles) and runs
the staged sharded search (vlr_coarse_stage1/2, vlr_search_stage3) with the
two coarse exchanges and the result exchange done by dist.all_gather, then
merges the gathered partial top-k with vlr_merge_partials. Every rank
must hold the single-GPU result bitwise, and the result must pass the oracle
rules R1-R4. This is the multi-process plumbing of bench.py's N > 1 path
without NCCL (NCCL refuses two ranks on one device).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather(t, world):
    """rank-ordered stack of every rank's CUDA tensor t (through host memory: gloo)."""
    c = t.cpu()
    parts = [torch.empty_like(c) for _ in range(world)]
    dist.all_gather(parts, c)
    return torch.stack(parts).cuda()


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import datagen
        import oracle
        import paper_2504_08930_b200 as vlr
        from parity import check
        c = datagen.CONFIGS["C1"]
        ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"])
        Q = datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, alpha=c["alpha"])
        Qd = torch.from_numpy(Q).cuda()
        h = vlr.Index.from_arrays(ix, rank=rank, world=world, device=0)
        ids, dd, miss, probes = h.search_staged(Qd, c["nprobe"], c["k"], lambda t: _gather(t, world))
        mi, md = vlr.merge_partials(_gather(ids, world), _gather(dd, world))
        torch.cuda.synchronize()
        got = dict(ids=mi.cpu().numpy(), dist=md.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())
        h.close()
        h1 = vlr.Index.from_arrays(ix, device=0)
        ref = h1.search(Qd, c["nprobe"], c["k"], sync=True)
        h1.close()
        bit = all(np.array_equal(got[key], r.cpu().numpy()) for key, r in zip(("ids", "dist", "miss", "probes"), ref))
        o = oracle.search(ix, Q, c["nprobe"], c["k"], nthreads=2)
        errs = check(ix, Q, got, o, idmap=oracle.IdMap(ix))
        out_q.put((rank, bit, errs[:3]))
    except Exception as e:  # report instead of hanging the parent
        out_q.put((rank, False, [repr(e)]))
    finally:
        dist.destroy_process_group()


def test_two_process_staged_search_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, bit, errs in res:
        assert not errs, (rank, errs)
        assert bit, f"rank {rank}: staged two-process result differs from the single-GPU search"


def _p2p_worker(rank, world, port, out_q, pipelined=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import datagen
        import oracle
        import paper_2504_08930_b200 as vlr
        from parity import check
        c = datagen.CONFIGS["C1"]
        ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"])
        Q = datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, alpha=c["alpha"])
        Qd = torch.from_numpy(Q).cuda()
        h = vlr.Index.from_arrays(ix, rank=rank, world=world, device=0)
        if pipelined:  # two workspace slots = two inbox regions; searches alternate over two streams
            h.set_pipeline(2, 8)
        h.reserve(c["batch"], c["nprobe"], c["k"])
        mine = h.p2p_export()
        handles = [None] * world
        dist.all_gather_object(handles, mine)
        h.p2p_connect(handles)
        dist.barrier()
        outs = []
        if pipelined:
            ss = [torch.cuda.Stream(), torch.cuda.Stream()]
            for it in range(6):  # slots 0,1,0,1,...: batch i+1 enqueued before batch i completes
                outs.append(h.search(Qd, c["nprobe"], c["k"], stream=ss[it % 2]))
            torch.cuda.synchronize()
        else:
            for it in range(3):  # collective searches over the peer inboxes (epochs advance together)
                outs.append(h.search(Qd, c["nprobe"], c["k"], sync=True))
        got = dict(ids=outs[-1][0].cpu().numpy(), dist=outs[-1][1].cpu().numpy(), miss=outs[-1][2].cpu().numpy(),
                   probes=outs[-1][3].cpu().numpy())
        dist.barrier()
        h.close()
        h1 = vlr.Index.from_arrays(ix, device=0)
        ref = h1.search(Qd, c["nprobe"], c["k"], sync=True)
        h1.close()
        bit = all(np.array_equal(got[key], r.cpu().numpy()) for key, r in zip(("ids", "dist", "miss", "probes"), ref))
        bit = bit and all(torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1]) for o in outs)
        o = oracle.search(ix, Q, c["nprobe"], c["k"], nthreads=2)
        errs = check(ix, Q, got, o, idmap=oracle.IdMap(ix))
        out_q.put((rank, bit, errs[:3]))
    except Exception as e:
        out_q.put((rank, False, [repr(e)]))
    finally:
        dist.destroy_process_group()


def _run_p2p(pipelined):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, pipelined)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_two_process_peer_exchange_pipelined_one_gpu():
    """Cross-batch pipelining over the peer exchange (vlr_set_pipeline(2, 8)): six
    collective searches alternate over two streams per rank, so batch i+1's coarse
    stage and its stage-1/2 exchanges run while batch i is still in flight; each
    slot exchanges through its own inbox region. Every row equals the single-GPU
    search bitwise and passes R1-R4."""
    for rank, bit, errs in _run_p2p(True):
        assert not errs, (rank, errs)
        assert bit, f"rank {rank}: pipelined peer-exchange result differs from the single-GPU search"


def test_two_process_nvlink_peer_exchange_one_gpu():
    """The peer-exchange transport (vlr_p2p_export / connect): two processes on
    one GPU map each other's inboxes with CUDA IPC; every search is collective,
    the producer kernels store their slabs into both inboxes and raise epoch
    flags, the consumers wait on them. Final rows equal the single-GPU search
    bitwise on both ranks, over repeated searches (epochs), and pass R1-R4."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, bit, errs in res:
        assert not errs, (rank, errs)
        assert bit, f"rank {rank}: peer-exchange result differs from the single-GPU search"
