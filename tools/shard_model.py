"""Per-rank device time of the sharded search at G ranks, measured on ONE GPU.

The G ranks are G shard-only handles of the same index (each holds its dealt
hot lists and filters its own 128-centroid tiles). Their staged calls run one
after another on one stream, so CUDA events around each rank's call measure
exactly that rank's kernels:
  stage1 = qprep + K1 (its tiles) + K2 stage 1
  stage2 = K2 stage 2 + K3a + K3b local
  stage3 = K3b merge + route + K4b + (LUT join) + K6 scan + K7
A ~5 ms spin kernel heads each batch so that all its launches are queued
before the first event fires (device time, not host enqueue time).
The exchanges (3 all-gathers on NVLink at G > 1) are not measurable on one
GPU; the line reports them as a separate term. Output: one JSON line.

  python tools/shard_model.py --config C4 --G 8 --batches 10
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--batches", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=2504_08930)
    ap.add_argument("--backlog-cycles", type=int, default=10_000_000)
    ap.add_argument("--deal", default="paper", choices=["paper", "traffic"],
                    help="hot-list deal: the paper's size round-robin (P:339) or the traffic-aware LPT deal on "
                         "size x access count of a 4096-query calibration stream (stream 1, disjoint; NEXT-2)")
    ap.add_argument("--pipe-reserve", default="0,8,16,24,32",
                    help="scan reserves for the pipelined single-rank pass ('' = skip)")
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    from paper_2504_08930_b200 import build
    build.build()
    c = datagen.CONFIGS[a.config]
    B, K = c["batch"], c["k"]
    t = time.time()
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], seed=a.seed, device="cuda")
    gen_s = time.time() - t
    pool = datagen.make_queries(c["N"], c["d"], c["nlist"], (a.warmup + a.batches) * B, seed=a.seed, stream=2,
                                alpha=c["alpha"], device="cuda")
    Qd = torch.from_numpy(pool).cuda().reshape(-1, B, c["d"])
    G = a.G
    owners = None
    if a.deal == "traffic":
        Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 4096, seed=a.seed, stream=1, alpha=c["alpha"],
                                  device="cuda")
        cnt = datagen.access_counts(ix.centroids, Qc, c["nprobe"], device="cuda")
        owners = vlr.deal_owners(ix.list_offsets, np.arange(c["nlist"], dtype=np.int32), G, counts=cnt)
    hs = [vlr.Index.from_arrays(ix, rank=r, world=G, hot_owner=owners) for r in range(G)]
    h1 = vlr.Index.from_arrays(ix)
    for h in hs + [h1]:
        h.reserve(B, c["nprobe"], K)
    s = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        return e

    rows = []
    xs = []  # per batch: (x1_all, x2_all), replayed by the pipelined single-rank pass
    for b in range(a.warmup + a.batches):
        Q = Qd[b]
        # backlog the stream (~5 ms spin) so every launch of the batch is queued before the first event
        # fires: the events then time device work only, not the host's enqueue of the staged calls
        torch.cuda._sleep(a.backlog_cycles)
        e1 = []
        x1 = []
        for h in hs:
            e0 = ev()
            x1.append(h.coarse_stage1(Q, c["nprobe"], stream=s))
            e1.append((e0, ev()))
        x1_all = torch.stack(x1)
        e2, x2 = [], []
        for h in hs:
            e0 = ev()
            x2.append(h.coarse_stage2(Q, c["nprobe"], x1_all, stream=s))
            e2.append((e0, ev()))
        x2_all = torch.stack(x2)
        xs.append((x1_all, x2_all))
        e3, parts = [], []
        for h in hs:
            h.set_profiling(2)
            e0 = ev()
            parts.append(h.search_stage3(Q, c["nprobe"], K, x2_all, stream=s))
            e3.append((e0, ev()))
        e0 = ev()
        mi, md = vlr.merge_partials(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]), stream=s)
        em = (e0, ev())
        torch.cuda.synchronize()
        scan = [h.stage_times(0)["scan"] for h in hs]
        for h in hs:
            h.set_profiling(0)
        # single-GPU reference on the same batch: bitwise equality + its stage breakdown
        h1.set_profiling(1)
        ids1, d1, m1, p1 = h1.search(Q, c["nprobe"], K, sync=True)
        st1 = h1.stage_times(0)
        h1.set_profiling(0)
        same = bool(torch.equal(ids1, mi) and torch.equal(d1, md) and torch.equal(p1, parts[0][3]))
        if b < a.warmup:
            continue
        t1 = [x.elapsed_time(y) for x, y in e1]
        t2 = [x.elapsed_time(y) for x, y in e2]
        t3 = [x.elapsed_time(y) for x, y in e3]
        rows.append(dict(t1=t1, t2=t2, t3=t3, scan=scan, merge=em[0].elapsed_time(em[1]), same=same, single=st1))
    T1, T2, T3, SC = (np.array([r[k] for r in rows]) for k in ("t1", "t2", "t3", "scan"))
    nonscan = T1 + T2 + T3 - SC  # [batches, G] ms
    single = {k: float(np.mean([r["single"][k] for r in rows])) for k in rows[0]["single"]}
    out = {
        "tool": "tools/shard_model.py", "config": a.config, "G": G, "deal": a.deal, "batch": B, "nprobe": c["nprobe"], "k": K,
        "batches": a.batches, "gen_s": round(gen_s, 1),
        "bitwise_equal_to_single_gpu": all(r["same"] for r in rows),
        "per_rank_ms": {"stage1_mean": float(T1.mean()), "stage2_mean": float(T2.mean()),
                        "stage3_minus_scan_mean": float((T3 - SC).mean()), "scan_mean": float(SC.mean()),
                        "scan_max_rank_mean": float(SC.max(1).mean()),
                        "nonscan_mean": float(nonscan.mean()), "nonscan_max_rank_mean": float(nonscan.max(1).mean()),
                        "step_kernels_max_rank_mean": float((T1 + T2 + T3).max(1).mean())},
        "merge_ms": float(np.mean([r["merge"] for r in rows])),
        "single_gpu_stage_ms": single,
        "model": "step(G) = max over ranks of (stage1 + stage2 + stage3) + 3 all-gathers (x1 nq*np*4 B, x2 "
                 "nq*np*16 B, results nq*k*16 B per rank; NVLink latency, not measurable on one GPU) + K8 merge",
    }
    if a.pipe_reserve:
        out["pipelined_rank"] = pipelined_rank(a, c, hs, Qd, xs, int(np.argmax((T1 + T2 + T3).mean(0))))
    print(json.dumps(out), flush=True)


def pipelined_rank(a, c, hs, Qd, xs, r):
    """One rank's step with cross-batch pipelining (vlr_set_pipeline(2, R)): rank r's staged calls of
    consecutive batches alternate over two streams; the exchanges are replaced by the gathered x1_all /
    x2_all the serial pass produced (zero-latency transport), so the loop holds exactly rank r's kernels
    (+ two small D2D copies of the gathered slabs per batch). Device ms per batch from CUDA events around
    the whole loop; R = SMs the scan leaves to the other stream's coarse stage."""
    B, K = c["batch"], c["k"]
    h = hs[r]
    n = a.warmup + a.batches
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]

    def loop(alt):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ss[0]):
            torch.cuda._sleep(2 * a.backlog_cycles)  # backlog: the whole loop is enqueued before e0 fires
        e0.record(ss[0])
        ss[1].wait_event(e0)
        for b in range(n):
            st = ss[b % 2] if alt else ss[0]
            h.coarse_stage1(Qd[b], c["nprobe"], stream=st)
            h.coarse_stage2(Qd[b], c["nprobe"], xs[b][0], stream=st)
            h.search_stage3(Qd[b], c["nprobe"], K, xs[b][1], stream=st)
        ss[0].wait_stream(ss[1])
        e1.record(ss[0])
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    res = {"rank": r}
    h.set_pipeline(1, 0)
    loop(False)
    res["serial_ms"] = min(loop(False) for _ in range(3))
    for R in [int(x) for x in a.pipe_reserve.split(",")]:
        h.set_pipeline(2, R)
        loop(True)
        res[f"pipelined_R{R}_ms"] = min(loop(True) for _ in range(3))
    h.set_pipeline(1, 0)
    res["how"] = pipelined_rank.__doc__.split("\n")[0]
    return res


if __name__ == "__main__":
    main()
