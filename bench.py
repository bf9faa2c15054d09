#!/usr/bin/env python
"""bench.py -- batched IVF-PQ hot-partition search throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl vlr|reference]

One step = one batch search (coarse quantizer K1-K3, route K4, LUT K5, ADC
scan K6, merges K7/K8) over `batch` synthetic queries of BASELINE.json's
128M-vector config (C4 by default), inputs resident in HBM. N > 1: launched
by torchrun, one rank per GPU; hot lists dealt over the ranks, every rank
runs the SPMD search and the partial top-k are merged over NCCL (strong
scaling: the index and the batch are fixed). Rank 0 prints ONE JSON line.
--impl reference times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

UNIT = "queries/s"


def metric_name(B, nprobe, k):
    return f"IVF-PQ search queries/s (batch {B}, nprobe {nprobe}, k {k})"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="vlr", choices=["vlr", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--N", type=int, default=None, help="override vector count (testing only)")
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--nprobe", type=int, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--hot-mass", type=float, default=1.0)
    p.add_argument("--alpha", type=float, default=None)
    p.add_argument("--seed", type=int, default=2504_08930)
    p.add_argument("--metric", type=int, default=0, choices=[0, 1], help="0 squared L2, 1 inner product (NEXT-3)")
    p.add_argument("--by-residual", type=int, default=1, choices=[0, 1], help="1 residual PQ codes (NEXT-3: 0)")
    p.add_argument("--nbits", type=int, default=8, choices=[4, 8], help="bits per PQ sub-code (NEXT-3: 4)")
    p.add_argument("--m", type=int, default=None, help="override PQ sub-quantizer count")
    p.add_argument("--no-oracle", action="store_true")
    p.add_argument("--oracle-seconds", type=float, default=15.0)
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--ncu", action="store_true", help="short run for ncu: no e2e/oracle/clocks")
    p.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampling")
    p.add_argument("--dump-lat", default=None, help="diagnostics: write per-step latencies (ms) and scan times here")
    p.add_argument("--dry-run-1gpu", action="store_true",
                   help="N > 1 plumbing on ONE shared GPU: gloo process group, shard-only handles, the staged "
                        "sharded search with the exchanges over gloo (host), vlr_merge_partials; timing is not a "
                        "multi-GPU number")
    p.add_argument("--exchange", default="p2p", choices=["p2p", "nccl", "staged"],
                   help="N > 1 transport: p2p = the NVLink peer-exchange kernels (vlr_p2p_*; default), nccl = "
                        "ncclAllGather on the search stream, staged = the staged C-ABI with the caller's transport "
                        "(dry run only)")
    p.add_argument("--lat-batches", type=int, default=1000,
                   help="latency pass: CUDA-graph closed-loop batches per batch size (SURVEY §8(d): >= 1000)")
    p.add_argument("--sustained-s", type=float, default=10.0, help="sustained pass length (s), batch of the config")
    p.add_argument("--pipeline", type=int, default=-1, choices=[-1, 0, 1],
                   help="1: cross-batch pipelining (vlr_set_pipeline: two workspace slots, batches alternate over "
                        "two streams, batch i+1's coarse stage beside batch i's scan); 0: one stream; -1 (default): "
                        "on at N > 1 only (one GPU: no gain measured, DESIGN.md §5b)")
    p.add_argument("--scan-reserve", type=int, default=-1,
                   help="SMs the scan leaves to the other stream's coarse stage when pipelining (-1: default)")
    p.add_argument("--deal", default="paper", choices=["paper", "traffic"],
                   help="N > 1 hot-list deal: the paper's size round-robin (P:339, default) or the traffic-aware "
                        "LPT deal on size x access count of the calibration stream (NEXT-2, vlr_deal_owners)")
    p.add_argument("--sweep-out", default=None,
                   help="also run the C5 batch x nprobe sweep on the same index and write JSON lines here")
    return p.parse_args()


# ---------------------------------------------------------------- helpers
def default_reserve(world):
    """SMs the scan leaves to the next batch's coarse stage when pipelining (tools/overlap_probe.py)."""
    return 8 if world == 1 else 16


def cfg_of(a):
    import datagen
    c = dict(datagen.CONFIGS[a.config])
    for key in ("N", "batch", "nprobe", "k", "alpha", "m"):
        v = getattr(a, key)
        if v is not None:
            c[key] = v
    c["hot_mass"] = a.hot_mass
    c["metric"] = a.metric
    c["by_residual"] = a.by_residual
    c["nbits"] = a.nbits
    return c


def workload_name(c, name):
    hot = "all lists resident" if c["hot_mass"] >= 1 else f"hot set = {c['hot_mass']:.0%} of access mass"
    var = ""
    if c.get("metric", 0) == 1 or c.get("by_residual", 1) == 0:
        var = ", " + ("inner product" if c.get("metric", 0) == 1 else "L2") + \
              ("" if c.get("by_residual", 1) else ", non-residual PQ")
    return (f"{name}: {c['N'] / 1e6:g}M x d{c['d']}, IVF{c['nlist']}, PQ{c['m']}x{c.get('nbits', 8)}, nprobe {c['nprobe']}, "
            f"k {c['k']}, batch {c['batch']}, Zipf alpha {c['alpha']}, {hot}{var}")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def f16_peak():
    """Dense fp16 tensor peak (K1 runs kind::f16): the measured cuBLAS bf16 burst
    figure (MEASURED_PEAKS.json; fp16 and bf16 share the nominal 2.25 PF/s rate,
    B200_PROFILING.md), else the guide's fallback 1.59 PF/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), "of measured (MEASURED_PEAKS.json bf16_tflops; fp16 = bf16 nominal rate)"
    except Exception:
        return 1590.0, "of fallback (B200_PROFILING.md 1.59 PFLOP/s bf16/fp16 burst)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) == 7]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_median": float(np.median(pw)) if pw else None,
                "power_w_max": max(pw) if pw else None}


def dist_setup(dry=False):
    """One process per GPU (torchrun env). dry: every rank on cuda:0 with a gloo group."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if dry else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _coll_dev():
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=_coll_dev(), dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_stack(t, world):
    """rank-ordered stack [world, *t.shape] of every rank's CUDA tensor t (the
    dry run's transport: host memory over gloo)."""
    import torch
    import torch.distributed as dist
    c = t.cpu() if _coll_dev() == "cpu" else t.contiguous()
    parts = [torch.empty_like(c) for _ in range(world)]
    dist.all_gather(parts, c)
    return torch.stack(parts).cuda()


def all_objects(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def gen_index(c, seed, rank, world, hot=None, gt_queries=None, owner_table=None):
    """Generate this rank's shard of the synthetic index on the GPU (TOOLING).
    VLR_GEN_CACHE=<dir> reuses arrays saved by an earlier process of the same
    command sequence (never relied on for timing: only generation time)."""
    import datagen
    sizes = datagen.list_sizes(c["N"], c["d"], c["nlist"], seed, device="cuda")
    owned = None
    if world > 1:
        own = owner_table if owner_table is not None else datagen.deal_owners(
            sizes, np.arange(c["nlist"]) if hot is None else hot, world)
        owned = own == rank
    t = time.time()
    cache = os.environ.get("VLR_GEN_CACHE")
    key = f"g3_{c['N']}_{c['d']}_{c['nlist']}_{c['m']}_{seed}_{world}_{rank}_{'all' if hot is None else len(hot)}"
    if owner_table is not None:
        import hashlib
        key += f"_own{hashlib.md5(np.ascontiguousarray(owner_table).tobytes()).hexdigest()[:10]}"
    key += f"_mt{c['metric']}_br{c['by_residual']}_nb{c['nbits']}"
    if gt_queries is not None:
        import hashlib
        key += f"_gt{len(gt_queries)}_{hashlib.md5(gt_queries.tobytes()).hexdigest()[:10]}"
    names = ["centroids", "codebooks", "list_offsets", "ids", "codes"] + (["gt_ids", "gt_dist"] if gt_queries is not None
                                                                          else [])
    if cache:
        path = os.path.join(cache, key)
        if os.path.exists(os.path.join(path, "done")):
            f = {n: np.ascontiguousarray(np.load(os.path.join(path, n + ".npy"), mmap_mode="r")) for n in names}
            gt, gtd = f.pop("gt_ids", None), f.pop("gt_dist", None)
            ix = datagen.IndexArrays(d=c["d"], nlist=c["nlist"], m=c["m"], seed=seed, metric=c["metric"],
                                     by_residual=c["by_residual"], nbits=c["nbits"], **f)
            if gt is not None:
                ix.gt_ids, ix.gt_dist = gt, gtd
            return ix, time.time() - t
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], seed=seed, device="cuda", owned=owned,
                            gt_queries=gt_queries, metric=c["metric"], by_residual=c["by_residual"],
                            nbits=c["nbits"])
    if cache:
        os.makedirs(path, exist_ok=True)
        for n in names:
            np.save(os.path.join(path, n + ".npy"), getattr(ix, n))
        open(os.path.join(path, "done"), "w").close()
    return ix, time.time() - t


def calib_hot(c, seed):
    """Hot set from a calibration stream (seed stream 1, disjoint from the test
    stream): shortest prefix of the access ranking holding
    hot_mass of the accesses (TOOLING)."""
    import datagen
    if c["hot_mass"] >= 1.0:
        return None, None
    ncal = 10_000
    C = datagen.centroids(c["N"], c["d"], c["nlist"], seed, device="cuda")
    Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], ncal, seed=seed, stream=1, alpha=c["alpha"], device="cuda")
    counts = datagen.access_counts(C, Qc, c["nprobe"], device="cuda", metric=c["metric"])
    return datagen.hot_from_mass(counts, c["hot_mass"]), counts


# ---------------------------------------------------------------- reference arm
def run_reference(a):
    """The oracle, as it stands, on host cores: each step a bounded sample of
    the workload (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    import datagen
    import oracle
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    c = cfg_of(a)
    oracle.build()
    hot, _ = calib_hot(c, a.seed)
    ix, gen_s = gen_index(c, a.seed, 0, 1, hot=hot)
    B = c["batch"]
    pool = datagen.make_queries(c["N"], c["d"], c["nlist"], (a.warmup + a.steps) * B, seed=a.seed, stream=2,
                                alpha=c["alpha"], device="cuda")
    cores = oracle.default_threads()
    # sample size per step: ~1 s of oracle work on the host cores
    t = time.time()
    oracle.search(ix, pool[:cores], c["nprobe"], c["k"], hot=hot, nthreads=cores)
    per_q = (time.time() - t) / cores
    S = int(max(1, min(B, round(max(1.0, 2.0 * cores * per_q) / per_q))))
    S = max(cores, (S // cores) * cores) if S >= cores else S
    times = []
    for i in range(a.warmup + a.steps):
        Q = pool[i * B:i * B + S]
        t = time.time()
        oracle.search(ix, Q, c["nprobe"], c["k"], hot=hot, nthreads=cores)
        if i >= a.warmup:
            times.append(time.time() - t)
    tot = sum(times)
    val = a.steps * S / tot
    line = {"impl": "reference", "metric": metric_name(B, c["nprobe"], c["k"]), "value": val, "unit": UNIT, "n_gpus": 1, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded clustered embeddings, Zipf queries)",
            "config": {"workload": workload_name(c, a.config), "seed": a.seed, "sample_queries_per_step": S},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{S} of the {B} queries of each step's batch, oracle/oracle.c fp64, OpenMP"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gen_s": gen_s}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import datagen
    import paper_2504_08930_b200 as vlr
    from paper_2504_08930_b200 import build as vbuild

    dry = bool(a.dry_run_1gpu)
    rank, world, local = dist_setup(dry)
    dry = dry and world > 1
    if world != a.gpus and rank == 0:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if rank == 0:
        vbuild.build()
    barrier(world)
    c = cfg_of(a)
    B, NP, K = c["batch"], min(c["nprobe"], c["nlist"]), c["k"]
    # ---- index (tooling), shard residency (vlr_load_index)
    t0 = time.time()
    hot, counts = calib_hot(c, a.seed)
    # query stream (test stream) first: ground truth of the first timed batch is
    # accumulated while the index vectors are generated (N = 1 only)
    pool = datagen.make_queries(c["N"], c["d"], c["nlist"], (a.warmup + a.steps) * B, seed=a.seed, stream=2,
                                alpha=c["alpha"], device="cuda")
    # ground truth of the first timed batch, accumulated while the vectors are generated (N > 1: each rank
    # over its own lists, merged below)
    gtq = pool[a.warmup * B:(a.warmup + 1) * B] if not a.ncu else None
    # hot-list deal (N > 1): the paper's round-robin by size, or the traffic-aware LPT deal on the calibration
    # stream's access counts (owner per cluster; -1 = cold)
    owner_table, hot_owner = None, None
    if world > 1 and a.deal == "traffic":
        sizes0 = datagen.list_sizes(c["N"], c["d"], c["nlist"], a.seed, device="cuda")
        offs0 = np.concatenate([[0], np.cumsum(sizes0)]).astype(np.int64)
        if counts is None:
            C0 = datagen.centroids(c["N"], c["d"], c["nlist"], a.seed, device="cuda")
            Qc0 = datagen.make_queries(c["N"], c["d"], c["nlist"], 10_000, seed=a.seed, stream=1, alpha=c["alpha"],
                                       device="cuda")
            counts = datagen.access_counts(C0, Qc0, c["nprobe"], device="cuda")
        hot_ids = np.arange(c["nlist"], dtype=np.int32) if hot is None else np.asarray(hot, np.int32)
        hot_owner = vlr.deal_owners(offs0, hot_ids, world, counts=counts)
        owner_table = np.full(c["nlist"], -1, np.int32)
        owner_table[hot_ids] = hot_owner
    ix, gen_s = gen_index(c, a.seed, rank, world, hot=hot, gt_queries=gtq, owner_table=owner_table)
    nccl_id = None
    if world > 1 and not dry:
        import torch.distributed as dist
        obj = [vlr.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t1 = time.time()
    h = vlr.Index.from_arrays(ix, hot=hot, hot_owner=hot_owner, rank=rank, world=world, device=local, nccl_id=nccl_id)
    load_s = time.time() - t1
    owners = h.owners()
    exp_own = owner_table if owner_table is not None else datagen.deal_owners(
        ix.list_sizes, np.arange(c["nlist"]) if hot is None else hot, world)
    assert np.array_equal(owners, exp_own), "owner table differs from the documented deal"
    info = h.info()
    # ---- queries (test stream), resident in HBM
    Qdev = torch.from_numpy(pool).cuda().reshape(a.warmup + a.steps, B, c["d"])
    xchg = a.exchange if world > 1 else "none"
    if dry and xchg == "nccl":
        xchg = "p2p"  # NCCL refuses two ranks on one device
    # cross-batch pipelining: not for the staged dry-run transport (host-synchronous gloo
    # exchanges) nor NCCL (the communicator serialises its collectives across streams)
    pipe = (a.pipeline == 1 or (a.pipeline < 0 and world > 1)) and xchg in ("none", "p2p")
    reserve = a.scan_reserve if a.scan_reserve >= 0 else default_reserve(world)
    if pipe:
        h.set_pipeline(2, reserve)
    h.reserve(B, NP, K)
    if xchg == "p2p":  # inboxes IPC-mapped across the ranks: exchanges inside the kernels, no NCCL calls
        if dry:
            mine = h.p2p_export()
            handles = all_objects(mine, world)
            h.p2p_connect(handles)
        else:
            h.p2p_setup()
        barrier(world)
    outs = [(torch.empty(B, K, dtype=torch.int64, device="cuda"), torch.empty(B, K, device="cuda"),
             torch.empty(B, NP, dtype=torch.uint8, device="cuda"), torch.empty(B, NP, dtype=torch.int32, device="cuda"))
            for _ in range(a.steps)]
    stream = torch.cuda.current_stream()
    streams = [stream, torch.cuda.Stream()] if pipe else [stream, stream]

    def step(Q, out, stream=stream):
        """one batch search: the collective NCCL search, or (dry run) the staged sharded search with the
        exchanges over gloo and the partial top-k merged by vlr_merge_partials"""
        if xchg != "staged":
            h.search(Q, c["nprobe"], K, out=out, stream=stream)
            return
        ids, dd, miss, prb = h.search_staged(Q, c["nprobe"], K, lambda t: gather_stack(t, world), stream=stream)
        mi, md = vlr.merge_partials(gather_stack(ids, world), gather_stack(dd, world), stream=stream)
        out[0].copy_(mi)
        out[1].copy_(md)
        out[2].copy_(miss)
        out[3].copy_(prb)

    for i in range(a.warmup):
        step(Qdev[i], outs[i % 2], streams[i % 2])
    torch.cuda.synchronize()
    launches = h.last_launch_count
    clocks = Clocks(local)
    if not a.ncu and not a.no_clocks:
        clocks.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    # ---- the timed region: K batches back to back (pipelined: alternating over two streams, two workspace
    # slots; each batch's whole hot path runs inside the region), device-timed from the first launch to
    # the completion of the last batch on both streams
    e0.record(stream)
    streams[1].wait_event(e0)
    for i in range(a.steps):
        step(Qdev[a.warmup + i], outs[i], streams[i % 2])
    stream.wait_stream(streams[1])
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop() if not a.ncu and not a.no_clocks else None
    ms_total = allmax(e0.elapsed_time(e1), world)
    # ---- serial pass on one stream with the scan on every SM (reserve 0): per-batch latency (launch ->
    # completion, no queueing behind another batch) and the scan kernel's own duration for the roofline
    # (CUDA events around the scan on its launch stream; in the pipelined region the scan of batch i+1
    # starts on SMs while batch i's still runs, so its event interval is not its duration)
    if pipe:
        h.set_pipeline(2, 0)
    for i in range(2):
        step(Qdev[i], outs[0])
    torch.cuda.synchronize()
    h.set_profiling(2)  # only the two events around the scan
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    es0.record(stream)
    for i in range(a.steps):
        ev[i][0].record(stream)
        step(Qdev[a.warmup + i], outs[i])
        ev[i][1].record(stream)
    es1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms_serial = allmax(es0.elapsed_time(es1), world)
    lat = np.array([s.elapsed_time(e) for s, e in ev])
    nrec = min(a.steps, 64)
    scan_ms = np.array([h.stage_times(back=j)["scan"] for j in range(nrec)][::-1])  # oldest first
    if a.dump_lat and rank == 0:
        with open(a.dump_lat, "w") as f:
            json.dump({"lat_ms": lat.tolist(), "scan_ms_last64": scan_ms.tolist()}, f)
    # ---- stage breakdown: a separate, untimed pass with events at every stage boundary
    h.set_profiling(1)
    nprof = min(a.steps, 16)
    for i in range(nprof):
        step(Qdev[a.warmup + i], outs[i])
    torch.cuda.synchronize()
    h.set_profiling(False)
    stages = [h.stage_times(back=j) for j in range(nprof)]
    stage_mean = {k2: float(np.mean([s[k2] for s in stages])) for k2 in stages[0]}
    # ---- algorithmic scan bytes: sum over owned hot probes of n_l * (m + 4)
    sizes = ix.list_sizes
    per_vec = (c["m"] * c["nbits"] + 7) // 8 + 4
    step_bytes, hit = [], []
    for i in range(a.steps):
        prb = outs[i][3].cpu().numpy()
        miss = outs[i][2].cpu().numpy()
        own = owners[prb] == rank
        step_bytes.append(float((sizes[prb] * own).sum()) * per_vec)
        hit.append(1.0 - miss.mean(axis=1))
    step_bytes = np.array(step_bytes)
    bytes_rec = step_bytes[a.steps - nrec:]
    achieved = float(bytes_rec.sum() / (scan_ms.sum() * 1e-3) / 1e9)
    peak, peak_src = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_scan_latest.json")) as f:
            tj = json.load(f)
        same = (tj.get("config") == a.config and tj.get("batch") == B and tj.get("nbits", 8) == c["nbits"]
                and tj.get("m", datagen.CONFIGS[a.config]["m"]) == c["m"] and tj.get("metric", 0) == c["metric"])
        if same:
            traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass
    # ---- e2e through the C-ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not a.ncu and not dry:
        ne = a.e2e_steps or a.steps
        hq = torch.from_numpy(pool[: B * ne].reshape(ne, B, c["d"]).copy()).pin_memory()
        hid = torch.empty(B, K, dtype=torch.int64).pin_memory()
        hd = torch.empty(B, K, dtype=torch.float32).pin_memory()
        hm = torch.empty(B, NP, dtype=torch.uint8).pin_memory()
        # the serving pipeline below alternates two streams with two workspace slots when the timed region
        # does (N > 1); on one GPU it stays on one stream: two slots there measured slower (127-136k vs
        # 139-143k q/s, profiles/r02/bench_c4_{o,p}.json vs bench_c4_m.json: the next batch's kernels start
        # inside the persistent scan's tail and its static split loses balance)
        e2e_pipe = pipe
        e2e_streams = [stream, torch.cuda.Stream()] if e2e_pipe else [stream, stream]
        if e2e_pipe:
            h.set_pipeline(2, reserve)
        for i in range(min(3, ne)):
            h.search_host_ptr(hq[i].data_ptr(), B, c["nprobe"], K, hid.data_ptr(), hd.data_ptr(), hm.data_ptr(), None)
        barrier(world)
        t = time.perf_counter()
        for i in range(ne):
            h.search_host_ptr(hq[i].data_ptr(), B, c["nprobe"], K, hid.data_ptr(), hd.data_ptr(), hm.data_ptr(), None)
        el_block = allmax(time.perf_counter() - t, world)
        # serving pipeline: vlr_search_host_async back to back (pipelined: alternating over two streams,
        # two workspace slots; each step's H2D, search and D2H enqueued; one synchronisation at the end),
        # per-step output buffers
        pid_ = torch.empty(ne, B, K, dtype=torch.int64).pin_memory()
        pdd_ = torch.empty(ne, B, K, dtype=torch.float32).pin_memory()
        pmm_ = torch.empty(ne, B, NP, dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        barrier(world)
        t = time.perf_counter()
        for i in range(ne):
            h.search_host_ptr_async(hq[i].data_ptr(), B, c["nprobe"], K, pid_[i].data_ptr(), pdd_[i].data_ptr(),
                                    pmm_[i].data_ptr(), None, stream=e2e_streams[i % 2])
        torch.cuda.synchronize()
        el = allmax(time.perf_counter() - t, world)
        e2e_same = bool(torch.equal(pid_[ne - 1], hid) and torch.equal(pdd_[ne - 1], hd))
        e2e = {"value": ne * B / el, "unit": UNIT, "h2d_bytes_per_step": B * c["d"] * 4,
               "d2h_bytes_per_step": B * K * 12 + B * NP,
               "how": ("vlr_search_host_async per step (pinned host queries in, ids/dist/miss out), "
                       + ("alternating over two streams with two workspace slots (copies overlap the other "
                          "batch's kernels)" if e2e_pipe else "back to back on one stream")
                       + "; wall clock from the first call to the final synchronisation"),
               "blocking_value": ne * B / el_block,
               "blocking_how": "vlr_search_host (synchronous: H2D, search, D2H, stream sync) per step",
               "async_equal_to_blocking": e2e_same}
        if e2e_pipe:
            h.set_pipeline(2, 0)
    # ---- NEXT-4 early per-query release (the paper's dispatcher ablation, Fig. 14):
    # host-observed latency of each query from launch to its release flag, against the same batches
    # searched with the batch barrier (launch -> stream sync). Untimed by the headline metric.
    release = None
    if world == 1 and not a.ncu:
        release = release_leg(a, c, h, Qdev, outs, K)
    # ---- latency pass: CUDA-graph closed loop of >= 1000 batches per batch size, p50/p99 over
    # batches; then a sustained run of the config's batch (q/s after the power cap settles)
    latency = None
    if world == 1 and not a.ncu and a.lat_batches > 0:
        latency = latency_leg(a, c, h, pool, K, local)
    # ---- NEXT-2: GPU access profile of a calibration stream -> per-rank work share of the paper's deal vs
    # the traffic-aware deal at G = 2/4/8 (over the timed batches' probes), and a full-shard refresh time
    shards = None
    if world == 1 and not a.ncu:
        shards = shard_leg(a, c, h, ix, hot, outs, K)
    # ---- oracle: cpu_baseline + sampled full-size parity (rank 0, N = 1)
    cpu = None
    par = None
    if rank == 0 and world == 1 and not a.no_oracle and not a.ncu:
        cpu, par = oracle_leg(a, c, ix, hot, pool, outs)
    if world > 1 and not a.no_oracle and not a.ncu:
        par = dist_parity_leg(a, c, ix, hot, pool, outs, owners, rank, world)
    recall = None
    if getattr(ix, "gt_ids", None) is not None:
        # the generator regenerates all N vectors for the ground truth on every rank (also when it encodes
        # only the rank's lists or the hot subset), so each rank's GT is the global one: no merge
        gt_ids = ix.gt_ids
        got = outs[0][0].cpu().numpy()
        kk = min(10, K)
        r = [len(set(g[:kk].tolist()) & set(t[:kk].tolist())) / kk for g, t in zip(got, gt_ids)]
        recall = {"recall_at_10": float(np.mean(r)), "queries": len(r),
                  "ground_truth": "exact fp32 flat search over all N float vectors (regenerated during index "
                                  "generation"
                                  + ("; the search covers the GPU-resident hot lists only" if hot is not None else "")
                                  + "), first timed batch"}
    # ---- coarse contraction (K1, tcgen05 kind::f16): 2*B*L*d flops per launch; the stage
    # also holds the tiny q-prep kernel, so this understates K1's own rate slightly
    cf_ms = float(stage_mean["coarse_filter"]) if stage_mean else None
    coarse_roof = None
    if cf_ms:
        tp, tp_src = f16_peak()
        fl = 2.0 * B * c["nlist"] * c["d"]
        tfs = fl / (cf_ms * 1e-3) / 1e12
        # bytes K1 moves: the pre-tiled fp16 centroid stream (L x d8 x 2, read once per batch) + the fp32 filter
        # matrix it writes (B x L x 4; most of it is consumed by K2 from L2) + the fp16 queries
        cbytes = c["nlist"] * ((c["d"] + 7) // 8 * 8) * 2 + B * c["nlist"] * 4 + B * c["d"] * 2
        coarse_roof = {"bound": "tensor", "dtype": "f16 (power-of-two scaled operands, fp32 accumulate)", "achieved": tfs, "peak": tp, "unit": "TFLOP/s",
                       "frac": tfs / tp, "peak_source": tp_src, "flops_per_launch": fl,
                       "ms_per_launch": cf_ms, "hbm_gbs": cbytes / (cf_ms * 1e-3) / 1e9,
                       "hbm_bytes_per_launch": cbytes,
                       "hbm_bytes_how": "fp16 centroid tiles (L*d8*2) + fp32 filter writes (B*L*4) + fp16 queries",
                       "kernel": "k_qprep + k_filter_tc (K1)"}
    # ---- residency (P:214 hit rate eta_q = 1 - sum_p miss / nprobe'; rho = resident share of the index)
    hq = np.concatenate(hit)
    sizes_all = ix.list_sizes
    hot_ids = np.arange(c["nlist"]) if hot is None else np.asarray(hot)
    residency = {"lists": float(len(hot_ids) / c["nlist"]),
                 "vectors": float(sizes_all[hot_ids].sum() / max(1, sizes_all.sum())),
                 "eta_q": {"mean": float(hq.mean()), "p10": float(np.percentile(hq, 10)),
                           "p50": float(np.percentile(hq, 50)), "p90": float(np.percentile(hq, 90)),
                           "all_hit_share": float((hq == 1.0).mean()), "all_miss_share": float((hq == 0.0).mean())},
                 "calibration_mass": c["hot_mass"]}
    value = a.steps * B / (ms_total * 1e-3)
    # per-rank work share (the size-based deal balances bytes, not traffic)
    shares = np.array(all_objects(float(step_bytes.sum()), world))
    work_share = float(shares.max() / max(shares.mean(), 1.0))
    if rank == 0:
        line = {
            "metric": metric_name(B, c["nprobe"], K), "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_total / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "dry_run": dry, "data": "synthetic (seeded clustered embeddings, Zipf-skewed queries; generated on the GPU)",
            "config": {"workload": workload_name(c, a.config), "N": c["N"], "d": c["d"], "nlist": c["nlist"], "m": c["m"],
                       "nprobe": c["nprobe"], "k": K, "batch": B, "alpha": c["alpha"], "hot_mass": c["hot_mass"],
                       "seed": a.seed,
                       "parallelism": (f"hot-list shards x{world} ("
                                       + ("size round-robin deal, P:339" if a.deal == "paper"
                                          else "traffic-aware LPT deal") + "), centroid-sharded coarse stage, "
                                       + {"p2p": "NVLink peer-exchange kernels (IPC-mapped inboxes, epoch flags)",
                                          "nccl": "NCCL all-gathers + GPU merge-select",
                                          "staged": "staged C-ABI, exchanges over gloo through host memory"}[xchg]
                                       + (", all ranks on ONE GPU (dry run)" if dry else "")) if world > 1
                                      else "one GPU",
                       "l2": "inputs larger than L2 (index %.1f GB/GPU, %.2f GB scanned per batch)" % (
                           info["bytes_on_device"] / 1e9, float(step_bytes.mean()) / 1e9)},
            "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
            "lat_ms_top5": [round(float(x), 4) for x in np.sort(lat)[::-1][:5]],
            "gpu_launches": int(launches * a.steps),
            "pipeline": {"on": pipe, "slots": 2 if pipe else 1, "scan_reserve_sms": reserve if pipe else 0,
                         "serial_value": a.steps * B / (ms_serial * 1e-3), "serial_ms_per_step": ms_serial / a.steps,
                         "how": "timed region: batches alternate over two streams (vlr_set_pipeline(2, R)); "
                                "serial pass: one stream, R = 0 (p50/p99 and the scan roofline come from it)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": "k_scan (K6 ADC scan)", "peak_source": peak_src,
                         "bytes_per_launch": float(bytes_rec.mean()), "ms_per_launch": float(scan_ms.mean())},
            "coarse_roofline": coarse_roof,
            "stage_ms": stage_mean,
            "stage_ms_source": "separate untimed pass (16 searches) with CUDA events at every stage boundary; "
                               "the timed region records only the two events around the scan",
            "hit_rate_mean": float(np.mean(np.concatenate(hit))),
            "work_share_max_over_mean": work_share,
            "residency": residency,
            "e2e": e2e, "clocks": clk, "cpu_baseline": cpu, "parity_sample": par, "recall": recall,
            "release": release,
            "latency": latency,
            "shards": shards,
            "gen_s": round(gen_s, 1), "load_s": round(load_s, 1),
        }
        if counts is not None:
            line["top20_share"] = datagen.topk_share(counts)
        print(json.dumps(line), flush=True)
    if a.sweep_out:
        sweep(a, c, h, pool, world, rank, gt=getattr(ix, "gt_ids", None))
    h.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def shard_leg(a, c, h, ix, hot, outs, K):
    import torch
    import datagen
    import paper_2504_08930_b200 as vlr
    B = outs[0][0].shape[0]
    ncal = 16
    Qc = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], ncal * B, seed=a.seed, stream=1,
                                               alpha=c["alpha"], device="cuda")).cuda().reshape(ncal, B, c["d"])
    counts = torch.zeros(c["nlist"], dtype=torch.int64, device="cuda")
    for i in range(ncal):
        _, _, _, prb = h.search(Qc[i].contiguous(), c["nprobe"], K, sync=True)
        h.access_counts(prb, counts)
    counts = counts.cpu().numpy()
    hot_ids = np.arange(c["nlist"], dtype=np.int32) if hot is None else np.asarray(hot, np.int32)
    sizes = ix.list_sizes.astype(np.float64)
    probes = np.concatenate([o[3].cpu().numpy().reshape(-1) for o in outs])
    per_list = np.bincount(probes, minlength=c["nlist"]).astype(np.float64) * sizes  # vectors scanned per list
    bal = {}
    for G in (2, 4, 8):
        row = {}
        for name, cnt in (("paper_round_robin", None), ("traffic_aware", counts)):
            own = np.full(c["nlist"], -1, np.int64)
            own[hot_ids] = vlr.deal_owners(ix.list_offsets, hot_ids, G, counts=cnt)
            load = np.bincount(own[own >= 0], weights=per_list[own >= 0], minlength=G)
            row[name] = float(load.max() / load.mean())
        bal[str(G)] = row
    t = time.perf_counter()
    h.update_hot_arrays(ix, hot=hot)
    reload_s = time.perf_counter() - t
    return {"work_share_max_over_mean": bal,
            "how": "vectors each rank would scan for the timed batches' probes; owners from vlr_deal_owners "
                   "(paper: size-descending round-robin, P:339; traffic-aware: LPT on size x access count of a "
                   "%d-query calibration stream profiled on the GPU with vlr_access_counts)" % (ncal * B),
            "refresh_s": reload_s,
            "refresh_how": "vlr_update_hot of this rank's whole shard (host arrays -> new device residency, swap; "
                           "the paper reports <10 s per shard, P:421)"}


def latency_leg(a, c, h, pool, K, device):
    """Per batch size B in (32, 64, 128, 256) (and the config's batch): the search captured ONCE in a CUDA
    graph (torch.cuda.graph on a side stream; the library's K5 fork/join is captured with it), replayed
    closed-loop for a.lat_batches batches; each replay's queries are copied into the graph's static input
    first (inside the replay's event pair: the latency is input-in-HBM to result-in-HBM). CUDA events around
    every replay -> p50 / p99 / p99.9 / max over >= 1000 batches; q/s = queries / summed device time.
    Then a sustained loop of the config's batch for a.sustained_s seconds (q/s of the last half, after
    the power cap settles) and, for the outlier question, the same closed loop with the nvidia-smi sampler
    running next to it."""
    import torch
    out = {"how": __doc_latency__, "by_batch": {}}
    qd = torch.from_numpy(pool).cuda()
    nb_pool = len(pool)
    NP = min(c["nprobe"], c["nlist"])
    batches = sorted({32, 64, 128, 256, c["batch"]})
    graphs = {}
    for B in batches:
        if B > nb_pool:
            continue
        h.reserve(B, NP, K)
        qin = torch.empty(B, c["d"], device="cuda")
        o = (torch.empty(B, K, dtype=torch.int64, device="cuda"), torch.empty(B, K, device="cuda"),
             torch.empty(B, NP, dtype=torch.uint8, device="cuda"), torch.empty(B, NP, dtype=torch.int32, device="cuda"))
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for i in range(3):  # eager warm-up on the capture stream (module loads, workspace)
                qin.copy_(qd[i * B % (nb_pool - B + 1):][:B])
                h.search(qin, c["nprobe"], K, out=o, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            h.search(qin, c["nprobe"], K, out=o, stream=s)
        graphs[B] = (g, qin, o, s)

    def loop(B, n, sampler=None):
        g, qin, o, s = graphs[B]
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        nstart = max(1, nb_pool // B)
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
            time.sleep(0.3)
        with torch.cuda.stream(s):
            for i in range(n):
                ev[i][0].record(s)
                j = (i % nstart) * B
                qin.copy_(qd[j:j + B])
                g.replay()
                ev[i][1].record(s)
        torch.cuda.synchronize()
        clk = sampler.stop() if sampler else None
        lat = np.array([x.elapsed_time(y) for x, y in ev])
        return lat, clk

    for B in graphs:
        lat, _ = loop(B, a.lat_batches)
        out["by_batch"][str(B)] = {"batches": len(lat), "qps": float(B * len(lat) / (lat.sum() * 1e-3)),
                                   "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
                                   "p999_ms": float(np.percentile(lat, 99.9)), "max_ms": float(lat.max()),
                                   "mean_ms": float(lat.mean()),
                                   "outlier_at_batch": [int(i) for i in np.nonzero(lat > 1.5 * np.median(lat))[0][:32]]}
    B = c["batch"]
    if B in graphs and a.sustained_s > 0:
        per = max(1e-4, out["by_batch"][str(B)]["mean_ms"] * 1e-3)
        n = int(a.sustained_s / per)
        lat, clk = loop(B, n, sampler=Clocks(device))
        half = lat[len(lat) // 2:]
        out["sustained"] = {"batch": B, "seconds": float(lat.sum() * 1e-3), "batches": int(n),
                            "qps_all": float(B * len(lat) / (lat.sum() * 1e-3)),
                            "qps_last_half": float(B * len(half) / (half.sum() * 1e-3)),
                            "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
                            "max_ms": float(lat.max()), "clocks": clk,
                            "outliers_gt_1p5x_median": int((lat > 1.5 * np.median(lat)).sum()),
                            # when they happen (device time since the loop start, s) and how long they are:
                            # periodic outliers point at power / clock management, not at the search
                            "outlier_at_s": [round(float(t), 4) for t in (np.cumsum(lat) * 1e-3)[lat > 1.5 * np.median(lat)][:32]],
                            "outlier_ms": [round(float(x), 3) for x in lat[lat > 1.5 * np.median(lat)][:32]],
                            "how": "same graph closed loop for sustained_s seconds with the nvidia-smi sampler "
                                   "(-lms 100) running; compare p99/max with by_batch (no sampler)"}
    return out


__doc_latency__ = ("torch CUDA graph of one vlr_search_async per batch size, replayed closed-loop; per replay a "
                   "D2D copy of that batch's queries into the graph input then the replay, CUDA events around both")


def release_leg(a, c, h, Qdev, outs, K):
    import torch
    R = min(a.steps, 20)
    batch_ms, q_ms, last_ms, equal = [], [], [], True
    scan_plain, scan_rel = [], []
    h.set_profiling(2)
    # untimed warm-up of both paths: the first release call on a fresh process pays one-time costs
    # (lazy module load of k_scan<REL> / k_release_merge, pinned row buffers) that are not per-query latency
    for i in range(min(a.warmup, 3)):
        h.search(Qdev[i], c["nprobe"], K, out=outs[0], sync=True)
        h.search_release(Qdev[i], c["nprobe"], K)
        torch.cuda.synchronize()
    for i in range(R):
        Q = Qdev[a.warmup + i]
        torch.cuda.synchronize()
        t0 = time.monotonic_ns()
        h.search(Q, c["nprobe"], K, out=outs[i], sync=True)
        batch_ms.append((time.monotonic_ns() - t0) / 1e6)
        scan_plain.append(h.stage_times(0)["scan"])
        torch.cuda.synchronize()
        ids, dist, _, _, t = h.search_release(Q, c["nprobe"], K)
        torch.cuda.synchronize()
        scan_rel.append(h.stage_times(0)["scan"])
        lat = (np.asarray(t, np.int64) - t.t0) / 1e6
        q_ms.append(lat)
        last_ms.append(float(lat.max()))
        equal &= bool(torch.equal(ids, outs[i][0].cpu()) and torch.equal(dist, outs[i][1].cpu()))
    h.set_profiling(False)
    ql = np.concatenate(q_ms)
    bm = np.array(batch_ms)
    return {"per_query_ms": {"mean": float(ql.mean()), "p50": float(np.percentile(ql, 50)),
                             "p99": float(np.percentile(ql, 99))},
            "batch_ms": {"mean": float(bm.mean()), "p50": float(np.percentile(bm, 50)),
                         "p99": float(np.percentile(bm, 99))},
            "last_release_ms_mean": float(np.mean(last_ms)),
            "scan_ms_device": {"batch": float(np.mean(scan_plain)), "release": float(np.mean(scan_rel))},
            "mean_latency_reduction": float(1.0 - ql.mean() / bm.mean()),
            "bitwise_equal_to_batch_search": equal, "batches": R,
            "how": "host CLOCK_MONOTONIC from launch to the query's release flag (vlr_poll_ready) vs launch to "
                   "stream completion of vlr_search on the same batch; rows in pinned host memory"}


def sweep(a, c, h, pool, world, rank, gt=None):
    """C5: batch x nprobe sweep on the loaded index (device-timed, CUDA events,
    max over ranks); one JSON line per point in --sweep-out. With ground truth
    (N = 1), each nprobe also gets recall@10 of the ground-truth batch against
    exact flat search (recall monotone in nprobe)."""
    import torch
    K = c["k"]
    recall_at = {}
    if gt is not None and rank == 0:
        Bg = c["batch"]
        qg = torch.from_numpy(pool[a.warmup * Bg:(a.warmup + 1) * Bg].copy()).cuda()
        for npb in [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]:
            ids, _, _, _ = h.search(qg, npb, 10, sync=True)
            got = ids.cpu().numpy()
            recall_at[npb] = float(np.mean([len(set(g.tolist()) & set(t[:10].tolist())) / 10
                                            for g, t in zip(got, gt)]))
    batches = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    nprobes = [16, 32, 64, 128, 256, 512]
    qd = torch.from_numpy(pool).cuda()
    lines = []
    for npb in nprobes:
        for B in batches:
            if B > len(pool):
                continue
            NP = min(npb, c["nlist"])
            h.reserve(B, NP, K)
            out = (torch.empty(B, K, dtype=torch.int64, device="cuda"), torch.empty(B, K, device="cuda"),
                   torch.empty(B, NP, dtype=torch.uint8, device="cuda"), None)
            steps = max(10, min(200, int(2000 / max(B, 1))))
            nb = len(pool) // B
            for i in range(3):
                h.search(qd[(i % nb) * B:(i % nb + 1) * B], npb, K, out=out)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            barrier(world)
            torch.cuda.synchronize()
            for i in range(steps):
                ev[i][0].record()
                h.search(qd[(i % nb) * B:(i % nb + 1) * B], npb, K, out=out)
                ev[i][1].record()
            torch.cuda.synchronize()
            lat = np.array([e0.elapsed_time(e1) for e0, e1 in ev])
            tot = allmax(float(lat.sum()), world)
            if rank == 0:
                lines.append({"batch": B, "nprobe": npb, "k": K, "n_gpus": world, "qps": steps * B / (tot * 1e-3),
                              "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
            "lat_ms_top5": [round(float(x), 4) for x in np.sort(lat)[::-1][:5]],
                              "steps": steps})
                if B == c["batch"] and npb in recall_at:
                    lines[-1]["recall_at_10"] = recall_at[npb]
    if rank == 0:
        if recall_at:
            lines.append({"recall_at_10_by_nprobe": {str(k2): v for k2, v in recall_at.items()}, "batch": c["batch"],
                          "ground_truth": "exact fp32 flat search over all N vectors, the bench's first timed batch"})
        with open(a.sweep_out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


def dist_parity_leg(a, c, ix, hot, pool, outs, owners, rank, world, S=32):
    """N > 1 sampled parity (the hybrid = monolithic rule S:473): every rank runs the
    oracle over the lists it owns (its codes are the only ones generated on it), computes dist_ref of the
    returned ids it owns, and rank 0 merges the rank partials into the oracle over all resident lists and
    checks the GPU's final rows (identical on every rank) with rules R1-R4."""
    import oracle
    from parity import check, merge_partials_np
    oracle.build()
    B = c["batch"]
    S = min(S, B)
    Qs = pool[a.warmup * B:a.warmup * B + S]
    mine = np.nonzero(owners == rank)[0].astype(np.int32)
    t = time.time()
    part = oracle.search(ix, Qs, c["nprobe"], c["k"], hot=mine, nthreads=max(1, oracle.default_threads() // 2))
    el = time.time() - t
    g = outs[0]
    gpu = dict(ids=g[0].cpu().numpy()[:S], dist=g[1].cpu().numpy()[:S], miss=g[2].cpu().numpy()[:S],
               probes=g[3].cpu().numpy()[:S])
    valid = gpu["ids"] >= 0
    rows = np.repeat(np.arange(S)[:, None], gpu["ids"].shape[1], 1)[valid]
    idmap = oracle.IdMap(ix)
    ok, lst, _ = idmap.locate(gpu["ids"][valid])
    here = ok & (owners[lst] == rank)
    ref = np.full(len(rows), np.nan)
    if here.any():
        ref[here] = oracle.dist_ref(ix, Qs, rows[here], gpu["ids"][valid][here], idmap=idmap)
    parts = all_objects(dict(part=part, ref=ref, here=here, el=el), world)
    if rank != 0:
        return None
    orc = merge_partials_np([p["part"] for p in parts], c["k"])
    ref_all = np.full(len(rows), np.nan)
    for p in parts:
        ref_all[p["here"]] = p["ref"][p["here"]]
    errs = check(ix, Qs, gpu, orc, hot=hot, idmap=idmap, ref=ref_all)
    return {"queries": S, "ranks": world,
            "rules": "R1 probes+mask bit-exact, R2 dist 1e-5 rel, R3 id sets, R4 order/padding; oracle run per "
                     "rank over its own lists and merged on rank 0 (hybrid = monolithic)",
            "pass": not errs, "errors": errs[:3], "oracle_s_max_rank": max(p["el"] for p in parts)}


def oracle_leg(a, c, ix, hot, pool, outs):
    import oracle
    from parity import check
    oracle.build()
    cores = oracle.default_threads()
    B = c["batch"]
    first = pool[a.warmup * B:(a.warmup + 1) * B]  # the first timed batch
    # size the sample to ~oracle_seconds of CPU work
    t = time.time()
    o = oracle.search(ix, first[:cores], c["nprobe"], c["k"], hot=hot, nthreads=cores)
    dt = time.time() - t
    S = int(min(B, max(cores, cores * math.floor(a.oracle_seconds / max(dt, 1e-3)))))
    t = time.time()
    o = oracle.search(ix, first[:S], c["nprobe"], c["k"], hot=hot, nthreads=cores)
    el = time.time() - t
    cpu = {"value": S / el, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"first {S} queries of the first timed batch (same index and queries), oracle/oracle.c fp64"}
    g = outs[0]
    gpu = dict(ids=g[0].cpu().numpy()[:S], dist=g[1].cpu().numpy()[:S], miss=g[2].cpu().numpy()[:S],
               probes=g[3].cpu().numpy()[:S])
    errs = check(ix, first, gpu, o, hot=hot, idmap=oracle.IdMap(ix) if ix.N <= 200_000_000 else None,
                 qsel=np.arange(S))
    par = {"queries": S, "rules": "R1 probes+mask bit-exact, R2 dist 1e-5 rel, R3 id sets, R4 order/padding",
           "pass": not errs, "errors": errs[:3]}
    return cpu, par


if __name__ == "__main__":
    main()
