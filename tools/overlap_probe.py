"""Cross-batch pipelining on one GPU (vlr_set_pipeline): batches alternate
over two streams with two workspace slots, the scan's persistent grid leaving
R SMs to the other stream's coarse stage. Prints device ms/batch (CUDA events
around the whole loop) for the serial single-stream loop and the alternating
loop at each R, and whether the rows are bitwise equal.
  python tools/overlap_probe.py --config C4 --reserve 0,4,8,12,16"""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--reserve", default="0,4,8,12,16")
    ap.add_argument("--prio", type=int, default=0)
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    c = datagen.CONFIGS[a.config]
    B, K, NP = c["batch"], c["k"], min(c["nprobe"], c["nlist"])
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], seed=2504_08930, device="cuda")
    pool = datagen.make_queries(c["N"], c["d"], c["nlist"], a.batches * B, seed=2504_08930, stream=2,
                                alpha=c["alpha"], device="cuda")
    Qd = torch.from_numpy(pool).cuda().reshape(-1, B, c["d"])
    h = vlr.Index.from_arrays(ix)
    h.set_pipeline(2, 0)
    h.reserve(B, NP, K)
    outs = [[torch.empty(B, K, dtype=torch.int64, device="cuda"), torch.empty(B, K, device="cuda"),
             torch.empty(B, NP, dtype=torch.uint8, device="cuda"),
             torch.empty(B, NP, dtype=torch.int32, device="cuda")] for _ in range(a.batches)]
    ss = [torch.cuda.Stream(priority=-a.prio), torch.cuda.Stream(priority=-a.prio)]

    def run(alt):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ss[0])
        ss[1].wait_event(e0)
        for i in range(a.batches):
            j = i % 2 if alt else 0
            h.search(Qd[i], c["nprobe"], K, out=outs[i], stream=ss[j])
        ss[0].wait_stream(ss[1])
        e1.record(ss[0])
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.batches

    h.set_pipeline(1, 0)
    run(False)
    ref = [o[0].clone() for o in outs], [o[1].clone() for o in outs]
    res = {"config": a.config, "batch": B, "batches": a.batches, "prio": a.prio,
           "serial_ms": min(run(False) for _ in range(3))}
    for R in [int(x) for x in a.reserve.split(",")]:
        h.set_pipeline(2, R)
        run(True)
        ms = min(run(True) for _ in range(3))
        same = all(torch.equal(o[0], r) and torch.equal(o[1], d) for o, r, d in zip(outs, *ref))
        res[f"alt_R{R}_ms"] = ms
        res[f"alt_R{R}_bitwise"] = same
        h.set_pipeline(1, R)
        res[f"serial_R{R}_ms"] = min(run(False) for _ in range(2))
    print(json.dumps(res), flush=True)
    h.close()


if __name__ == "__main__":
    main()
