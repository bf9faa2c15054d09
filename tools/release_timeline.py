"""NEXT-4 device timeline (variant build with -DVLR_SCAN_TRACE, tools/variants.py scantrace
VLR_SCAN_TRACE=1): for release searches at a config (default C4, batch 256), the scan CTAs' end times,
the first k_release_rest CTA start, the merger's end, and every query's release time (device
globaltimer at its flag store) with who released it (merger / rest kernel); for the plain search the
scan CTAs' end and the K7 time. All times in us from the first scan CTA's start. One JSON line.

  python tools/release_timeline.py --config C4"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--runs", type=int, default=6)
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    vlr.LIB_PATH = os.path.join(ROOT, "tools", "_variants", "scantrace", "libvlr.so")
    c = datagen.CONFIGS[a.config]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
    Q = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, device="cuda")).cuda()
    L = vlr.lib()
    L.vlr_debug_scan_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.vlr_debug_rel_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    h = vlr.Index.from_arrays(ix)
    nq = c["batch"]
    out = {"config": a.config, "batch": nq, "release": [], "plain": []}
    for it in range(a.runs):
        # plain: scan CTAs + stage times (K7)
        h.set_profiling(1)
        h.search(Q, c["nprobe"], c["k"], sync=True)
        st = h.stage_times(0)
        t = np.zeros((148, 6), np.uint64)
        assert L.vlr_debug_scan_trace(t.ctypes.data, 148) == 0
        t = t.astype(np.int64)
        t0 = t[:, 0].min()
        end = (t[:, 1] - t0) / 1e3
        if it >= 2:
            out["plain"].append({"scan_end_us": [float(end.min()), float(np.median(end)), float(end.max())],
                                 "k7_us": 1e3 * st["rank_merge"], "scan_event_us": 1e3 * st["scan"]})
        # release
        h.set_profiling(0)
        assert L.vlr_debug_rel_trace(None, 0, None) == 0
        h.search_release_launch(Q, c["nprobe"], c["k"])
        torch.cuda.synchronize()
        t = np.zeros((147, 6), np.uint64)
        assert L.vlr_debug_scan_trace(t.ctypes.data, 147) == 0
        t = t.astype(np.int64)
        r = np.zeros((nq, 2), np.uint64)
        misc = np.zeros(4, np.uint64)
        assert L.vlr_debug_rel_trace(r.ctypes.data, nq, misc.ctypes.data) == 0
        r = r.astype(np.int64)
        misc = misc.astype(np.int64)
        t0 = t[:, 0].min()
        end = (t[:, 1] - t0) / 1e3
        rel = (r[:, 0] - t0) / 1e3
        who = r[:, 1]
        if it >= 2:
            out["release"].append({
                "scan_end_us": [float(end.min()), float(np.median(end)), float(end.max())],
                "rest_start_us": float((misc[0] - t0) / 1e3), "merger_end_us": float((misc[1] - t0) / 1e3),
                "before_fork_us": float((misc[2] - t0) / 1e3), "after_join_us": float((misc[3] - t0) / 1e3),
                "release_us": {"p10": float(np.percentile(rel, 10)), "p50": float(np.percentile(rel, 50)),
                               "p90": float(np.percentile(rel, 90)), "p99": float(np.percentile(rel, 99)),
                               "max": float(rel.max())},
                "by_merger": int((who == 1).sum()), "by_rest": int((who == 2).sum()),
                "after_scan_end": int((rel > end.max()).sum())})
    h.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
