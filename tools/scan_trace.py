"""K6 per-CTA timeline (variant build with -DVLR_SCAN_TRACE, tools/variants.py scantrace
VLR_SCAN_TRACE=1): kernel span, per-CTA start skew / duration / LUT-wait / segments,
and the end spread (the tail), at a config (default C4) with G shard ranks
(rank 0's shard traced). JSON on stdout.

  python tools/variants.py scantrace VLR_SCAN_TRACE=1
  python tools/scan_trace.py --config C4 --G 1
"""
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
    ap.add_argument("--G", default="1,8", help="shard counts (rank 0's shard traced)")
    ap.add_argument("--release", action="store_true", help="trace the NEXT-4 release scan (REL waves) too")
    ap.add_argument("--lib", default="scantrace", help="variant under tools/_variants/ (built with VLR_SCAN_TRACE=1)")
    ap.add_argument("--release-nowait", action="store_true",
                    help="launch the release search without waiting for the flags (VLR_REL_EXPERIMENT=1 runs)")
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    vlr.LIB_PATH = os.path.join(ROOT, "tools", "_variants", a.lib, "libvlr.so")
    c = datagen.CONFIGS[a.config]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
    Q = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, device="cuda")).cuda()
    L = vlr.lib()
    L.vlr_debug_scan_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    for G in [int(x) for x in a.G.split(",")]:
        h = vlr.Index.from_arrays(ix) if G == 1 else vlr.Index.from_arrays(ix, rank=0, world=G)
        print(json.dumps(trace(h, c, Q, L, a.config, G)), flush=True)
        if a.release:
            print(json.dumps(trace(h, c, Q, L, a.config, G, release=True, nowait=a.release_nowait)), flush=True)
        h.close()


def vlr_lib_path():
    import paper_2504_08930_b200 as vlr
    return vlr.LIB_PATH


def trace(h, c, Q, L, config, G, release=False, nowait=False):
    out = {"config": config, "G": G, "release": release, "lib": os.path.basename(os.path.dirname(vlr_lib_path())), "env": {k: v for k, v in os.environ.items()
                                                                  if k.startswith("VLR_")}, "runs": []}
    for it in range(6):
        h.set_profiling(2)
        if release and nowait:
            h.search_release_launch(Q, c["nprobe"], c["k"])
            torch.cuda.synchronize()
        elif release:
            h.search_release(Q, c["nprobe"], c["k"])
            torch.cuda.synchronize()
        else:
            h.search(Q, c["nprobe"], c["k"], sync=True)
        scan_ms = h.stage_times(0)["scan"]
        # the scan's grid: SMs - VLR_SCAN_RESERVE, and the release scan leaves one more SM to the merger CTA
        n = 148 - int(os.environ.get("VLR_SCAN_RESERVE", "0")) - (1 if release else 0)
        t = np.zeros((n, 6), np.uint64)
        assert L.vlr_debug_scan_trace(t.ctypes.data, n) == 0
        t = t.astype(np.int64)
        t0 = t[:, 0].min()
        st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        dur = en - st
        if it >= 2:
            out["runs"].append({"scan_ms_events": scan_ms, "span_us": float(en.max()),
                                "start_skew_us": [float(np.percentile(st, 50)), float(st.max())],
                                "end_us_p0_p50_p100": [float(en.min()), float(np.percentile(en, 50)), float(en.max())],
                                "dur_us_mean": float(dur.mean()), "dur_us_cv": float(dur.std() / dur.mean()),
                                "lut_wait_us_mean": float(t[:, 2].mean() / 1e3), "segments_mean": float(t[:, 3].mean()),
                                "groups_per_cta_mean": float(t[:, 5].mean()),
                                "us_per_group_mean": float((dur / np.maximum(t[:, 5], 1)).mean())})
    return out


if __name__ == "__main__":
    main()
