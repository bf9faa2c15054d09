"""Plain-scan device time (CUDA events around K6, profiling mode 2) of one library at a config: median
over 30 searches of one batch rotation. python tools/scan_ab.py [product|VARIANT] [--config C4]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", default="product")
    ap.add_argument("--config", default="C4")
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    if a.lib != "product":
        vlr.LIB_PATH = os.path.join(ROOT, "tools", "_variants", a.lib, "libvlr.so")
    c = datagen.CONFIGS[a.config]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
    Q = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], 4 * c["batch"], stream=2,
                                              device="cuda")).cuda().reshape(4, c["batch"], c["d"])
    h = vlr.Index.from_arrays(ix)
    h.set_profiling(2)
    ms = []
    for i in range(34):
        h.search(Q[i % 4], c["nprobe"], c["k"], sync=True)
        if i >= 4:
            ms.append(h.stage_times(0)["scan"])
    h.close()
    print(json.dumps({"lib": a.lib, "scan_ms_median": float(np.median(ms)), "scan_ms_min": float(np.min(ms))}))


if __name__ == "__main__":
    main()
