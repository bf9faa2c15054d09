"""Per-stage device times for a few batch sizes on a generated config (diagnostics)."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--N", type=int, default=None)
p.add_argument("--batches", default="1,8,32,256")
p.add_argument("--nprobe", type=int, default=None)
p.add_argument("--lib", default=None, help="comma-separated alternative libvlr.so paths (tools/variants.py); "
                                          "'product' = the in-tree library")
p.add_argument("--reps", type=int, default=10)
a = p.parse_args()
c = dict(datagen.CONFIGS[a.config])
if a.N:
    c["N"] = a.N
npb = a.nprobe or c["nprobe"]
ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
pool = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], 4096, stream=2, device="cuda")).cuda()
PRODUCT = vlr.LIB_PATH
for libp in (a.lib or "product").split(","):
    vlr.LIB_PATH = PRODUCT if libp == "product" else libp
    vlr._lib = None
    h = vlr.Index.from_arrays(ix)
    for B in [int(x) for x in a.batches.split(",")]:
        for i in range(3):
            h.search(pool[i * B:(i + 1) * B], npb, 10, sync=True)
        h.set_profiling(True)
        res = []
        for i in range(a.reps):
            j = i % max(1, 4096 // B)
            h.search(pool[j * B:(j + 1) * B], npb, 10, sync=True)
            res.append(h.stage_times())
        h.set_profiling(False)
        mean = {k: round(float(np.mean([r[k] for r in res])) * 1000, 1) for k in res[0]}
        print(json.dumps({"lib": libp, "batch": B, "nprobe": npb, "stage_us": mean,
                          "total_us": round(sum(mean.values()), 1)}), flush=True)
    h.close()
