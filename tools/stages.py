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
a = p.parse_args()
c = dict(datagen.CONFIGS[a.config])
if a.N:
    c["N"] = a.N
npb = a.nprobe or c["nprobe"]
ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
h = vlr.Index.from_arrays(ix)
pool = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], 4096, stream=2, device="cuda")).cuda()
for B in [int(x) for x in a.batches.split(",")]:
    for i in range(3):
        h.search(pool[i * B:(i + 1) * B], npb, 10, sync=True)
    h.set_profiling(True)
    res = []
    for i in range(10):
        h.search(pool[i * B:(i + 1) * B], npb, 10, sync=True)
        res.append(h.stage_times())
    h.set_profiling(False)
    mean = {k: round(float(np.mean([r[k] for r in res])) * 1000, 1) for k in res[0]}
    print(json.dumps({"batch": B, "nprobe": npb, "stage_us": mean, "total_us": round(sum(mean.values()), 1)}))
