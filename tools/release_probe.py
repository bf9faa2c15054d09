"""NEXT-4 probe: device scan time of the release-mode scan vs the plain scan
on one index (default C2 shape), printed as JSON; run under ncu to compare
the two kernels. Usage: python tools/release_probe.py [N d nlist m nprobe batch]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [10_000_000, 768, 4096, 96, 64, 256]
N, d, L, m, P, B = args
ix = datagen.make_index(N, d, L, m, device="cuda")
h = vlr.Index.from_arrays(ix)
Q = torch.from_numpy(datagen.make_queries(N, d, L, B * 4, stream=2)).cuda().reshape(4, B, d)
h.set_profiling(2)
res = {"plain": [], "release": []}
for it in range(6):
    for i in range(4):
        h.search(Q[i], P, 10, sync=True)
        res["plain"].append(h.stage_times(0)["scan"])
        h.search_release(Q[i].contiguous(), P, 10)
        torch.cuda.synchronize()
        res["release"].append(h.stage_times(0)["scan"])
print(json.dumps({k: float(np.median(v[4:])) for k, v in res.items()} | {"waves": os.environ.get("VLR_RELEASE_WAVES")}))
