"""Sustained-load comparison of libvlr variants (diagnostics): for each lib,
`steps` back-to-back 256-query searches at C4 on one stream, per-search CUDA
event times; reports the mean of the first 20 and of the last 100 searches
(power capping shows up as a drift between the two)."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--steps", type=int, default=300)
p.add_argument("--lib", default="product")
p.add_argument("--rounds", type=int, default=2)
p.add_argument("--cool", type=float, default=5.0)
a = p.parse_args()
c = datagen.CONFIGS[a.config]
ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
B = c["batch"]
pool = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], 16 * B, stream=2, device="cuda")).cuda()
PRODUCT = vlr.LIB_PATH
hs = {}
for libp in a.lib.split(","):
    vlr.LIB_PATH = PRODUCT if libp == "product" else libp
    vlr._lib = None
    hs[libp] = (vlr._lib, vlr.Index.from_arrays(ix))
    hs[libp] = (vlr.lib(), hs[libp][1])
s = torch.cuda.current_stream()
for r in range(a.rounds):
    for libp, (L, h) in hs.items():
        vlr._lib = L
        h.reserve(B, c["nprobe"], 10)
        outs = [torch.empty(B, 10, dtype=torch.int64, device="cuda"), torch.empty(B, 10, device="cuda"),
                torch.empty(B, c["nprobe"], dtype=torch.uint8, device="cuda"),
                torch.empty(B, c["nprobe"], dtype=torch.int32, device="cuda")]
        time.sleep(a.cool)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        torch.cuda.synchronize()
        for i in range(a.steps):
            ev[i][0].record(s)
            h.search(pool[(i % 16) * B:(i % 16 + 1) * B], c["nprobe"], 10, out=outs, stream=s)
            ev[i][1].record(s)
        torch.cuda.synchronize()
        lat = np.array([x.elapsed_time(y) for x, y in ev])
        print(json.dumps({"round": r, "lib": libp, "first20_ms": round(float(lat[:20].mean()), 4),
                          "last100_ms": round(float(lat[-100:].mean()), 4), "mean_ms": round(float(lat.mean()), 4)}),
              flush=True)
