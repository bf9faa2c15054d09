"""Debug: the sharded coarse stage vs the single-GPU path on C1 (x1 rows, candidates, probes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

c = datagen.CONFIGS["C1"]
ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"])
Q = datagen.make_queries(c["N"], c["d"], c["nlist"], 20, stream=2)
Qd = torch.from_numpy(Q).cuda()
np_, G = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 4
h1 = vlr.Index.from_arrays(ix)
ref = h1.search(Qd, np_, 10, sync=True)
hs = [vlr.Index.from_arrays(ix, rank=r, world=G) for r in range(G)]
x1 = torch.stack([h.coarse_stage1(Qd, np_) for h in hs])
torch.cuda.synchronize()
C = torch.from_numpy(ix.centroids).cuda().double()
q = Qd.double()
dt = (C * C).sum(1)[None, :] - 2 * q @ C.T  # fp64 emulation (filter = this +- Delta)
T = (c["nlist"] + 127) // 128
for r in range(G):
    lo, hi = min(c["nlist"], r * T // G * 128), min(c["nlist"], (r + 1) * T // G * 128)
    exp = torch.sort(dt[0, lo:hi]).values[:np_].cpu().numpy()
    got = np.sort(x1[r, 0].cpu().numpy())
    n = min(len(exp), np_)
    print("rank", r, "range", lo, hi, "max|x1-exp| over", n, float(np.abs(got[:n] - exp[:n]).max()) if n else None,
          "x1 inf count", int(np.isinf(got).sum()), "first", got[:3], exp[:3])
x2 = torch.stack([h.coarse_stage2(Qd, np_, x1) for h in hs])
torch.cuda.synchronize()
e = x2.view(torch.uint8).cpu().numpy().reshape(G, 20, np_, 16)
ls = e[..., 8:12].copy().view(np.int32)[..., 0]
print("valid x2 entries per rank (q0):", [(int((ls[r, 0] >= 0).sum())) for r in range(G)])
outs = [h.search_stage3(Qd, np_, 10, x2) for h in hs]
torch.cuda.synchronize()
pr = outs[0][3].cpu().numpy()
rp = ref[3].cpu().numpy()
print("probes equal:", np.array_equal(pr, rp))
for qq in range(3):
    if not np.array_equal(pr[qq], rp[qq]):
        print("q", qq, "sharded", pr[qq][:12], "... -1 count", int((pr[qq] < 0).sum()))
        print("q", qq, "single ", rp[qq][:12])
        miss = sorted(set(rp[qq].tolist()) - set(pr[qq].tolist()))
        print("  missing from sharded:", miss[:20], "owners", [min(G - 1, (l // 128) * G // T) for l in miss[:20]])
