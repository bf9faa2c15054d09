"""Candidate-band diagnostics for the coarse filter: for a batch of
queries, how many centroids pass {dt <= theta' + 2 Delta*} (the K3 workload),
versus theta~ (the exact nprobe'-th filter value) instead of the group-minima
theta', and versus the ideal nprobe'. The filter values are emulated in torch
(fp16-rounded, power-of-two-scaled operands, fp32 GEMM)."""
import argparse
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--nq", type=int, default=256)
a = p.parse_args()
c = datagen.CONFIGS[a.config]
g = None
C = datagen.layout(c["N"], c["d"], c["nlist"], device="cuda")["centroids"]
C = torch.as_tensor(C, device="cuda", dtype=torch.float32)
Q = torch.from_numpy(datagen.make_queries(c["N"], c["d"], c["nlist"], a.nq, stream=2, device="cuda")).cuda()
d = c["d"]
np_ = c["nprobe"]


def f16s(x, rowwise):
    m = x.abs().amax(dim=1, keepdim=True) if rowwise else x.abs().amax().reshape(1, 1)
    e = torch.where(m > 0, 14 - torch.frexp(m).exponent, torch.zeros_like(m, dtype=torch.int32)).clamp(-60, 60)
    s = torch.pow(2.0, e.float())
    return (x * s).half().float() / s


cq, qq = f16s(C, False), f16s(Q, True)
torch.backends.cuda.matmul.allow_tf32 = False
cn = (C.double() ** 2).sum(1).float()
dt = cn[None, :] - 2 * (qq @ cq.T)
qn = Q.double().norm(dim=1).float()
cmax = float(C.double().norm(dim=1).max())
u = 2.0 ** -24
e_dot = 2 * 2.0 ** -11 + 2.0 ** -22 + 1.01 * d * 2.0 ** -23
delta = 2 * (2 * (e_dot + 2 * u) * qn * cmax + 4 * u * (cmax ** 2 + qn ** 2))
L = C.shape[0]
gmin = dt.view(a.nq, L // 32, 32).amin(2)
theta_p = gmin.sort(1).values[:, np_ - 1]
theta_t = dt.sort(1).values[:, np_ - 1]
n_p = (dt <= (theta_p + 2 * delta)[:, None]).sum(1).float()
n_t = (dt <= (theta_t + 2 * delta)[:, None]).sum(1).float()
exact = ((Q.double()[:, None, :] - C.double()[None, :, :]) ** 2).sum(2) if L * a.nq * d < 2e9 else None
out = {"config": a.config, "nq": a.nq, "nprobe": np_, "delta_mean": float(delta.mean()),
       "cand_mean_theta_groupmin": float(n_p.mean()), "cand_max_theta_groupmin": float(n_p.max()),
       "cand_mean_theta_exact": float(n_t.mean()), "theta_gap_mean": float((theta_p - theta_t).mean()),
       "dist_spread_top_np": float((dt.sort(1).values[:, np_ - 1] - dt.sort(1).values[:, 0]).mean())}
print(json.dumps(out))
