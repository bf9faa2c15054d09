"""Run one search configuration (for compute-sanitizer / debugging)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--N", type=int, default=100_000)
p.add_argument("--d", type=int, default=128)
p.add_argument("--nlist", type=int, default=1024)
p.add_argument("--m", type=int, default=16)
p.add_argument("--nq", type=int, default=24)
p.add_argument("--nprobe", type=int, default=64)
p.add_argument("--k", type=int, default=10)
a = p.parse_args()
ix = datagen.make_index(a.N, a.d, a.nlist, a.m)
Q = datagen.make_queries(a.N, a.d, a.nlist, a.nq, stream=2)
h = vlr.Index.from_arrays(ix)
ids, dist, miss, probes = h.search(torch.from_numpy(Q).cuda(), a.nprobe, a.k, sync=True)
torch.cuda.synchronize()
print("ok", ids[0].tolist(), dist[0].tolist())
