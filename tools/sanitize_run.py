"""Driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on C1-sized inputs.

Runs every search path once, small: the plain search (K1 one-CTA filter,
K2, K3a/K3b, K4b, K5 on its side stream, K6, K7), the early-release search
(NEXT-4: REL scan + resident merger CTA, rows in pinned host memory), the
staged sharded coarse stage (G = 2 shard-only handles; K3b merges by rank), the large-k path,
the pipelined search (two workspace slots on two streams)
(DUMP scan + k_select_large + large merge), a 4-bit index, and -- selected by
the environment of the run -- the K1 variants (VLR_FILTER_CLUSTER,
VLR_FILTER_PAIR, VLR_FILTER_PERSISTENT). Exits non-zero if a result differs
from the plain search (the sanitizer's own exit code reports its findings).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import datagen
    import paper_2504_08930_b200 as vlr
    torch.cuda.set_device(0)
    ix = datagen.make_index(20_000, 64, 256, 16, seed=31)
    Q = torch.from_numpy(datagen.make_queries(20_000, 64, 256, 24, seed=31, stream=2)).cuda()
    h = vlr.Index.from_arrays(ix)
    a = h.search(Q, 16, 10, sync=True)
    ok = True
    # NEXT-4 release path
    ids, dist, _, _, _ = h.search_release(Q, 16, 10)
    ok &= torch.equal(ids, a[0].cpu()) and torch.equal(dist, a[1].cpu())
    # large k
    big = h.search(Q, 64, 100, sync=True)
    ref64 = h.search(Q, 64, 10, sync=True)
    ok &= torch.equal(big[0][:, :10], ref64[0]) and torch.equal(big[1][:, :10], ref64[1])
    # cross-batch pipelining: two workspace slots, searches alternating over two streams, scan reserve
    h.set_pipeline(2, 8)
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [h.search(Q, 16, 10, stream=ss[i % 2]) for i in range(4)]
    torch.cuda.synchronize()
    ok &= all(torch.equal(o[0], a[0]) and torch.equal(o[1], a[1]) for o in outs)
    h.close()
    # sharded coarse stage, 2 shard-only handles, exchanges by stacking
    hs = [vlr.Index.from_arrays(ix, rank=r, world=2) for r in range(2)]
    x1 = torch.stack([hh.coarse_stage1(Q, 16) for hh in hs])
    x2 = torch.stack([hh.coarse_stage2(Q, 16, x1) for hh in hs])
    parts = [hh.search_stage3(Q, 16, 10, x2) for hh in hs]
    mi, md = vlr.merge_partials(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]))
    torch.cuda.synchronize()
    ok &= torch.equal(mi, a[0]) and torch.equal(md, a[1]) and torch.equal(parts[0][3], a[3])
    for hh in hs:
        hh.close()
    # 4-bit index
    i4 = datagen.make_index(8_000, 32, 64, 16, seed=33, nbits=4)
    h4 = vlr.Index.from_arrays(i4)
    h4.search(torch.from_numpy(datagen.make_queries(8_000, 32, 64, 8, seed=33, stream=2)).cuda(), 8, 10, sync=True)
    h4.close()
    torch.cuda.synchronize()
    print("SANITIZE_RUN", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
