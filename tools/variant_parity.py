"""Bitwise check of a tuning variant of libvlr.so (tools/_variants/NAME) against the product library:
each runs in its own process on the same seeded C1-sized index and queries (plain, hot subset, G = 4
shard-only staged search), results compared exactly. python tools/variant_parity.py NAME"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, out):
    import torch
    sys.path.insert(0, ROOT)
    import datagen
    import paper_2504_08930_b200 as vlr
    if lib != "product":
        vlr.LIB_PATH = os.path.join(ROOT, "tools", "_variants", lib, "libvlr.so")
    ix = datagen.make_index(200_000, 128, 1024, 16, seed=11)
    Q = torch.from_numpy(datagen.make_queries(200_000, 128, 1024, 256, seed=11, stream=2)).cuda()
    res = {}
    h = vlr.Index.from_arrays(ix)
    for npb in (16, 64):
        ids, dist, miss, prb = h.search(Q, npb, 10, sync=True)
        res[f"ids{npb}"], res[f"dist{npb}"] = ids.cpu().numpy(), dist.cpu().numpy()
    h.close()
    h = vlr.Index.from_arrays(ix, hot=np.arange(0, 1024, 3))
    ids, dist, miss, prb = h.search(Q, 32, 10, sync=True)
    res["hot_ids"], res["hot_dist"] = ids.cpu().numpy(), dist.cpu().numpy()
    h.close()
    hs = [vlr.Index.from_arrays(ix, rank=r, world=4) for r in range(4)]
    x1 = torch.stack([hh.coarse_stage1(Q, 32) for hh in hs])
    x2 = torch.stack([hh.coarse_stage2(Q, 32, x1) for hh in hs])
    parts = [hh.search_stage3(Q, 32, 10, x2) for hh in hs]
    for r, p in enumerate(parts):
        res[f"g4_ids{r}"], res[f"g4_dist{r}"] = p[0].cpu().numpy(), p[1].cpu().numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    name = sys.argv[1]
    outs = {}
    for lib in ("product", name):
        out = f"/tmp/vp_{lib}.npz"
        subprocess.run([sys.executable, __file__, "--child", lib, out], check=True)
        outs[lib] = np.load(out)
    a, b = outs["product"], outs[name]
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print({"variant": name, "arrays": len(a.files), "bitwise_equal": not bad, "differ": bad})
    sys.exit(1 if bad else 0)
