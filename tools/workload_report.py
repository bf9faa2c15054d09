"""Workload characterisation of a generated config.

For one BASELINE config, on one GPU:
  * list-size statistics of the k-means lists (max/mean, coefficient of variation);
  * access skew: share of the probes falling on the top-20% clusters (P:180:
    ~0.60 for Wiki-All, > 0.93 for ORCAS) for calibration streams at several
    Zipf alpha (nprobe of the config, 10k queries);
  * recall@10 of the library's search at nprobe 1..512 against
      - exact flat search over all N float vectors (fp32, ground truth of the
        query batch accumulated during generation), and
      - exhaustive PQ (the exact top-10 over all N PQ reconstructions
        c_l + yhat_i, decoded on the GPU in chunks; configs up to --pq-gt-max-n
        vectors): the quantity of reading A14, monotone in nprobe per query.
One JSON line on stdout.

  python tools/workload_report.py --config C2
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def exhaustive_pq_gt(ix, Q, k=10, chunk=1 << 16):
    """top-k over all N reconstructions (fp32 GEMM, tooling; ties unresolved)."""
    dev = "cuda"
    C = torch.from_numpy(ix.centroids).to(dev)
    cb = torch.from_numpy(ix.codebooks).to(dev)
    m, ksub, dsub = cb.shape
    q = torch.from_numpy(Q).to(dev)
    qn = (q * q).sum(1)
    best_d = torch.full((len(Q), k), float("inf"), device=dev)
    best_i = torch.full((len(Q), k), -1, dtype=torch.int64, device=dev)
    offs = ix.list_offsets
    lists = np.repeat(np.arange(ix.nlist), np.diff(offs))
    ids = torch.from_numpy(ix.ids).to(dev)
    jj = torch.arange(m, device=dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for a in range(0, ix.N, chunk):
            b = min(a + chunk, ix.N)
            codes = torch.from_numpy(ix.codes[a:b]).to(dev).long()
            if ix.nbits == 4:
                lo, hi = codes & 15, codes >> 4
                codes = torch.stack([lo, hi], 2).reshape(b - a, -1)[:, :m]
            xh = cb[jj[None, :], codes].reshape(b - a, m * dsub)
            if ix.by_residual:
                xh = xh + C[torch.from_numpy(lists[a:b]).to(dev)]
            dd = (xh * xh).sum(1)[None, :] - 2.0 * (q @ xh.T) + qn[:, None]
            vd, vi = torch.topk(dd, min(k, b - a), dim=1, largest=False)
            cd = torch.cat([best_d, vd], 1)
            ci = torch.cat([best_i, ids[a:b][vi]], 1)
            o = torch.topk(cd, k, dim=1, largest=False).indices
            best_d, best_i = torch.gather(cd, 1, o), torch.gather(ci, 1, o)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return best_i.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--nq", type=int, default=256)
    ap.add_argument("--seed", type=int, default=2504_08930)
    ap.add_argument("--alphas", default="0.6,0.8,1.0,1.2,1.4,1.6")
    ap.add_argument("--pq-gt-max-n", type=int, default=40_000_000)
    a = ap.parse_args()
    import datagen
    import paper_2504_08930_b200 as vlr
    from paper_2504_08930_b200 import build
    build.build()
    c = datagen.CONFIGS[a.config]
    N, d, L, m = c["N"], c["d"], c["nlist"], c["m"]
    t = time.time()
    Q = datagen.make_queries(N, d, L, a.nq, seed=a.seed, stream=2, alpha=c["alpha"], device="cuda")
    ix = datagen.make_index(N, d, L, m, seed=a.seed, device="cuda", gt_queries=Q)
    gen_s = time.time() - t
    sizes = ix.list_sizes
    out = {"tool": "tools/workload_report.py", "config": a.config, "N": N, "d": d, "nlist": L, "m": m,
           "gen_s": round(gen_s, 1),
           "list_sizes": {"mean": float(sizes.mean()), "max_over_mean": float(sizes.max() / sizes.mean()),
                          "cv": float(sizes.std() / sizes.mean()), "empty": int((sizes == 0).sum())}}
    skew = {}
    for al in [float(x) for x in a.alphas.split(",")]:
        Qc = datagen.make_queries(N, d, L, 10_000, seed=a.seed, stream=1, alpha=al, device="cuda")
        cnt = datagen.access_counts(ix.centroids, Qc, c["nprobe"], device="cuda")
        hot50 = datagen.hot_from_mass(cnt, 0.5)
        skew[str(al)] = {"top20_share": datagen.topk_share(cnt), "lists_for_50pct_mass": float(len(hot50) / L)}
    out["access_skew"] = {"nprobe": c["nprobe"], "calibration_queries": 10_000, "by_alpha": skew}
    h = vlr.Index.from_arrays(ix)
    Qd = torch.from_numpy(Q).cuda()
    gt_pq = exhaustive_pq_gt(ix, Q) if N <= a.pq_gt_max_n else None
    rec_exact, rec_pq = {}, {}
    for npb in [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]:
        if npb > L:
            break
        ids = h.search(Qd, npb, 10, sync=True)[0].cpu().numpy()
        rec_exact[str(npb)] = float(np.mean([len(set(g.tolist()) & set(t_.tolist())) / 10
                                             for g, t_ in zip(ids, ix.gt_ids)]))
        if gt_pq is not None:
            rec_pq[str(npb)] = float(np.mean([len(set(g.tolist()) & set(t_.tolist())) / 10
                                              for g, t_ in zip(ids, gt_pq)]))
    h.close()
    out["recall_at_10"] = {"queries": a.nq, "vs_exact_flat": rec_exact,
                           "vs_exhaustive_pq": rec_pq if gt_pq is not None else None,
                           "exhaustive_pq_how": "top-10 over all N reconstructions c_l + yhat_i (fp32 GEMM on the "
                                                "GPU, tooling)" if gt_pq is not None else
                           f"skipped (N > {a.pq_gt_max_n}: one full decode of the index per report)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
