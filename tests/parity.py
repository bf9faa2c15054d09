"""GPU-vs-oracle comparison rules R1-R4.

Test infrastructure (imports oracle/). Used by tests/ and by bench.py's
sampled parity check at full size.
"""
from __future__ import annotations

import numpy as np

import oracle

REL = 1e-5       # BASELINE.json north_star: "distances within 1e-5 relative in fp32"
FLOOR = 0.25     # absolute floor 1e-5 * 0.25 * ||q||^2 (DESIGN reading A11)


def tol(ref, qn2):
    # |ref|: inner-product distances (-<q, x>, NEXT-3) are negative
    return REL * np.maximum(np.abs(ref), FLOOR * qn2)


def check(index, Q, gpu, orc, hot=None, idmap=None, qsel=None, max_report=5, ref=None):
    """Compare GPU outputs with oracle outputs on the queries `qsel` (rows of
    Q; default all). gpu/orc: dicts with ids, dist, miss, probes (numpy,
    row-aligned with qsel). ref: optional precomputed dist_ref of the GPU's
    valid (id >= 0) entries in row-major order (a multi-rank check assembles it
    from the ranks that hold the codes). Returns a list of failure strings
    (empty = pass).
    """
    errs = []
    qsel = np.arange(len(Q)) if qsel is None else np.asarray(qsel)
    Qs = Q[qsel].astype(np.float64)
    qn2 = (Qs * Qs).sum(1)
    # R1: probes and mask bit-exact
    if gpu.get("probes") is not None and not np.array_equal(gpu["probes"], orc["probes"]):
        bad = np.nonzero((gpu["probes"] != orc["probes"]).any(1))[0]
        errs.append(f"R1 probes differ on {len(bad)} queries, first {qsel[bad[:max_report]].tolist()}")
    if not np.array_equal(gpu["miss"], orc["miss"]):
        bad = np.nonzero((gpu["miss"] != orc["miss"]).any(1))[0]
        errs.append(f"R1 miss mask differs on {len(bad)} queries")
    k = orc["ids"].shape[1]
    gids, gd = gpu["ids"], gpu["dist"].astype(np.float64)
    # R4: ascending, padding identical
    if np.any(np.diff(np.where(np.isinf(gd), np.inf, gd), axis=1) < 0):
        errs.append("R4 GPU distances not non-decreasing")
    if not np.array_equal(gids < 0, orc["ids"] < 0):
        bad = np.nonzero((gids < 0) != (orc["ids"] < 0))[0]
        errs.append(f"R4 padding differs on queries {qsel[np.unique(bad)[:max_report]].tolist()}")
    if np.any(np.isinf(gd) != (gids < 0)):
        errs.append("R4 padding slots must be exactly (-1, +inf)")
    # R2: every returned distance vs dist_ref
    valid = gids >= 0
    rows = np.repeat(qsel[:, None], k, 1)[valid]
    if ref is None:
        ref = oracle.dist_ref(index, Q, rows, gids[valid], idmap=idmap)
    if np.any(np.isnan(ref)):
        errs.append("R2 GPU returned unknown ids")
    qn2v = np.repeat(qn2[:, None], k, 1)[valid]
    dev = np.abs(gd[valid] - ref)
    t = tol(ref, qn2v)
    if np.any(dev > t):
        i = int(np.argmax(dev / t))
        errs.append(f"R2 distance off: max |gpu-ref|/tol = {float((dev / t)[i]):.3g} (gpu {gd[valid][i]!r}, ref {ref[i]!r})")
    # candidates must come from probed, resident lists of that query
    if idmap is not None and valid.any():
        ok, lst, _ = idmap.locate(gids[valid])
        prb = np.repeat(np.arange(len(qsel))[:, None], k, 1)[valid]
        hotm = np.ones(index.nlist, bool) if hot is None else np.isin(np.arange(index.nlist), hot)
        probed = np.array([l in set(orc["probes"][r].tolist()) for r, l in zip(prb, lst)]) if len(lst) < 200000 else None
        if probed is not None and not probed.all():
            errs.append("GPU returned a vector from a list that was not probed")
        if not hotm[lst].all():
            errs.append("GPU returned a vector from a non-resident list")
    # R3: id sets
    for r in range(len(qsel)):
        od = orc["dist"][r]
        oid = orc["ids"][r]
        nvalid = int((oid >= 0).sum())
        if nvalid == 0:
            continue
        rk = od[nvalid - 1]
        rk1 = orc["kth1"][r] if nvalid == k else np.inf
        tk = tol(rk, qn2[r])
        gset = set(gids[r][gids[r] >= 0].tolist())
        oset = set(oid[oid >= 0].tolist())
        if rk1 - rk > tk:
            if gset != oset:
                errs.append(f"R3 id set differs for query {int(qsel[r])}: missing {sorted(oset - gset)[:4]}")
        else:
            must = set(oid[(oid >= 0) & (od < rk - tk)].tolist())
            if not must <= gset:
                errs.append(f"R3 query {int(qsel[r])} lost a clear winner")
        if len(errs) > 20:
            break
    # R3 (tie branch) second half: every GPU id within r_k + tol
    row_of = np.repeat(np.arange(len(qsel))[:, None], k, 1)[valid]
    nv = (orc["ids"] >= 0).sum(1)
    rk_all = np.array([orc["dist"][r][max(n - 1, 0)] if n else np.inf for r, n in enumerate(nv)])
    lim = rk_all[row_of] + tol(rk_all[row_of], qn2[row_of])
    full = nv[row_of] == k
    if np.any(full & (ref > lim)):
        errs.append("R3 GPU returned an id beyond r_k + tol")
    return errs


def merge_partials_np(parts, k):
    """Merge rank-partial oracle results (dicts with ids, dist, kth1; the same
    probes/miss on every rank) into the result over the union of the ranks'
    lists: the k smallest by (dist, id), padded (-1, +inf); kth1 = the
    (k+1)-th smallest of the union of every rank's top-k and (k+1)-th (
    the hybrid = monolithic rule S:473)."""
    nq = parts[0]["ids"].shape[0]
    # a probe is a miss iff no rank holds it (each rank's oracle saw only its own lists as resident)
    out = dict(ids=np.full((nq, k), -1, np.int64), dist=np.full((nq, k), np.inf), kth1=np.full(nq, np.inf),
               probes=parts[0]["probes"], miss=np.minimum.reduce([p["miss"] for p in parts]))
    big = np.iinfo(np.int64).max
    for q in range(nq):
        i = np.concatenate([p["ids"][q] for p in parts])
        dv = np.concatenate([p["dist"][q] for p in parts])
        o = np.lexsort((np.where(i < 0, big, i), dv))
        sel = o[:k]
        out["ids"][q], out["dist"][q] = i[sel], dv[sel]
        extra = np.concatenate([dv[o[k:]], [p["kth1"][q] for p in parts]])
        out["kth1"][q] = extra.min() if len(extra) else np.inf
    return out
