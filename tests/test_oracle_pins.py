"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names the passage / reading it follows (DESIGN.md §Oracle pins).
A plausible mistake in the oracle -- a dropped term (c_l, a sub-space), a
wrong sign or index, transposed codebook axes, a wrong tie-break, a summation
in the wrong order, an off-by-one in the list offsets, a wrong mask polarity
-- fails at least one of them.
"""
import numpy as np
import pytest

import datagen
import oracle
from conftest import fval, golden_index, load_golden


# --- hand-derived golden fixture (DESIGN readings A2/A5/A7) ---
def test_golden_tiny_hand_example():
    g = load_golden("tiny_hand.json")
    ix = golden_index(g)
    Q = np.array(g["queries"], np.float32)
    for case in g["cases"]:
        r = oracle.search(ix, Q, case["nprobe"], case["k"], hot=case["hot"])
        assert r["probes"].tolist() == case["probes"]
        assert r["miss"].tolist() == case["miss"]
        assert r["ids"].tolist() == case["ids"]
        exp = np.array([[fval(x) for x in row] for row in case["dist"]])
        assert np.array_equal(r["dist"], exp)
        if "coarse" in case:
            p, dd = oracle.coarse(Q, ix.centroids, case["nprobe"])
            assert p.tolist() == case["probes"]
            assert np.array_equal(dd, np.array(case["coarse"]))


# --- O2: sequential fp64 summation order (DESIGN reading "O2 order") -------
def test_coarse_sum_is_sequential_in_dimension_order():
    # squares (2^54, 1, 1, 1): left-to-right fp64 gives 2^54 exactly
    # (each +1 rounds away); any other order gives 2^54 + 4.
    q = np.array([[2.0 ** 27, 1, 1, 1]], np.float32)
    c = np.zeros((1, 4), np.float32)
    _, dd = oracle.coarse(q, c, 1)
    assert dd[0, 0] == 2.0 ** 54
    rev = 1.0 + 1.0 + 1.0 + 2.0 ** 54
    assert rev != 2.0 ** 54


# --- O3 special cases ---------------------------------------
def test_query_equal_to_centroid_is_first_probe(small_index):
    C = small_index.centroids
    p, dd = oracle.coarse(C[[5, 17, 40]], C, 1)
    assert p[:, 0].tolist() == [5, 17, 40]
    assert np.all(dd[:, 0] == 0.0)


def test_full_nprobe_is_sorted_permutation(small_index, small_queries):
    C = small_index.centroids
    p, dd = oracle.coarse(small_queries[:8], C, 10 ** 6)  # clamped to nlist
    assert p.shape == (8, C.shape[0])
    for row, drow in zip(p, dd):
        assert sorted(row.tolist()) == list(range(C.shape[0]))
        assert np.all(np.diff(drow) >= 0)
        ties = np.nonzero(np.diff(drow) == 0)[0]
        assert np.all(row[ties] < row[ties + 1])


def test_duplicate_centroids_ordered_by_id():
    rng = np.random.default_rng(0)
    C = rng.standard_normal((10, 8)).astype(np.float32)
    C[7] = C[2]
    C[9] = C[2]
    p, dd = oracle.coarse(C[2:3] + np.float32(0.25), C, 10)
    pos = [p[0].tolist().index(i) for i in (2, 7, 9)]
    assert pos == sorted(pos) and pos[2] - pos[0] == 2
    assert dd[0, pos[0]] == dd[0, pos[1]] == dd[0, pos[2]]


# --- O2 against a different formula (closed form ||q||^2+||c||^2-2<q,c>) ---
def test_coarse_matches_expanded_closed_form(small_index, small_queries):
    C = small_index.centroids.astype(np.float64)
    Q = small_queries.astype(np.float64)
    p, dd = oracle.coarse(small_queries, small_index.centroids, 64)
    expand = (Q * Q).sum(1)[:, None] + (C * C).sum(1)[None, :] - 2.0 * Q @ C.T
    got = np.take_along_axis(expand, p.astype(np.int64), 1)
    scale = (Q * Q).sum(1)[:, None] + (C * C).sum(1)[p]
    assert np.all(np.abs(got - dd) <= 1e-12 * scale)
    # and the probe set is the argsort of the closed form up to 1e-12 near-ties
    srt = np.sort(expand, axis=1)
    assert np.all(np.abs(srt - dd) <= 1e-12 * (1 + np.abs(srt)))


def test_coarse_translation_and_scaling(small_index):
    # integer-valued data: translation by 0.5 and scaling by 2 are exact in fp32
    rng = np.random.default_rng(1)
    C = rng.integers(-20, 20, (50, 16)).astype(np.float32)
    Q = rng.integers(-20, 20, (6, 16)).astype(np.float32)
    p0, d0 = oracle.coarse(Q, C, 50)
    p1, d1 = oracle.coarse(Q + np.float32(0.5), C + np.float32(0.5), 50)
    p2, d2 = oracle.coarse(Q * np.float32(2), C * np.float32(2), 50)
    assert np.array_equal(p0, p1) and np.array_equal(d0, d1)
    assert np.array_equal(p0, p2) and np.array_equal(d2, 4 * d0)


# --- O6: ADC by definition vs the LUT decomposition identity (reading A2) ---
def _recon(ix, pos):
    lst = np.searchsorted(ix.list_offsets, pos, side="right") - 1
    codes = ix.codes[pos].astype(np.int64)
    yhat = ix.codebooks[np.arange(ix.m)[None, :], codes].reshape(len(pos), ix.d).astype(np.float64)
    return ix.centroids[lst].astype(np.float64), yhat, lst


def test_adc_equals_lut_decomposition(small_index, small_queries):
    ix, Q = small_index, small_queries
    rng = np.random.default_rng(2)
    pos = rng.integers(0, ix.N, 400)
    qi = rng.integers(0, len(Q), 400)
    got = oracle.dist_ref(ix, Q, qi, ix.ids[pos])
    c, y, _ = _recon(ix, pos)
    q = Q[qi].astype(np.float64)
    dsub = ix.d // ix.m
    # term1 + b_i + sum_j LUT_q[j][code_ij] with LUT = -2<q_j, y_j>
    term1 = ((q - c) ** 2).sum(1)
    b = (y * y).sum(1) + 2 * (c * y).sum(1)
    lut = -2 * (q * y).reshape(-1, ix.m, dsub).sum(2).sum(1)
    ref = term1 + b + lut
    assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))


# --- Exhaustive reduction: nprobe = nlist, hot = all -> flat PQ search ------
def _flat_pq_topk(ix, Q, k):
    pos = np.arange(ix.N)
    c, y, _ = _recon(ix, pos)
    X = c + y
    Qd = Q.astype(np.float64)
    D = (Qd * Qd).sum(1)[:, None] + (X * X).sum(1)[None, :] - 2 * Qd @ X.T
    out = []
    for row in D:
        o = np.lexsort((ix.ids, row))[:k]
        out.append((ix.ids[o], row[o]))
    return out


def test_full_probe_equals_exhaustive_pq(small_index, small_queries):
    ix, Q = small_index, small_queries[:16]
    k = 10
    r = oracle.search(ix, Q, ix.nlist, k)
    flat = _flat_pq_topk(ix, Q, k + 1)
    for qi, (fid, fd) in enumerate(flat):
        assert np.allclose(r["dist"][qi], fd[:k], rtol=1e-10, atol=1e-12)
        gap = fd[k] - fd[k - 1]
        if gap > 1e-9:
            assert set(r["ids"][qi].tolist()) == set(fid[:k].tolist())
        assert abs(r["kth1"][qi] - fd[k]) <= 1e-10 * max(1.0, fd[k])
    assert np.all(r["miss"] == 0)
    assert np.all(r["ncand"] == ix.N)


# --- Exact kNN on lossless-PQ data vs sklearn brute force (library routine) ---
def test_lossless_pq_full_probe_is_exact_knn():
    from sklearn.neighbors import NearestNeighbors
    ix = datagen.make_index(3000, 16, 32, 4, seed=11, lossless=True)
    Q = datagen.make_queries(3000, 16, 32, 40, seed=11, stream=2)
    X = ix.vectors  # generation order == list order; ids are a permutation
    nn = NearestNeighbors(n_neighbors=11, algorithm="brute", metric="sqeuclidean").fit(X.astype(np.float64))
    dist, ind = nn.kneighbors(Q.astype(np.float64))
    r = oracle.search(ix, Q, ix.nlist, 10)
    for qi in range(len(Q)):
        # X rows were rounded to fp32, the oracle reconstructs in fp64: agree to ~1e-7
        assert np.allclose(r["dist"][qi], dist[qi, :10], rtol=2e-6, atol=2e-7)
        if dist[qi, 10] - dist[qi, 9] > 1e-5:
            assert set(r["ids"][qi].tolist()) == set(ix.ids[ind[qi, :10]].tolist())


# --- Recall@k monotone in nprobe against exhaustive PQ (theorem, reading A14) ---
def test_recall_vs_exhaustive_pq_monotone_in_nprobe(small_index, small_queries):
    ix, Q = small_index, small_queries
    k = 10
    full = oracle.search(ix, Q, ix.nlist, k)
    prev = None
    for npb in (1, 2, 4, 8, 16, 32, 64):
        r = oracle.search(ix, Q, npb, k)
        rec = np.array([len(set(a.tolist()) & set(b.tolist())) for a, b in zip(r["ids"], full["ids"])])
        if prev is not None:
            assert np.all(rec >= prev)  # per query, not only on average
        prev = rec
    assert np.all(prev == k)


# --- Mask / hit rate ---------------------------
def test_mask_all_hot_and_empty_hot(small_index, small_queries):
    ix, Q = small_index, small_queries[:12]
    a = oracle.search(ix, Q, 8, 5)
    b = oracle.search(ix, Q, 8, 5, hot=np.arange(ix.nlist))
    assert np.all(a["miss"] == 0) and np.array_equal(a["ids"], b["ids"])
    e = oracle.search(ix, Q, 8, 5, hot=[])
    assert np.all(e["miss"] == 1)
    assert np.all(e["ids"] == -1) and np.all(np.isinf(e["dist"]))
    assert np.all(e["ncand"] == 0)


def test_mean_hitrate_equals_coverage(small_index):
    ix = small_index
    Qc = datagen.make_queries(6000, 32, 64, 500, seed=7, stream=1, alpha=1.2)
    probes, _ = oracle.coarse(Qc, ix.centroids, 8)
    counts = datagen.access_counts(ix.centroids, Qc, 8, probes=probes.astype(np.int64))
    for mass in (0.3, 0.5, 0.7):
        hot = datagen.hot_from_mass(counts, mass)
        r = oracle.search(ix, Qc, 8, 1, hot=hot)
        eta = 1.0 - r["miss"].mean(axis=1)
        assert abs(eta.mean() - datagen.coverage_mean_hitrate(counts, hot)) < 1e-12
        assert datagen.coverage_mean_hitrate(counts, hot) >= mass


# --- Hot/cold decomposition: hybrid = monolithic -------------
def test_hot_cold_merge_equals_full(small_index, small_queries):
    ix, Q = small_index, small_queries
    k, npb = 10, 12
    rng = np.random.default_rng(3)
    hot = np.sort(rng.choice(ix.nlist, ix.nlist // 3, replace=False))
    cold = np.setdiff1d(np.arange(ix.nlist), hot)
    h = oracle.search(ix, Q, npb, k, hot=hot)
    c = oracle.search(ix, Q, npb, k, hot=cold)
    f = oracle.search(ix, Q, npb, k)
    assert np.array_equal(h["miss"] + c["miss"], np.ones_like(h["miss"]))
    for qi in range(len(Q)):
        ids = np.concatenate([h["ids"][qi], c["ids"][qi]])
        dd = np.concatenate([h["dist"][qi], c["dist"][qi]])
        o = np.lexsort((np.where(ids < 0, np.iinfo(np.int64).max, ids), dd))[:k]
        assert np.array_equal(ids[o], f["ids"][qi])
        assert np.array_equal(dd[o], f["dist"][qi])


# --- k >= candidates, duplicate vectors, empty / single-vector lists --------
def test_padding_and_ties_and_empty_lists():
    rng = np.random.default_rng(4)
    C = rng.standard_normal((4, 8)).astype(np.float32)
    cb = rng.standard_normal((2, 256, 4)).astype(np.float32)
    code = np.array([[3, 7]], np.uint8)
    lists = [([5, 2, 9], np.repeat(code, 3, 0)),   # three identical vectors
             ([], np.zeros((0, 2), np.uint8)),      # empty list
             ([1], np.array([[0, 0]], np.uint8)),   # single-vector list
             ([4, 3], rng.integers(0, 256, (2, 2)).astype(np.uint8))]
    ix = datagen.index_from_parts(C, cb, lists)
    Q = rng.standard_normal((3, 8)).astype(np.float32)
    r = oracle.search(ix, Q, 4, 10)
    for qi in range(3):
        ids = r["ids"][qi].tolist()
        assert ids[6:] == [-1] * 4 and np.all(np.isinf(r["dist"][qi, 6:]))
        got = [i for i in ids if i in (2, 5, 9)]
        assert got == [2, 5, 9]  # equal distances -> ascending id
        assert sorted(i for i in ids if i >= 0) == [1, 2, 3, 4, 5, 9]
        assert np.all(np.diff(r["dist"][qi, :6]) >= 0)


# --- workload skew of the generator -------------------
def test_zipf_stream_skew(small_index):
    ix = small_index
    # (at 64 lists / 16 topics the latent query noise spreads probes over neighbouring clusters: alpha 1.5
    # for > 50%; the calibrated per-config shares are in profiles/workload_*.json)
    Qz = datagen.make_queries(6000, 32, 64, 4000, seed=7, stream=1, alpha=1.5)
    Qu = datagen.make_queries(6000, 32, 64, 4000, seed=7, stream=1, alpha=0.0, dup_frac=0.0)
    cz = datagen.access_counts(ix.centroids, Qz, 1)
    cu = datagen.access_counts(ix.centroids, Qu, 1)
    assert datagen.topk_share(cz) > 0.5
    assert datagen.topk_share(cu) < 0.4


# --- NEXT-3 variants: inner-product metric and by_residual = 0 -------------
# ("independent of the distance metric"; DESIGN readings A1', A2')
def test_golden_tiny_variants():
    g = load_golden("tiny_variants.json")
    ix = golden_index(load_golden(g["index"]))
    Q = np.array(load_golden(g["index"])["queries"], np.float32)
    for case in g["cases"]:
        r = oracle.search(ix, Q, case["nprobe"], case["k"], hot=case["hot"], metric=case["metric"],
                          by_residual=case["by_residual"])
        assert r["probes"].tolist() == case["probes"], case
        assert r["miss"].tolist() == case["miss"], case
        assert r["ids"].tolist() == case["ids"], case
        exp = np.array([[fval(x) for x in row] for row in case["dist"]])
        assert np.array_equal(r["dist"], exp), case
        if "coarse" in case:
            p, dd = oracle.coarse(Q, ix.centroids, case["nprobe"], metric=case["metric"])
            assert p.tolist() == case["probes"]
            assert np.array_equal(dd, np.array(case["coarse"]))


def test_ip_coarse_matches_numpy_ranking(small_index, small_queries):
    # the IP coarse key is -<q, c>; against an fp64 numpy matmul + lexsort
    C, Q = small_index.centroids, small_queries
    p, dd = oracle.coarse(Q, C, C.shape[0], metric=1)
    ref = -(Q.astype(np.float64) @ C.astype(np.float64).T)
    for qi in range(len(Q)):
        assert np.allclose(dd[qi], ref[qi, p[qi]], rtol=0, atol=1e-12)
        o = np.lexsort((np.arange(C.shape[0]), ref[qi]))
        gaps = np.diff(ref[qi, o])
        clear = np.concatenate([[True], gaps > 1e-12]) & np.concatenate([gaps > 1e-12, [True]])
        assert np.array_equal(p[qi][clear], o[clear])
    # a query equal to a unit-norm centroid direction probes it first
    u = C[7] / np.linalg.norm(C[7])
    p1, _ = oracle.coarse((u * 3.0)[None, :].astype(np.float32), C / np.linalg.norm(C, axis=1, keepdims=True), 1,
                          metric=1)
    assert p1[0, 0] == 7


def _flat_topk_variant(ix, Q, k, metric, by_residual):
    c, y, _ = _recon(ix, np.arange(ix.N))
    X = c + y if by_residual else y
    Qd = Q.astype(np.float64)
    if metric == 1:
        D = -(Qd @ X.T)
    else:
        D = (Qd * Qd).sum(1)[:, None] + (X * X).sum(1)[None, :] - 2 * Qd @ X.T
    out = []
    for row in D:
        o = np.lexsort((ix.ids, row))[:k]
        out.append((ix.ids[o], row[o]))
    return out


@pytest.mark.parametrize("metric,by_residual", [(1, 1), (0, 0), (1, 0)])
def test_variant_full_probe_equals_exhaustive(small_index, small_queries, metric, by_residual):
    ix, Q = small_index, small_queries[:16]
    k = 10
    r = oracle.search(ix, Q, ix.nlist, k, metric=metric, by_residual=by_residual)
    flat = _flat_topk_variant(ix, Q, k + 1, metric, by_residual)
    for qi, (fid, fd) in enumerate(flat):
        assert np.allclose(r["dist"][qi], fd[:k], rtol=1e-10, atol=1e-12)
        if fd[k] - fd[k - 1] > 1e-9:
            assert set(r["ids"][qi].tolist()) == set(fid[:k].tolist())


def test_variant_dist_identities(small_index, small_queries):
    # ||q - x||^2 = ||q||^2 + ||x||^2 - 2<q, x> links the L2 and IP branches;
    # the residual and plain branches differ exactly by the centroid term
    ix, Q = small_index, small_queries
    rng = np.random.default_rng(5)
    pos = rng.integers(0, ix.N, 300)
    qi = rng.integers(0, len(Q), 300)
    c, y, _ = _recon(ix, pos)
    q = Q[qi].astype(np.float64)
    d = {(mt, br): oracle.dist_ref(ix, Q, qi, ix.ids[pos], metric=mt, by_residual=br) for mt in (0, 1) for br in (0, 1)}
    for br, X in ((1, c + y), (0, y)):
        lhs = d[(0, br)] - (q * q).sum(1) - (X * X).sum(1)
        assert np.allclose(lhs, 2.0 * d[(1, br)], rtol=1e-9, atol=1e-9)
    assert np.allclose(d[(1, 1)] - d[(1, 0)], -(q * c).sum(1), rtol=1e-9, atol=1e-12)
    # the GPU's LUT decomposition (second path): term1 + b + sum_j LUT
    dsub = ix.d // ix.m
    lut_ip = -(q * y).reshape(-1, ix.m, dsub).sum(2).sum(1)
    assert np.allclose(d[(1, 1)], -(q * c).sum(1) + lut_ip, rtol=1e-12, atol=1e-12)
    assert np.allclose(d[(0, 0)], (q * q).sum(1) + (y * y).sum(1) + 2 * lut_ip, rtol=1e-12, atol=1e-12)


def test_lossless_plain_pq_is_exact_knn_both_metrics():
    from sklearn.neighbors import NearestNeighbors
    ix = datagen.make_index(3000, 16, 32, 4, seed=13, lossless=True, by_residual=0)
    Q = datagen.make_queries(3000, 16, 32, 40, seed=13, stream=2)
    X = ix.vectors.astype(np.float64)  # x_i := yhat_i
    nn = NearestNeighbors(n_neighbors=11, algorithm="brute", metric="sqeuclidean").fit(X)
    dist, ind = nn.kneighbors(Q.astype(np.float64))
    r = oracle.search(ix, Q, ix.nlist, 10)
    assert ix.by_residual == 0 and ix.metric == 0
    for qi in range(len(Q)):
        assert np.allclose(r["dist"][qi], dist[qi, :10], rtol=2e-6, atol=2e-7)
        if dist[qi, 10] - dist[qi, 9] > 1e-5:
            assert set(r["ids"][qi].tolist()) == set(ix.ids[ind[qi, :10]].tolist())
    # maximum inner product: scikit-learn's cosine on rows of equal norm ranks as IP;
    # here a direct argsort of X q (library matmul) is the reference
    ri = oracle.search(ix, Q, ix.nlist, 10, metric=1)
    S = Q.astype(np.float64) @ X.T
    for qi in range(len(Q)):
        o = np.argsort(-S[qi], kind="stable")[:11]
        assert np.allclose(ri["dist"][qi], -S[qi, o[:10]], rtol=2e-6, atol=2e-7)
        if S[qi, o[9]] - S[qi, o[10]] > 1e-5:
            assert set(ri["ids"][qi].tolist()) == set(ix.ids[o[:10]].tolist())


# --- NEXT-3: 4-bit PQ (reading A4') -----------------------
def _unpack4(codes, m):
    j = np.arange(m)
    return (codes[:, j // 2] >> (4 * (j % 2))) & 15


def test_golden_tiny_pq4_hand_packed():
    from conftest import golden_pq4_index
    ix, g = golden_pq4_index()
    Q = np.array(g["queries"], np.float32)
    for case in g["cases"]:
        r = oracle.search(ix, Q, case["nprobe"], case["k"], hot=case["hot"])
        assert r["probes"].tolist() == case["probes"]
        assert r["miss"].tolist() == case["miss"]
        assert r["ids"].tolist() == case["ids"]
        assert np.array_equal(r["dist"], np.array([[fval(x) for x in row] for row in case["dist"]]))


def test_pack_nibbles_layout():
    import torch
    cc = torch.tensor([[1, 2, 3], [15, 0, 7]], dtype=torch.uint8)
    assert datagen.pack_nibbles(cc).tolist() == [[0x21, 0x03], [0x0F, 0x07]]


@pytest.mark.parametrize("metric,by_residual", [(0, 1), (1, 1), (0, 0)])
def test_pq4_full_probe_equals_exhaustive(metric, by_residual):
    ix = datagen.make_index(5000, 32, 48, 8, seed=17, nbits=4, metric=metric, by_residual=by_residual)
    assert ix.codes.shape == (5000, 4) and ix.codebooks.shape == (8, 16, 4)
    Q = datagen.make_queries(5000, 32, 48, 16, seed=17, stream=2)
    codes = _unpack4(ix.codes, ix.m).astype(np.int64)
    y = ix.codebooks[np.arange(ix.m)[None, :], codes].reshape(ix.N, ix.d).astype(np.float64)
    lst = np.searchsorted(ix.list_offsets, np.arange(ix.N), side="right") - 1
    X = ix.centroids[lst].astype(np.float64) + y if by_residual else y
    Qd = Q.astype(np.float64)
    D = -(Qd @ X.T) if metric else (Qd * Qd).sum(1)[:, None] + (X * X).sum(1)[None, :] - 2 * Qd @ X.T
    r = oracle.search(ix, Q, ix.nlist, 10)
    for qi in range(len(Q)):
        o = np.lexsort((ix.ids, D[qi]))[:11]
        assert np.allclose(r["dist"][qi], D[qi, o[:10]], rtol=1e-10, atol=1e-12)
        if D[qi, o[10]] - D[qi, o[9]] > 1e-9:
            assert set(r["ids"][qi].tolist()) == set(ix.ids[o[:10]].tolist())


def test_pq4_lossless_is_exact_knn():
    from sklearn.neighbors import NearestNeighbors
    ix = datagen.make_index(3000, 16, 32, 4, seed=19, lossless=True, nbits=4)
    Q = datagen.make_queries(3000, 16, 32, 40, seed=19, stream=2)
    nn = NearestNeighbors(n_neighbors=11, algorithm="brute", metric="sqeuclidean").fit(ix.vectors.astype(np.float64))
    dist, ind = nn.kneighbors(Q.astype(np.float64))
    r = oracle.search(ix, Q, ix.nlist, 10)
    for qi in range(len(Q)):
        assert np.allclose(r["dist"][qi], dist[qi, :10], rtol=2e-6, atol=2e-7)
        if dist[qi, 10] - dist[qi, 9] > 1e-5:
            assert set(r["ids"][qi].tolist()) == set(ix.ids[ind[qi, :10]].tolist())
