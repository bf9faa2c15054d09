"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
element by element on the same seeded inputs (rules R1-R5).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2504_08930_b200 as vlr
from conftest import fval, golden_index, load_golden
from parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2504_08930_b200 import build
    build.build()
    assert torch.cuda.is_available()


def gpu_search(index_handle, Q, nprobe, k):
    Qd = torch.from_numpy(np.ascontiguousarray(Q, np.float32)).cuda()
    ids, dist, miss, probes = index_handle.search(Qd, nprobe, k, sync=True)
    torch.cuda.synchronize()
    return dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=probes.cpu().numpy())


def run_parity(ix, Q, nprobe, k, hot=None, idmap=None):
    h = vlr.Index.from_arrays(ix, hot=hot)
    g = gpu_search(h, Q, nprobe, k)
    o = oracle.search(ix, Q, nprobe, k, hot=hot)
    errs = check(ix, Q, g, o, hot=hot, idmap=idmap or oracle.IdMap(ix))
    h.close()
    return errs, g, o


# --------------------------------------------------------------- golden
def test_golden_tiny_on_gpu():
    gd = load_golden("tiny_hand.json")
    ix = golden_index(gd)
    Q = np.array(gd["queries"], np.float32)
    for case in gd["cases"]:
        h = vlr.Index.from_arrays(ix, hot=case["hot"])
        g = gpu_search(h, Q, case["nprobe"], case["k"])
        assert g["probes"].tolist() == case["probes"]
        assert g["miss"].tolist() == case["miss"]
        assert g["ids"].tolist() == case["ids"]
        exp = np.array([[fval(x) for x in row] for row in case["dist"]], np.float32)
        assert np.array_equal(g["dist"], exp)  # every value here is exact in fp32
        h.close()


# --------------------------------------------------------------- C1
def test_c1_parity_all_hot(c1_index, c1_queries):
    c = datagen.CONFIGS["C1"]
    errs, g, o = run_parity(c1_index, c1_queries, c["nprobe"], c["k"])
    assert not errs, errs
    assert np.all(g["miss"] == 0)


def test_c1_parity_hot_half_mass(c1_index, c1_queries):
    c = datagen.CONFIGS["C1"]
    Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 2000, stream=1, alpha=c["alpha"])
    counts = datagen.access_counts(c1_index.centroids, Qc, c["nprobe"])
    hot = datagen.hot_from_mass(counts, 0.5)
    errs, g, o = run_parity(c1_index, c1_queries, c["nprobe"], c["k"], hot=hot)
    assert not errs, errs
    assert 0 < g["miss"].mean() < 1


@pytest.mark.parametrize("nprobe,k", [(1, 1), (4, 32), (64, 10), (300, 7), (1024, 10), (5000, 3)])
def test_c1_parity_nprobe_k(c1_index, c1_queries, nprobe, k):
    errs, g, o = run_parity(c1_index, c1_queries[:24], nprobe, k)
    assert not errs, errs


def test_c1_determinism_and_shard_invariance(c1_index, c1_queries):
    c = datagen.CONFIGS["C1"]
    h = vlr.Index.from_arrays(c1_index)
    a = gpu_search(h, c1_queries, c["nprobe"], c["k"])
    b = gpu_search(h, c1_queries, c["nprobe"], c["k"])
    for key in a:
        assert np.array_equal(a[key], b[key])  # R5: repeated runs bitwise identical
    h.close()
    Qd = torch.from_numpy(c1_queries).cuda()
    for G in (2, 3, 4, 8):
        parts_i, parts_d = [], []
        owners = None
        for r in range(G):
            hs = vlr.Index.from_arrays(c1_index, rank=r, world=G)
            ids, dist, miss, probes = hs.search(Qd, c["nprobe"], c["k"], sync=True)
            parts_i.append(ids)
            parts_d.append(dist)
            assert np.array_equal(miss.cpu().numpy(), a["miss"])
            assert np.array_equal(probes.cpu().numpy(), a["probes"])
            own = hs.owners()
            owners = own if owners is None else owners
            assert np.array_equal(own, owners)
            hs.close()
        mi, md = vlr.merge_partials(torch.stack(parts_i), torch.stack(parts_d))
        torch.cuda.synchronize()
        assert np.array_equal(mi.cpu().numpy(), a["ids"]), f"G={G} ids differ"
        assert np.array_equal(md.cpu().numpy(), a["dist"]), f"G={G} dist differ"
        # size-descending round-robin deal: shard sizes differ by at most one list
        counts = np.bincount(owners[owners >= 0], minlength=G)
        assert counts.max() - counts.min() <= 1


def test_search_host_matches_device(c1_index, c1_queries):
    c = datagen.CONFIGS["C1"]
    h = vlr.Index.from_arrays(c1_index)
    a = gpu_search(h, c1_queries, c["nprobe"], c["k"])
    ids, dist, miss, probes = h.search_host(c1_queries, c["nprobe"], c["k"])
    assert np.array_equal(ids, a["ids"]) and np.array_equal(dist, a["dist"])
    assert np.array_equal(miss, a["miss"]) and np.array_equal(probes, a["probes"])
    assert h.last_launch_count >= 8
    h.close()


def test_nonfinite_query_reported(c1_index, c1_queries):
    h = vlr.Index.from_arrays(c1_index)
    Q = c1_queries[:4].copy()
    Q[2, 7] = np.nan
    with pytest.raises(vlr.VlrError) as e:
        gpu_search(h, Q, 8, 5)
    assert e.value.name == "NONFINITE"
    g = gpu_search(h, c1_queries[:4], 8, 5)  # the handle stays usable
    assert g["ids"].shape == (4, 5)
    h.close()


def test_batch_sizes(c1_index, c1_queries):
    h = vlr.Index.from_arrays(c1_index)
    big = datagen.make_queries(100_000, 128, 1024, 513, stream=3)
    for nq in (1, 2, 33, 513):
        Q = big[:nq]
        g = gpu_search(h, Q, 16, 10)
        o = oracle.search(c1_index, Q, 16, 10)
        assert not check(c1_index, Q, g, o)
    Qd = torch.zeros(0, 128, device="cuda")
    ids, dist, miss, probes = h.search(Qd, 16, 10, sync=True)
    assert ids.shape == (0, 10)
    h.close()


def test_small_batch_wide_merge():
    """Batches 1-8 over long lists: one query spans all scan CTAs, so K7 runs
    its multi-warp path (up to 32 warps, sort-merge and insertion offers)."""
    ix = datagen.make_index(2_000_000, 128, 1024, 16, device="cuda")
    h = vlr.Index.from_arrays(ix)
    Qa = datagen.make_queries(2_000_000, 128, 1024, 16, stream=2)
    for nq, k in ((1, 10), (1, 32), (1, 1), (3, 10), (8, 32)):
        Q = Qa[:nq]
        g = gpu_search(h, Q, 64, k)
        o = oracle.search(ix, Q, 64, k)
        assert not check(ix, Q, g, o), (nq, k)
    h.close()


# --------------------------------------------------------------- shapes / m_pad variants
@pytest.mark.parametrize("d,m,L", [(32, 4, 50), (64, 32, 40), (96, 48, 33), (128, 64, 64), (192, 96, 40),
                                   (256, 128, 70), (40, 20, 17), (64, 16, 1030)])
def test_m_variants(d, m, L):
    ix = datagen.make_index(4000, d, L, m, seed=d + m)
    Q = datagen.make_queries(4000, d, L, 20, seed=d + m, stream=2)
    hot = np.arange(0, L, 2)
    for npb, hh in ((8, None), (min(L, 1000), hot)):
        errs, g, o = run_parity(ix, Q, npb, 10, hot=hh)
        assert not errs, (d, m, L, errs)


# --------------------------------------------------------------- adversarial
def _rand_index(rng, L, d, m, sizes, dup_centroids=()):
    C = rng.standard_normal((L, d)).astype(np.float32)
    for a, b in dup_centroids:
        C[b] = C[a]
    Y = (0.3 * rng.standard_normal((m, 256, d // m))).astype(np.float32)
    ids = rng.permutation(10 * sum(sizes) + 10)[: sum(sizes)]
    lists, o = [], 0
    for s in sizes:
        lists.append((ids[o:o + s], rng.integers(0, 256, (s, m)).astype(np.uint8)))
        o += s
    return datagen.index_from_parts(C, Y, lists)


def test_adversarial_empty_single_duplicate():
    rng = np.random.default_rng(5)
    sizes = [0, 1, 0, 33, 64, 1, 0, 31, 32, 95]
    ix = _rand_index(rng, 10, 16, 4, sizes, dup_centroids=[(3, 7), (3, 9)])
    # duplicate vectors inside a list (same code) -> ties broken by id
    ix.codes[ix.list_offsets[4]:ix.list_offsets[4] + 5] = ix.codes[ix.list_offsets[4]]
    Q = np.concatenate([ix.centroids[[3, 7, 0]], rng.standard_normal((13, 16)).astype(np.float32)])
    for npb in (1, 3, 10, 50):
        for k in (1, 5, 32):
            for hot in (None, [1, 3, 4, 9], []):
                errs, g, o = run_parity(ix, Q, npb, k, hot=hot)
                assert not errs, (npb, k, hot, errs)


def test_adversarial_equidistant_centroids():
    # centroids +-e_i around the origin: every query at the origin sees all
    # of them at distance 1 -> probes must be ordered by cluster id (A7)
    d = 16
    C = np.concatenate([np.eye(d), -np.eye(d)]).astype(np.float32)
    rng = np.random.default_rng(6)
    Y = (0.1 * rng.standard_normal((4, 256, 4))).astype(np.float32)
    lists = [(np.arange(i * 40, i * 40 + 40), rng.integers(0, 256, (40, 4)).astype(np.uint8)) for i in range(2 * d)]
    ix = datagen.index_from_parts(C, Y, lists)
    Q = np.zeros((3, d), np.float32)
    Q[1, 0] = 1e-3
    Q[2] = 0.5
    for npb in (1, 5, 32):
        errs, g, o = run_parity(ix, Q, npb, 10)
        assert not errs, errs
    assert g["probes"][0].tolist()[:5] == [0, 1, 2, 3, 4]


def test_adversarial_identical_centroids_many():
    # 200 identical centroids: the band holds all of them; order by id
    rng = np.random.default_rng(8)
    c = rng.standard_normal(8).astype(np.float32)
    C = np.repeat(c[None], 200, 0)
    C[150:] += np.float32(1.0)
    Y = (0.2 * rng.standard_normal((2, 256, 4))).astype(np.float32)
    lists = [(np.arange(i * 3, i * 3 + 3), rng.integers(0, 256, (3, 2)).astype(np.uint8)) for i in range(200)]
    ix = datagen.index_from_parts(C, Y, lists)
    Q = (c + 0.01 * rng.standard_normal((5, 8))).astype(np.float32)
    for npb in (16, 150, 160):
        errs, g, o = run_parity(ix, Q, npb, 10)
        assert not errs, errs


def test_offset_data_stress():
    # reading A3: data with a large common offset; the LUT decomposition loses
    # fp32 accuracy there. Documented limit: parity is still required at the
    # 1e-5 relative rule because distances scale with the offset as well.
    ix = datagen.make_index(3000, 32, 20, 8, seed=12)
    off = np.float32(3.0)
    ix.centroids = ix.centroids + off
    Q = datagen.make_queries(3000, 32, 20, 16, seed=12, stream=2) + off
    errs, g, o = run_parity(ix, Q, 6, 10)
    assert not errs, errs


def test_candidate_overflow_rescan_path():
    # 9000 identical centroids: every one lies inside the filter band, so the
    # candidate list (capacity 8192) overflows and K3 takes the rescan path.
    rng = np.random.default_rng(9)
    L, d = 9000, 8
    c = rng.standard_normal(d).astype(np.float32)
    C = np.repeat(c[None], L, 0)
    C[8990:] += np.float32(2.0)
    Y = (0.2 * rng.standard_normal((2, 256, 4))).astype(np.float32)
    lists = [(np.arange(i * 2, i * 2 + 2), rng.integers(0, 256, (2, 2)).astype(np.uint8)) for i in range(L)]
    ix = datagen.index_from_parts(C, Y, lists)
    Q = (c + 0.01 * rng.standard_normal((3, d))).astype(np.float32)
    for npb in (8, 700, 2048):
        errs, g, o = run_parity(ix, Q, npb, 10)
        assert not errs, errs
        assert g["probes"][0].tolist() == list(range(npb))  # equal distances -> ascending id


# --------------------------------------------------------------- full-size sampled parity
@pytest.mark.parametrize("cfg,hot_mass,nq", [("C2", 1.0, 24), ("C3", 0.5, 16)])
def test_full_size_sampled_parity(cfg, hot_mass, nq):
    """BASELINE configs at full size (generated on the GPU), the batch and launch
    configuration bench.py uses; the oracle checks a sample of queries."""
    c = datagen.CONFIGS[cfg]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], device="cuda")
    Q = datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, alpha=c["alpha"], device="cuda")
    hot = None
    if hot_mass < 1.0:
        Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 10_000, stream=1, alpha=c["alpha"], device="cuda")
        hot = datagen.hot_from_mass(datagen.access_counts(ix.centroids, Qc, c["nprobe"], device="cuda"), hot_mass)
    h = vlr.Index.from_arrays(ix, hot=hot)
    g = gpu_search(h, Q, c["nprobe"], c["k"])  # the full batch, as timed by bench.py
    h.close()
    sel = np.linspace(0, len(Q) - 1, nq).astype(np.int64)
    o = oracle.search(ix, Q[sel], c["nprobe"], c["k"], hot=hot)
    gs = {key: v[sel] for key, v in g.items()}
    errs = check(ix, Q, gs, o, hot=hot, idmap=oracle.IdMap(ix), qsel=sel)
    assert not errs, errs
    if hot is not None:
        assert 0.0 < g["miss"].mean() < 1.0


def test_hybrid_hot_gpu_plus_cold_cpu_equals_monolithic(c1_index, c1_queries):
    """NEXT-1 / S:473: the GPU result over the hot lists merged (on the
    GPU, vlr_merge_partials) with a cold-tier result over the remaining lists
    equals the search over all lists. The cold tier here is the oracle (the
    paper's CPU path)."""
    c = datagen.CONFIGS["C1"]
    ix, Q = c1_index, c1_queries
    rng = np.random.default_rng(11)
    hot = np.sort(rng.choice(ix.nlist, ix.nlist // 2, replace=False))
    cold = np.setdiff1d(np.arange(ix.nlist), hot)
    h = vlr.Index.from_arrays(ix, hot=hot)
    g = gpu_search(h, Q, c["nprobe"], c["k"])
    h.close()
    oc = oracle.search(ix, Q, c["nprobe"], c["k"], hot=cold)
    # cold-tier partial in the GPU's fp32 distance type
    parts_i = torch.from_numpy(np.stack([g["ids"], oc["ids"]])).cuda()
    parts_d = torch.from_numpy(np.stack([g["dist"], oc["dist"].astype(np.float32)])).cuda()
    mi, md = vlr.merge_partials(parts_i, parts_d)
    merged = dict(ids=mi.cpu().numpy(), dist=md.cpu().numpy(), miss=np.zeros_like(g["miss"]), probes=g["probes"])
    full = oracle.search(ix, Q, c["nprobe"], c["k"])
    errs = check(ix, Q, merged, full, idmap=oracle.IdMap(ix))
    assert not errs, errs
    assert np.array_equal(g["miss"], np.isin(g["probes"], cold).astype(np.uint8))


def test_access_counts_and_hot_set(c1_index):
    """NEXT-2: the GPU access profile of a calibration stream equals the count
    of the oracle's probes; the hot set chosen from it covers the target mass
    and its measured mean hit rate equals the coverage eta-bar."""
    c = datagen.CONFIGS["C1"]
    Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 1500, stream=1, alpha=1.2)
    h = vlr.Index.from_arrays(c1_index)
    g = gpu_search(h, Qc, c["nprobe"], 1)
    cnt = h.access_counts(torch.from_numpy(g["probes"]).cuda()).cpu().numpy()
    po, _ = oracle.coarse(Qc, c1_index.centroids, c["nprobe"])
    assert np.array_equal(cnt, np.bincount(po.reshape(-1), minlength=c1_index.nlist))
    hot = datagen.hot_from_mass(cnt, 0.5)
    h.close()
    h2 = vlr.Index.from_arrays(c1_index, hot=hot)
    g2 = gpu_search(h2, Qc, c["nprobe"], 1)
    h2.close()
    eta = 1.0 - g2["miss"].mean(axis=1)
    assert abs(eta.mean() - datagen.coverage_mean_hitrate(cnt, hot)) < 1e-12


def test_profiling_modes(c1_index, c1_queries):
    """Stage timing: mode 1 = every stage boundary, mode 2 = scan only (the
    bench's timed region); results do not depend on profiling."""
    h = vlr.Index.from_arrays(c1_index)
    Q = c1_queries[:64]
    base = gpu_search(h, Q, 16, 10)
    h.set_profiling(1)
    g1 = gpu_search(h, Q, 16, 10)
    st = h.stage_times()
    assert all(np.isfinite(v) and v >= 0 for v in st.values()), st
    assert st["scan"] > 0
    h.set_profiling(2)
    g2 = gpu_search(h, Q, 16, 10)
    st2 = h.stage_times()
    assert np.isfinite(st2["scan"]) and st2["scan"] > 0
    assert all(np.isnan(v) for k2, v in st2.items() if k2 != "scan"), st2
    assert h.stage_times(back=1)["select"] >= 0  # the mode-1 search is still in the ring
    h.set_profiling(False)
    with pytest.raises(vlr.VlrError):
        h.set_profiling(3)
    for g in (g1, g2):
        for key in base:
            assert np.array_equal(base[key], g[key]), key
    h.close()


# --------------------------------------------------------------- NEXT-3 variants
def test_golden_tiny_variants_on_gpu():
    gv = load_golden("tiny_variants.json")
    base = load_golden(gv["index"])
    ix = golden_index(base)
    Q = np.array(base["queries"], np.float32)
    for case in gv["cases"]:
        h = vlr.Index.from_arrays(ix, hot=case["hot"], metric=case["metric"], by_residual=case["by_residual"])
        g = gpu_search(h, Q, case["nprobe"], case["k"])
        h.close()
        assert g["probes"].tolist() == case["probes"], case
        assert g["miss"].tolist() == case["miss"], case
        assert g["ids"].tolist() == case["ids"], case
        exp = np.array([[fval(x) for x in row] for row in case["dist"]], np.float32)
        assert np.array_equal(g["dist"], exp), case  # every value here is exact in fp32


@pytest.fixture(scope="module")
def c1_variant_indexes():
    c = datagen.CONFIGS["C1"]
    return {(mt, br): datagen.make_index(c["N"], c["d"], c["nlist"], c["m"], metric=mt, by_residual=br)
            for mt, br in ((1, 1), (0, 0), (1, 0))}


@pytest.mark.parametrize("metric,by_residual", [(1, 1), (0, 0), (1, 0)])
def test_c1_variant_parity(c1_variant_indexes, c1_queries, metric, by_residual):
    """Inner-product metric and plain (non-residual) PQ: probes and mask
    bit-exact, distances within the R2 rule, id sets by R3 (DESIGN §2 A1', A2')."""
    c = datagen.CONFIGS["C1"]
    ix = c1_variant_indexes[(metric, by_residual)]
    errs, g, o = run_parity(ix, c1_queries, c["nprobe"], c["k"])
    assert not errs, errs
    hot = np.arange(0, ix.nlist, 3)
    for npb, k in ((1, 1), (64, 25), (1024, 10)):
        errs, g, o = run_parity(ix, c1_queries[:24], npb, k, hot=hot)
        assert not errs, (npb, k, errs)


@pytest.mark.parametrize("metric", [0, 1])
def test_paper_operating_point_nprobe_2048_k25(metric):
    """The paper's operating point nprobe = 2048, k = 25 on an index
    with nlist = 8192 > nprobe, so the coarse select keeps a strict subset."""
    ix = datagen.make_index(600_000, 64, 8192, 16, seed=21, device="cuda", metric=metric)
    Q = datagen.make_queries(600_000, 64, 8192, 40, seed=21, stream=2)
    hot = np.arange(0, 8192, 2)
    for hh in (None, hot):
        errs, g, o = run_parity(ix, Q, 2048, 25, hot=hh)
        assert not errs, errs
        assert g["probes"].shape == (40, 2048)


# --------------------------------------------------------------- NEXT-3: 4-bit PQ
def test_golden_tiny_pq4_on_gpu():
    from conftest import golden_pq4_index
    ix, g = golden_pq4_index()
    Q = np.array(g["queries"], np.float32)
    for case in g["cases"]:
        h = vlr.Index.from_arrays(ix, hot=case["hot"])
        r = gpu_search(h, Q, case["nprobe"], case["k"])
        h.close()
        assert r["probes"].tolist() == case["probes"]
        assert r["miss"].tolist() == case["miss"]
        assert r["ids"].tolist() == case["ids"]
        exp = np.array([[fval(x) for x in row] for row in case["dist"]], np.float32)
        assert np.array_equal(r["dist"], exp)


@pytest.mark.parametrize("m,metric,by_residual", [(32, 0, 1), (64, 0, 1), (32, 1, 1), (32, 0, 0)])
def test_c1_pq4_parity(c1_queries, m, metric, by_residual):
    """4-bit codes (nibble-packed, 16 codewords; reading A4') on the C1 shape."""
    c = datagen.CONFIGS["C1"]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], m, nbits=4, metric=metric, by_residual=by_residual)
    errs, g, o = run_parity(ix, c1_queries, c["nprobe"], c["k"])
    assert not errs, errs
    hot = np.arange(1, ix.nlist, 3)
    for npb, k in ((1, 1), (64, 25), (1024, 10)):
        errs, g, o = run_parity(ix, c1_queries[:24], npb, k, hot=hot)
        assert not errs, (npb, k, errs)


@pytest.mark.parametrize("d,m,L", [(32, 8, 50), (40, 20, 17), (64, 64, 40), (192, 96, 33), (128, 128, 64),
                                   (144, 144, 30), (192, 192, 40), (256, 256, 70)])
def test_pq4_m_variants(d, m, L):
    """Every 4-bit scan instantiation (padded sub-spaces 32, 64, 96, 128, 192, 256)."""
    ix = datagen.make_index(4000, d, L, m, seed=d + m, nbits=4)
    Q = datagen.make_queries(4000, d, L, 20, seed=d + m, stream=2)
    hot = np.arange(0, L, 2)
    for npb, hh in ((8, None), (L, hot)):
        errs, g, o = run_parity(ix, Q, npb, 10, hot=hh)
        assert not errs, (d, m, L, errs)


@pytest.fixture
def pq4_nibble_mode(monkeypatch):
    """4-bit nibble-slot scan (VLR_PQ4_NIBBLE=1, read at vlr_load_index) instead of the default pair tables."""
    monkeypatch.setenv("VLR_PQ4_NIBBLE", "1")


@pytest.mark.parametrize("d,m,L", [(32, 8, 50), (40, 20, 17), (64, 64, 40), (192, 96, 33), (128, 128, 64),
                                   (144, 144, 30), (192, 192, 40), (256, 256, 70)])
def test_pq4_nibble_mode_m_variants(pq4_nibble_mode, d, m, L):
    """The nibble-slot 4-bit scan (every instantiation) stays parity-green next to the default pair mode."""
    ix = datagen.make_index(4000, d, L, m, seed=d + m, nbits=4)
    Q = datagen.make_queries(4000, d, L, 20, seed=d + m, stream=2)
    for npb, hh in ((8, None), (L, np.arange(0, L, 2))):
        errs, g, o = run_parity(ix, Q, npb, 10, hot=hh)
        assert not errs, (d, m, L, errs)


def test_pq4_pair_and_nibble_modes_agree(c1_queries, monkeypatch):
    """Pair tables (LUT2[j'][b] = LUT[2j'][b&15] + LUT[2j'+1][b>>4]) and nibble
    slots sum the same terms in different fp32 orders: identical probes and
    masks, distances within the parity tolerance of each other, both green."""
    c = datagen.CONFIGS["C1"]
    ix = datagen.make_index(c["N"], c["d"], c["nlist"], 64, nbits=4)
    errs, gp, _ = run_parity(ix, c1_queries, c["nprobe"], c["k"])
    assert not errs, errs
    monkeypatch.setenv("VLR_PQ4_NIBBLE", "1")
    errs, gn, _ = run_parity(ix, c1_queries, c["nprobe"], c["k"])
    assert not errs, errs
    assert np.array_equal(gp["probes"], gn["probes"]) and np.array_equal(gp["miss"], gn["miss"])
    tol = 1e-5 * np.maximum(np.abs(gn["dist"]), 0.25)
    assert np.all(np.abs(gp["dist"] - gn["dist"]) <= 2 * tol)


def test_update_hot_refresh_equals_fresh_load(c1_index, c1_queries):
    """NEXT-2 shard refresh: after vlr_update_hot to a new hot set
    the handle answers exactly like a handle freshly loaded with that set
    (bitwise), and the oracle agrees; a mismatched index is refused and leaves
    the handle unchanged."""
    import threading
    c = datagen.CONFIGS["C1"]
    ix, Q = c1_index, c1_queries
    rng = np.random.default_rng(5)
    hot_a = np.sort(rng.choice(ix.nlist, ix.nlist // 3, replace=False))
    hot_b = np.sort(rng.choice(ix.nlist, ix.nlist // 2, replace=False))
    h = vlr.Index.from_arrays(ix, hot=hot_a)
    ga = gpu_search(h, Q, c["nprobe"], c["k"])
    # serve from another thread while the refresh builds
    stop, errs_bg = threading.Event(), []
    Qd = torch.from_numpy(Q).cuda()

    def serve():
        s = torch.cuda.Stream()
        try:
            while not stop.is_set():
                with torch.cuda.stream(s):
                    h.search(Qd, c["nprobe"], c["k"], stream=s, sync=True)
        except Exception as e:  # pragma: no cover
            errs_bg.append(e)
    t = threading.Thread(target=serve)
    t.start()
    h.update_hot_arrays(ix, hot=hot_b)
    stop.set()
    t.join()
    assert not errs_bg, errs_bg
    gb = gpu_search(h, Q, c["nprobe"], c["k"])
    f = vlr.Index.from_arrays(ix, hot=hot_b)
    gf = gpu_search(f, Q, c["nprobe"], c["k"])
    f.close()
    for key in gf:
        assert np.array_equal(gb[key], gf[key]), key
    o = oracle.search(ix, Q, c["nprobe"], c["k"], hot=hot_b)
    assert not check(ix, Q, gb, o, hot=hot_b, idmap=oracle.IdMap(ix))
    assert not np.array_equal(ga["miss"], gb["miss"])
    other = datagen.make_index(20_000, 64, 128, 16, seed=3)
    with pytest.raises(vlr.VlrError) as e:
        h.update_hot_arrays(other)
    assert e.value.name == "INVALID_ARG"
    gb2 = gpu_search(h, Q, c["nprobe"], c["k"])
    assert np.array_equal(gb2["ids"], gb["ids"])
    h.close()


def test_traffic_aware_deal_shards_equal_monolithic(c1_index, c1_queries):
    """A traffic-aware owner assignment (vlr_deal_owners with access counts)
    shards the hot lists differently but the merged shard results are bitwise
    the single-GPU result (R5)."""
    c = datagen.CONFIGS["C1"]
    Qc = datagen.make_queries(c["N"], c["d"], c["nlist"], 1000, stream=1, alpha=1.2)
    counts = datagen.access_counts(c1_index.centroids, Qc, c["nprobe"])
    hot = np.arange(c1_index.nlist, dtype=np.int32)
    G = 4
    own = vlr.deal_owners(c1_index.list_offsets, hot, G, counts=counts)
    assert not np.array_equal(own, vlr.deal_owners(c1_index.list_offsets, hot, G))
    h = vlr.Index.from_arrays(c1_index)
    a = gpu_search(h, c1_queries, c["nprobe"], c["k"])
    h.close()
    Qd = torch.from_numpy(c1_queries).cuda()
    pi, pd = [], []
    for r in range(G):
        hs = vlr.Index.from_arrays(c1_index, hot=hot, hot_owner=own, rank=r, world=G)
        assert np.array_equal(hs.owners(), own)
        ids, dist, _, _ = hs.search(Qd, c["nprobe"], c["k"], sync=True)
        pi.append(ids)
        pd.append(dist)
        hs.close()
    mi, md = vlr.merge_partials(torch.stack(pi), torch.stack(pd))
    assert np.array_equal(mi.cpu().numpy(), a["ids"]) and np.array_equal(md.cpu().numpy(), a["dist"])


def test_search_host_async_pipeline_matches_blocking(c1_index):
    """vlr_search_host_async back to back on one stream (pinned buffers, one
    final sync) returns, per batch, exactly what the blocking call returns."""
    h = vlr.Index.from_arrays(c1_index)
    Qs = datagen.make_queries(100_000, 128, 1024, 4 * 48, stream=4).reshape(4, 48, 128)
    ref = [h.search_host(Q, 16, 10) for Q in Qs]
    hq = torch.from_numpy(Qs.copy()).pin_memory()
    ids = torch.empty(4, 48, 10, dtype=torch.int64).pin_memory()
    dist = torch.empty(4, 48, 10, dtype=torch.float32).pin_memory()
    miss = torch.empty(4, 48, 16, dtype=torch.uint8).pin_memory()
    prb = torch.empty(4, 48, 16, dtype=torch.int32).pin_memory()
    for i in range(4):
        h.search_host_ptr_async(hq[i].data_ptr(), 48, 16, 10, ids[i].data_ptr(), dist[i].data_ptr(),
                                miss[i].data_ptr(), prb[i].data_ptr())
    torch.cuda.current_stream().synchronize()
    for i in range(4):
        assert np.array_equal(ids[i].numpy(), ref[i][0]) and np.array_equal(dist[i].numpy(), ref[i][1])
        assert np.array_equal(miss[i].numpy(), ref[i][2]) and np.array_equal(prb[i].numpy(), ref[i][3])
    h.close()


def test_cuda_graph_capture_and_replay(c1_index):
    """include/vlr.h: vlr_search_async is CUDA-graph capturable once
    vlr_reserve has sized the workspace; replays give the eager results for
    new query contents in the same buffers."""
    h = vlr.Index.from_arrays(c1_index)
    B, npb, k = 48, 16, 10
    h.reserve(B, npb, k)
    Qs = datagen.make_queries(100_000, 128, 1024, 3 * B, stream=5).reshape(3, B, 128)
    ref = [gpu_search(h, Q, npb, k) for Q in Qs]
    Qd = torch.from_numpy(Qs[0].copy()).cuda()
    out = (torch.empty(B, k, dtype=torch.int64, device="cuda"), torch.empty(B, k, dtype=torch.float32, device="cuda"),
           torch.empty(B, npb, dtype=torch.uint8, device="cuda"), torch.empty(B, npb, dtype=torch.int32, device="cuda"))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h.search(Qd, npb, k, out=out, stream=s)  # warm-up on the capture stream
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h.search(Qd, npb, k, out=out, stream=s)
    for i in (1, 2, 0):
        Qd.copy_(torch.from_numpy(Qs[i]))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy(), ref[i]["ids"])
        assert np.array_equal(out[1].cpu().numpy(), ref[i]["dist"])
        assert np.array_equal(out[3].cpu().numpy(), ref[i]["probes"])
    del g
    h.close()


def test_nccl_exchange_path_single_rank(c1_index, c1_queries, monkeypatch):
    """The G > 1 exchange path (K7 into packed 16-B entries -> ncclAllGather on
    the search stream -> K8 merge-select) run on one GPU through a 1-rank NCCL
    communicator (VLR_FORCE_EXCHANGE=1): bitwise the plain search."""
    c = datagen.CONFIGS["C1"]
    h = vlr.Index.from_arrays(c1_index)
    a = gpu_search(h, c1_queries, c["nprobe"], c["k"])
    n_plain = h.last_launch_count
    h.close()
    monkeypatch.setenv("VLR_FORCE_EXCHANGE", "1")
    monkeypatch.setenv("VLR_COARSE_REPLICATED", "1")  # the replicated coarse stage: only the result exchange
    hx = vlr.Index.from_arrays(c1_index, nccl_id=vlr.nccl_unique_id())
    b = gpu_search(hx, c1_queries, c["nprobe"], c["k"])
    assert hx.last_launch_count == n_plain + 1  # + K8
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    hx.close()
    # and directly against the oracle (rules R1-R4), not only against the plain search
    o = oracle.search(c1_index, c1_queries, c["nprobe"], c["k"])
    errs = check(c1_index, c1_queries, b, o, idmap=oracle.IdMap(c1_index))
    assert not errs, errs


@pytest.mark.parametrize("flag,val", [("VLR_FILTER_PERSISTENT", "1"), ("VLR_FILTER_CLUSTER", "2"),
                                      ("VLR_FILTER_CLUSTER", "4"), ("VLR_FILTER_PAIR", "1"), ("VLR_EXACT_CFG", "4,4"),
                                      ("VLR_EXACT_CFG", "2,8"), ("VLR_EXACT_CFG", "2,2"), ("VLR_EXACT_CFG", "3,2,2"),
                                      ("VLR_EXACT_CFG", "3,4,2"), ("VLR_EXACT_CFG", "5,2,2"), ("VLR_EXACT_CFG", "16,1"),
                                      ("VLR_EXACT_CFG", "32,1"), ("VLR_FILTER_BTILED", "0")])
def test_filter_variant_parity(flag, val):
    """K1 experiment kernels (persistent k_filter_tc_p; query-tile multicast
    over 2- or 4-CTA clusters; the CTA-pair cta_group::2 kernel) and K3a (stages, warps) configurations other
    than the product's (3, 4), flags read once per process: probes stay
    bit-exact and results pass the parity rules, for batches 1, 64 and 200
    (nN 16, 64, 208). Runs in a subprocess so the flag does not leak."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, 'tests');"
        "import datagen, oracle, paper_2504_08930_b200 as vlr; from parity import check;"
        "ix = datagen.make_index(100_000, 128, 1024, 16);"
        "Q = datagen.make_queries(100_000, 128, 1024, 200, stream=2);"
        "h = vlr.Index.from_arrays(ix);"
        "bad = 0\n"
        "for nq, npb in ((1, 16), (64, 16), (200, 300)):\n"
        "    ids, dist, miss, prb = h.search(torch.from_numpy(Q[:nq]).cuda(), npb, 10, sync=True)\n"
        "    g = dict(ids=ids.cpu().numpy(), dist=dist.cpu().numpy(), miss=miss.cpu().numpy(), probes=prb.cpu().numpy())\n"
        "    bad += len(check(ix, Q[:nq], g, oracle.search(ix, Q[:nq], npb, 10), idmap=oracle.IdMap(ix)))\n"
        "sys.exit(1 if bad else 0)\n")
    import os
    env = dict(os.environ, **{flag: val})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_lut_side_stream_equals_serial(c1_index, c1_queries, monkeypatch):
    """K5 on its forked side stream (default) vs the serial order
    (VLR_LUT_SERIAL=1): bitwise-identical results, also for back-to-back
    searches with different query batches on one stream without a sync in
    between (the fork must order K5 after the previous search's scan, which
    read the same LUT buffer)."""
    c = datagen.CONFIGS["C1"]
    Qa = torch.from_numpy(np.ascontiguousarray(c1_queries)).cuda()
    Qb = torch.from_numpy(np.ascontiguousarray(c1_queries[::-1])).cuda()
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("VLR_LUT_SERIAL", mode)  # read once per handle at its first search
        h = vlr.Index.from_arrays(c1_index)
        outs = []
        for Q in (Qa, Qb, Qa, Qb):
            outs.append(h.search(Q, c["nprobe"], c["k"], sync=False))
        torch.cuda.synchronize()
        res[mode] = [[t.cpu().numpy() for t in o] for o in outs]
        h.close()
    for a, b in zip(res["0"], res["1"]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for i in (0, 1):  # the repeated batches agree with their first run
        for x, y in zip(res["0"][i], res["0"][i + 2]):
            assert np.array_equal(x, y)
    errs = check(c1_index, c1_queries, dict(zip(("ids", "dist", "miss", "probes"), res["0"][0])),
                 oracle.search(c1_index, c1_queries, c["nprobe"], c["k"]), idmap=oracle.IdMap(c1_index))
    assert not errs, errs
