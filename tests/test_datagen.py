"""Seeded input generator (TOOLING) properties: determinism, per-shard
generation equals the full generation, ground-truth kNN equals a library
brute force, deal of hot lists."""
import numpy as np

import datagen


def test_generation_is_deterministic():
    a = datagen.make_index(3000, 16, 20, 4, seed=1)
    b = datagen.make_index(3000, 16, 20, 4, seed=1)
    for f in ("centroids", "codebooks", "list_offsets", "ids", "codes"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    qa = datagen.make_queries(3000, 16, 20, 50, seed=1, stream=2)
    qb = datagen.make_queries(3000, 16, 20, 50, seed=1, stream=2)
    assert np.array_equal(qa, qb)
    qc = datagen.make_queries(3000, 16, 20, 50, seed=1, stream=1)
    assert not np.array_equal(qa, qc)  # calibration and test streams are disjoint


def test_ids_are_a_permutation_and_duplicates_exist():
    ix = datagen.make_index(4000, 16, 20, 4, seed=2)
    assert np.array_equal(np.sort(ix.ids), np.arange(ix.N))
    Q = datagen.make_queries(4000, 16, 20, 400, seed=2, stream=2)
    nunique = len(np.unique(Q, axis=0))
    assert 300 < nunique < 400  # ~10% repeats


def test_ground_truth_matches_sklearn():
    from sklearn.neighbors import NearestNeighbors
    Q = datagen.make_queries(5000, 32, 40, 20, seed=3, stream=2)
    ix = datagen.make_index(5000, 32, 40, 8, seed=3, gt_queries=Q, chunk=1000)
    nn = NearestNeighbors(n_neighbors=10, algorithm="brute").fit(ix.vectors.astype(np.float64))
    _, i = nn.kneighbors(Q.astype(np.float64))
    rec = np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ix.ids[i], ix.gt_ids)])
    assert rec > 0.99


def test_deal_owners_round_robin_by_size():
    sizes = np.array([10, 8, 6, 4, 2])
    own = datagen.deal_owners(sizes, np.arange(5), 2)
    assert own.tolist() == [0, 1, 0, 1, 0]  # S:395 example: {10,6,2} and {8,4}
    own = datagen.deal_owners(np.array([5, 5, 5, 1]), np.array([3, 2, 1, 0]), 3)
    assert own.tolist() == [0, 1, 2, 0]  # equal sizes: ascending cluster id
    own = datagen.deal_owners(sizes, np.array([1, 3]), 2)
    assert own.tolist() == [-1, 0, -1, 1, -1]
