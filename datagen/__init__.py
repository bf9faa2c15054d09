"""Seeded synthetic inputs for the IVF-PQ hot-partition search (TOOLING).

This package is the ONLY code shared by the CUDA path's tests/bench and the
oracle: it produces input arrays (centroids, PQ codebooks, inverted lists,
query streams, hot sets). It holds none of the search method's arithmetic
(no coarse distances used as results, no LUTs, no ADC, no top-k of search);
index *construction* (k-means for PQ codebooks, nearest-codeword encoding) is
input preparation, as in PAPER.md:141-142 (§II.A) where the index is built
before search.
"""
from .gen import (  # noqa: F401
    CONFIGS,
    IndexArrays,
    make_index,
    make_queries,
    access_counts,
    hot_from_mass,
    coverage_mean_hitrate,
    topk_share,
    index_from_parts,
    list_sizes,
    centroids,
    layout,
    deal_owners,
    pack_nibbles,
)
