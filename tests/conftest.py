import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_index(g):
    """IndexArrays from the hand fixture tests/golden/tiny_hand.json."""
    import datagen
    cb = np.zeros((g["m"], 256, g["dsub"]), np.float32)
    for j, s, y in g["codewords_nonzero"]["entries"]:
        cb[j, s] = y
    lists = [(l["ids"], np.array(l["codes"], np.uint8)) for l in g["lists"]]
    return datagen.index_from_parts(np.array(g["centroids"], np.float32), cb, lists)


def fval(x):
    return np.inf if x == "inf" else float(x)


@pytest.fixture(scope="session")
def small_index():
    """A small clustered index (fast on CPU): N=6000, d=32, nlist=64, m=4."""
    import datagen
    return datagen.make_index(6000, 32, 64, 4, seed=7)


@pytest.fixture(scope="session")
def small_queries():
    import datagen
    return datagen.make_queries(6000, 32, 64, 48, seed=7, stream=2)


@pytest.fixture(scope="session")
def c1_index():
    import datagen
    c = datagen.CONFIGS["C1"]
    return datagen.make_index(c["N"], c["d"], c["nlist"], c["m"])


@pytest.fixture(scope="session")
def c1_queries():
    import datagen
    c = datagen.CONFIGS["C1"]
    return datagen.make_queries(c["N"], c["d"], c["nlist"], c["batch"], stream=2, alpha=c["alpha"])


def golden_pq4_index():
    """4-bit IndexArrays from tests/golden/tiny_pq4.json (hand-packed codes)."""
    import datagen
    g4 = load_golden("tiny_pq4.json")
    g = load_golden(g4["index"])
    cb = np.zeros((g["m"], g4["ksub"], g["dsub"]), np.float32)
    for j, s, y in g["codewords_nonzero"]["entries"]:
        cb[j, s] = y
    codes = np.array([row for lst in g4["codes_packed_per_list"] for row in lst], np.uint8)
    sizes = [len(lst) for lst in g4["codes_packed_per_list"]]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ids = np.array([i for l in g["lists"] for i in l["ids"]], np.int64)
    return datagen.IndexArrays(d=g["d"], nlist=g["nlist"], m=g["m"], centroids=np.array(g["centroids"], np.float32),
                               codebooks=cb, list_offsets=offs, ids=ids, codes=codes, nbits=4), g
