"""Shared test setup: the ``gpu`` marker, repo-root imports, fixtures.

``-m "not gpu"`` tests run on the CPU build container (oracle vs golden
vectors, integer preprocessing, C-ABI symbol checks); ``-m gpu`` tests call
the CUDA path through the C ABI and compare it with the oracle.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: config-1 sized checks (seconds to a minute)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


# destination-grouped toy edge list of the reference (tests/conftest.py:44-78)
TOY_EDGES = [
    (1, 0), (2, 0), (0, 1), (3, 1), (4, 2), (3, 2), (2, 3), (5, 3),
    (0, 4), (1, 4), (4, 4), (2, 5), (4, 5), (5, 5), (6, 5), (3, 6),
    (4, 6), (7, 6), (3, 7),
]
TOY_OWNER = np.array([0, 0, 0, 0, 1, 1, 2, 2], dtype=np.int64)
TOY_RANGES = [[(0, 2), (2, 4)], [(0, 1), (1, 2)], [(0, 1), (1, 2)]]


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_toy():
    return load_json("toy.json")


@pytest.fixture(scope="session")
def golden_small():
    meta = load_json("small.json")
    arr = dict(np.load(os.path.join(GOLDEN, "small.npz")))
    return meta, arr


@pytest.fixture(scope="session")
def golden_gat():
    meta = load_json("gat.json")
    arr = dict(np.load(os.path.join(GOLDEN, "gat.npz")))
    return meta, arr


@pytest.fixture(scope="session")
def golden_sets():
    return load_json("sets.json")


def random_set_instances(count=200, seed=123):
    """Same recipe and draw order as make_golden.set_instances."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(1, 5))
        n = int(rng.integers(1, 7))
        universe = int(rng.integers(8, 40))
        owner = rng.integers(0, m, size=universe)
        nbrs = []
        for _i in range(m):
            row = []
            for _j in range(n):
                k = int(rng.integers(0, max(2, universe // 2)))
                row.append(np.unique(rng.integers(0, universe, size=k)))
            nbrs.append(row)
        out.append((nbrs, owner))
    return out


def random_graph(rng, num_vertices=None, num_edges=None):
    """Random directed multigraph (reference tests/conftest.py:85-91 recipe)."""
    import paper_2311_14898_b200 as H
    V = int(rng.integers(4, 40)) if num_vertices is None else num_vertices
    E = int(rng.integers(V, 6 * V)) if num_edges is None else num_edges
    src = rng.integers(0, V, size=E)
    dst = rng.integers(0, V, size=E)
    return H.from_edges(src, dst, num_vertices=V)


def random_two_level(g, rng, m, n):
    import paper_2311_14898_b200 as H
    owner = rng.permutation(np.arange(g.num_vertices, dtype=np.int64) % m)
    return H.split_chunks(g, H.PartitionAssignment(owner=owner, m=m), n)
