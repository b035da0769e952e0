"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU.

The CPU oracle (oracle/, test infrastructure) is the checker; golden vectors
come from the Python reference itself (tests/golden/make_golden.py)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

TWO_COMMUNITIES = [
    (0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7),
    (1, 2), (1, 4), (1, 7), (2, 8), (4, 7),
    (8, 9),
    (9, 10), (9, 11), (9, 12), (9, 13),
    (10, 11), (10, 12), (10, 13), (11, 12), (11, 13), (12, 13),
]
SHARED_MEMBER_EDGES = [(0, 1), (0, 2), (1, 2), (2, 3), (3, 4), (4, 5), (4, 6), (5, 6)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


class Golden:
    def __init__(self):
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
            self.meta = json.load(f)
        self.arr = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))

    def cases(self):
        for k, c in enumerate(self.meta["cases"]):
            yield k, c

    def edges(self, k):
        return self.arr[f"g{k}_edges"]

    def get(self, k, name):
        return self.arr[f"g{k}_{name}"]

    def has(self, k, name):
        return f"g{k}_{name}" in self.arr.files


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.load()
    return oracle


def make_graph(n, edges):
    """A package Graph built by the CPU oracle's build_graph restatement
    (test helper, so CPU tests need no device)."""
    from oracle import oracle
    from paper_2311_12281_b200.graph import Graph

    c = oracle.CSR(n, np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    return Graph(n=c.n, m=c.m, vertex_offsets=c.vertex_offsets, adjacency=c.adjacency,
                 edge_ids=c.edge_ids, edge_list=c.edge_list, orig_ids=c.orig_ids)


def normalise_on_host(u, v):
    """graph.py:98-118's normalisation (sorted unique ids, self-loops dropped,
    duplicates merged) in numpy -- the CPU tier's checker for the parser, in
    place of the device normaliser the product calls (gs_normalize_sparse)."""
    from paper_2311_12281_b200.graph import EdgeList

    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    ids = np.unique(np.concatenate([u, v]))
    du, dv = np.searchsorted(ids, u), np.searchsorted(ids, v)
    keep = du != dv
    lo, hi = np.minimum(du, dv)[keep], np.maximum(du, dv)[keep]
    key = np.unique(lo * (len(ids) + 1) + hi)
    edges = np.stack([key // (len(ids) + 1), key % (len(ids) + 1)], axis=1).astype(np.int32)
    return EdgeList(n_hint=len(ids), edges=edges, orig_ids=ids.astype(np.uint32))


@pytest.fixture
def host_normaliser(monkeypatch):
    """CPU tier: parse_edge_list's normalisation step served by the numpy
    checker above (the product raises without a device)."""
    import paper_2311_12281_b200.graph as graph

    monkeypatch.setattr(graph, "_normalize", normalise_on_host)


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
