"""Generate the golden fixtures from the Python reference itself.

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py            (writes tests/golden/golden.npz
                                                   and tests/golden/golden.json)

It imports graphscan from /root/reference/pkg/src (read-only) and records, per
graph and (epsilon, mu):
  * build_graph's arrays (graph.py:162-259) for a subset of graphs,
  * edge_similarities (oracle.py:47-55),
  * serial_scan in canonical form: role letters and cluster id =
    min core id of the class / min eligible label for members,
  * the reference engine (scan_in_memory, workers=1) internal roles, raw
    parent ids and its counters (sim_evals, adj_probes, union_retries,
    probe_bound_violations).
The GPU box never reads /root/reference; tests use these committed files.
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from graphscan import EdgeList, build_graph, edge_similarities, serial_scan  # noqa: E402
from graphscan.scan import (  # noqa: E402
    StatsReport,
    classify_hub_outlier,
    detect_clusters,
    identify_core,
    init_state,
)

from oracle import oracle as orc  # noqa: E402  (generator only: same R-MAT stream)

EPS_GRID = ["0.2", "0.3", "0.4", "0.5", "0.6", "0.7", "0.8"]
MU_GRID = [2, 3, 6, 10]
DENSITY_FACTORS = [0.5, 1, 2, 4, 8]
ROLE_CODE = {"core": 1, "member": 3, "hub": 5, "outlier": 6}

TWO_COMMUNITIES = [
    (0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7),
    (1, 2), (1, 4), (1, 7), (2, 8), (4, 7),
    (8, 9),
    (9, 10), (9, 11), (9, 12), (9, 13),
    (10, 11), (10, 12), (10, 13), (11, 12), (11, 13), (12, 13),
]
SHARED_MEMBER_EDGES = [(0, 1), (0, 2), (1, 2), (2, 3), (3, 4), (4, 5), (4, 6), (5, 6)]


def corpus_edges(seed: int):
    """test_acceptance.py:39-46"""
    rng = random.Random(1000 + seed)
    n = rng.randint(20, 200)
    factor = DENSITY_FACTORS[seed % len(DENSITY_FACTORS)]
    m = min(int(n * factor), n * (n - 1) // 2)
    pairs = [(u, v) for u in range(n) for v in range(u + 1, n)]
    return n, sorted(rng.sample(pairs, m))


def gnm_edges(n: int, m: int, seed: int):
    """conftest.py:20-25"""
    rng = random.Random(seed)
    all_pairs = [(u, v) for u in range(n) for v in range(u + 1, n)]
    return n, sorted(rng.sample(all_pairs, min(m, len(all_pairs))))


def canonical(o, n: int):
    roles = np.full(n, 6, dtype=np.uint8)
    cl = np.full(n, -1, dtype=np.int32)
    label_of = {}
    for label, vs in o.clusters.items():
        for v in vs & o.cores:
            label_of[v] = label
    for v in range(n):
        if v in o.cores:
            roles[v] = 1
            cl[v] = label_of[v]
        elif o.memberships.get(v):
            roles[v] = 3
            cl[v] = min(o.memberships[v])
        elif v in o.hubs:
            roles[v] = 5
        else:
            assert v in o.outliers
    return roles, cl


def engine_raw(g, mu: int, eps: str):
    st = init_state(g)
    stats = StatsReport(n=g.n, m=g.m)
    identify_core(g, mu, eps, st, workers=1, stats=stats)
    detect_clusters(g, eps, st, workers=1, stats=stats)
    classify_hub_outlier(g, st, workers=1, stats=stats)
    roles = np.frombuffer(bytes(st.role), dtype=np.uint8).copy()
    parent = np.array(st.parent, dtype=np.int32)
    cl = np.where(parent >= 0, parent, -1).astype(np.int32)
    ctr = dict(sim_evals=stats.sim_evals, adj_probes=stats.adj_probes,
               union_retries=stats.union_retries,
               probe_bound_violations=stats.probe_bound_violations)
    return roles, cl, ctr


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    index = []

    def add_case(name, n, edges, configs, keep_build=False, engine_configs=None):
        t0 = time.time()
        k = len(index)
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        g = build_graph(EdgeList(n_hint=n, edges=[tuple(map(int, p)) for p in e]))
        arrays[f"g{k}_edges"] = e
        commons = edge_similarities(g)
        arrays[f"g{k}_commons"] = np.asarray(commons, dtype=np.int32)
        if keep_build:
            arrays[f"g{k}_offsets"] = np.asarray(g.vertex_offsets, dtype=np.int64)
            arrays[f"g{k}_adjacency"] = np.asarray(g.adjacency, dtype=np.int32)
            arrays[f"g{k}_edge_ids"] = np.asarray(g.edge_ids, dtype=np.int32)
            arrays[f"g{k}_edge_list"] = np.asarray(g.edge_list, dtype=np.int32)
        cfgs = []
        for j, (eps, mu) in enumerate(configs):
            o = serial_scan(g, mu, eps, commons=commons)
            roles, cl = canonical(o, g.n)
            arrays[f"g{k}_c{j}_roles"] = roles
            arrays[f"g{k}_c{j}_cluster"] = cl
            entry = {"eps": eps, "mu": mu}
            if engine_configs is None or (eps, mu) in engine_configs:
                r_roles, r_cl, ctr = engine_raw(g, mu, eps)
                arrays[f"g{k}_c{j}_ref_roles"] = r_roles
                arrays[f"g{k}_c{j}_ref_cluster"] = r_cl
                entry["ref"] = ctr
            entry["n_core"] = int((roles == 1).sum())
            entry["n_member"] = int((roles == 3).sum())
            entry["n_hub"] = int((roles == 5).sum())
            cfgs.append(entry)
        index.append({"name": name, "n": g.n, "m": g.m, "build": keep_build, "configs": cfgs})
        print(f"{name}: n={g.n} m={g.m} configs={len(cfgs)} {time.time() - t0:.1f}s", flush=True)

    grid = [(e, mu) for e in EPS_GRID for mu in MU_GRID]
    add_case("two_communities", 14, sorted(TWO_COMMUNITIES), grid + [("0.6", 3)], keep_build=True)
    add_case("shared_member", 7, SHARED_MEMBER_EDGES, grid + [("0.5", 4)], keep_build=True)
    add_case("triangle", 3, [(0, 1), (0, 2), (1, 2)], [("0.5", 2)], keep_build=True)
    add_case("clique50", 50, [(u, v) for u in range(50) for v in range(u + 1, 50)],
             [("0.1", 3), ("0.9", 3)], keep_build=True)
    add_case("path64", 64, [(i, i + 1) for i in range(63)], [("0.5", 2), ("0.7", 2)],
             keep_build=True)
    add_case("pendant", 5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4)],
             [("0.8", 3)], keep_build=True)
    add_case("isolated", 4, [(0, 1)], [("0.5", 2)], keep_build=True)
    add_case("empty", 0, [], [("0.5", 2)], keep_build=True)
    add_case("edgeless5", 5, [], [("0.5", 2)], keep_build=True)
    add_case("threshold_exact", 14, sorted(TWO_COMMUNITIES),
             [("0.5", 2), ("0.500000000000001", 2), ("1", 2), (str(0.6), 3)], keep_build=False)
    for seed in range(40):
        n, edges = corpus_edges(seed)
        add_case(f"corpus{seed}", n, edges, grid, keep_build=seed < 5)
    for seed in range(8):
        n, edges = gnm_edges(40, 120, seed)
        add_case(f"gnm40_{seed}", n, edges, [("0.4", 3), ("0.25", 2), ("0.75", 2)])
    rmat_cfgs = [(e, mu) for e in ["0.2", "0.3", "0.4", "0.5", "0.6"] for mu in (3, 5)]
    n, edges = orc.rmat(10, seed=1)
    add_case("rmat10", n, edges, rmat_cfgs, keep_build=True)
    n, edges = orc.rmat(12, seed=7)
    add_case("rmat12", n, edges, rmat_cfgs, engine_configs={("0.2", 3), ("0.5", 5)})
    n, edges = orc.rmat(14, seed=1)
    add_case("rmat14", n, edges,
             [("0.6", 3), ("0.2", 3), ("0.2", 5), ("0.3", 3), ("0.3", 5), ("0.4", 3), ("0.4", 5),
              ("0.5", 5)],
             engine_configs={("0.6", 3), ("0.2", 3)})
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/pkg/src/graphscan", "cases": index}, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
