"""Generate the GSCP spill fixtures from the Python reference itself.

Run in the build container, where the reference is importable:

    python tests/golden/make_spill_golden.py     (writes tests/golden/spill/)

For each case it runs the reference's ``partition_graph(g, budget, spill_dir)``
(partition.py:231-333) and keeps what it wrote: the partition files
``part-NNNNN.bin`` (GSCP, partition.py:336-375) and ``plan.manifest``
(partition.py:318-333), plus ``case.json`` with the edge list and budget.  It
then runs the reference's ``scan_out_of_core`` over that plan and records its
roles, and the InfeasibleBudgetError it raises for a budget just too small.
The GPU box never reads /root/reference; tests use these committed files.
"""

from __future__ import annotations

import json
import os
import random
import shutil
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "spill")

from graphscan import EdgeList, build_graph  # noqa: E402
from graphscan.partition import (  # noqa: E402
    GraphMeta,
    InfeasibleBudgetError,
    estimate_memory,
    partition_graph,
    scan_out_of_core,
)

TWO_COMMUNITIES = [
    (0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7),
    (1, 2), (1, 4), (1, 7), (2, 8), (4, 7),
    (8, 9),
    (9, 10), (9, 11), (9, 12), (9, 13),
    (10, 11), (10, 12), (10, 13), (11, 12), (11, 13), (12, 13),
]


def sparse_gnm(n: int, m: int, seed: int):
    """tests/test_acceptance.py:49-57 of the reference."""
    rng = random.Random(seed)
    edges = set()
    while len(edges) < m:
        u = rng.randrange(n)
        v = rng.randrange(n)
        if u != v:
            edges.add((u, v) if u < v else (v, u))
    return sorted(edges)


def skewed(n: int, m: int, seed: int):
    """A few hubs plus a sparse rest: closures of very different sizes."""
    rng = random.Random(seed)
    edges = set()
    while len(edges) < m:
        u = rng.randrange(8) if rng.random() < 0.3 else rng.randrange(n)
        v = rng.randrange(n)
        if u != v:
            edges.add((u, v) if u < v else (v, u))
    return sorted(edges)


def cases():
    yield "fig1", 14, TWO_COMMUNITIES, lambda g: 15 * g.n + 420, (3, "0.6")
    e = sparse_gnm(300, 900, 404)
    yield "gnm300", 300, e, None, (3, "0.5")
    e = skewed(400, 1500, 7)
    yield "skewed400", 400, e, None, (3, "0.4")


def main() -> None:
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    for name, n, edges, budget_fn, (mu, eps) in cases():
        g = build_graph(EdgeList(n_hint=n, edges=edges))
        # the acceptance test's budget, 15n + est/3 (test_acceptance.py:140-183)
        budget = budget_fn(g) if budget_fn else 15 * g.n + estimate_memory(g) // 3
        d = os.path.join(OUT, name)
        plan = partition_graph(g, budget, spill_dir=d)
        res, stats = scan_out_of_core(GraphMeta.from_graph(g), plan, mu, eps)
        # the spill files as partition_graph wrote them (scan_out_of_core's
        # store_sim rewrote the sim sections; they start all SIM_UNKNOWN = 0)
        for p in plan.partitions:
            with open(p.path, "r+b") as f:
                f.seek(-p.m_local, os.SEEK_END)
                f.write(bytes(p.m_local))
        case = {"n": n, "edges": [list(x) for x in edges], "budget": budget, "mu": mu,
                "eps": eps, "partitions": len(plan.partitions),
                "roles": "".join(r.name[0] for r in res.roles),
                "cluster_ids": list(res.cluster_id)}
        try:  # the reference's InfeasibleBudgetError for a budget just too small
            partition_graph(g, 15 * g.n + 200, spill_dir=os.path.join(d, "_x"))
            infeasible = None
        except InfeasibleBudgetError as exc:
            infeasible = {"budget": exc.budget_bytes, "edge": list(exc.edge),
                          "required": exc.required_bytes}
        shutil.rmtree(os.path.join(d, "_x"), ignore_errors=True)
        case["infeasible"] = infeasible
        with open(os.path.join(d, "case.json"), "w") as f:
            json.dump(case, f)
        print(name, "n", g.n, "m", g.m, "budget", budget, "partitions", len(plan.partitions),
              "sim_evals", stats.sim_evals)


if __name__ == "__main__":
    main()
