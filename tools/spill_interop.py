"""Spill-file interoperability with the reference, both directions (run with
the reference package on PYTHONPATH: baseline/_ref/pkg/src).

1. The reference's partition_graph writes GSCP files; this package's
   scan_out_of_core executes that reference PartitionPlan (its files are the
   only graph it is given) -- roles and canonical ids equal to the oracle.
2. This package's partition_graph writes the files; the reference's own
   scan_out_of_core executes our PartitionPlan (its load_partition reading our
   files) -- its result equivalent to the oracle (results_equivalent).
Prints one JSON line; exit 1 on any mismatch."""

import json
import os
import random
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from graphscan import EdgeList as RefEdgeList, build_graph as ref_build  # noqa: E402
from graphscan.oracle import results_equivalent, serial_scan as ref_serial  # noqa: E402
from graphscan.partition import (GraphMeta as RefMeta, estimate_memory as ref_est,  # noqa: E402
                                 partition_graph as ref_partition,
                                 scan_out_of_core as ref_ooc)

import paper_2311_12281_b200 as gs  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def gnm(n, m, seed):
    rng = random.Random(seed)
    e = set()
    while len(e) < m:
        u, v = rng.randrange(n), rng.randrange(n)
        if u != v:
            e.add((min(u, v), max(u, v)))
    return sorted(e)


def main():
    out = {"cases": []}
    ok = True
    for n, m, seed, mu, eps in ((600, 2400, 11, 3, "0.4"), (1500, 4500, 12, 2, "0.5")):
        edges = gnm(n, m, seed)
        rg = ref_build(RefEdgeList(n_hint=n, edges=edges))
        budget = 15 * n + ref_est(rg) // 4
        roles, cids = orc.serial_scan(orc.CSR(n, np.asarray(edges, np.int32)), mu, eps)
        case = {"n": n, "m": m, "mu": mu, "eps": eps, "budget": budget}
        with tempfile.TemporaryDirectory() as d:
            # 1. the reference's plan and files -> this engine
            rplan = ref_partition(rg, budget, spill_dir=os.path.join(d, "ref"))
            rplan.budget_bytes = 64 << 20  # the device's cap (the files keep the host budget)
            res, st = gs.scan_out_of_core(RefMeta.from_graph(rg), rplan, mu, eps)
            a = bool(np.array_equal(res.role_codes, roles) and np.array_equal(res.cluster_ids, cids))
            case["reference_plan_on_engine"] = {"partitions": len(rplan.partitions), "identical": a}
            # 2. this package's plan and files -> the reference's scan_out_of_core
            g = gs.build_graph(gs.EdgeList(n_hint=n, edges=np.asarray(edges, np.int32)))
            plan = gs.partition_graph(g, budget, spill_dir=os.path.join(d, "ours"))
            rres, _ = ref_ooc(RefMeta.from_graph(rg), plan, mu, eps)
            oracle_res = ref_serial(rg, mu, eps)
            eq = results_equivalent(rres, oracle_res)
            b = bool(eq.ok if hasattr(eq, "ok") else eq)
            case["engine_plan_on_reference"] = {"partitions": len(plan.partitions), "equivalent": b}
            ok = ok and a and b
        out["cases"].append(case)
    out["ok"] = ok
    print(json.dumps(out))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
