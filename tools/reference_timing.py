"""Time the REFERENCE's own CPU path -- graphscan.scan_in_memory (scan.py:965-982)
and the oracle serial_scan (oracle.py:97-190) from baseline/_ref, unmodified --
on the box's host cores, beside the B200 engine on the same graphs
(BASELINE.md section 3 step 1).

    python tools/reference_timing.py [--scales 12 14 16] [--eps 0.5] [--mu 5]
        [--extrapolate 24]

Per scale: R-MAT (the same counter-based generator as the device, host side),
the reference's own build_graph, then scan_in_memory with workers=1 and
workers=os.cpu_count() (a ThreadPoolExecutor under the GIL), serial_scan, and
the engine's scan_in_memory on the same Graph; results compared with the
reference's results_equivalent.  ns per adjacency probe is fitted from the
reference's own counters; --extrapolate S prices scale S with the probe count
of the C restatement of the reference engine (oracle/, exact counters), which
is labelled as an extrapolation.  One JSON line per measurement."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", type=int, nargs="+", default=[12, 14, 16])
    ap.add_argument("--eps", default="0.5")
    ap.add_argument("--mu", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--extrapolate", type=int, default=0)
    ap.add_argument("--no-threads", action="store_true", help="skip workers=cpu_count")
    args = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "graphscan")):
        print(json.dumps({"unavailable": "baseline/_ref/graphscan not present"}))
        return 1
    sys.path.insert(0, REF)
    import graphscan
    from graphscan.graph import EdgeList as RefEdgeList
    from graphscan.graph import build_graph as ref_build
    from graphscan.oracle import results_equivalent, serial_scan

    import paper_2311_12281_b200 as gs
    from oracle import oracle as orc

    cores = os.cpu_count()
    fits = []
    for s in args.scales:
        n, edges = orc.rmat(s, seed=args.seed)
        el = RefEdgeList(n_hint=n, edges=[(int(u), int(v)) for u, v in edges])
        t0 = time.perf_counter()
        g = ref_build(el)
        t_build = time.perf_counter() - t0
        rec = {"graph": f"R-MAT s{s} ef16 seed {args.seed}", "n": g.n, "m": g.m,
               "eps": args.eps, "mu": args.mu, "host_cores": cores,
               "ref_build_graph_s": round(t_build, 3)}
        t0 = time.perf_counter()
        res1, st1 = graphscan.scan_in_memory(g, args.mu, args.eps, workers=1)
        rec["ref_scan_in_memory_workers1_s"] = round(time.perf_counter() - t0, 3)
        rec["ref_adj_probes"] = st1.adj_probes
        rec["ref_sim_evals"] = st1.sim_evals
        if not args.no_threads:
            t0 = time.perf_counter()
            graphscan.scan_in_memory(g, args.mu, args.eps, workers=cores)
            rec[f"ref_scan_in_memory_workers{cores}_s"] = round(time.perf_counter() - t0, 3)
        t0 = time.perf_counter()
        oracle_res = serial_scan(g, args.mu, args.eps)
        rec["ref_serial_scan_s"] = round(time.perf_counter() - t0, 3)
        rec["ref_equivalent_to_serial_scan"] = bool(results_equivalent(res1, oracle_res))
        rec["ref_ns_per_probe"] = round(1e9 * rec["ref_scan_in_memory_workers1_s"] /
                                        max(1, st1.adj_probes), 1)
        fits.append((st1.adj_probes, st1.sim_evals, rec["ref_scan_in_memory_workers1_s"]))
        if gs._lib.load().gs_device_count() == 0:
            print(json.dumps(rec), flush=True)
            continue
        # the engine on the reference's own Graph object (first call warms the context)
        gs.scan_in_memory(g, args.mu, args.eps)
        t0 = time.perf_counter()
        res, st = gs.scan_in_memory(g, args.mu, args.eps)
        rec["engine_scan_in_memory_wall_s"] = round(time.perf_counter() - t0, 4)
        ref_view = graphscan.ClusteringResult(
            n=res.n, roles=[graphscan.Role(r.value) for r in res.roles],
            cluster_id=list(res.cluster_id), orig_ids=list(res.orig_ids))
        rep = results_equivalent(ref_view, oracle_res)
        rec["engine_equivalent_to_serial_scan"] = bool(rep)
        rec["speedup_engine_vs_ref_workers1"] = round(
            rec["ref_scan_in_memory_workers1_s"] / rec["engine_scan_in_memory_wall_s"], 1)
        print(json.dumps(rec), flush=True)
    if args.extrapolate and fits:
        # the probe loop is the reference's runtime (99.5%): price
        # the target's probes at the largest measured scale's s/probe
        spp = fits[-1][2] / max(1, fits[-1][0])
        s = args.extrapolate
        n, edges = orc.rmat(s, seed=args.seed)
        t0 = time.perf_counter()
        c = orc.CSR(n, edges)
        _, _, cnt = orc.ref_scan(c, args.mu, args.eps)
        t_c = time.perf_counter() - t0
        est = float(spp * cnt["adj_probes"])
        print(json.dumps({
            "graph": f"R-MAT s{s} ef16 seed {args.seed}", "n": c.n, "m": c.m, "eps": args.eps,
            "mu": args.mu, "kind": "EXTRAPOLATION (not a measurement)",
            "fit": {"ns_per_probe": round(1e9 * spp, 1), "from_scale": args.scales[-1],
                    "ns_per_probe_by_scale": [round(1e9 * t / max(1, p), 1)
                                              for p, _, t in fits]},
            "probes_from": "oracle/ C restatement of scan_in_memory(workers=1), exact counters "
                           f"({t_c:.0f} s incl. build)",
            "adj_probes": cnt["adj_probes"], "sim_evals": cnt["sim_evals"],
            "ref_scan_in_memory_workers1_s_extrapolated": round(est, 1),
            "ref_scan_in_memory_workers1_days_extrapolated": round(est / 86400, 2)}),
            flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
