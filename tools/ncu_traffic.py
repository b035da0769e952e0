"""DRAM traffic of the identify pass per kernel class, from an ncu launch list
of ONE bench step, stamped with the engine's source hash (bench.py refuses a
record taken on other sources: `roofline.traffic` is then null).

    GS_NO_WARMUP=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --print-units base --csv --log-file L.csv \
        python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0
    python tools/ncu_traffic.py L.csv --config "s24 eps=0.5 mu=5" [--out profiles/sim_traffic.json]

Classes (gs_stats.kernel_bytes order): 0 prep (thresholds, degree tables,
hub split, sketch build, Lemma-1 pre-pass), 1 k_sim_hash<1024,true>,
2 k_sim_hash<1024,false>, 3 k_sim_hash<512,false>, 4 k_sim_warp, 5 k_sim_tiny,
6 identify stage 1 (k_p1_items, k_p1_owner, k_sk_filter).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PREP = ("k_thresholds", "k_degree_tables", "k_hubsplit", "k_sk_sizes", "k_sk_warp", "k_sk_cta",
        "k_sk_bytes", "k_prepass_bs")


def kernel_class(name: str):
    # ncu prints template flags as 0 / 1
    if "k_sim_hash<1024, 1>" in name or "k_sim_hash<1024, true>" in name:
        return 1
    if "k_sim_hash<1024, 0>" in name or "k_sim_hash<1024, false>" in name:
        return 2
    if "k_sim_hash<512, 0>" in name or "k_sim_hash<512, false>" in name:
        return 3
    if "k_sim_warp" in name:
        return 4
    if "k_sim_tiny" in name:
        return 5
    if any(k in name for k in ("k_sk_filter", "k_p1_items", "k_p1_owner")):
        return 6
    if any(k in name for k in PREP):
        return 0
    return None


def to_base(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    return x * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sim_traffic.json"))
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    h = rows[0]
    K, M, V, U, ID = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"), h.index("ID"))
    classes: dict = {}
    for r in rows[1:]:
        c = kernel_class(r[K])
        if c is None:
            continue
        d = classes.setdefault(str(c), {"dram_bytes": 0.0, "ns": 0.0, "launches": set()})
        d["launches"].add(r[ID])
        v = to_base(r[V], r[U])
        if r[M] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            d["dram_bytes"] += v
        elif r[M] == "gpu__time_duration.sum":
            d["ns"] += v
    from bench import source_hash

    out = {"config": a.config, "source_hash": source_hash(),
           "when": time.strftime("%Y-%m-%dT%H:%MZ", time.gmtime()),
           "source": f"{os.path.basename(a.csv)}: ncu --metrics gpu__time_duration.sum,"
                     "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none of one "
                     "bench step (serialised, cold-cache launches)",
           "classes": {k: {"dram_bytes": v["dram_bytes"], "ncu_ms": v["ns"] / 1e6,
                           "launches": len(v["launches"])} for k, v in sorted(classes.items())}}
    out["identify_dram_bytes"] = sum(v["dram_bytes"] for v in out["classes"].values())
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
