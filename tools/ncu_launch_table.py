"""Per-kernel table (launches, time, share, DRAM GB) of an ncu --metrics launch list.

    python tools/ncu_launch_table.py launches.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
K, M, V, I = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg, seen = OrderedDict(), {}
for r in rows[1:]:
    name = r[K].split("(")[0][:60]
    a = agg.setdefault(name, {"n": set(), "t": 0.0, "rd": 0.0, "wr": 0.0})
    a["n"].add(r[I])
    v = float(r[V].replace(",", ""))
    if r[M] == "gpu__time_duration.sum":
        a["t"] += v
    elif r[M] == "dram__bytes_read.sum":
        a["rd"] += v
    elif r[M] == "dram__bytes_write.sum":
        a["wr"] += v
tot = sum(a["t"] for a in agg.values())
unit = 1e6  # ns -> ms
print("| kernel | launches | time ms | share | DRAM read GB | DRAM write GB |")
print("|---|---|---|---|---|---|")
for k, a in agg.items():
    print(f"| `{k}` | {len(a['n'])} | {a['t'] / unit:.2f} | {100 * a['t'] / tot:.1f}% | "
          f"{a['rd'] / 1e9:.2f} | {a['wr'] / 1e9:.2f} |")
print(f"| total | | {tot / unit:.2f} | | | |")
