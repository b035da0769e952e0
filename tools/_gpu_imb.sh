# per-kernel SM-time imbalance (max / avg of sm__cycles_active) of the identify kernels at eps $1
mkdir -p gpurun_out
GS_NO_WARMUP=1 timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,sm__cycles_active.min,smsp__warps_active.avg.pct_of_peak_sustained_active --clock-control none --print-units base --csv --log-file gpurun_out/imb_$1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --python-ref-seconds 0 --eps $1 > /dev/null 2>&1
python - $1 <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/imb_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; K, M, V, ID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    if "k_sim" in r[K] or "k_sk_filter" in r[K]:
        d.setdefault((r[ID], r[K][:34]), {})[r[M]] = float(r[V].replace(",", ""))
for (i, k), v in d.items():
    t = v.get("gpu__time_duration.sum", 0) / 1e6
    if t < 0.05: continue
    print(f"{k:36s} {t:8.3f} ms  max/avg {v['sm__cycles_active.max'] / max(1, v['sm__cycles_active.avg']):.2f}  min/avg {v['sm__cycles_active.min'] / max(1, v['sm__cycles_active.avg']):.2f}  warps {v['smsp__warps_active.avg.pct_of_peak_sustained_active']:.0f}%")
PY
