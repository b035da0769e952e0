"""Stall samples / executed instructions per CUDA source line of one kernel
(ncu cuda,sass view).  python tools/ncu_line_stalls.py rep kernel-regex [skip] [top]"""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{pat}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr and r[0] and len(r) >= 8:  # a CUDA line row: aggregated metrics
        key = f"{fname}:{r[0]}"
        f = lambda x: float(x) if x not in ("", "-") else 0.0
        try:
            st, ex = f(r[4]), f(r[7])
        except ValueError:
            continue
        agg[key] = (st, ex, r[1].strip()[:80])
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts:.3g}, warp instructions {te:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / ts:5.1f}% stall {100 * v[1] / te:5.1f}% inst  {k:18s} {v[2]}")
