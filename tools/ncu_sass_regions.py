"""Aggregate SASS executions/stall samples of one kernel into address bins
(basic-block-ish regions) to see which code region dominates.
   python tools/ncu_sass_regions.py rep kernel-substring [bin]"""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kern, hdr, ins = None, None, []
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]; hdr = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if kern and pat in kern and hdr and r:
        ins.append(dict(zip(hdr, r)))
tot_e = sum(float(i["Instructions Executed"] or 0) for i in ins)
tot_s = sum(float(i["Warp Stall Sampling (All Samples)"] or 0) for i in ins)
# regions: split where the execution count changes by > 3x between consecutive instructions
regs, cur = [], []
prev = None
for i in ins:
    e = float(i["Instructions Executed"] or 0)
    if prev is not None and cur and (e > 3 * prev + 1 or prev > 3 * e + 1):
        regs.append(cur); cur = []
    cur.append(i); prev = e
if cur: regs.append(cur)
print(f"total exe {tot_e:.3g} samples {tot_s:.3g}")
rs = []
for g in regs:
    e = sum(float(i["Instructions Executed"] or 0) for i in g)
    s = sum(float(i["Warp Stall Sampling (All Samples)"] or 0) for i in g)
    rs.append((s, e, g))
for s, e, g in sorted(rs, key=lambda x: -x[0])[:14]:
    first = g[0]; mx = max(float(i["Instructions Executed"] or 0) for i in g)
    print(f"{100*s/tot_s:5.1f}% stall {100*e/tot_e:5.1f}% exe  n={len(g):3d} x{mx:.3g}  {first['Address'][-5:]}  {first['Source'].strip()[:60]}")
