"""Summarise an ncu report's SASS source page: per kernel, the hottest
instructions by warp-stall samples and executions.

    python tools/ncu_sass_summary.py gpurun_out/x.ncu-rep [kernel-substring] [top]
"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kern = None
    blocks = {}
    hdr = None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kern = r[1]
            blocks[kern] = []
            hdr = None
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if kern and hdr and r:
            blocks[kern].append(dict(zip(hdr, r)))
    for k, ins in blocks.items():
        if pat and pat not in k:
            continue
        tot = sum(float(i.get("Warp Stall Sampling (All Samples)", 0) or 0) for i in ins)
        texe = sum(float(i.get("Instructions Executed", 0) or 0) for i in ins)
        print(f"=== {k}\n    samples {tot:.0f}  warp-instructions {texe:.3g}")
        ins_sorted = sorted(ins, key=lambda i: -float(i.get("Warp Stall Sampling (All Samples)", 0) or 0))
        for i in ins_sorted[:top]:
            s = float(i.get("Warp Stall Sampling (All Samples)", 0) or 0)
            e = float(i.get("Instructions Executed", 0) or 0)
            print(f"  {100 * s / max(tot, 1):5.1f}%  exe {e:10.3g}  {i['Address'][-5:]}  {i['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
