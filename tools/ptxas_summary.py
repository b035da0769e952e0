"""Registers and spills per kernel from the ptxas -v logs of the build
(paper_2311_12281_b200/csrc/*.ptxas.log).

    python tools/ptxas_summary.py [sim|build|...]
"""
import glob
import os
import re
import subprocess
import sys

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2311_12281_b200", "csrc")


def main():
    pats = sys.argv[1:] or ["*"]
    for pat in pats:
        for path in sorted(glob.glob(os.path.join(CSRC, f"{pat}.ptxas.log"))):
            cur = None
            spill = ""
            for line in open(path):
                m = re.search(r"Compiling entry function '(\S+)'", line)
                if m:
                    cur = m.group(1)
                    try:
                        cur = subprocess.run(["c++filt", cur], capture_output=True,
                                             text=True).stdout.strip()
                    except OSError:
                        pass
                m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
                if m:
                    spill = f"spill {m.group(1)}/{m.group(2)}"
                m = re.search(r"Used (\d+) registers", line)
                if m and cur:
                    print(f"{os.path.basename(path)[:-10]:8s} {m.group(1):>4s} regs  {spill:16s} {cur[:110]}")
                    cur = None


if __name__ == "__main__":
    main()
