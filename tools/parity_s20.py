"""One-off parity check at R-MAT s20 (16.8 M edges) against the C oracle,
through the pinned/pageable host CSR path and the edge-list path.

    python tools/parity_s20.py [scale] [eps:mu,eps:mu...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

import paper_2311_12281_b200 as gs  # noqa: E402
from conftest import make_graph  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    n, e = orc.rmat(scale, seed=7)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    cfgs = (("0.15", 3), ("0.3", 4), ("0.5", 5), ("0.75", 2))
    if len(sys.argv) > 2:  # e.g. "0.5:5,0.2:5"
        cfgs = tuple((c.split(":")[0], int(c.split(":")[1])) for c in sys.argv[2].split(","))
    for eps, mu in cfgs:
        t0 = time.time()
        roles, cl = orc.serial_scan(c, mu, eps)
        t1 = time.time()
        r, s = gs.scan_in_memory(g, mu, eps)
        r2, _ = gs.scan_edges(n, e, mu, eps)
        ok = (np.array_equal(r.role_codes, roles) and np.array_equal(r.cluster_ids, cl)
              and np.array_equal(r2.role_codes, roles) and np.array_equal(r2.cluster_ids, cl))
        print(f"s{scale} eps={eps} mu={mu}: {'IDENTICAL' if ok else 'MISMATCH'} "
              f"(cores {int((roles == 1).sum())}, clusters {len(set(cl[roles == 1].tolist()))}, "
              f"hubs {int((roles == 5).sum())}; oracle {t1 - t0:.1f}s)", flush=True)
        if not ok:
            sys.exit(1)


if __name__ == "__main__":
    main()
