"""Cold-process latency of the first scan_in_memory call (the reference's
acceptance test allows 1.0 s, test_acceptance.py:104)."""
import os, sys, time
t0 = time.monotonic()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2311_12281_b200 as gs
t1 = time.monotonic()
from oracle import oracle as orc
edges = np.array([(0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7), (1, 2), (1, 4), (1, 7),
                  (2, 8), (4, 7), (8, 9), (9, 10), (9, 11), (9, 12), (9, 13), (10, 11), (10, 12),
                  (10, 13), (11, 12), (11, 13), (12, 13)], dtype=np.int32)
c = orc.CSR(14, edges)
g = gs.Graph(n=c.n, m=c.m, vertex_offsets=c.vertex_offsets, adjacency=c.adjacency,
             edge_ids=c.edge_ids, edge_list=c.edge_list, orig_ids=c.orig_ids)
t2 = time.monotonic()
r, _ = gs.scan_in_memory(g, 3, "0.6")
t3 = time.monotonic()
r, _ = gs.scan_in_memory(g, 3, "0.6")
t4 = time.monotonic()
print(f"import {t1 - t0:.3f}s  first scan {t3 - t2:.3f}s  second {1000 * (t4 - t3):.2f}ms")
