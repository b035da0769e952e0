"""One-off parity check at R-MAT s20 (16.8 M edges) against the C oracle,
through the pinned/pageable host CSR path, the edge-list path and the
device-CSR path (the bench's fused relabel + sort build).

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


def device_csr_scan(g, mu, eps):
    """gs_engine_load_csr from device-resident reference arrays + gs_engine_scan."""
    import ctypes

    import torch

    from paper_2311_12281_b200 import _lib

    lib = _lib.load()
    off = torch.from_numpy(np.asarray(g.vertex_offsets, dtype=np.int64)).cuda()
    adj = torch.from_numpy(np.asarray(g.adjacency, dtype=np.int32)).cuda()
    torch.cuda.synchronize()
    eng = _lib.Engine()
    try:
        _lib.check(lib.gs_engine_load_csr(eng.handle, g.n, g.m, off.data_ptr(), adj.data_ptr(), 1))
        roles = np.empty(g.n, np.uint8)
        cl = np.empty(g.n, np.int32)
        eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps))
        _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), roles.ctypes.data,
                                      cl.ctypes.data, 0, None))
        return roles, cl
    finally:
        eng.close()


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
        r3 = device_csr_scan(g, mu, eps)  # the bench's path: fused relabel + sort build
        ok = (np.array_equal(r.role_codes, roles) and np.array_equal(r.cluster_ids, cl)
              and np.array_equal(r2.role_codes, roles) and np.array_equal(r2.cluster_ids, cl)
              and np.array_equal(r3[0], roles) and np.array_equal(r3[1], cl))
        print(f"s{scale} eps={eps} mu={mu}: {'IDENTICAL' if ok else 'MISMATCH'} "
              f"(cores {int((roles == 1).sum())}, clusters {len(set(cl[roles == 1].tolist()))}, "
              f"hubs {int((roles == 5).sum())}; oracle {t1 - t0:.1f}s)", flush=True)
        if not ok:
            sys.exit(1)


if __name__ == "__main__":
    main()
