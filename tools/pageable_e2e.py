"""scan_in_memory on the s24 graph from PAGEABLE host arrays (what a caller of
the reference API passes: numpy / array.array), against the pinned path.

    python tools/pageable_e2e.py [scale]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_12281_b200 as gs  # noqa: E402
from paper_2311_12281_b200 import _lib  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    lib = _lib.load()
    n, cnt = 1 << scale, 16 << scale
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_rmat_generate(scale, 16, 1, src.data_ptr(), dst.data_ptr(), None))
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    mm = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(mm), None))
    m = mm.value
    del src, dst
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off.data_ptr(), adj.data_ptr(), None))
    torch.cuda.synchronize()

    class G:
        pass

    g = G()
    g.n, g.m = n, m
    g.vertex_offsets = off.cpu().numpy()
    g.adjacency = adj.cpu().numpy()
    g.orig_ids = np.arange(n, dtype=np.uint32)
    if os.environ.get("GS_PROFILE"):
        import cProfile
        import pstats

        gs.scan_in_memory(g, 5, "0.5")
        pr = cProfile.Profile()
        pr.enable()
        gs.scan_in_memory(g, 5, "0.5")
        pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
        return
    for i in range(4):
        t0 = time.perf_counter()
        r, s = gs.scan_in_memory(g, 5, "0.5")
        t1 = time.perf_counter()
        print(f"pageable scan_in_memory: {1e3 * (t1 - t0):.1f} ms wall "
              f"(build {s.extra['build_us'] / 1e3:.1f} ms, scan {s.phases['identify'] / 1e3:.1f} ms)",
              flush=True)


if __name__ == "__main__":
    main()
