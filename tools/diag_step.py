"""Where does a bench step's time go?  Host wall time per C-ABI call (with a
stream sync on each side) against the engine's own phase events.

    python tools/diag_step.py [scale] [steps] [eps] [mu]
"""

import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_12281_b200 import _lib  # noqa: E402
from fractions import Fraction  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    eps = sys.argv[3] if len(sys.argv) > 3 else "0.5"
    mu = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    lib = _lib.load()
    n = 1 << scale
    cnt = 16 << scale
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_rmat_generate(scale, 16, 1, src.data_ptr(), dst.data_ptr(), None))
    torch.cuda.synchronize()
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    mm = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(mm), None))
    m = mm.value
    del src, dst
    csr = os.environ.get("GS_DIAG_EDGES") is None  # default: the bench's CSR call
    if csr:
        off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        adj = torch.empty(2 * m, dtype=torch.int32, device="cuda")
        _lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off.data_ptr(), adj.data_ptr(),
                                           None))
    torch.cuda.synchronize()
    eng = _lib.Engine()
    eps2 = _lib.eps2_struct(Fraction(eps))
    role = torch.empty(n, dtype=torch.uint8, device="cuda")
    clus = torch.empty(n, dtype=torch.int32, device="cuda")
    st = _lib.GsStats()
    for i in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if csr:
            _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off.data_ptr(), adj.data_ptr(), 1))
        else:
            _lib.check(lib.gs_engine_load_edges(eng.handle, n, m, uv.data_ptr(), 1))
        t1 = time.perf_counter()
        _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), role.data_ptr(),
                                      clus.data_ptr(), 1, ctypes.byref(st)))
        t2 = time.perf_counter()
        ph = [round(st.phase_ms[k], 2) for k in range(9)]
        print(f"step {i}: load {1e3 * (t1 - t0):.1f} ms (build ev {ph[1]}), scan {1e3 * (t2 - t1):.1f} ms "
              f"(phases {ph[2:8]}), launches {st.kernel_launches}, evals {st.sim_evals} "
              f"inters {st.sim_intersections} probes {st.adj_probes}", flush=True)


if __name__ == "__main__":
    main()
