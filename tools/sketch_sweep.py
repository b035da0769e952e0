"""Sketch-bound sweep: identify time and decisions with the neighbourhood
sketches off / at k = 4, 8, 16 bits per neighbour, per epsilon, on one
R-MAT graph loaded once.  Every setting's roles and cluster ids must equal
the sketch-off result (the bound only ever proves dissimilarity).

    python tools/sketch_sweep.py [scale] [mu] [eps,eps,...] [k,k,...]

Prints one JSON line per (eps, k): identify ms of a scan on a fresh load
(sketch built inside) and of a repeated scan (sketch cached), counters.
"""

import ctypes
import json
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_12281_b200 import _lib  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    mu = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    epss = (sys.argv[3] if len(sys.argv) > 3 else "0.2,0.3,0.5,0.8").split(",")
    ks = (sys.argv[4] if len(sys.argv) > 4 else "0,4,8,16").split(",")
    lib = _lib.load()
    try:
        import pynvml
        pynvml.nvmlInit()
        hdl = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clock = lambda: pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)  # noqa: E731
    except Exception:
        clock = lambda: None  # noqa: E731
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
    del uv
    eng = _lib.Engine()
    role = torch.empty(n, dtype=torch.uint8, device="cuda")
    clus = torch.empty(n, dtype=torch.int32, device="cuda")
    st = _lib.GsStats()
    for eps in epss:
        eps2 = _lib.eps2_struct(Fraction(eps))
        ref = None
        for k in ks:
            os.environ["GS_SKETCH"] = k
            res = []
            for rep in range(3):
                if rep == 0:
                    _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off.data_ptr(),
                                                      adj.data_ptr(), 1))
                _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), role.data_ptr(),
                                              clus.data_ptr(), 1, ctypes.byref(st)))
                res.append(round(st.phase_ms[_lib.GS_PH_IDENTIFY], 2))
            out = (role.clone(), clus.clone())
            if ref is None:
                ref = out
            same = bool(torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1]))
            print(json.dumps({"scale": scale, "eps": eps, "mu": mu, "k": int(k),
                              "identify_ms_fresh": res[0], "identify_ms_cached": res[1:],
                              "sketch_decided": int(st.sim_decided_by_sketch),
                              "intersections": int(st.sim_intersections),
                              "adj_probes": int(st.adj_probes), "sim_evals": int(st.sim_evals),
                              "cores": int(st.n_core), "clusters": int(st.n_clusters),
                              "equal_to_k0": same, "sm_mhz": clock()}), flush=True)
    os.environ.pop("GS_SKETCH", None)


if __name__ == "__main__":
    main()
