"""Out-of-core benchmark: R-MAT scale-27 (>= 1.8B edges) clustered under a
2 GB HBM cap, the CSR streamed from pinned host memory (BASELINE configs[3]).

    python tools/ooc_bench.py [--scale 27] [--cap 2000000000] [--eps 0.5] [--mu 5] [--verify]

Input preparation (generation, normalisation, CSR build) runs on the device
without a cap and is NOT part of the measured run; the CSR is then moved to
pinned host memory and every device byte the partitioned scan allocates is
counted against the cap by the engine allocator.  nvidia-smi memory.used is
sampled during the run as independent evidence.  --verify re-runs the same
graph with the in-HBM engine and compares roles and cluster ids.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_12281_b200 as gs  # noqa: E402
from paper_2311_12281_b200 import _lib  # noqa: E402


def smi_used_mib():
    out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=memory.used",
                          "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
    return int(out.strip().splitlines()[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=27)
    ap.add_argument("--cap", type=int, default=2_000_000_000)
    ap.add_argument("--eps", default="0.5")
    ap.add_argument("--mu", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--verify", action="store_true")
    args = ap.parse_args()
    lib = _lib.load()
    n = 1 << args.scale
    cnt = 16 << args.scale
    t0 = time.time()
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_rmat_generate(args.scale, 16, args.seed, src.data_ptr(), dst.data_ptr(), None))
    torch.cuda.synchronize()
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    mm = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(mm), None))
    m = int(mm.value)
    del src, dst
    torch.cuda.empty_cache()
    off_d = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    adj_d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off_d.data_ptr(), adj_d.data_ptr(),
                                       None))
    torch.cuda.synchronize()
    del uv
    off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    adj_h = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
    off_h.copy_(off_d)
    adj_h.copy_(adj_d)
    dmax = int((off_d[1:] - off_d[:-1]).max().item())
    del off_d, adj_d
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    prep_s = time.time() - t0
    role = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    clus = torch.empty(n, dtype=torch.int32, pin_memory=True)
    eps2 = _lib.eps2_struct(gs.epsilon_fraction(args.eps), dmax)
    st = _lib.GsStats()
    base_mib = smi_used_mib()
    samp = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=memory.used",
                             "--format=csv,noheader,nounits", "-lms", "100"],
                            stdout=subprocess.PIPE, text=True)
    time.sleep(0.5)
    t1 = time.time()
    _lib.check(lib.gs_scan_partitioned(n, m, off_h.data_ptr(), adj_h.data_ptr(), args.mu,
                                       ctypes.byref(eps2), args.cap, role.data_ptr(),
                                       clus.data_ptr(), ctypes.byref(st)))
    wall = time.time() - t1
    time.sleep(0.3)
    samp.terminate()
    used = [int(x) for x in samp.stdout.read().split() if x.strip().isdigit()]
    line = {
        "workload": f"R-MAT scale-{args.scale} edgefactor 16 seed {args.seed}, eps={args.eps} "
                    f"mu={args.mu}, out-of-core under an HBM cap",
        "n": n, "m": m, "dmax": dmax, "cap_bytes": args.cap,
        "peak_engine_device_bytes": int(st.peak_device_bytes),
        "nvidia_smi_used_mib": {"before": base_mib, "max_during": max(used) if used else None,
                                "delta_mib": (max(used) - base_mib) if used else None},
        "partitions": int(st.partitions),
        "seconds": wall,
        "edges_per_s": m / wall,
        "phases_ms": {"sketch_prepass": st.phase_ms[1], "identify": st.phase_ms[2],
                      "cluster": st.phase_ms[4],
                      "classify": st.phase_ms[5], "total_device": st.phase_ms[7]},
        "counts": {"sim_evals": int(st.sim_evals), "decided_by_bound": int(st.sim_decided_by_bound),
                   "decided_by_sketch": int(st.sim_decided_by_sketch),
                   "intersections": int(st.sim_intersections), "adj_probes": int(st.adj_probes),
                   "cores": int(st.n_core), "members": int(st.n_member), "hubs": int(st.n_hub),
                   "outliers": int(st.n_outlier), "clusters": int(st.n_clusters)},
        "prep_s": prep_s,
        "kernel_launches": int(st.kernel_launches),
    }
    if args.verify:
        eng = _lib.Engine()
        r2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        c2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
        st2 = _lib.GsStats()
        t2 = time.time()
        _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_h.data_ptr(), adj_h.data_ptr(), 0))
        _lib.check(lib.gs_engine_scan(eng.handle, args.mu, ctypes.byref(eps2), r2.data_ptr(),
                                      c2.data_ptr(), 0, ctypes.byref(st2)))
        line["in_hbm_seconds"] = time.time() - t2
        line["verify_equal_to_in_hbm"] = bool(torch.equal(r2, role) and torch.equal(c2, clus))
        eng.close()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
