"""Parity at the scale of the BASELINE configs (VERDICT r01 "next round" #1).

    python tools/parity_scale.py rmat    --scale 24 [--seed 1] [--cfg 0.2:5,0.5:5,...]
    python tools/parity_scale.py chunglu --logn 22 --samples 80000000 [--wmax 6e4] [--cfg ...]
    python tools/parity_scale.py ooc     --scale 24 --cap 2000000000 [--cfg ...] [--oracle]

rmat / chunglu: the device result (three input paths: the drop-in
``scan_in_memory`` on pageable host arrays, the device-CSR call the bench
times, and the device edge-list build) against the C oracle's
``serial_scan`` (oracle.py:97-190 restated in oracle/, pinned to the
reference's goldens).  One common-neighbour pass of the oracle
(``commons_marked``) serves every (eps, mu) of the sweep.

ooc: the out-of-core engine under an HBM cap (gs_scan_partitioned, CSR in
pinned host memory) against the in-HBM engine on the same CSR and, with
--oracle, against serial_scan as well.

Each configuration prints one JSON line; "identical" is true only when roles
and canonical cluster ids match bit for bit.  Exit status 1 on any mismatch.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2311_12281_b200 as gs  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2311_12281_b200 import _lib  # noqa: E402


def parse_cfg(s: str):
    return [(c.split(":")[0], int(c.split(":")[1])) for c in s.split(",")]


def summary(roles, cl):
    core = roles == 1
    return {"cores": int(core.sum()), "clusters": int(len(np.unique(cl[core]))),
            "members": int((roles == 3).sum()), "hubs": int((roles == 5).sum()),
            "outliers": int((roles == 6).sum())}


def device_csr_scan(n, m, off, adj, mu, eps):
    """The bench's call: gs_engine_load_csr from device arrays + gs_engine_scan."""
    import torch

    lib = _lib.load()
    off_d = torch.from_numpy(off).cuda()
    adj_d = torch.from_numpy(adj).cuda()
    torch.cuda.synchronize()
    eng = _lib.Engine()
    try:
        _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_d.data_ptr(), adj_d.data_ptr(), 1))
        roles = np.empty(n, np.uint8)
        cl = np.empty(n, np.int32)
        eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps))
        _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), roles.ctypes.data,
                                      cl.ctypes.data, 0, None))
        return roles, cl
    finally:
        eng.close()
        del off_d, adj_d
        torch.cuda.empty_cache()


def compare_all(tag, n, edges, cfgs, extra=None):
    t0 = time.time()
    c = orc.CSR(n, edges)
    t1 = time.time()
    cm = orc.commons_marked(c)
    t2 = time.time()
    head = {"graph": tag, "n": n, "m": c.m, "dmax": c.deg_max,
            "oracle_build_s": round(t1 - t0, 1), "oracle_commons_s": round(t2 - t1, 1)}
    if extra:
        head.update(extra)
    print(json.dumps(head), flush=True)
    g = gs.Graph(n=n, m=c.m, vertex_offsets=c.vertex_offsets, adjacency=c.adjacency,
                 edge_ids=c.edge_ids, edge_list=c.edge_list, orig_ids=c.orig_ids)
    ok_all = True
    for eps, mu in cfgs:
        t3 = time.time()
        roles, cl = orc.serial_scan(c, mu, eps, commons=cm)
        t4 = time.time()
        r1, s1 = gs.scan_in_memory(g, mu, eps)                      # drop-in, pageable host
        t5 = time.time()
        r2 = device_csr_scan(n, c.m, c.vertex_offsets, c.adjacency, mu, eps)  # bench path
        r3, _ = gs.scan_edges(n, edges, mu, eps)                     # device edge-list build
        paths = {"scan_in_memory_host": (r1.role_codes, r1.cluster_ids),
                 "device_csr": r2, "device_edges": (r3.role_codes, r3.cluster_ids)}
        same = {k: bool(np.array_equal(v[0], roles) and np.array_equal(v[1], cl))
                for k, v in paths.items()}
        ok = all(same.values())
        ok_all &= ok
        line = {"graph": tag, "eps": eps, "mu": mu, "identical": ok, "paths": same,
                **summary(roles, cl), "oracle_s": round(t4 - t3, 1),
                "scan_in_memory_wall_s": round(t5 - t4, 2),
                "device_sim_evals": s1.sim_evals}
        print(json.dumps(line), flush=True)
    return ok_all


def cmd_rmat(a):
    t0 = time.time()
    n, e = orc.rmat(a.scale, seed=a.seed)
    return compare_all(f"R-MAT s{a.scale} ef16 seed {a.seed}", n, e, parse_cfg(a.cfg),
                       {"gen_s": round(time.time() - t0, 1)})


def device_graph(kind, a):
    """Normalised edges generated on the device (R-MAT or Chung-Lu), as host numpy."""
    import torch

    lib = _lib.load()
    if kind == "chunglu":
        n, cnt = 1 << a.logn, a.samples
    else:
        n, cnt = 1 << a.scale, 16 << a.scale
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    if kind == "chunglu":
        _lib.check(lib.gs_chunglu_generate(a.logn, a.gamma, a.wmax, cnt, a.seed, src.data_ptr(),
                                           dst.data_ptr(), None))
    else:
        _lib.check(lib.gs_rmat_generate(a.scale, 16, a.seed, src.data_ptr(), dst.data_ptr(),
                                        None))
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    mm = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(mm), None))
    m = int(mm.value)
    e = uv[: 2 * m].view(-1, 2).cpu().numpy()
    del src, dst, uv
    torch.cuda.empty_cache()
    return n, np.ascontiguousarray(e)


def cmd_chunglu(a):
    n, e = device_graph("chunglu", a)
    return compare_all(f"Chung-Lu 2^{a.logn} gamma {a.gamma} wmax {a.wmax:g} samples {a.samples} "
                       f"seed {a.seed}", n, e, parse_cfg(a.cfg))


def cmd_ooc(a):
    import torch

    lib = _lib.load()
    n, e = device_graph("rmat", a)
    m = e.shape[0]
    # reference-layout CSR on the device (uncapped input preparation), then pinned host
    uv = torch.from_numpy(e.reshape(-1)).cuda()
    off_d = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    adj_d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off_d.data_ptr(), adj_d.data_ptr(),
                                       None))
    torch.cuda.synchronize()
    off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    adj_h = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
    off_h.copy_(off_d)
    adj_h.copy_(adj_d)
    dmax = int((off_d[1:] - off_d[:-1]).max().item())
    del uv, off_d, adj_d
    torch.cuda.empty_cache()
    cm = c = None
    if a.oracle:
        c = orc.CSR(n, e)
        cm = orc.commons_marked(c)
    ok_all = True
    for eps, mu in parse_cfg(a.cfg):
        eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps), dmax)
        r_o = np.empty(n, np.uint8)
        c_o = np.empty(n, np.int32)
        st = _lib.GsStats()
        t0 = time.time()
        _lib.check(lib.gs_scan_partitioned(n, m, off_h.data_ptr(), adj_h.data_ptr(), mu,
                                           ctypes.byref(eps2), a.cap, r_o.ctypes.data,
                                           c_o.ctypes.data, ctypes.byref(st)))
        t_ooc = time.time() - t0
        eng = _lib.Engine()
        r_h = np.empty(n, np.uint8)
        c_h = np.empty(n, np.int32)
        t1 = time.time()
        _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_h.data_ptr(), adj_h.data_ptr(), 0))
        _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), r_h.ctypes.data,
                                      c_h.ctypes.data, 0, None))
        t_hbm = time.time() - t1
        eng.close()
        same = {"ooc_vs_in_hbm": bool(np.array_equal(r_o, r_h) and np.array_equal(c_o, c_h))}
        if c is not None:
            roles, cl = orc.serial_scan(c, mu, eps, commons=cm)
            same["ooc_vs_oracle"] = bool(np.array_equal(r_o, roles) and np.array_equal(c_o, cl))
        ok = all(same.values())
        ok_all &= ok
        print(json.dumps({"graph": f"R-MAT s{a.scale} ef16 seed {a.seed}", "n": n, "m": m,
                          "eps": eps, "mu": mu, "cap_bytes": a.cap, "identical": ok,
                          "checks": same, **summary(r_o, c_o),
                          "partitions": int(st.partitions),
                          "peak_device_bytes": int(st.peak_device_bytes),
                          "ooc_s": round(t_ooc, 2), "in_hbm_s": round(t_hbm, 2)}), flush=True)
    return ok_all


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("rmat")
    r.add_argument("--scale", type=int, default=24)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--cfg", default="0.2:5,0.3:5,0.4:5,0.5:5,0.6:5,0.7:5,0.8:5,0.15:3,0.25:3")
    cl = sub.add_parser("chunglu")
    cl.add_argument("--logn", type=int, default=22)
    cl.add_argument("--samples", type=int, default=80_000_000)
    cl.add_argument("--gamma", type=float, default=2.1)
    cl.add_argument("--wmax", type=float, default=6e4)
    cl.add_argument("--seed", type=int, default=1)
    cl.add_argument("--cfg", default="0.2:5,0.5:5,0.15:3,0.3:3")
    o = sub.add_parser("ooc")
    o.add_argument("--scale", type=int, default=24)
    o.add_argument("--seed", type=int, default=1)
    o.add_argument("--cap", type=int, default=2_000_000_000)
    o.add_argument("--cfg", default="0.5:5,0.2:5,0.15:3")
    o.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    ok = {"rmat": cmd_rmat, "chunglu": cmd_chunglu, "ooc": cmd_ooc}[a.cmd](a)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
