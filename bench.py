#!/usr/bin/env python
"""Headline benchmark: SCAN end-to-end on R-MAT scale-24 (eps=0.5, mu=5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one clustering call of the hot path, exactly what
scan_in_memory(g, mu, eps) does through the C-ABI (gs_engine_load_csr +
gs_engine_scan): the reference Graph's CSR (vertex_offsets i64, adjacency
i32) in, degree-rank relabel + identify + cluster + classify, roles and
cluster ids out -- over the synthetic R-MAT s24 graph (BASELINE.json
configs[1], the in-HBM config the metric is quoted on).  Inputs exceed L2
(2.2 GB CSR vs 126 MB), so no flush is needed between steps.

  value   edges/s = m / device time per step, CSR resident in HBM, results
          left in HBM (CUDA events on the engine stream)
  e2e     same metric through the same call with HOST buffers: pinned CSR
          streamed H2D (overlapped with the relabel) + scan + roles/cluster
          ids D2H inside the timed region
  build_from_edges_ms  the edge-list -> CSR build (build_graph's job, timed
          separately; not part of scan_in_memory)
  roofline  similarity pass (identify) algorithmic bytes W_sim
          / its measured time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference hot loop (_eval_edge, scan.py:203-233, C port in
          oracle/) on a bounded uniform edge sample, all host threads
--impl reference times that CPU port alone (rank 0), same metric and config.
"""

from __future__ import annotations

import argparse
import ctypes
import glob
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SCAN end-to-end sec & edges/sec (R-MAT s24 ε=0.5 μ=5); HBM GB/s vs peak, 1-8 GPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--eps", default="0.5")
    ap.add_argument("--mu", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--input", choices=["csr", "edges"], default=None,
                    help="csr: scan_in_memory's call on the reference CSR (default below "
                         "scale 27); edges: build from the device edge list inside the step "
                         "(default from scale 27: the CSR copy would not fit beside the engine)")
    ap.add_argument("--python-ref-seconds", type=float, default=8.0,
                    help="seconds of the reference's own Python _eval_edge (baseline/_ref) "
                         "timed on sampled edges of the same graph (0: skip)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU phase path even with one process")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this command as N
    ranks (one per GPU, NCCL) through torch.distributed.run.  Fails loudly when
    fewer GPUs are visible -- never falls back to fewer ranks."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}; "
              "refusing to run fewer ranks", file=sys.stderr)
        return 2
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator log (nranks) for the record
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def source_hash() -> str:
    """Hash of the engine's sources: a traffic record taken on other sources is stale."""
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2311_12281_b200", "csrc", "*.cu")) +
                   glob.glob(os.path.join(ROOT, "paper_2311_12281_b200", "csrc", "*.cuh")))
    for f in files + [os.path.join(ROOT, "include", "gscan.h")]:
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def workload_config(args, n: int, m: int) -> dict:
    """The `config` object, identical in both arms (the driver compares them)."""
    return {
        "workload": f"R-MAT scale-{args.scale} edgefactor {args.edgefactor}, eps={args.eps} "
                    f"mu={args.mu} (BASELINE configs[1])" if args.scale == 24 else
                    f"R-MAT scale-{args.scale} edgefactor {args.edgefactor}, eps={args.eps} "
                    f"mu={args.mu}",
        "n": n, "m": m, "seed": args.seed,
        "l2": "inputs larger than L2 (CSR 8(n+1) + 8m bytes), no flush",
        "step": "one clustering call (scan_in_memory, scan.py:965-982): degree-rank relabel "
                "+ identify + cluster + classify, roles and cluster ids out",
    }


def python_reference_rate(csr, eps, seconds: float):
    """The reference's own hot loop -- graphscan.scan._eval_edge from
    baseline/_ref, unmodified -- on uniformly sampled edges of the same graph,
    one core (the GIL), for about `seconds`.  None when baseline/_ref is absent."""
    import random
    from array import array

    import numpy as np

    ref = os.path.join(ROOT, "baseline", "_ref")
    if seconds <= 0 or not os.path.isdir(os.path.join(ref, "graphscan")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from graphscan.scan import _epsilon_squared, _eval_edge
    except ImportError:
        return None
    off_np = np.asarray(csr.vertex_offsets, dtype=np.int64)
    adj = array("i", np.asarray(csr.adjacency, dtype=np.int32).tobytes())
    p, q = _epsilon_squared(eps)
    rng = random.Random(0)
    n_edges = probes = 0
    secs = 0.0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        slot = rng.randrange(len(adj))
        v = adj[slot]
        u = int(np.searchsorted(off_np, slot, side="right") - 1)
        ou, ov = int(off_np[u]), int(off_np[v])
        du, dv = int(off_np[u + 1]) - ou, int(off_np[v + 1]) - ov
        if (dv, v) < (du, u):  # the low-(degree, id) side probes (scan.py:252-254)
            ou, du, ov, dv = ov, dv, ou, du
        t1 = time.perf_counter()
        _, pr = _eval_edge(adj, ou, ou + du, ov, ov + dv, p, q)
        secs += time.perf_counter() - t1  # the reference call alone, not the sampling
        probes += pr
        n_edges += 1
    return {"edges_per_s": n_edges / secs, "probes_per_s": probes / secs, "cores": 1,
            "sample": f"{n_edges} uniformly sampled edges in {secs:.1f}s, {probes} probes: "
                      "graphscan.scan._eval_edge (scan.py:203-233) from baseline/_ref, "
                      "unmodified, one core (GIL)",
            "ms_per_step_extrapolated": 1000.0 * csr.m * secs / max(n_edges, 1)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    One long-lived `nvidia-smi -lms 200` process (started before the timed
    region) writes CSV to a file; no fork happens while timing."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._path = os.path.join("/tmp", f"gs_clocks_{os.getpid()}_{index}.csv")

    def __enter__(self):
        try:
            self._f = open(self._path, "w")
            self._p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self._f,
                stderr=subprocess.DEVNULL)
            time.sleep(0.5)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._f.close()
            with open(self._path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 6:
                        self.samples.append(parts)
            os.unlink(self._path)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_sample(csr, eps, seconds, threads, rng_seed=0):
    """Reference hot loop on uniformly sampled edges for ~`seconds`."""
    import numpy as np

    from oracle import oracle as orc

    rng = np.random.default_rng(rng_seed)
    probe = rng.integers(0, 2 * csr.m, 2000)
    t, _, _ = orc.sample_eval_slots(csr, eps, probe, threads)
    rate = len(probe) / max(t, 1e-6)
    count = int(max(2000, min(rate * seconds, 50_000_000)))
    slots = rng.integers(0, 2 * csr.m, count)
    secs, probes, similar = orc.sample_eval_slots(csr, eps, slots, threads)
    return count, secs, probes, similar


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as orc

    threads = orc.max_threads()
    t0 = time.time()
    n, edges = orc.rmat(args.scale, seed=args.seed, edgefactor=args.edgefactor)
    csr = orc.PlainCSR(n, edges)
    prep = time.time() - t0
    m = csr.m
    per_step = min(args.cpu_seconds, max(2.0, min(20.0, 150.0 / (args.steps + args.warmup))))
    vals = []
    tot_edges = 0
    tot_secs = 0.0
    for i in range(args.warmup + args.steps):
        cnt, secs, probes, _ = cpu_sample(csr, args.eps, per_step, threads, rng_seed=i)
        if i >= args.warmup:
            vals.append(cnt / secs)
            tot_edges += cnt
            tot_secs += secs
    value = tot_edges / tot_secs
    pyref = python_reference_rate(csr, args.eps, args.python_ref_seconds)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "edges/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * m / value,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic R-MAT (Graph500 a,b,c,d=.57,.19,.19,.05, scrambled ids), generated "
                "on the host by the same counter-based generator as the device",
        "config": workload_config(args, n, m),
        "parallelism": f"{threads} host threads",
        "cpu_baseline": {
            "value": value, "unit": "edges/s", "cores": threads, "kind": "port",
            "sample": f"{tot_edges} uniformly sampled edges over {args.steps} timed steps; the "
                      f"reference's hot loop _eval_edge (scan.py:203-233, 99.5% of its runtime) "
                      f"restated in C (oracle/), all {threads} host threads; value and "
                      f"ms_per_step are EXTRAPOLATED from the sample to all m={m} edges "
                      "(the full reference call would take days at this scale)",
            "reference_python": pyref,
        },
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "prep_s": round(prep, 1),
    }
    print(json.dumps(line), flush=True)


def eng_build_ms(eng) -> float:
    """Device time of the engine's last load (gs_stats.phase_ms[BUILD] via a
    stats-only call)."""
    from paper_2311_12281_b200 import _lib

    st = _lib.GsStats()
    _lib.check(_lib.load().gs_engine_phase_stats(eng.handle, ctypes.byref(st)))
    return float(st.phase_ms[_lib.GS_PH_BUILD])


def run_ours(args):
    import numpy as np
    import torch

    import paper_2311_12281_b200 as gs
    from paper_2311_12281_b200 import _lib

    rank, world, local = dist_env()
    # GS_DIST_BACKEND=gloo runs N ranks on fewer GPUs (ranks share devices):
    # a functional check of the multi-process path on a one-GPU box, not a
    # scaling measurement (NCCL refuses two ranks on one device).
    backend = os.environ.get("GS_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    lib = _lib.load()
    f = gs.epsilon_fraction(args.eps)
    eps2 = _lib.eps2_struct(f)

    # ---- synthetic input, generated and normalised on the device (not timed)
    n = 1 << args.scale
    cnt = args.edgefactor << args.scale
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_rmat_generate(args.scale, args.edgefactor, args.seed, src.data_ptr(),
                                    dst.data_ptr(), None))
    torch.cuda.synchronize()
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    mm = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(mm), None))
    del src, dst
    m = int(mm.value)
    uv = uv[: 2 * m].clone()
    torch.cuda.empty_cache()

    eng = _lib.Engine(device=local)
    stream = torch.cuda.ExternalStream(eng.stream())
    role_d = torch.empty(n, dtype=torch.uint8, device="cuda")
    clus_d = torch.empty(n, dtype=torch.int32, device="cuda")
    st = _lib.GsStats()
    shard = None
    if world > 1 or args.sharded:
        # strong scaling: every rank owns 1/world of the edges of the same graph
        from paper_2311_12281_b200.dist import ShardedScan

        if dist is None:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
        shard = ShardedScan(eng, n)

    def scan_call(role_ptr, clus_ptr, on_dev, stats):
        if shard is None:
            _lib.check(lib.gs_engine_scan(eng.handle, args.mu, ctypes.byref(eps2), role_ptr,
                                          clus_ptr, on_dev, ctypes.byref(stats)))
        else:
            shard.run(args.mu, eps2, role_ptr, clus_ptr, on_dev, stats)

    # the reference Graph's CSR of the same graph (build_graph's output)
    if args.input == "csr":
        off_d = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        adj_d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
        _lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off_d.data_ptr(), adj_d.data_ptr(),
                                           None))
        torch.cuda.synchronize()

    def step_device():
        if args.input == "csr" and shard is not None:  # partitioned build + row exchange
            shard.load_csr(m, off_d.data_ptr(), adj_d.data_ptr(), 1)
        elif args.input == "csr":
            _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_d.data_ptr(), adj_d.data_ptr(),
                                              1))
        else:
            _lib.check(lib.gs_engine_load_edges(eng.handle, n, m, uv.data_ptr(), 1))
        scan_call(role_d.data_ptr(), clus_d.data_ptr(), 1, st)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step_device()
    sim_ms, ident_ms, launches, phase = [], [], 0, {}
    NK = len(_lib.KERNEL_CLASSES)
    cls_ms = [[] for _ in range(NK)]
    barrier()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
            ident_ms.append(st.phase_ms[_lib.GS_PH_IDENTIFY])
            for c in range(NK):
                cls_ms[c].append(st.phase_ms[_lib.GS_PH_K_PREP + c])
            launches += int(st.kernel_launches)
        e1.record(stream)
        barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    stats = gs.scan.stats_from_native(st, n, m, 1)
    value = m / (ms_step / 1000.0)  # one graph, sharded over the ranks
    for k in range(_lib.GS_PH_COUNT):
        phase[k] = round(st.phase_ms[k], 3)

    # ---- roofline: identify-pass kernel classes (algorithmic bytes counted on
    # the device, per class, over the class's own CUDA-event time)
    peak, peak_src = peaks()
    t_sim = statistics.median(ident_ms) / 1000.0
    kernels = []
    for c in range(NK):
        t = statistics.median(cls_ms[c]) / 1000.0
        b = int(st.kernel_bytes[c])
        kernels.append({"kernel": _lib.KERNEL_CLASSES[c], "ms": round(t * 1000, 3), "bytes": b,
                        "achieved_gbs": b / t / 1e9 if t > 0 else None,
                        "frac": b / t / 1e9 / peak if t > 0 else None})
    dom = max(range(NK), key=lambda c: kernels[c]["ms"])
    pass_bytes = sum(k["bytes"] for k in kernels)
    traffic, traffic_note = None, "no ncu record for these sources (tools/ncu_traffic.py)"
    tf = os.path.join(ROOT, "profiles", "sim_traffic.json")
    if os.path.exists(tf):
        with open(tf) as fh:
            td = json.load(fh)
        want = f"s{args.scale} eps={args.eps} mu={args.mu}"
        if td.get("source_hash") != source_hash() or td.get("config") != want:
            traffic_note = (f"stale: profiles/sim_traffic.json is for sources "
                            f"{td.get('source_hash')} / {td.get('config')}, not "
                            f"{source_hash()} / {want}")
        else:
            tk = td.get("classes", {}).get(str(dom))
            traffic = tk.get("dram_bytes") if tk else None
            traffic_note = (f"ncu dram__bytes_read.sum + dram__bytes_write.sum of the {dom}-th "
                            f"class's launches, {td.get('when')}, sources {td.get('source_hash')}")
            for c in range(NK):
                tc = td.get("classes", {}).get(str(c))
                if tc:
                    kernels[c]["dram_bytes_ncu"] = tc.get("dram_bytes")

    # ---- the edge-list -> CSR build, timed on its own (build_graph's job)
    eb = []
    for _ in range(3):
        _lib.check(lib.gs_engine_load_edges(eng.handle, n, m, uv.data_ptr(), 1))
        eb.append(eng_build_ms(eng))
    build_edges_ms = statistics.median(eb)

    # ---- e2e through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e and args.input == "csr":
        off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        adj_h = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
        off_h.copy_(off_d)
        adj_h.copy_(adj_d)
        role_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        clus_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
        st2 = _lib.GsStats()

        def step_host():
            if shard is not None:
                shard.load_csr(m, off_h.data_ptr(), adj_h.data_ptr(), 0)
            else:
                _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_h.data_ptr(),
                                                  adj_h.data_ptr(), 0))
            scan_call(role_h.data_ptr(), clus_h.data_ptr(), 0, st2)

        for _ in range(max(1, args.warmup)):
            step_host()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step_host()
        e1.record(stream)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        # parity of the two paths on the same input
        assert torch.equal(role_h, role_d.cpu()) and torch.equal(clus_h, clus_d.cpu())
        e2e = {"value": m / (ms_e2e / 1000.0), "unit": "edges/s",
               "ms_per_step": ms_e2e, "h2d_bytes_per_step": 8 * (n + 1) + 8 * m,
               "d2h_bytes_per_step": 5 * n,
               "input": "the reference Graph's CSR in pinned host memory (scan_in_memory's input)"}
        del off_h, adj_h

    # ---- e2e from a pinned (m, 2) edge array (SURVEY 8(d)'s definition):
    # build_graph + scan_in_memory in one call (gs_engine_load_edges from host)
    if not args.no_e2e and shard is None:
        uv_h = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
        uv_h.copy_(uv)
        role_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        clus_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
        st3 = _lib.GsStats()

        def step_edges_host():
            _lib.check(lib.gs_engine_load_edges(eng.handle, n, m, uv_h.data_ptr(), 0))
            scan_call(role_h.data_ptr(), clus_h.data_ptr(), 0, st3)

        for _ in range(max(1, args.warmup)):
            step_edges_host()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step_edges_host()
        e1.record(stream)
        barrier()
        ms_e = e0.elapsed_time(e1) / args.steps
        assert torch.equal(role_h, role_d.cpu()) and torch.equal(clus_h, clus_d.cpu())
        ee = {"value": m / (ms_e / 1000.0), "unit": "edges/s", "ms_per_step": ms_e,
              "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 5 * n,
              "input": "normalised (m, 2) int32 edge array in pinned host memory (build_graph "
                       "+ scan_in_memory)"}
        if e2e is None:
            e2e = ee
        else:
            e2e["from_edge_array"] = ee
        del uv_h

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as orc

        edges = uv.view(-1, 2).cpu().numpy()
        csr = orc.PlainCSR(n, edges)
        threads = orc.max_threads()
        count, secs, probes, _ = cpu_sample(csr, args.eps, args.cpu_seconds, threads)
        cpu = {"value": count / secs, "unit": "edges/s", "cores": threads, "kind": "port",
               "sample": f"{count} uniformly sampled edges of the same s{args.scale} graph, "
                         f"reference _eval_edge (scan.py:203-233) C port, {secs:.1f}s; "
                         f"{probes / max(count, 1):.0f} probes/edge; edges/s extrapolates the "
                         f"sample to the whole call",
               "reference_python": python_reference_rate(csr, args.eps, args.python_ref_seconds)}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "edges/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic R-MAT (Graph500 a,b,c,d=.57,.19,.19,.05, scrambled ids), "
                    "generated + normalised on the device" + (
                        "; the reference-layout CSR built once on the device "
                        "(gs_build_csr_device) before timing" if args.input == "csr" else ""),
            "config": workload_config(args, n, m),
            "parallelism": (f"edge-sharded x{world} (b % world), build partitioned by "
                            f"rank-space rows; {backend.upper()} broadcast/all-reduce/all-gather"
                            + ("" if backend == "nccl" else
                               f" (ranks sharing {torch.cuda.device_count()} GPU(s): "
                               "functional check, not a scaling number)")
                            if shard is not None else "single GPU"),
            "input": ("the reference CSR resident in HBM (gs_engine_load_csr: relabel + "
                      "per-run sort inside the step)") if args.input == "csr" else
                     "the normalised device edge list (gs_engine_load_edges: CSR build inside "
                     "the step)",
            "roofline": {"bound": "hbm", "achieved": kernels[dom]["achieved_gbs"], "peak": peak,
                         "unit": "GB/s", "frac": kernels[dom]["frac"], "traffic": traffic,
                         "kernel": kernels[dom]["kernel"],
                         "traffic_source": traffic_note,
                         "alg_bytes_per_launch": kernels[dom]["bytes"],
                         "t_ms": kernels[dom]["ms"],
                         "note": "achieved = algorithmic bytes counted on the device for this "
                                 "kernel class (every global element of graph, sketch and "
                                 "state data it reads or writes, at its size, early exits "
                                 "where they stop; DESIGN.md 5) / the class's CUDA-event time "
                                 "inside the timed steps",
                         "identify_pass": {"ms": t_sim * 1000, "bytes": pass_bytes,
                                           "achieved_gbs": pass_bytes / t_sim / 1e9,
                                           "frac": pass_bytes / t_sim / 1e9 / peak},
                         "kernels": kernels,
                         "w_sim_survey": {"bytes": int(st.wsim_bytes),
                                          "note": "SURVEY 8(d) W_sim (4 min(d) per edge the O(1) "
                                                  "bounds leave): NOT what the kernels read -- "
                                                  "the sketch bound and the early exit read ~3% "
                                                  "of it; kept for comparison with round 1"},
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "build_from_edges_ms": build_edges_ms,
            "clocks": clk.summary(),
            "phases_ms": {"h2d": phase[0], "build": phase[1], "identify": phase[2],
                          "cleanup": phase[3], "cluster": phase[4], "classify": phase[5],
                          "d2h": phase[6], "scan_total": phase[7]},
            "counts": {"sim_evals": stats.sim_evals, "sim_evals_avoided": m - stats.sim_evals,
                       "decided_by_bound": stats.extra["sim_decided_by_bound"],
                       "intersections": stats.extra["sim_intersections"],
                "decided_by_sketch": stats.extra["sim_decided_by_sketch"],
                       "adj_probes": stats.adj_probes, "cores": int(st.n_core),
                       "members": int(st.n_member), "hubs": int(st.n_hub),
                       "outliers": int(st.n_outlier), "clusters": int(st.n_clusters)},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None and dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.input is None:
        args.input = "csr" if args.scale < 27 else "edges"
    rank, world, _ = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
