"""Sharded multi-GPU scan: one process per GPU, NCCL over
NVLink through torch.distributed for the three exchanges, the engine's
sm_100a kernels for everything else.

Every rank loads the same graph (degree-rank layout is deterministic, so
rank-space vertex ids agree across ranks) and owns the oriented edges whose
high endpoint b satisfies ``b % world == rank`` (round-robin over the
degree-sorted order, which balances the heavy tail).  Lemma-1 bounds built
from a subset of the edges are still valid bounds, so each rank prunes with
its own counts during identify; the exact global state is then rebuilt by

  1. all-reduce(SUM) of per-vertex similar / dissimilar counts  -> roles
  2. all-gather of each rank's (core, local root) pairs           -> merged
     union-find forest (identical on every rank), canonical labels
  3. all-reduce(MIN / MAX) of member labels                       -> members,
     shared members, then hub / outlier classification

With world = 1 the same phases run with no exchange and reproduce
``scan_in_memory`` exactly (tests/test_gpu_shards.py checks world 2 and 3).
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch
import torch.distributed as dist

from . import _lib


def all_gather_varlen(t: torch.Tensor, n_valid: int, group=None) -> torch.Tensor:
    """Concatenate the first ``n_valid`` rows of ``t`` from every rank (rank
    order).  Pads to the longest contribution so NCCL sees equal sizes."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([n_valid], dtype=torch.int64, device=t.device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    mx = max(sizes)
    if mx == 0:
        return t[:0]
    buf = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    buf[:n_valid] = t[:n_valid]
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:s] for o, s in zip(out, sizes)])


def exchange_row_slices(buf: torch.Tensor, bounds, group=None) -> None:
    """Part k's slice buf[bounds[k]:bounds[k+1]] is broadcast from rank k, so
    every rank ends with the whole buffer (the partitioned build's exchange)."""
    world = dist.get_world_size(group)
    for k in range(world):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        if hi > lo:
            src = dist.get_global_rank(group, k) if group is not None else k
            dist.broadcast(buf[lo:hi], src=src, group=group)


def all_ok(rc: int, device, group=None) -> bool:
    """True iff every rank's return code is GS_OK (so all ranks fail together)."""
    ok = torch.tensor([1 if rc == _lib.GS_OK else 0], dtype=torch.int32, device=device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    return int(ok.item()) == 1


def reduce_stats(st: _lib.GsStats, group=None) -> _lib.GsStats:
    """Sum the per-rank counters, max the timings (whole-job view)."""
    ints = ["sim_evals", "adj_probes", "union_retries", "probe_bound_violations",
            "sim_decided_by_bound", "sim_intersections", "alg_bytes_sim", "kernel_launches",
            "sim_decided_by_sketch"]
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([getattr(st, k) for k in ints], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    ph = torch.tensor(list(st.phase_ms), dtype=torch.float64, device=dev)
    dist.all_reduce(ph, op=dist.ReduceOp.MAX, group=group)
    for k, v in zip(ints, t.tolist()):
        setattr(st, k, int(v))
    kb = torch.tensor(list(st.kernel_bytes) + [st.wsim_bytes, st.pcie_bytes], dtype=torch.int64,
                      device=dev)
    dist.all_reduce(kb, op=dist.ReduceOp.SUM, group=group)
    kbl = kb.tolist()
    nk = len(st.kernel_bytes)
    for i in range(nk):
        st.kernel_bytes[i] = int(kbl[i])
    st.wsim_bytes, st.pcie_bytes = int(kbl[nk]), int(kbl[nk + 1])
    for i, v in enumerate(ph.tolist()):
        st.phase_ms[i] = v
    return st


class ShardedScan:
    """Run the phases of one engine as this rank's shard of a scan.

    ``load_csr`` is the partitioned build: each rank relabels and sorts 1/world
    of the rank-space rows, the row slices are broadcast from their owners
    (NCCL), and every rank finishes the same full CSR -- the build's work
    divides by world instead of being replicated."""

    def __init__(self, engine: _lib.Engine, n: int, group=None):
        self.eng = engine
        self.n = int(n)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.lib = _lib.load()
        _lib.check(self.lib.gs_engine_set_shard(engine.handle, self.rank, self.world))
        dev = torch.device("cuda", torch.cuda.current_device())
        # the engine works on its own non-blocking stream; collectives run on
        # (or are waited for by) torch's current stream
        self.estream = torch.cuda.ExternalStream(engine.stream(), device=dev)
        self.counts = torch.empty(2 * max(self.n, 1), dtype=torch.int32, device=dev)
        self.pairs = torch.empty((max(self.n, 1), 2), dtype=torch.int32, device=dev)
        self.labels = torch.empty(2 * max(self.n, 1), dtype=torch.int32, device=dev)

    def _after_collective(self) -> None:
        """Order the engine stream after the exchange just issued: every
        gs_engine_phase_* call that reads an exchanged buffer runs on the
        engine's own non-blocking stream, which is not implicitly ordered
        after torch's current stream (where NCCL's / gloo's work is waited
        for).  Device-side wait, no host synchronisation.  (The engine side
        synchronises its stream before returning a buffer to exchange.)"""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.estream.wait_event(ev)

    def load_csr(self, m: int, offsets: int, adjacency: int, on_device: int) -> None:
        """Partitioned gs_engine_load_csr (the reference CSR at the given
        pointers, host or device) with the row slices exchanged by broadcast."""
        lib, h, n, g = self.lib, self.eng.handle, self.n, self.group
        dev = torch.device("cuda", torch.cuda.current_device())
        if getattr(self, "adj", None) is None or self.adj.numel() != max(2 * m, 1):
            self.adj = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
        bounds = (ctypes.c_int64 * (self.world + 1))()
        rc = lib.gs_engine_load_csr_part(h, n, m, offsets, adjacency, on_device, self.rank,
                                         self.world, self.adj.data_ptr(), bounds)
        everyone_ok = all_ok(rc, dev, g)  # every rank fails together
        if rc != _lib.GS_OK:
            _lib.check(rc)
        if not everyone_ok:
            raise ValueError("invalid graph (detected by another rank's part)")
        exchange_row_slices(self.adj, list(bounds), g)                     # exchange 0
        if self.world > 1:
            self._after_collective()
            _lib.check(lib.gs_engine_load_finish(h))

    def run(self, mu: int, eps2: _lib.GsEps2, role_out: int, cluster_out: int,
            out_on_device: int, stats: Optional[_lib.GsStats] = None) -> _lib.GsStats:
        lib, h, n, g = self.lib, self.eng.handle, self.n, self.group
        st = stats if stats is not None else _lib.GsStats()
        _lib.check(lib.gs_engine_phase_begin(h, int(mu), ctypes.byref(eps2)))
        _lib.check(lib.gs_engine_phase_identify(h, self.counts.data_ptr()))
        dist.all_reduce(self.counts[: 2 * n], op=dist.ReduceOp.SUM, group=g)    # exchange 1
        self._after_collective()
        nc = ctypes.c_int64(0)
        _lib.check(lib.gs_engine_phase_resolve(h, self.counts.data_ptr(), ctypes.byref(nc)))
        labels_ptr = None
        if nc.value > 0:  # no core anywhere: nothing to merge or attach
            npairs = ctypes.c_int64(0)
            _lib.check(lib.gs_engine_phase_union(h, self.pairs.data_ptr(), ctypes.byref(npairs)))
            allp = all_gather_varlen(self.pairs, npairs.value, g).contiguous()  # exchange 2
            self._after_collective()
            _lib.check(lib.gs_engine_phase_merge(h, allp.data_ptr() if len(allp) else None,
                                                 len(allp)))
            _lib.check(lib.gs_engine_phase_attach(h, self.labels.data_ptr()))
            dist.all_reduce(self.labels[:n], op=dist.ReduceOp.MIN, group=g)      # exchange 3
            dist.all_reduce(self.labels[n: 2 * n], op=dist.ReduceOp.MAX, group=g)
            self._after_collective()
            labels_ptr = self.labels.data_ptr()
        else:
            _lib.check(lib.gs_engine_phase_merge(h, None, 0))
        _lib.check(lib.gs_engine_phase_finish(h, labels_ptr, role_out, cluster_out,
                                              out_on_device, ctypes.byref(st)))
        return reduce_stats(st, g)


def init_from_env() -> tuple[int, int, int]:
    """Join the process group torchrun set up (RANK / WORLD_SIZE / LOCAL_RANK),
    one GPU per rank over NCCL (GS_DIST_BACKEND=gloo: ranks may share a GPU, a
    functional check).  Returns (rank, world, local device)."""
    import os

    backend = os.environ.get("GS_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise RuntimeError("the sharded scan needs CUDA devices; none is visible")
    if backend == "nccl" and local >= ndev:
        raise RuntimeError(f"rank {local} has no GPU of its own ({ndev} visible)")
    local %= ndev
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size(), local


def scan_sharded(g, mu: int, epsilon, *, workers: int = 1, group=None):
    """scan_in_memory (scan.py:965-982) over the ranks of an initialised
    process group: every rank passes the same graph and gets the same
    (ClusteringResult, StatsReport); the edges are split b % world, the build
    by rank-space rows, and the four exchanges run over NCCL."""
    import numpy as np

    from .graph import as_array, graph_arrays
    from .scan import ClusteringResult, _validate, stats_from_native

    f = _validate(mu, workers, epsilon)
    n, m, off, adj = graph_arrays(g)
    orig = as_array(g.orig_ids, np.uint32) if n else np.empty(0, np.uint32)
    roles = np.empty(n, dtype=np.uint8)
    cids = np.empty(n, dtype=np.int32)
    st = _lib.GsStats()
    if n:
        eng = _lib.Engine(device=torch.cuda.current_device())
        try:
            shard = ShardedScan(eng, n, group)
            shard.load_csr(m, off.ctypes.data, adj.ctypes.data, 0)
            eps2 = _lib.eps2_struct(f, int(np.diff(off).max()))
            shard.run(int(mu), eps2, roles.ctypes.data, cids.ctypes.data, 0, st)
        finally:
            eng.close()
    stats = stats_from_native(st, n, m, workers)
    stats.extra["devices"] = dist.get_world_size(group)
    return ClusteringResult(n, roles, cids, orig), stats
