"""Host mirror of the reference's out-of-core API (graphscan/partition.py).

``partition_graph(g, budget_bytes)`` plans the run (``gs_plan_partitions``,
host only) and ``scan_out_of_core(meta, plan, mu, epsilon)`` executes exactly
that plan on the device (``gs_scan_partitioned_plan``: partition.py:666-757
iterates ``plan.partitions``) under an HBM cap of ``budget_bytes``.

The reference spills edge-extended subgraphs (Def. 9) to disk and re-reads
them per pass (partition.py:231-446); its greedy closure planner is O(sum d^2)
and replicates R-MAT edges 181-1,993x.  Here the graph stays in
(pinned) host memory: partitions are contiguous ranges of high endpoints whose
adjacency slice is streamed into HBM, the low endpoint's list is gathered
zero-copy, and only per-vertex state (13 bytes/vertex) is resident.  The plan
object keeps the reference's reporting surface (partitions, budget, manifest
lines) so callers and stats look the same.

Budget semantics differ from the reference on purpose: the budget is the HBM
cap and the resident state is what the device holds, 13 bytes per vertex
(degree 4 + role 1 + bounds 8, later forest 4 + labels 4), not the reference's
15 (partition.py:70, its Python ClusterState).  With 15 the s27 state alone
(2.01 GB) would not fit the 2 GB cap BASELINE configs[3] asks for.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from .graph import as_array, graph_arrays
from .scan import ClusteringResult, EpsilonLike, _validate, stats_from_native

VERTEX_STATE_BYTES = 13  # degree 4 + role 1 + bounds 8 (or forest 4 + labels 4)
EDGE_BYTES = 25  # the reference's per-edge estimate (partition.py:70-72), reporting only
VERTEX_BYTES = 4


class InfeasibleBudgetError(ValueError):
    """The resident state or the largest adjacency list cannot fit the budget
    (partition.py:79-89)."""

    def __init__(self, edge: tuple, required_bytes: int, budget_bytes: int, msg: str = ""):
        self.edge = edge
        self.required_bytes = required_bytes
        self.budget_bytes = budget_bytes
        super().__init__(msg or (f"edge {edge} needs {required_bytes} bytes against a budget of "
                                 f"{budget_bytes}; no partitioning can satisfy this"))


@dataclass
class StreamSlice:
    """One device streaming slice: high endpoints [lo, hi), adjacency [a0, a1).

    What the device executes (gs_scan_partitioned_plan).  Without spill files
    a plan's ``partitions`` are these slices, and the reference's fields map
    as: ``owned_lo``/``owned_hi`` -> the vertex range [lo, hi) whose lists
    are streamed (the reference's are edge-id ranges of its closure
    partitions); ``n_local`` -> hi - lo; ``m_local`` -> the adjacency
    elements streamed, a1 - a0; ``path`` -> None (nothing on disk)."""

    index: int
    lo: int
    hi: int
    a0: int
    a1: int

    @property
    def estimate_bytes(self) -> int:
        return 4 * (self.a1 - self.a0) + 8 * (self.hi - self.lo + 1)

    @property
    def owned_lo(self) -> int:
        return self.lo

    @property
    def owned_hi(self) -> int:
        return self.hi

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    @property
    def m_local(self) -> int:
        return self.a1 - self.a0

    @property
    def path(self) -> Optional[str]:
        return None


@dataclass
class PartitionInfo:
    """Spill-side metadata of one sealed partition (partition.py:122-132):
    owned edge ids [owned_lo, owned_hi), its closure's n_local vertices and
    m_local edges, and the GSCP file at ``path``."""

    index: int
    path: str
    n_local: int
    m_local: int
    owned_lo: int
    owned_hi: int
    estimate_bytes: int


@dataclass
class EdgeExtendedSubgraph:
    """One loaded partition (partition.py:92-119): owned edges plus their
    closure.  ``vmap[l]`` is the global id of local vertex l (ascending),
    ``emap[k]`` the global edge id of local edge k, ``owned_local`` the owned
    local edge ids sorted by global id, ``sim_local`` one byte per local edge."""

    index: int
    owned_lo: int
    owned_hi: int
    local_graph: object
    vmap: np.ndarray
    emap: np.ndarray
    sim_local: bytearray
    owned_local: list


@dataclass
class GraphMeta:
    """The globally resident slice of a graph (partition.py:143-160)."""

    n: int
    m: int
    degrees: np.ndarray
    orig_ids: np.ndarray
    graph: object = field(default=None, repr=False)

    @classmethod
    def from_graph(cls, g) -> "GraphMeta":
        n, m, off, _ = graph_arrays(g)
        orig = as_array(g.orig_ids, np.uint32) if n else np.empty(0, np.uint32)
        return cls(n=n, m=m, degrees=np.diff(off).astype(np.int64), orig_ids=orig, graph=g)


@dataclass
class PartitionPlan:
    """A budgeted run (partition.py:134-141).  ``partitions`` are the device's
    streaming slices, or -- with a spill directory -- the reference's closure
    partitions written there (GSCP files), which the device reads the graph
    back from when the plan carries no in-memory graph.  ``slices`` is the
    cut the device executes (None: derived from the budget at scan time)."""

    n: int
    m: int
    budget_bytes: int
    partitions: list
    spill_dir: Optional[str] = None
    manifest_path: Optional[str] = None
    graph: object = field(default=None, repr=False)
    slices: Optional[list] = field(default=None, repr=False)
    state_bytes_per_vertex: int = VERTEX_STATE_BYTES

    @property
    def global_state_bytes(self) -> int:
        return self.state_bytes_per_vertex * self.n

    def manifest(self) -> str:
        """The manifest text: the reference's format (partition.py:318-333)
        for spilled partitions, slice bounds otherwise."""
        lines = [f"n={self.n}", f"m={self.m}", f"budget_bytes={self.budget_bytes}",
                 f"global_state_bytes={self.global_state_bytes}",
                 f"partitions={len(self.partitions)}"]
        for p in self.partitions:
            if isinstance(p, StreamSlice):
                lines.append(f"{p.index}\t{p.lo}\t{p.hi}\t{p.a0}\t{p.a1}\t{p.estimate_bytes}")
            else:
                lines.append(f"{p.index}\t{os.path.basename(p.path)}\t{p.n_local}\t{p.m_local}"
                             f"\t{p.owned_lo}\t{p.owned_hi}\t{p.estimate_bytes}")
        return "\n".join(lines) + "\n"


def estimate_memory(s) -> int:
    """``25*|E_s| + 4*|V_s|`` (partition.py:163-171), the reference's formula,
    for a subgraph, a partition record or a graph."""
    if isinstance(s, EdgeExtendedSubgraph):
        return EDGE_BYTES * int(s.local_graph.m) + VERTEX_BYTES * int(s.local_graph.n)
    if isinstance(s, (PartitionInfo, StreamSlice)):
        return s.estimate_bytes
    return EDGE_BYTES * int(s.m) + VERTEX_BYTES * int(s.n)


def _stream_slices(n: int, off: np.ndarray, budget_bytes: int) -> list:
    """The device's cut (gs_plan_partitions): high-endpoint ranges whose
    adjacency fits the two streaming buffers the budget leaves after the
    resident state."""
    parts = []
    if not n:
        return parts
    lib = _lib.load()
    nparts = ctypes.c_int64(0)
    elems = ctypes.c_int64(0)
    try:
        _lib.check(lib.gs_plan_partitions(n, off.ctypes.data, int(budget_bytes), None, 0,
                                          ctypes.byref(nparts), ctypes.byref(elems)))
    except _lib.InfeasibleBudget as exc:
        raise InfeasibleBudgetError((-1, -1), VERTEX_STATE_BYTES * n + (2 << 20), budget_bytes,
                                    str(exc)) from None
    bounds = np.empty(nparts.value + 1, dtype=np.int64)
    _lib.check(lib.gs_plan_partitions(n, off.ctypes.data, int(budget_bytes),
                                      bounds.ctypes.data, nparts.value,
                                      ctypes.byref(nparts), ctypes.byref(elems)))
    for k in range(nparts.value):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        parts.append(StreamSlice(k, lo, hi, int(off[lo]), int(off[hi])))
    return parts


def partition_graph(g, budget_bytes: int, spill_dir: Optional[str] = None) -> PartitionPlan:
    """Plan a budgeted run (partition.py:231-333).  Raises InfeasibleBudgetError
    like the reference.

    Without ``spill_dir``: validate the budget and cut the high-endpoint range
    into streaming slices (the graph stays in pinned host memory; 13 bytes of
    resident state per vertex).  With ``spill_dir``: the reference's plan
    exactly -- its greedy closure planner with its 15 bytes per vertex
    (native, gs_plan_closure), each partition sealed into a GSCP file and the
    manifest written, byte for byte what the reference writes (the local
    graphs are built on the device)."""
    if budget_bytes <= 0:
        raise ValueError(f"budget_bytes must be positive, got {budget_bytes}")
    n, m, off, _ = graph_arrays(g)
    if spill_dir is None:
        state = VERTEX_STATE_BYTES * n
        if state > budget_bytes:
            raise InfeasibleBudgetError((-1, -1), state, budget_bytes)
        parts = _stream_slices(n, off, budget_bytes)
        return PartitionPlan(n=n, m=m, budget_bytes=int(budget_bytes), partitions=parts,
                             graph=g, slices=parts)
    state = REF_VERTEX_STATE_BYTES * n
    if state > budget_bytes:
        raise InfeasibleBudgetError((-1, -1), state, budget_bytes)
    os.makedirs(spill_dir, exist_ok=True)
    records = _plan_closure(g, int(budget_bytes), state)
    parts = [_seal_partition(g, k, lo, hi, nl, ml, int(budget_bytes), spill_dir)
             for k, (lo, hi, nl, ml) in enumerate(records)]
    plan = PartitionPlan(n=n, m=m, budget_bytes=int(budget_bytes), partitions=parts,
                         spill_dir=spill_dir,
                         manifest_path=os.path.join(spill_dir, "plan.manifest"), graph=g,
                         state_bytes_per_vertex=REF_VERTEX_STATE_BYTES)
    _write_manifest(plan)
    return plan


# --- the reference's spill format (GSCP, partition.py:336-446) ---------------

REF_VERTEX_STATE_BYTES = 15  # partition.py:70, the reference's resident state per vertex
_SPILL_MAGIC = b"GSCP"
_SPILL_VERSION = 1
# magic, version, index, nL, mL, budget, owned_lo, owned_hi (partition.py:76)
_SPILL_HEADER = struct.Struct("<4sII5Q")
# sections of a GSCP file after the header (partition.py:362-375): name, dtype,
# and the element count as (per vertex, constant, per edge)
_SPILL_SECTIONS = (("vmap", "<u4", 1, 0, 0), ("emap", "<i4", 0, 0, 1),
                   ("vertex_offsets", "<i8", 1, 1, 0), ("adjacency", "<i4", 0, 0, 2),
                   ("edge_ids", "<i4", 0, 0, 2), ("edge_list", "<i4", 0, 0, 2),
                   ("orig_ids", "<u4", 1, 0, 0))


def _plan_closure(g, budget_bytes: int, state_bytes: int) -> list:
    """The reference's greedy closure planner (partition.py:245-312) in native
    code: [(owned_lo, owned_hi, n_local, m_local)] per partition."""
    n, m, off, adj = graph_arrays(g)
    if not m:
        return []
    eids = as_array(g.edge_ids, np.int32)
    el = as_array(g.edge_list, np.int32)
    lib = _lib.load()
    cap = 1024
    while True:
        bounds = np.empty(cap + 1, dtype=np.int64)
        nl = np.empty(cap, dtype=np.int64)
        ml = np.empty(cap, dtype=np.int64)
        nparts = ctypes.c_int64(0)
        bad = np.zeros(3, dtype=np.int64)
        rc = lib.gs_plan_closure(n, m, off.ctypes.data, adj.ctypes.data, eids.ctypes.data,
                                 el.ctypes.data, budget_bytes, state_bytes, bounds.ctypes.data,
                                 nl.ctypes.data, ml.ctypes.data, cap, ctypes.byref(nparts),
                                 bad.ctypes.data)
        if rc == _lib.GS_EBUDGET:
            raise InfeasibleBudgetError((int(bad[0]), int(bad[1])), int(bad[2]), budget_bytes)
        _lib.check(rc)
        if nparts.value <= cap:
            k = nparts.value
            return [(int(bounds[i]), int(bounds[i + 1]), int(nl[i]), int(ml[i]))
                    for i in range(k)]
        cap = nparts.value


def _run_positions(off: np.ndarray, verts: np.ndarray) -> np.ndarray:
    """Adjacency positions of every run of ``verts`` (concatenated)."""
    lo = off[verts]
    lens = off[verts + 1] - lo
    total = int(lens.sum())
    starts = np.repeat(lo - np.concatenate(([0], np.cumsum(lens)[:-1])), lens)
    return starts + np.arange(total, dtype=np.int64)


def _seal_partition(g, index: int, owned_lo: int, owned_hi: int, n_local: int, m_local: int,
                    budget_bytes: int, spill_dir: str) -> PartitionInfo:
    """partition.py:177-216: the closure of the owned edges as a local graph
    (vertices in ascending global order, built by build_graph -- on the
    device), its edge map, the owned local edges, and the GSCP file."""
    from .graph import EdgeList, build_graph

    n, m, off, adj = graph_arrays(g)
    el = as_array(g.edge_list, np.int32).reshape(-1, 2)
    eids = as_array(g.edge_ids, np.int32)
    ends = np.unique(el[owned_lo:owned_hi].ravel()).astype(np.int64)
    pos = _run_positions(off, ends)
    vmap = np.unique(np.concatenate((ends, adj[pos].astype(np.int64)))).astype(np.uint32)
    edges = np.unique(eids[pos]).astype(np.int64)
    if len(vmap) != n_local or len(edges) != m_local:
        raise RuntimeError(f"partition {index}: closure has {len(vmap)} vertices / "
                           f"{len(edges)} edges, the planner counted {n_local} / {m_local}")
    ge = el[edges]
    lu = np.searchsorted(vmap, ge[:, 0].astype(np.uint32)).astype(np.int64)
    lv = np.searchsorted(vmap, ge[:, 1].astype(np.uint32)).astype(np.int64)
    a, b = np.minimum(lu, lv), np.maximum(lu, lv)
    pairs = np.stack((a, b), axis=1).astype(np.int32)
    lg = build_graph(EdgeList(n_hint=len(vmap), edges=pairs, orig_ids=vmap))
    keys = a * len(vmap) + b
    order = np.argsort(keys)
    lel = lg.edge_list.reshape(-1, 2).astype(np.int64)
    lk = np.minimum(lel[:, 0], lel[:, 1]) * len(vmap) + np.maximum(lel[:, 0], lel[:, 1])
    emap = edges[order[np.searchsorted(keys[order], lk)]].astype(np.int32)
    sub = EdgeExtendedSubgraph(index=index, owned_lo=owned_lo, owned_hi=owned_hi, local_graph=lg,
                               vmap=vmap, emap=emap, sim_local=bytearray(lg.m),
                               owned_local=_owned_local(emap, owned_lo, owned_hi))
    path = os.path.join(spill_dir, f"part-{index:05d}.bin")
    _write_spill(path, sub, budget_bytes)
    return PartitionInfo(index=index, path=path, n_local=lg.n, m_local=lg.m, owned_lo=owned_lo,
                         owned_hi=owned_hi, estimate_bytes=estimate_memory(sub))


def _owned_local(emap: np.ndarray, owned_lo: int, owned_hi: int) -> list:
    """partition.py:219-222: owned local edge ids sorted by global id."""
    emap = np.asarray(emap, dtype=np.int64)
    ks = np.nonzero((emap >= owned_lo) & (emap < owned_hi))[0]
    return [int(k) for k in ks[np.argsort(emap[ks], kind="stable")]]


def _write_manifest(plan: PartitionPlan) -> None:
    """partition.py:318-333."""
    with open(plan.manifest_path, "w", encoding="utf-8") as f:
        f.write(plan.manifest())


def _write_spill(path: str, sub: EdgeExtendedSubgraph, budget_bytes: int) -> None:
    """partition.py:356-375: header, the seven arrays little-endian, sim bytes."""
    lg = sub.local_graph
    arrays = {"vmap": sub.vmap, "emap": sub.emap, "vertex_offsets": lg.vertex_offsets,
              "adjacency": lg.adjacency, "edge_ids": lg.edge_ids, "edge_list": lg.edge_list,
              "orig_ids": lg.orig_ids}
    with open(path, "wb") as f:
        f.write(_SPILL_HEADER.pack(_SPILL_MAGIC, _SPILL_VERSION, sub.index, lg.n, lg.m,
                                   budget_bytes, sub.owned_lo, sub.owned_hi))
        for name, dt, _, _, _ in _SPILL_SECTIONS:
            f.write(np.ascontiguousarray(arrays[name]).astype(dt, copy=False).tobytes())
        f.write(bytes(sub.sim_local))


def load_partition(info) -> EdgeExtendedSubgraph:
    """partition.py:378-433: materialise a spilled partition, with the
    reference's checks and messages (ValueError for a bad or mismatched file,
    OSError naming the partition for I/O failures)."""
    from .graph import Graph

    try:
        with open(info.path, "rb") as f:
            header = f.read(_SPILL_HEADER.size)
            if len(header) != _SPILL_HEADER.size:
                raise ValueError("truncated partition header")
            magic, version, index, n, m, _budget, owned_lo, owned_hi = (
                _SPILL_HEADER.unpack(header))
            if magic != _SPILL_MAGIC:
                raise ValueError("not a partition spill file")
            if version != _SPILL_VERSION:
                raise ValueError(f"unsupported partition format version {version}")
            if index != info.index or n != info.n_local or m != info.m_local:
                raise ValueError(
                    f"partition file {info.path} does not match plan entry {info.index}")
            arrs = {}
            for name, dt, per_v, const, per_e in _SPILL_SECTIONS:
                size = (per_v * n + const + per_e * m) * np.dtype(dt).itemsize
                data = f.read(size)
                if len(data) != size:
                    raise ValueError("truncated partition file")
                arrs[name] = np.frombuffer(data, dtype=dt)
            sim_local = bytearray(f.read(m))
            if len(sim_local) != m:
                raise ValueError("truncated similarity section")
    except OSError as exc:
        raise OSError(f"partition {info.index}: cannot load {info.path}: {exc}") from exc
    lg = Graph(n=n, m=m, vertex_offsets=arrs["vertex_offsets"].astype(np.int64),
               adjacency=arrs["adjacency"].astype(np.int32),
               edge_ids=arrs["edge_ids"].astype(np.int32),
               edge_list=arrs["edge_list"].astype(np.int32),
               orig_ids=arrs["orig_ids"].astype(np.uint32))
    return EdgeExtendedSubgraph(index=index, owned_lo=owned_lo, owned_hi=owned_hi, local_graph=lg,
                                vmap=arrs["vmap"].astype(np.uint32),
                                emap=arrs["emap"].astype(np.int32), sim_local=sim_local,
                                owned_local=_owned_local(arrs["emap"], owned_lo, owned_hi))


def store_sim(info, sub: EdgeExtendedSubgraph) -> None:
    """partition.py:436-446: persist the partition's similarity bytes in place."""
    try:
        with open(info.path, "r+b") as f:
            f.seek(-sub.local_graph.m, os.SEEK_END)
            f.write(bytes(sub.sim_local))
    except OSError as exc:
        raise OSError(f"partition {info.index}: cannot store {info.path}: {exc}") from exc


def _graph_from_spill(meta, plan):
    """The global graph read back from a plan's spill files: every partition's
    owned edges (their global ids and endpoints via emap / vmap), rebuilt by
    build_graph on the device.  This is how a plan without an in-memory graph
    -- e.g. one the reference's own partition_graph wrote -- is executed."""
    from .graph import EdgeList, build_graph

    n, m = int(meta.n), int(meta.m)
    pairs = np.full((m, 2), -1, dtype=np.int64)
    for info in plan.partitions:
        sub = load_partition(info)
        own = np.asarray(sub.owned_local, dtype=np.int64)
        lel = sub.local_graph.edge_list.reshape(-1, 2)[own].astype(np.int64)
        ends = sub.vmap.astype(np.int64)[lel]
        pairs[sub.emap[own].astype(np.int64)] = np.sort(ends, axis=1)
    if m and pairs.min() < 0:
        raise ValueError("the plan's spill files do not cover every edge of the graph")
    orig = np.asarray(meta.orig_ids, dtype=np.uint32) if n else None
    g = build_graph(EdgeList(n_hint=n, edges=pairs.astype(np.int32), orig_ids=orig))
    got = np.sort(g.edge_list.reshape(-1, 2).astype(np.int64), axis=1)
    if g.n != n or g.m != m or not np.array_equal(got, pairs):
        raise ValueError("the plan's spill files do not describe the plan's graph")
    return g


def scan_out_of_core(meta: GraphMeta, plan: PartitionPlan, mu: int, epsilon: EpsilonLike, *,
                     workers: int = 1):
    """Cluster under the plan's HBM budget (partition.py:666-757).  Same
    results as ``scan_in_memory`` (canonical ids), same error behaviour.

    The device executes the plan's streaming slices as given; a spill plan
    (this package's or the reference's own PartitionPlan) is executed from its
    files when it carries no in-memory graph, under a device cut of the same
    budget.  The spill files' similarity sections are not rewritten: the
    streamed device scan keeps no per-edge state (they stay SIM_UNKNOWN)."""
    f = _validate(mu, workers, epsilon)
    if plan.n != meta.n or plan.m != meta.m:
        raise ValueError(f"plan is for a different graph: plan n={plan.n} m={plan.m}, "
                         f"graph n={meta.n} m={meta.m}")
    g = getattr(plan, "graph", None)
    if g is None:
        g = getattr(meta, "graph", None)
    if g is None:
        g = _graph_from_spill(meta, plan)
    n, m, off, adj = graph_arrays(g)
    parts = list(plan.partitions)
    slices = getattr(plan, "slices", None)
    if slices is None:
        if parts and all(isinstance(p, StreamSlice) for p in parts):
            slices = parts
        else:
            slices = _stream_slices(n, off, plan.budget_bytes)
    degrees = np.asarray(meta.degrees)
    eps2 = _lib.eps2_struct(f, int(degrees.max()) if n else 0)
    roles = np.empty(n, dtype=np.uint8)
    cids = np.empty(n, dtype=np.int32)
    st = _lib.GsStats()
    if n:
        lib = _lib.load()
        # the slices are executed as given (validated on the device side: a
        # slice that does not fit the cap raises InfeasibleBudgetError)
        bounds = np.array([p.lo for p in slices] + [n], dtype=np.int64)
        if len(slices) == 0 or bounds[0] != 0:
            raise ValueError("plan has no partitions covering the graph")
        try:
            _lib.check(lib.gs_scan_partitioned_plan(n, m, off.ctypes.data, adj.ctypes.data,
                                                    int(mu), ctypes.byref(eps2),
                                                    int(plan.budget_bytes), len(slices),
                                                    bounds.ctypes.data, roles.ctypes.data,
                                                    cids.ctypes.data, ctypes.byref(st)))
        except _lib.InfeasibleBudget as exc:
            raise InfeasibleBudgetError((-1, -1), VERTEX_STATE_BYTES * n, plan.budget_bytes,
                                        str(exc)) from None
    stats = stats_from_native(st, n, m, workers)
    stats.extra["partitions"] = len(parts) if n else 0
    stats.extra["stream_slices"] = int(st.partitions) if n else 0
    stats.extra["pcie_bytes"] = int(st.pcie_bytes) if n else 0
    orig = np.asarray(meta.orig_ids, dtype=np.uint32) if n else np.empty(0, np.uint32)
    return ClusteringResult(n, roles, cids, orig), stats
