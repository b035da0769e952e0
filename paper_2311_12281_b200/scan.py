"""Host mirror of the reference clustering call (graphscan/scan.py).

``scan_in_memory(g, mu, epsilon, *, workers=1)`` keeps the reference
signature, validation and error behaviour (scan.py:965-982) and returns the
same result/stat types; the three phases run on the B200 through
libgscan.so (``gs_engine_load_csr`` + ``gs_engine_scan``).  There is no CPU
path: without the shared library the import of ``_lib`` fails.

Cluster ids are canonical: the smallest core vertex id of the
cluster, and for a border vertex eligible for several clusters the smallest
such cluster.  The reference's own ids are union-find roots; both are valid
under ``results_equivalent`` (oracle.py:220-297) and the canonical form is
additionally bit-exact against ``serial_scan``.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction
from typing import Optional, Union

import numpy as np

from . import _lib
from .graph import as_array, graph_arrays

EpsilonLike = Union[str, float, int, Fraction]

# byte codes (scan.py:38-56)
SIM_UNKNOWN, SIM_SIMILAR, SIM_DISSIMILAR = 0, 1, 2
ROLE_UNKNOWN, ROLE_CORE, ROLE_NONCORE, ROLE_MEMBER = 0, 1, 2, 3
ROLE_MEMBER_SHARED, ROLE_HUB, ROLE_OUTLIER = 4, 5, 6
PARENT_NONE, PARENT_HUB = -2, -1


class Role(Enum):
    UNKNOWN = "unknown"
    CORE = "core"
    NONCORE = "noncore"
    MEMBER = "member"
    HUB = "hub"
    OUTLIER = "outlier"


_PUBLIC_ROLE = {
    ROLE_UNKNOWN: Role.UNKNOWN,
    ROLE_CORE: Role.CORE,
    ROLE_NONCORE: Role.NONCORE,
    ROLE_MEMBER: Role.MEMBER,
    ROLE_MEMBER_SHARED: Role.MEMBER,
    ROLE_HUB: Role.HUB,
    ROLE_OUTLIER: Role.OUTLIER,
}
ROLE_LETTERS = {Role.CORE: "C", Role.MEMBER: "M", Role.HUB: "H", Role.OUTLIER: "O"}


def epsilon_fraction(epsilon: EpsilonLike) -> Fraction:
    """scan.py:137-152: validate epsilon, exact Fraction in (0, 1]."""
    if isinstance(epsilon, Fraction):
        f = epsilon
    elif isinstance(epsilon, (str, int)) and not isinstance(epsilon, bool):
        try:
            f = Fraction(epsilon)
        except (ValueError, ZeroDivisionError):
            raise ValueError(f"epsilon is not a number: {epsilon!r}") from None
    elif isinstance(epsilon, float):
        f = Fraction(epsilon)  # exact binary value
    else:
        raise TypeError(f"unsupported epsilon type: {type(epsilon).__name__}")
    if not 0 < f <= 1:
        raise ValueError(f"epsilon must be in (0, 1], got {epsilon!r}")
    return f


class ClusteringResult:
    """Per-vertex roles and cluster ids (scan.py:858-908).

    Backed by the device output arrays; ``roles`` / ``cluster_id`` are
    materialised as the reference's Python lists on first access (they stay
    mutable, as the reference's are).
    """

    def __init__(self, n: int, role_codes: np.ndarray, cluster_ids: np.ndarray,
                 orig_ids: np.ndarray):
        self.n = int(n)
        self.role_codes = role_codes
        self.cluster_ids = cluster_ids
        self._orig = orig_ids
        self._roles: Optional[list] = None
        self._cluster: Optional[list] = None
        self._orig_list: Optional[list] = None

    @property
    def roles(self) -> list:
        if self._roles is None:
            self._roles = [_PUBLIC_ROLE[int(c)] for c in self.role_codes]
        return self._roles

    @roles.setter
    def roles(self, value: list) -> None:
        self._roles = value

    @property
    def cluster_id(self) -> list:
        if self._cluster is None:
            self._cluster = self.cluster_ids.tolist()
        return self._cluster

    @cluster_id.setter
    def cluster_id(self, value: list) -> None:
        self._cluster = value

    @property
    def orig_ids(self) -> list:
        if self._orig_list is None:
            self._orig_list = np.asarray(self._orig).tolist()
        return self._orig_list

    def _codes(self) -> np.ndarray:
        if self._roles is None:
            return self.role_codes
        letters = {Role.CORE: ROLE_CORE, Role.MEMBER: ROLE_MEMBER, Role.HUB: ROLE_HUB,
                   Role.OUTLIER: ROLE_OUTLIER, Role.UNKNOWN: ROLE_UNKNOWN,
                   Role.NONCORE: ROLE_NONCORE}
        return np.array([letters[r] for r in self._roles], dtype=np.uint8)

    def _ids(self) -> np.ndarray:
        if self._cluster is None:
            return self.cluster_ids
        return np.asarray(self._cluster, dtype=np.int64)

    def _set(self, code: int) -> set[int]:
        c = self._codes()
        if code == ROLE_MEMBER:
            mask = (c == ROLE_MEMBER) | (c == ROLE_MEMBER_SHARED)
        else:
            mask = c == code
        return set(np.flatnonzero(mask).tolist())

    def core_set(self) -> set[int]:
        return self._set(ROLE_CORE)

    def member_set(self) -> set[int]:
        return self._set(ROLE_MEMBER)

    def hub_set(self) -> set[int]:
        return self._set(ROLE_HUB)

    def outlier_set(self) -> set[int]:
        return self._set(ROLE_OUTLIER)

    def core_equivalence(self) -> set[frozenset[int]]:
        codes, ids = self._codes(), self._ids()
        classes: dict[int, set[int]] = {}
        for v in np.flatnonzero(codes == ROLE_CORE).tolist():
            classes.setdefault(int(ids[v]), set()).add(v)
        return {frozenset(s) for s in classes.values()}

    def to_bytes(self) -> bytes:
        """to_text() as ASCII bytes, formatted by libgscan (gs_format_result)."""
        if self.n == 0:
            return b""
        codes = np.ascontiguousarray(self._codes(), dtype=np.uint8)
        ids = np.ascontiguousarray(self._ids(), dtype=np.int32)
        orig = np.ascontiguousarray(self._orig, dtype=np.uint32)
        cap = 25 * self.n
        buf = np.empty(cap, dtype=np.uint8)
        ln = ctypes.c_int64(0)
        lib = _lib.load()
        _lib.check(lib.gs_format_result(self.n, codes.ctypes.data, ids.ctypes.data,
                                        orig.ctypes.data, 0, buf.ctypes.data, cap,
                                        ctypes.byref(ln)))
        return buf[: ln.value].tobytes()

    def to_text(self) -> str:
        """``orig<TAB>role<TAB>orig(cluster)|-1`` per vertex (scan.py:892-904)."""
        return self.to_bytes().decode("ascii")

    def write(self, path: str) -> None:
        with open(path, "wb") as f:
            f.write(self.to_bytes())


@dataclass
class StatsReport:
    """Operation counts and phase timings (scan.py:911-947)."""

    n: int = 0
    m: int = 0
    workers: int = 1
    sim_evals: int = 0
    adj_probes: int = 0
    union_retries: int = 0
    probe_bound_violations: int = 0
    phases: dict = field(default_factory=dict)  # name -> microseconds
    extra: dict = field(default_factory=dict)

    def to_text(self) -> str:
        lines = [
            f"n={self.n}",
            f"m={self.m}",
            f"workers={self.workers}",
            f"sim_evals={self.sim_evals}",
            f"adj_probes={self.adj_probes}",
            f"union_retries={self.union_retries}",
            f"probe_bound_violations={self.probe_bound_violations}",
        ]
        lines.extend(f"phase_{name}_us={us}" for name, us in self.phases.items())
        lines.extend(f"{key}={val}" for key, val in sorted(self.extra.items()))
        return "\n".join(lines) + "\n"

    def write(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as f:
            f.write(self.to_text())


def stats_from_native(st: _lib.GsStats, n: int, m: int, workers: int) -> StatsReport:
    ph = st.phase_ms
    us = lambda i: int(round(ph[i] * 1000.0))  # noqa: E731
    rep = StatsReport(n=n, m=m, workers=workers, sim_evals=int(st.sim_evals),
                      adj_probes=int(st.adj_probes), union_retries=int(st.union_retries),
                      probe_bound_violations=int(st.probe_bound_violations))
    rep.phases = {
        "identify": us(_lib.GS_PH_IDENTIFY),
        "cleanup": us(_lib.GS_PH_CLEANUP),
        "cluster": us(_lib.GS_PH_CLUSTER),
        "classify": us(_lib.GS_PH_CLASSIFY),
        "total": us(_lib.GS_PH_TOTAL),
    }
    rep.extra = {
        "build_us": us(_lib.GS_PH_BUILD),
        "h2d_us": us(_lib.GS_PH_H2D),
        "d2h_us": us(_lib.GS_PH_D2H),
        "sim_evals_avoided": m - int(st.sim_evals),
        "sim_decided_by_bound": int(st.sim_decided_by_bound),
        "sim_intersections": int(st.sim_intersections),
        "hbm_bytes_alg": int(st.alg_bytes_sim) + 9 * int(st.sim_evals) + 8 * (n + 1),
        "clusters": int(st.n_clusters),
        "kernel_launches": int(st.kernel_launches),
        "peak_device_bytes": int(st.peak_device_bytes),
        "sim_decided_by_sketch": int(st.sim_decided_by_sketch),
    }
    if st.partitions:
        rep.extra["partitions"] = int(st.partitions)
    return rep


def _validate(mu: int, workers: int, epsilon: EpsilonLike) -> Fraction:
    if mu < 2:
        raise ValueError(f"mu must be >= 2, got {mu}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    return epsilon_fraction(epsilon)


def _dmax(off: np.ndarray) -> int:
    return int(np.diff(off).max()) if len(off) > 1 else 0


def scan_in_memory(g, mu: int, epsilon: EpsilonLike, *, workers: int = 1):
    """Run the three-phase pipeline on the device (scan.py:965-982).

    ``g`` is any reference-layout graph (this package's ``Graph`` or the
    reference's).  ``workers`` is accepted and validated for signature
    compatibility; the device schedule is data-parallel regardless and the
    canonical output does not depend on it.
    """
    f = _validate(mu, workers, epsilon)
    n, m, off, adj = graph_arrays(g)
    orig = as_array(g.orig_ids, np.uint32) if n else np.empty(0, np.uint32)
    eps2 = _lib.eps2_struct(f, lambda: _dmax(off))
    roles = np.empty(n, dtype=np.uint8)
    cids = np.empty(n, dtype=np.int32)
    st = _lib.GsStats()
    if n:
        lib = _lib.load()
        eng = _lib.thread_engine()
        _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off.ctypes.data, adj.ctypes.data, 0))
        _lib.check(lib.gs_engine_scan(eng.handle, int(mu), ctypes.byref(eps2), roles.ctypes.data,
                                      cids.ctypes.data, 0, ctypes.byref(st)))
        st.phase_ms[_lib.GS_PH_TOTAL] += st.phase_ms[_lib.GS_PH_H2D] + st.phase_ms[_lib.GS_PH_BUILD]
    stats = stats_from_native(st, n, m, workers)
    return ClusteringResult(n, roles, cids, orig), stats


def scan_edges(n: int, edges: np.ndarray, mu: int, epsilon: EpsilonLike,
               orig_ids: Optional[np.ndarray] = None):
    """build_graph + scan_in_memory in one device call from a normalised
    edge array (m, 2) int32 with u < v (gs_scan_edges)."""
    f = _validate(mu, 1, epsilon)
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
    m = int(e.shape[0])
    roles = np.empty(n, dtype=np.uint8)
    cids = np.empty(n, dtype=np.int32)
    st = _lib.GsStats()
    eps2 = _lib.eps2_struct(f)
    if n:
        lib = _lib.load()
        _lib.check(lib.gs_scan_edges(n, m, e.ctypes.data, int(mu), ctypes.byref(eps2),
                                     roles.ctypes.data, cids.ctypes.data, ctypes.byref(st)))
    orig = np.arange(n, dtype=np.uint32) if orig_ids is None else np.asarray(orig_ids, np.uint32)
    return ClusteringResult(n, roles, cids, orig), stats_from_native(st, n, m, 1)


# check_sim has its own engine per host thread (scan_in_memory loads other
# graphs into the scan engine) and remembers the graph it holds by identity:
# the cache keeps the graph object and the exact arrays it loaded alive, so
# neither an address reused after a free nor a temporary conversion can make a
# different graph look loaded.
_check_tls = threading.local()


def _check_engine(g) -> _lib.Engine:
    n, m, off, adj = graph_arrays(g)
    eng = getattr(_check_tls, "engine", None)
    if eng is None:
        eng = _check_tls.engine = _lib.Engine()
        _check_tls.held = None
    held = _check_tls.held
    # Same graph object (held alive, so its id cannot be reused) and the same
    # buffers (the held arrays keep them alive, so their addresses cannot be
    # reused either): the engine already holds this graph.
    if (held is None or held[0] is not g or held[1].ctypes.data != off.ctypes.data
            or held[2].ctypes.data != adj.ctypes.data):
        _check_tls.held = None
        _lib.check(_lib.load().gs_engine_load_csr(eng.handle, n, m, off.ctypes.data,
                                                  adj.ctypes.data, 0))
        _check_tls.held = (g, off, adj)
    return eng


def check_sim(g, u: int, v: int, epsilon: EpsilonLike) -> bool:
    """scan.py:241-258: exact similarity test of an existing edge (device).
    Out-of-range ids raise IndexError (edge_index, graph.py:268-269); u == v
    and non-adjacent pairs raise ValueError."""
    f = epsilon_fraction(epsilon)
    if not (0 <= u < g.n and 0 <= v < g.n):
        raise IndexError(f"vertex id out of range: ({u}, {v})")
    if u == v:
        raise ValueError(f"({u}, {v}) is not an edge")
    eng = _check_engine(g)
    uu = np.array([u], dtype=np.int32)
    vv = np.array([v], dtype=np.int32)
    out = np.empty(1, dtype=np.int8)
    eps2 = _lib.eps2_struct(f, g.deg_max if hasattr(g, "deg_max") else None)
    lib = _lib.load()
    _lib.check(lib.gs_engine_check_sim(eng.handle, 1, uu.ctypes.data, vv.ctypes.data,
                                       ctypes.byref(eps2), out.ctypes.data))
    if out[0] < 0:
        raise ValueError(f"({u}, {v}) is not an edge")
    return bool(out[0])


def structural_similarity(g, u: int, v: int) -> float:
    """scan.py:164-200: float sigma over closed neighbourhoods (diagnostic,
    host-side as in the reference; the engine uses the exact predicate)."""
    if not (0 <= u < g.n and 0 <= v < g.n):
        raise IndexError(f"vertex id out of range: ({u}, {v})")
    if u == v:
        return 1.0
    n, m, off, adj = graph_arrays(g)
    nu = adj[off[u]:off[u + 1]]
    nv = adj[off[v]:off[v + 1]]
    common = len(np.intersect1d(nu, nv, assume_unique=True))
    adjacent = bool(np.any(nu == v))
    inter = common + (2 if adjacent else 0)
    return inter / ((len(nu) + 1) * (len(nv) + 1)) ** 0.5


# --- phase-level API (scan.py:87-134, 390-412, 452-564, 701-852, 950-962) -----
#
# The reference exposes its three phases over a mutable ClusterState.  Here
# the state lives on the device (the engine that ran the phase); the host
# arrays of ClusterState are a snapshot exported after each phase
# (gs_engine_export_state) in the reference layout, indexed by caller ids.
# find_root / union_roots are the reference's host utilities over those
# arrays (the device clustering uses its own lock-free union-find).


class SimilarityStatus(int, Enum):
    UNKNOWN = SIM_UNKNOWN
    SIMILAR = SIM_SIMILAR
    DISSIMILAR = SIM_DISSIMILAR


@dataclass
class ClusterState:
    """Working state shared by the phases (scan.py:87-107): ``lower``/``upper``
    bound the similar-neighbourhood size (both include the vertex), ``parent``
    is the cluster forest (vertex id; -1 hub; -2 none), ``height`` the
    union-by-height rank, ``sim`` one status byte per edge of ``edge_list``."""

    n: int
    m: int
    lower: np.ndarray
    upper: np.ndarray
    role: np.ndarray
    parent: np.ndarray
    height: np.ndarray
    sim: np.ndarray
    _engine: Optional[_lib.Engine] = field(default=None, repr=False, compare=False)
    _stage: int = field(default=-1, repr=False, compare=False)  # last finished phase
    _mu: int = field(default=0, repr=False, compare=False)
    _eps: Optional[Fraction] = field(default=None, repr=False, compare=False)


def init_vertex_state(n: int, degrees, m: int, with_sim: bool) -> ClusterState:
    """scan.py:117-134: lower=1, upper=deg+1, role/sim unknown, parent=-2."""
    deg = np.asarray(degrees, dtype=np.int64).reshape(-1)
    if deg.shape[0] != n:
        raise ValueError(f"{deg.shape[0]} degrees for {n} vertices")
    return ClusterState(
        n=int(n), m=int(m),
        lower=np.ones(n, dtype=np.int32),
        upper=(deg + 1).astype(np.int32),
        role=np.zeros(n, dtype=np.uint8),
        parent=np.full(n, PARENT_NONE, dtype=np.int32),
        height=np.ones(n, dtype=np.int32),
        sim=np.zeros(m if with_sim else 0, dtype=np.uint8),
    )


def init_state(g) -> ClusterState:
    """scan.py:110-114: fresh state for graph ``g``."""
    n, m, off, _ = graph_arrays(g)
    return init_vertex_state(n, np.diff(off) if n else np.empty(0, np.int64), m, True)


def _export(g, st: ClusterState, stage: int) -> None:
    """Device state -> the host arrays of ``st`` (reference layout)."""
    n, m = st.n, st.m
    lib = _lib.load()
    lower = np.empty(n, np.int32)
    upper = np.empty(n, np.int32)
    role = np.empty(n, np.uint8)
    parent = np.empty(n, np.int32)
    sim = np.empty(m, np.uint8)
    pairs = np.empty((m, 2), np.int32)
    if n:
        _lib.check(lib.gs_engine_export_state(st._engine.handle, stage, lower.ctypes.data,
                                              upper.ctypes.data, role.ctypes.data,
                                              parent.ctypes.data, sim.ctypes.data,
                                              pairs.ctypes.data))
    st.lower, st.upper, st.role, st.parent = lower, upper, role, parent
    if m and len(st.sim) == m:
        # reference edge k = the k-th (a, b) pair in (a, b) order (graph.py:218-231)
        order = np.lexsort((pairs[:, 1], pairs[:, 0]))
        st.sim[:] = sim[order]
    st._stage = stage


def identify_core(g, mu: int, epsilon: EpsilonLike, st: ClusterState, *, workers: int = 1,
                  stats: Optional[StatsReport] = None, on_edge=None) -> None:
    """scan.py:452-492: decide Core/NonCore for every vertex on the device
    (pre-pass, bound-pruned sweep, then the cleanup sweep of unresolved roles).

    ``on_edge`` is the reference's observability hook; the device sweep has no
    per-edge host callback, so it is called once after the sweep and once
    after the cleanup, each time with ``-1`` and ``st`` holding a consistent
    snapshot (the bounds sandwich |N_eps| at every step of the sweep)."""
    f = _validate(mu, workers, epsilon)
    n, m, off, adj = graph_arrays(g)
    if st.n != n or st.m != m:
        raise ValueError("state does not belong to this graph")
    if n == 0:
        st._stage = 0
        return
    lib = _lib.load()
    if st._engine is None:
        st._engine = _lib.Engine()
    h = st._engine.handle
    _lib.check(lib.gs_engine_load_csr(h, n, m, off.ctypes.data, adj.ctypes.data, 0))
    eps2 = _lib.eps2_struct(f, lambda: _dmax(off))
    _lib.check(lib.gs_engine_phase_begin(h, int(mu), ctypes.byref(eps2)))
    _lib.check(lib.gs_engine_phase_identify(h, None))
    if on_edge is not None:
        _export(g, st, 0)
        on_edge(-1)
    ncores = ctypes.c_int64(0)
    _lib.check(lib.gs_engine_phase_resolve(h, None, ctypes.byref(ncores)))
    st._mu, st._eps = int(mu), f
    _export(g, st, 0)
    if on_edge is not None:
        on_edge(-1)
    if stats is not None:
        _phase_stats(st, stats, ("identify", "cleanup"))


def _phase_stats(st: ClusterState, stats: StatsReport, names) -> None:
    """Counters and the device phase times of the engine's scan so far."""
    tmp = _lib.GsStats()
    lib = _lib.load()
    _lib.check(lib.gs_engine_phase_stats(st._engine.handle, ctypes.byref(tmp)))
    rep = stats_from_native(tmp, st.n, st.m, stats.workers)
    stats.sim_evals = rep.sim_evals
    stats.adj_probes = rep.adj_probes
    stats.union_retries = rep.union_retries
    stats.probe_bound_violations = rep.probe_bound_violations
    for k in names:
        stats.phases[k] = rep.phases[k]


def _require_stage(st: ClusterState, stage: int, what: str) -> None:
    if st._engine is None or st._stage < stage:
        raise RuntimeError(f"{what}: run the previous phases on this state first")


def detect_clusters(g, epsilon: EpsilonLike, st: ClusterState, *, workers: int = 1,
                    stats: Optional[StatsReport] = None) -> None:
    """scan.py:701-773: cluster forest over similar core-core edges, flatten,
    canonical labels, member attachment -- on the device."""
    f = epsilon_fraction(epsilon)
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if st.n == 0:
        st._stage = 1
        return
    _require_stage(st, 0, "detect_clusters")
    if f != st._eps:
        raise ValueError("detect_clusters must use the epsilon of identify_core")
    lib = _lib.load()
    h = st._engine.handle
    _lib.check(lib.gs_engine_phase_union(h, None, None))
    _lib.check(lib.gs_engine_phase_merge(h, None, 0))
    _lib.check(lib.gs_engine_phase_attach(h, None))
    _export(g, st, 1)
    if stats is not None:
        _phase_stats(st, stats, ("cluster",))


def classify_hub_outlier(g, st: ClusterState, *, workers: int = 1,
                         stats: Optional[StatsReport] = None) -> None:
    """scan.py:832-852: every unclustered vertex becomes Hub or Outlier."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if st.n == 0:
        st._stage = 2
        return
    _require_stage(st, 1, "classify_hub_outlier")
    if st._stage >= 2:  # idempotent (scan.py:832)
        return
    lib = _lib.load()
    tmp = _lib.GsStats()
    _lib.check(lib.gs_engine_phase_finish(st._engine.handle, None, None, None, 0,
                                          ctypes.byref(tmp)))
    _export(g, st, 2)
    if stats is not None:
        _phase_stats(st, stats, ("classify",))


def resolve_roles_from_bounds(st: ClusterState, mu: int, strict: bool = False) -> bool:
    """scan.py:390-412 over the host snapshot: Core if lower >= mu, NonCore if
    upper < mu; True when some role is still open, as in the reference
    (``strict`` raises instead)."""
    open_ = st.role == ROLE_UNKNOWN
    st.role[open_ & (st.lower >= mu)] = ROLE_CORE
    st.role[open_ & (st.lower < mu) & (st.upper < mu)] = ROLE_NONCORE
    left = int(np.count_nonzero(st.role == ROLE_UNKNOWN))
    if left and strict:
        raise RuntimeError(f"{left} vertices have unresolved roles")
    return left > 0


def _chase(parent, u: int) -> int:
    r = u
    nxt = parent[r]
    while nxt != r:
        r = int(nxt)
        nxt = parent[r]
    return int(r)


def find_root(st: ClusterState, u: int) -> int:
    """scan.py:507-511: root of u's cluster tree (read-only)."""
    if st.parent[u] < 0:
        raise ValueError(f"vertex {u} is not in any cluster tree")
    return _chase(st.parent, u)


def union_roots(st: ClusterState, u: int, v: int, *, lock=None, counters=None) -> None:
    """scan.py:514-564: union by height on the host forest of ``st`` (a tie
    links v's root under u's and bumps its height); with ``lock`` the link is
    validated under the lock and a lost race retries (counted)."""
    parent, height = st.parent, st.height
    while True:
        ru, rv = _chase(parent, u), _chase(parent, v)
        if ru == rv:
            return
        if lock is None:
            _link(parent, height, ru, rv)
            return
        with lock:
            if parent[ru] == ru and parent[rv] == rv:
                _link(parent, height, ru, rv)
                return
        if counters is not None:
            counters.union_retries += 1
        u, v = ru, rv


def _link(parent, height, ru: int, rv: int) -> None:
    hu, hv = int(height[ru]), int(height[rv])
    if hu < hv:
        parent[ru] = rv
    elif hv < hu:
        parent[rv] = ru
    else:
        parent[rv] = ru
        height[ru] = hu + 1


def build_result(st: ClusterState, orig_ids) -> ClusteringResult:
    """scan.py:950-962: freeze the state; MEMBER_SHARED reads as MEMBER,
    cluster_id = parent if >= 0 else -1."""
    role = np.asarray(st.role, dtype=np.uint8)
    bad = ~np.isin(role, [ROLE_CORE, ROLE_MEMBER, ROLE_MEMBER_SHARED, ROLE_HUB, ROLE_OUTLIER])
    if st.n and bad.any():
        v = int(np.flatnonzero(bad)[0])
        raise RuntimeError(f"vertex {v} finished with unresolved role {_PUBLIC_ROLE[int(role[v])]}")
    codes = np.where(role == ROLE_MEMBER_SHARED, ROLE_MEMBER, role).astype(np.uint8)
    par = np.asarray(st.parent, dtype=np.int32)
    cids = np.where(par >= 0, par, -1).astype(np.int32)
    orig = np.asarray(orig_ids, dtype=np.uint32) if st.n else np.empty(0, np.uint32)
    return ClusteringResult(st.n, codes, cids, orig)
