"""ctypes wrapper of the CPU oracle (oracle/liborc.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- as the checker or the timed
CPU baseline, never by the product package (paper_2311_12281_b200), which has
no CPU path.  Every function restates a reference function (file:line in
gscan_oracle.h) and is pinned against outputs of the Python reference itself
(tests/golden/, produced by tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liborc.so")

_lib = None


class Counters(ctypes.Structure):
    _fields_ = [
        ("sim_evals", ctypes.c_int64),
        ("adj_probes", ctypes.c_int64),
        ("union_retries", ctypes.c_int64),
        ("probe_bound_violations", ctypes.c_int64),
    ]


class Eps2(ctypes.Structure):
    _fields_ = [("p_lo", ctypes.c_uint64), ("p_hi", ctypes.c_uint64),
                ("q_lo", ctypes.c_uint64), ("q_hi", ctypes.c_uint64)]


def build() -> str:
    """Compile liborc.so from the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    lib = ctypes.CDLL(LIB)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    lib.orc_rmat_edges.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, I64, I64, P, P]
    lib.orc_rmat_edges.restype = None
    lib.orc_normalize.argtypes = [I64, P, P]
    lib.orc_normalize.restype = I64
    lib.orc_build_graph.argtypes = [I64, I64, P, P, P, P, P, P]
    lib.orc_build_graph.restype = ctypes.c_int
    lib.orc_edge_commons.argtypes = [I64, I64, P, P, P, P]
    lib.orc_edge_commons.restype = None
    lib.orc_serial_scan.argtypes = [I64, I64, P, P, P, ctypes.c_int32, Eps2, P, P]
    lib.orc_serial_scan.restype = ctypes.c_int
    lib.orc_ref_scan.argtypes = [I64, I64, P, P, P, ctypes.c_int32, Eps2, P, P,
                                 ctypes.POINTER(Counters)]
    lib.orc_ref_scan.restype = ctypes.c_int
    lib.orc_sample_eval.argtypes = [I64, I64, P, P, P, Eps2, P, I64, ctypes.c_int,
                                    ctypes.POINTER(I64), ctypes.POINTER(I64)]
    lib.orc_sample_eval.restype = ctypes.c_double
    lib.orc_build_csr.argtypes = [I64, I64, P, P, P, P]
    lib.orc_build_csr.restype = ctypes.c_int
    lib.orc_sample_eval_slots.argtypes = [I64, P, P, Eps2, P, I64, ctypes.c_int,
                                          ctypes.POINTER(I64), ctypes.POINTER(I64)]
    lib.orc_sample_eval_slots.restype = ctypes.c_double
    lib.orc_edge_commons_marked.argtypes = [I64, I64, P, P, P, P]
    lib.orc_edge_commons_marked.restype = None
    lib.orc_serial_scan_commons.argtypes = [I64, I64, P, P, P, P, ctypes.c_int32, Eps2, P, P]
    lib.orc_serial_scan_commons.restype = ctypes.c_int
    lib.orc_max_threads.argtypes = []
    lib.orc_max_threads.restype = ctypes.c_int
    lib.orc_set_threads.argtypes = [ctypes.c_int]
    lib.orc_set_threads.restype = None
    _lib = lib
    return lib


def eps2(epsilon) -> Eps2:
    f = Fraction(epsilon) if not isinstance(epsilon, Fraction) else epsilon
    f2 = f * f
    p, q = f2.numerator, f2.denominator
    if p >= 1 << 128 or q >= 1 << 128:
        raise ValueError("epsilon^2 exceeds 128-bit numerator/denominator")
    m = (1 << 64) - 1
    return Eps2(p & m, p >> 64, q & m, q >> 64)


def rmat(scale: int, seed: int = 1, edgefactor: int = 16) -> tuple[int, np.ndarray]:
    """Normalised R-MAT edge list (n = 2^scale, pairs u<v sorted unique)."""
    lib = load()
    cnt = edgefactor << scale
    src = np.empty(cnt, dtype=np.int32)
    dst = np.empty(cnt, dtype=np.int32)
    lib.orc_rmat_edges(scale, edgefactor, seed, 0, cnt, src.ctypes.data, dst.ctypes.data)
    m = lib.orc_normalize(cnt, src.ctypes.data, dst.ctypes.data)
    edges = np.stack([src[:m], dst[:m]], axis=1).astype(np.int32)
    return 1 << scale, np.ascontiguousarray(edges)


def rmat_raw(scale: int, seed: int = 1, edgefactor: int = 16, first: int = 0, count=None):
    lib = load()
    cnt = (edgefactor << scale) if count is None else count
    src = np.empty(cnt, dtype=np.int32)
    dst = np.empty(cnt, dtype=np.int32)
    lib.orc_rmat_edges(scale, edgefactor, seed, first, cnt, src.ctypes.data, dst.ctypes.data)
    return src, dst


class CSR:
    """Reference-layout graph built by the C restatement of build_graph."""

    def __init__(self, n: int, edges: np.ndarray):
        lib = load()
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        m = e.shape[0]
        eu = np.ascontiguousarray(e[:, 0])
        ev = np.ascontiguousarray(e[:, 1])
        self.n, self.m = int(n), int(m)
        self.vertex_offsets = np.zeros(n + 1, dtype=np.int64)
        self.adjacency = np.empty(2 * m, dtype=np.int32)
        self.edge_ids = np.empty(2 * m, dtype=np.int32)
        self.edge_list = np.empty(2 * m, dtype=np.int32)
        self.orig_ids = np.arange(n, dtype=np.uint32)
        rc = lib.orc_build_graph(n, m, eu.ctypes.data, ev.ctypes.data,
                                 self.vertex_offsets.ctypes.data, self.adjacency.ctypes.data,
                                 self.edge_ids.ctypes.data, self.edge_list.ctypes.data)
        if rc != 0:
            raise ValueError("invalid edge list")

    @property
    def deg_max(self) -> int:
        return int(np.diff(self.vertex_offsets).max()) if self.n else 0

    def _p(self):
        return (self.vertex_offsets.ctypes.data, self.adjacency.ctypes.data,
                self.edge_list.ctypes.data)


def commons(g: CSR) -> np.ndarray:
    out = np.empty(g.m, dtype=np.int32)
    load().orc_edge_commons(g.n, g.m, *g._p(), out.ctypes.data)
    return out


def commons_marked(g: CSR) -> np.ndarray:
    """Same counts as commons() (oracle.py:27-44), by per-vertex marking:
    sum of min degrees instead of sum of degree pairs (large-scale checks)."""
    out = np.empty(g.m, dtype=np.int32)
    load().orc_edge_commons_marked(g.n, g.m, g.vertex_offsets.ctypes.data,
                                   g.adjacency.ctypes.data, g.edge_ids.ctypes.data,
                                   out.ctypes.data)
    return out


def serial_scan(g: CSR, mu: int, epsilon, commons: np.ndarray | None = None
                ) -> tuple[np.ndarray, np.ndarray]:
    """Canonical (roles {1,3,5,6}, cluster ids) of oracle.serial_scan.  With
    ``commons`` (per edge_list edge) the count pass is skipped."""
    roles = np.empty(g.n, dtype=np.uint8)
    cl = np.empty(g.n, dtype=np.int32)
    if commons is not None:
        cm = np.ascontiguousarray(commons, dtype=np.int32)
        assert cm.shape == (g.m,)
        rc = load().orc_serial_scan_commons(g.n, g.m, *g._p(), cm.ctypes.data, mu,
                                            eps2(epsilon), roles.ctypes.data, cl.ctypes.data)
    else:
        rc = load().orc_serial_scan(g.n, g.m, *g._p(), mu, eps2(epsilon), roles.ctypes.data,
                                    cl.ctypes.data)
    if rc != 0:
        raise ValueError("serial_scan failed")
    return roles, cl


def ref_scan(g: CSR, mu: int, epsilon):
    """scan_in_memory(workers=1) restated: raw roles, raw ids, counters."""
    roles = np.empty(g.n, dtype=np.uint8)
    cl = np.empty(g.n, dtype=np.int32)
    c = Counters()
    rc = load().orc_ref_scan(g.n, g.m, *g._p(), mu, eps2(epsilon), roles.ctypes.data,
                             cl.ctypes.data, ctypes.byref(c))
    if rc != 0:
        raise RuntimeError(f"ref_scan failed ({rc})")
    return roles, cl, {"sim_evals": c.sim_evals, "adj_probes": c.adj_probes,
                       "union_retries": c.union_retries,
                       "probe_bound_violations": c.probe_bound_violations}


def sample_eval(g: CSR, epsilon, sample: np.ndarray, threads: int = 0):
    """Time the reference hot loop (_eval_edge) over sampled edge ids."""
    lib = load()
    s = np.ascontiguousarray(sample, dtype=np.int64)
    pr = ctypes.c_int64(0)
    sm = ctypes.c_int64(0)
    secs = lib.orc_sample_eval(g.n, g.m, *g._p(), eps2(epsilon), s.ctypes.data, len(s), threads,
                               ctypes.byref(pr), ctypes.byref(sm))
    return secs, pr.value, sm.value


class PlainCSR:
    """offsets + sorted adjacency only (parallel build), for CPU baselines."""

    def __init__(self, n: int, edges: np.ndarray):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        eu = np.ascontiguousarray(e[:, 0])
        ev = np.ascontiguousarray(e[:, 1])
        self.n, self.m = int(n), int(e.shape[0])
        self.vertex_offsets = np.zeros(n + 1, dtype=np.int64)
        self.adjacency = np.empty(2 * self.m, dtype=np.int32)
        if load().orc_build_csr(n, self.m, eu.ctypes.data, ev.ctypes.data,
                                self.vertex_offsets.ctypes.data, self.adjacency.ctypes.data):
            raise ValueError("invalid edge list")


def sample_eval_slots(g, epsilon, slots: np.ndarray, threads: int = 0):
    """Time _eval_edge over edges named by uniformly sampled adjacency slots."""
    s = np.ascontiguousarray(slots, dtype=np.int64)
    pr = ctypes.c_int64(0)
    sm = ctypes.c_int64(0)
    secs = load().orc_sample_eval_slots(g.n, g.vertex_offsets.ctypes.data, g.adjacency.ctypes.data,
                                        eps2(epsilon), s.ctypes.data, len(s), threads,
                                        ctypes.byref(pr), ctypes.byref(sm))
    return secs, pr.value, sm.value


def max_threads() -> int:
    return load().orc_max_threads()


def canonical_from_raw(roles: np.ndarray, cluster: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Public role codes of a raw engine result (MEMBER_SHARED -> MEMBER)."""
    r = roles.copy()
    r[r == 4] = 3
    return r, cluster
