"""Graph containers of the host mirror (graphscan/graph.py:37-276).

``Graph`` keeps the reference's field names and meaning (vertex_offsets,
adjacency, edge_ids, edge_list, orig_ids) as numpy arrays, so a reference
``Graph`` (``array.array`` fields) and this one are interchangeable inputs to
:func:`paper_2311_12281_b200.scan.scan_in_memory`.  ``build_graph`` runs on
the device (``gs_build_graph``); ``parse_edge_list`` is host ingest.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import BinaryIO, Optional, Union

import numpy as np

from . import _lib

MAX_VERTICES = 2**31 - 1  # graph.py:28-32
MAX_EDGES = 2**31 - 1
MAX_ORIGINAL_ID = 2**32 - 1


class ParseError(ValueError):
    """Malformed edge-list input, with the offending 1-based line number."""

    def __init__(self, message: str, line: Optional[int] = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


@dataclass
class EdgeList:
    """Normalised undirected edge list (graph.py:47-60): pairs u<v, unique,
    dense ids in [0, n_hint); ``orig_ids`` maps dense ids to input ids."""

    n_hint: int
    edges: object  # list[tuple[int,int]] or int array of shape (m, 2)
    orig_ids: Optional[object] = None

    def pairs(self) -> np.ndarray:
        """The edges as a C-contiguous int32 array of shape (m, 2)."""
        e = self.edges
        if isinstance(e, np.ndarray):
            arr = e.reshape(-1, 2)
        else:
            arr = np.asarray(list(e), dtype=np.int64).reshape(-1, 2)
        if arr.size and (arr.min() < 0 or arr.max() > MAX_VERTICES):
            raise ValueError("edge has an id outside the 4-byte vertex range")
        return np.ascontiguousarray(arr, dtype=np.int32)


def parse_edge_list(source: Union[bytes, str, BinaryIO]) -> EdgeList:
    """Text edge list -> EdgeList, the reference's rules (graph.py:63-118):
    '#' comments and blank lines skipped, self-loops dropped (vertex kept),
    duplicates merged, sparse ids remapped order-preservingly."""
    data = source.read() if hasattr(source, "read") else source
    if isinstance(data, bytes):
        try:
            text = data.decode("utf-8")
        except UnicodeDecodeError as exc:
            raise ParseError(f"input is not valid UTF-8 text: {exc}") from None
    else:
        text = data
    us: list[int] = []
    vs: list[int] = []
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 2:
            raise ParseError(f"expected two integer tokens, got {len(parts)}: {line!r}", lineno)
        try:
            u = int(parts[0])
            v = int(parts[1])
        except ValueError:
            raise ParseError(f"non-integer vertex id in {line!r}", lineno) from None
        if u < 0 or v < 0:
            raise ParseError(f"negative vertex id in {line!r}", lineno)
        if u > MAX_ORIGINAL_ID or v > MAX_ORIGINAL_ID:
            raise ParseError(f"vertex id exceeds 4-byte unsigned range in {line!r}", lineno)
        us.append(u)
        vs.append(v)
    u = np.asarray(us, dtype=np.int64)
    v = np.asarray(vs, dtype=np.int64)
    ids = np.unique(np.concatenate([u, v]))
    du = np.searchsorted(ids, u)
    dv = np.searchsorted(ids, v)
    keep = du != dv
    lo = np.minimum(du, dv)[keep]
    hi = np.maximum(du, dv)[keep]
    key = np.unique(lo * (len(ids) + 1) + hi)
    edges = np.stack([key // (len(ids) + 1), key % (len(ids) + 1)], axis=1).astype(np.int32)
    return EdgeList(n_hint=len(ids), edges=edges, orig_ids=ids.astype(np.uint32))


@dataclass
class Graph:
    """CSR-enhanced layout (graph.py:121-159), numpy-backed."""

    n: int
    m: int
    vertex_offsets: np.ndarray  # int64 [n+1]
    adjacency: np.ndarray  # int32 [2m]
    edge_ids: np.ndarray  # int32 [2m]
    edge_list: np.ndarray  # int32 [2m] flattened degree-oriented pairs
    orig_ids: np.ndarray  # uint32 [n]

    def degree(self, u: int) -> int:
        return int(self.vertex_offsets[u + 1] - self.vertex_offsets[u])

    def neighbors(self, u: int) -> list[int]:
        lo, hi = self.vertex_offsets[u], self.vertex_offsets[u + 1]
        return [int(x) for x in self.adjacency[lo:hi]]

    def endpoints(self, k: int) -> tuple[int, int]:
        return int(self.edge_list[2 * k]), int(self.edge_list[2 * k + 1])

    @property
    def deg_max(self) -> int:
        return int(np.diff(self.vertex_offsets).max()) if self.n else 0


def build_graph(el: EdgeList) -> Graph:
    """build_graph (graph.py:162-259) on the device: degree count, offsets,
    sorted runs, degree-oriented edge array and edge ids, bit-identical to the
    reference layout.  Raises ValueError for out-of-range ids, self-loops and
    duplicate edges (graph.py:181-195)."""
    pairs = el.pairs()
    m = int(pairs.shape[0])
    n = int(el.n_hint)
    if m:
        n = max(n, int(pairs.max()) + 1)
    if n > MAX_VERTICES:
        raise ValueError(f"vertex count {n} exceeds the 4-byte id range ({MAX_VERTICES})")
    if m > MAX_EDGES:
        raise ValueError(f"edge count {m} exceeds the 4-byte id range ({MAX_EDGES})")
    if el.orig_ids is not None:
        orig = np.asarray(el.orig_ids, dtype=np.uint32)
        if len(orig) != n:
            raise ValueError(f"orig_ids has {len(orig)} entries for {n} vertices")
    else:
        orig = np.arange(n, dtype=np.uint32)
    offsets = np.zeros(n + 1, dtype=np.int64)
    adjacency = np.empty(2 * m, dtype=np.int32)
    edge_ids = np.empty(2 * m, dtype=np.int32)
    edge_list = np.empty(2 * m, dtype=np.int32)
    if m:
        lib = _lib.load()
        _lib.check(
            lib.gs_build_graph(
                n, m, pairs.ctypes.data, offsets.ctypes.data, adjacency.ctypes.data,
                edge_ids.ctypes.data, edge_list.ctypes.data,
            )
        )
    return Graph(n=n, m=m, vertex_offsets=offsets, adjacency=adjacency, edge_ids=edge_ids,
                 edge_list=edge_list, orig_ids=orig)


def edge_index(g, u: int, v: int) -> Optional[int]:
    """graph.py:262-276: undirected edge id of {u, v} or None."""
    if not (0 <= u < g.n and 0 <= v < g.n):
        raise IndexError(f"vertex id out of range: ({u}, {v})")
    if u == v:
        return None
    off = as_array(g.vertex_offsets, np.int64)
    adj = as_array(g.adjacency, np.int32)
    lo, hi = int(off[u]), int(off[u + 1])
    s = lo + int(np.searchsorted(adj[lo:hi], v))
    if s < hi and adj[s] == v:
        return int(as_array(g.edge_ids, np.int32)[s])
    return None


def as_array(a, dtype) -> np.ndarray:
    """Zero-copy numpy view of a reference ``array.array`` or numpy array."""
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=dtype)
    arr = np.frombuffer(memoryview(a), dtype=dtype) if len(a) else np.empty(0, dtype=dtype)
    return arr


def graph_arrays(g) -> tuple[int, int, np.ndarray, np.ndarray]:
    """(n, m, offsets i64, adjacency i32) of any reference-layout graph."""
    n, m = int(g.n), int(g.m)
    off = as_array(g.vertex_offsets, np.int64)
    adj = as_array(g.adjacency, np.int32)
    if len(off) != n + 1 or len(adj) != 2 * m:
        raise ValueError("graph arrays do not match n and m")
    return n, m, off, adj


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data_as(ctypes.c_void_p).value or 0
