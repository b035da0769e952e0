"""Graph containers of the host mirror (graphscan/graph.py:37-276).

``Graph`` keeps the reference's field names and meaning (vertex_offsets,
adjacency, edge_ids, edge_list, orig_ids) as numpy arrays, so a reference
``Graph`` (``array.array`` fields) and this one are interchangeable inputs to
:func:`paper_2311_12281_b200.scan.scan_in_memory`.  ``build_graph`` runs on
the device (``gs_build_graph``); ``parse_edge_list`` is host ingest.
"""

from __future__ import annotations

import ctypes
import struct
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
    duplicates merged, sparse ids remapped order-preservingly.

    Native ingest: libgscan's multi-threaded parser (gs_parse_edge_text) reads
    the text, the device remaps and deduplicates (gs_normalize_sparse; no
    host path).  Input outside the parser's ASCII
    grammar -- malformed lines included -- goes through the reference-exact
    Python parser below, so errors (ParseError with the line number) and
    exotic-but-valid inputs behave exactly as in the reference."""
    data = source.read() if hasattr(source, "read") else source
    if isinstance(data, str):
        data = data.encode("utf-8")
    raw = _parse_native(bytes(data))
    if raw is None:
        return _parse_exact(data)
    return _normalize(*raw)


def _parse_native(data: bytes):
    lib = _lib.load()
    cap = data.count(b"\n") + data.count(b"\r") + 1
    u = np.empty(cap, dtype=np.uint32)
    v = np.empty(cap, dtype=np.uint32)
    cnt = ctypes.c_int64(0)
    err = ctypes.c_int64(-1)
    rc = lib.gs_parse_edge_text(data, len(data), 0, u.ctypes.data, v.ctypes.data, cap,
                                ctypes.byref(cnt), ctypes.byref(err))
    if rc == _lib.GS_EPARSE:
        return None
    _lib.check(rc)
    return u[: cnt.value], v[: cnt.value]


def _normalize(u: np.ndarray, v: np.ndarray) -> EdgeList:
    """Remap sparse ids order-preservingly, drop self-loops, merge duplicates
    (graph.py:98-118) on the device (gs_normalize_sparse).  There is no host
    path: without a CUDA device this raises."""
    u = np.ascontiguousarray(u, dtype=np.uint32)
    v = np.ascontiguousarray(v, dtype=np.uint32)
    count = int(len(u))
    if count == 0:
        return EdgeList(n_hint=0, edges=np.empty((0, 2), dtype=np.int32),
                        orig_ids=np.empty(0, dtype=np.uint32))
    lib = _lib.load()
    if lib.gs_device_count() <= 0:
        raise RuntimeError("parse_edge_list: normalising the edge list needs a CUDA device "
                           "(libgscan has no CPU path)")
    ids = np.empty(2 * count, dtype=np.uint32)
    edges = np.empty((count, 2), dtype=np.int32)
    n = ctypes.c_int64(0)
    m = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_sparse(count, u.ctypes.data, v.ctypes.data, ids.ctypes.data,
                                       ctypes.byref(n), edges.ctypes.data, ctypes.byref(m)))
    return EdgeList(n_hint=n.value, edges=edges[: m.value].copy(),
                    orig_ids=ids[: n.value].copy())


def _parse_exact(data: bytes) -> EdgeList:
    """graph.py:63-118 rule for rule (str.splitlines / strip / split / int)."""
    try:
        text = data.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise ParseError(f"input is not valid UTF-8 text: {exc}") from None
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
    return _normalize(np.asarray(us, dtype=np.uint32), np.asarray(vs, dtype=np.uint32))


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


# --- binary graph cache (graph.py:279-350): the GSCG format, byte-compatible -
#
#   magic "GSCG" | version u32 | n u64 | m u64      (little-endian)
#   vertex_offsets (n+1) x i64 | adjacency 2m x i32 | edge_ids 2m x i32
#   edge_list 2m x i32 | orig_ids n x u32
#
# Arrays are read with one bulk read each (np.fromfile), so a cached s24 graph
# (6.5 GB) loads at disk speed instead of through per-element Python code.

_GRAPH_MAGIC = b"GSCG"
_GRAPH_VERSION = 1
_HEADER = struct.Struct("<4sIQQ")
_LAYOUT = (("vertex_offsets", "<i8", 1, 0), ("adjacency", "<i4", 0, 2),
           ("edge_ids", "<i4", 0, 2), ("edge_list", "<i4", 0, 2), ("orig_ids", "<u4", 0, 0))


def _count(n: int, m: int, plus_one: int, per_edge: int) -> int:
    return (n + plus_one) if per_edge == 0 else per_edge * m


def save_graph(g, path: str) -> None:
    """graph.py:313-321: write the five layout arrays to a GSCG cache."""
    n, m = int(g.n), int(g.m)
    with open(path, "wb") as f:
        f.write(_HEADER.pack(_GRAPH_MAGIC, _GRAPH_VERSION, n, m))
        for name, dt, plus, per in _LAYOUT:
            a = np.ascontiguousarray(as_array(getattr(g, name), np.dtype(dt).newbyteorder("=")),
                                     dtype=dt)
            want = _count(n, m, plus, per)
            if len(a) != want:
                raise ValueError(f"{name} has {len(a)} entries, expected {want}")
            a.tofile(f)


def load_graph(path: str) -> Graph:
    """graph.py:324-350: read a GSCG cache written by save_graph (or by the
    reference); the same validation and error messages."""
    with open(path, "rb") as f:
        header = f.read(_HEADER.size)
        if len(header) != _HEADER.size:
            raise ValueError("truncated graph cache header")
        magic, version, n, m = _HEADER.unpack(header)
        if magic != _GRAPH_MAGIC:
            raise ValueError("not a graph cache file (bad magic)")
        if version != _GRAPH_VERSION:
            raise ValueError(f"unsupported graph cache version {version}")
        arrs = {}
        for name, dt, plus, per in _LAYOUT:
            cnt = (n + plus) if per == 0 else per * m
            a = np.fromfile(f, dtype=dt, count=cnt)
            if len(a) != cnt:
                raise ValueError("truncated graph cache")
            arrs[name] = a.astype(np.dtype(dt).newbyteorder("="), copy=False)
    off = arrs["vertex_offsets"]
    if off[0] != 0 or off[n] != 2 * m:
        raise ValueError("corrupt graph cache: bad offset bounds")
    if n and np.any(np.diff(off) < 0):
        raise ValueError("corrupt graph cache: offsets not monotone")
    return Graph(n=int(n), m=int(m), **arrs)


def is_graph_cache(path: str) -> bool:
    """graph.py:353-359: True if ``path`` starts with the GSCG magic."""
    try:
        with open(path, "rb") as f:
            return f.read(4) == _GRAPH_MAGIC
    except OSError:
        return False
