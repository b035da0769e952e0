"""The engine's CSR relabel-build (csrc/build.cu) on inputs that reach every
branch: host CSR streamed in many chunks (ring reuse, run-order checks across
chunk boundaries), every per-run sort class (2-32 warp registers, 33-256 warp
shared memory, 257-4095 the four CTA radix classes, >= 4096 the hub-run radix
sort) and the CTA scatter of hub runs.  Checked bit-exactly against the CPU
oracle and across the three input paths (host CSR, device CSR, edge list)."""

import os

import numpy as np
import pytest

from conftest import cuda_ok, make_graph

pytestmark = pytest.mark.gpu

if not cuda_ok():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2311_12281_b200 as gs  # noqa: E402


def _degree_class_graph(seed=3):
    """Vertices of chosen degrees in every sort class, over a sparse background."""
    rng = np.random.default_rng(seed)
    n = 30000
    edges = set()
    for _ in range(60000):
        u, v = rng.integers(0, n, size=2)
        if u != v:
            edges.add((int(min(u, v)), int(max(u, v))))
    centres = {}
    for k, d in enumerate((3, 20, 40, 200, 300, 700, 1500, 3000, 5000, 9000)):
        c = 100 + k
        for v in rng.choice(np.arange(200, n), size=d, replace=False):
            edges.add((c, int(v)))
        centres[c] = d
    # a dense block so some of them become cores at low eps
    block = np.arange(200, 260)
    for i in block:
        for j in block:
            if i < j:
                edges.add((int(i), int(j)))
    return n, np.array(sorted(edges), dtype=np.int32)


def _run(g, mu, eps):
    r, s = gs.scan_in_memory(g, mu, eps)
    return r.role_codes.copy(), r.cluster_ids.copy()


@pytest.fixture
def chunk_env():
    old = os.environ.get("GS_H2D_CHUNK")
    yield
    if old is None:
        os.environ.pop("GS_H2D_CHUNK", None)
    else:
        os.environ["GS_H2D_CHUNK"] = old


def test_every_sort_class_against_oracle(orc):
    n, e = _degree_class_graph()
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.1", 3), ("0.3", 2), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl = _run(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"{eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"{eps} {mu}")
        r, _ = gs.scan_edges(n, e, mu, eps)  # edge-list build path
        np.testing.assert_array_equal(r.role_codes, roles)
        np.testing.assert_array_equal(r.cluster_ids, cl)


@pytest.mark.parametrize("chunk,scale", [(64, 11), (1000, 14), (4093, 15), (1 << 16, 15)])
def test_host_csr_many_chunks(orc, chunk_env, chunk, scale):
    n, e = orc.rmat(scale, seed=4)
    g = make_graph(n, e)
    ref = _run(g, 3, "0.3")
    os.environ["GS_H2D_CHUNK"] = str(chunk)
    got = _run(g, 3, "0.3")
    np.testing.assert_array_equal(got[0], ref[0])
    np.testing.assert_array_equal(got[1], ref[1])
    roles, cl = orc.serial_scan(orc.CSR(n, e), 3, "0.3")
    np.testing.assert_array_equal(got[0], roles)
    np.testing.assert_array_equal(got[1], cl)


def _hub_graph(seed=5):
    """Hub runs on both sides of 16384 (the chunk pipeline's CTA sort and its
    segmented sort), spread over many chunks, on a sparse background."""
    rng = np.random.default_rng(seed)
    n = 60000
    edges = set()
    for _ in range(80000):
        u, v = rng.integers(0, n, size=2)
        if u != v:
            edges.add((int(min(u, v)), int(max(u, v))))
    for k, d in enumerate((4096, 6000, 16384, 16385, 21000, 40000)):
        c = 1000 * (k + 1) + 7
        for v in rng.choice(np.arange(0, n), size=d, replace=False):
            if v != c:
                edges.add((int(min(c, v)), int(max(c, v))))
    return n, np.array(sorted(edges), dtype=np.int32)


@pytest.mark.parametrize("hub_chunk", ["1", "0"])
@pytest.mark.parametrize("chunk", [4093, 1 << 15])
def test_host_csr_hub_runs_sorted_chunk_by_chunk(orc, chunk_env, monkeypatch, chunk, hub_chunk):
    """Runs >= 4096 sorted as their last chunk lands (GS_HUB_CHUNK=1, default)
    or at the end (0): the same graph and clustering as the oracle."""
    n, e = _hub_graph()
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    monkeypatch.setenv("GS_HUB_CHUNK", hub_chunk)
    os.environ["GS_H2D_CHUNK"] = str(chunk)
    for eps, mu in (("0.2", 3), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        got = _run(g, mu, eps)
        np.testing.assert_array_equal(got[0], roles, err_msg=f"{eps} {mu}")
        np.testing.assert_array_equal(got[1], cl, err_msg=f"{eps} {mu}")


@pytest.mark.parametrize("chunk", [4093, 1 << 15])
def test_host_csr_streamed_sketch_rows_equal_the_scan_built_ones(orc, chunk_env, monkeypatch,
                                                                  chunk):
    """Sketch rows built chunk by chunk while the CSR streams in (GS_SK_STREAM=1)
    or by the scan (0): the clustering equals the oracle's either way, and the
    sketch decides a similar number of edges (the counters are not exactly
    reproducible: pruning order varies run to run)."""
    n, e = _hub_graph()
    g = make_graph(n, e)
    os.environ["GS_H2D_CHUNK"] = str(chunk)
    for eps, mu in (("0.5", 5), ("0.35", 3), ("0.2", 3)):  # 0.2: k = 8, rebuilt by the scan
        out = {}
        for flag in ("1", "0"):
            monkeypatch.setenv("GS_SK_STREAM", flag)
            r, st = gs.scan_in_memory(g, mu, eps)
            out[flag] = (r.role_codes.copy(), r.cluster_ids.copy(),
                         st.extra["sim_decided_by_sketch"], st.sim_evals)
        a, b = out["1"][2], out["0"][2]
        assert abs(a - b) <= 0.02 * max(a, b) + 50, (eps, a, b)
        roles, cl = orc.serial_scan(orc.CSR(n, e), mu, eps)
        for flag in ("1", "0"):
            np.testing.assert_array_equal(out[flag][0], roles)
            np.testing.assert_array_equal(out[flag][1], cl)


@pytest.mark.parametrize("victim", [2007, 4007, 6007])  # degrees 6000, 16385, 40000
def test_host_csr_bad_hub_run_detected(chunk_env, victim):
    n, e = _hub_graph()
    g = make_graph(n, e)
    off = np.asarray(g.vertex_offsets).copy()
    lo, hi = int(off[victim]), int(off[victim + 1])
    assert hi - lo >= 6000
    os.environ["GS_H2D_CHUNK"] = "4093"
    for how in ("swap", "dup"):
        adj = np.asarray(g.adjacency).copy()
        mid = (lo + hi) // 2
        if how == "swap":
            adj[mid], adj[mid + 1] = adj[mid + 1], adj[mid]
        else:
            adj[mid + 1] = adj[mid]
        bad = _csr(n, [adj[off[v]:off[v + 1]] for v in range(n)])
        with pytest.raises(ValueError):
            gs.scan_in_memory(bad, 3, "0.5")


def _csr(n, runs):
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in runs])
    adj = np.concatenate([np.asarray(r, np.int32) for r in runs]) if off[-1] else np.empty(0, np.int32)

    class G:
        pass

    g = G()
    g.n, g.m = n, int(off[-1]) // 2
    g.vertex_offsets, g.adjacency = off, adj
    g.orig_ids = np.arange(n, dtype=np.uint32)
    return g


@pytest.mark.parametrize("chunk", [64, 97])
def test_invalid_csr_detected_across_chunks(chunk_env, chunk):
    os.environ["GS_H2D_CHUNK"] = str(chunk)
    n = 80
    base = [[w for w in range(n) if w != v and (w - v) % n in (1, n - 1, 2, n - 2)]
            for v in range(n)]
    g = _csr(n, base)
    gs.scan_in_memory(g, 2, "0.5")  # valid: ring lattice, 4 neighbours each
    bad = [list(r) for r in base]
    bad[40] = bad[40][::-1]  # a run out of order, mid-array
    with pytest.raises(ValueError):
        gs.scan_in_memory(_csr(n, bad), 2, "0.5")
    dup = [list(r) for r in base]
    dup[16] = sorted(dup[16][:-1] + [dup[16][0]])  # repeated neighbour
    with pytest.raises(ValueError):
        gs.scan_in_memory(_csr(n, dup), 2, "0.5")
    oor = [list(r) for r in base]
    oor[70][-1] = n + 5  # id out of range
    with pytest.raises(ValueError):
        gs.scan_in_memory(_csr(n, oor), 2, "0.5")


def _random_graph(rng, n, m):
    u = rng.integers(0, n, size=m)
    # skew: a third of the endpoints from a small hot set (hubs)
    hot = rng.integers(0, max(1, n // 50), size=m)
    v = np.where(rng.random(m) < 0.33, hot, rng.integers(0, n, size=m))
    keep = u != v
    a, b = np.minimum(u, v)[keep], np.maximum(u, v)[keep]
    key = np.unique(a.astype(np.int64) * n + b)
    return np.stack([key // n, key % n], 1).astype(np.int32)


@pytest.mark.parametrize("n", [5, 97, 1000, 4097, 30000, 65537, 262143, 262145, 300001])
def test_vertex_count_sweep_against_oracle(orc, n):
    """Sizes around the hub-bitmap (2^18 ranks) and alignment boundaries."""
    rng = np.random.default_rng(n)
    e = _random_graph(rng, n, min(8 * n, 1_500_000))
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 2), ("0.45", 4)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl = _run(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"n={n} {eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"n={n} {eps} {mu}")


@pytest.mark.parametrize("n", [4097, 30000, 262145])
def test_vertex_count_sweep_sharded_and_out_of_core(orc, n):
    """The same sizes through the sharded phases (2 and 3 simulated ranks) and
    the HBM-capped partitioned engine with several partitions."""
    from test_gpu_shards import sharded

    rng = np.random.default_rng(n + 1)
    e = _random_graph(rng, n, min(8 * n, 1_500_000))
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    roles, cl = orc.serial_scan(c, 2, "0.2")
    for world in (2, 3):
        for r_roles, r_cl, _ in sharded(g, 2, "0.2", world):
            np.testing.assert_array_equal(r_roles, roles, err_msg=f"n={n} w{world}")
            np.testing.assert_array_equal(r_cl, cl, err_msg=f"n={n} w{world}")
    dmax = int(np.diff(g.vertex_offsets).max())
    budget = 13 * n + (2 << 20) + 8 * (dmax + 1) + max(2 * g.m // 4 * 4 * 4 // 3, 8 * 4 * dmax)
    plan = gs.partition_graph(g, budget)
    r, s = gs.scan_out_of_core(gs.GraphMeta.from_graph(g), plan, 2, "0.2")
    assert s.extra["partitions"] >= 2
    np.testing.assert_array_equal(r.role_codes, roles, err_msg=f"n={n} ooc")
    np.testing.assert_array_equal(r.cluster_ids, cl, err_msg=f"n={n} ooc")


def _device_csr_scan(g, mu, eps):
    """gs_engine_load_csr from DEVICE arrays (the fused relabel + sort build)."""
    import ctypes

    import torch

    from paper_2311_12281_b200 import _lib

    lib = _lib.load()
    off = torch.from_numpy(np.asarray(g.vertex_offsets, dtype=np.int64)).cuda()
    adj = torch.from_numpy(np.asarray(g.adjacency, dtype=np.int32)).cuda()
    torch.cuda.synchronize()
    eng = _lib.Engine()
    try:
        _lib.check(lib.gs_engine_load_csr(eng.handle, g.n, g.m, off.data_ptr(), adj.data_ptr(), 1))
        roles = np.empty(g.n, np.uint8)
        cl = np.empty(g.n, np.int32)
        eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps))
        _lib.check(lib.gs_engine_scan(eng.handle, mu, ctypes.byref(eps2), roles.ctypes.data,
                                      cl.ctypes.data, 0, None))
        return roles, cl
    finally:
        eng.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_device_csr_every_sort_class(orc, monkeypatch, fused):
    """Device-resident reference CSR: fused relabel + per-run sort (and the
    unfused scatter-then-sort order) in every size class incl. the hub tail."""
    monkeypatch.setenv("GS_FUSED_BUILD", fused)
    n, e = _degree_class_graph(seed=5)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.1", 3), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl = _device_csr_scan(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"{fused} {eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"{fused} {eps} {mu}")


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("deg", [5, 100, 700, 3000, 6000])
def test_device_csr_invalid_runs_detected(monkeypatch, fused, deg):
    """A duplicate, a self-loop or an unsorted run is rejected (ValueError) in
    every size class of the device build."""
    monkeypatch.setenv("GS_FUSED_BUILD", fused)
    from paper_2311_12281_b200.graph import Graph

    n = deg + 10
    edges = [(0, v) for v in range(1, deg + 1)] + [(1, 2)]
    base = make_graph(n, np.array(edges, dtype=np.int32))
    for kind in ("dup", "self", "unsorted"):
        adj = np.asarray(base.adjacency, dtype=np.int32).copy()
        o = int(base.vertex_offsets[0])
        if kind == "dup":
            adj[o + 1] = adj[o]
        elif kind == "self":
            adj[o + deg // 2] = 0
        else:
            adj[o], adj[o + 1] = adj[o + 1], adj[o]
        g = Graph(n=base.n, m=base.m, vertex_offsets=base.vertex_offsets, adjacency=adj,
                  edge_ids=base.edge_ids, edge_list=base.edge_list, orig_ids=base.orig_ids)
        with pytest.raises(ValueError):
            _device_csr_scan(g, 2, "0.5")


@pytest.mark.parametrize("batch", ["5000", "1"])
def test_hub_runs_sorted_in_batches(orc, monkeypatch, batch):
    """The hub-run segmented sort split into many batches (large graphs need
    batches below 2^31 items): same result, duplicates still caught."""
    monkeypatch.setenv("GS_SEG_BATCH", batch)
    n, e = _degree_class_graph(seed=7)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    roles, cl = orc.serial_scan(c, 3, "0.1")
    for r_roles, r_cl in (_run(g, 3, "0.1"), _device_csr_scan(g, 3, "0.1")):
        np.testing.assert_array_equal(r_roles, roles)
        np.testing.assert_array_equal(r_cl, cl)
