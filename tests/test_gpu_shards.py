"""Sharded scan correctness on ONE GPU: W engines (one per simulated rank)
run the phases of dist.ShardedScan in lock-step; the three exchanges are
done here with torch ops on the device (sum / concat / min / max), i.e. what
NCCL computes.  Every rank must produce the single-GPU canonical result."""

import ctypes

import numpy as np
import pytest

from conftest import TWO_COMMUNITIES, cuda_ok, make_graph

pytestmark = pytest.mark.gpu

if not cuda_ok():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_2311_12281_b200 as gs  # noqa: E402
from paper_2311_12281_b200 import _lib  # noqa: E402


def partitioned_load(engs, g, on_device=False):
    """gs_engine_load_csr_part on every simulated rank, then the row slices
    copied owner -> everyone (what dist.ShardedScan.load_csr broadcasts)."""
    lib = _lib.load()
    n, m, world = g.n, g.m, len(engs)
    bufs = [torch.empty(max(2 * m, 1), dtype=torch.int32, device="cuda") for _ in engs]
    if on_device:
        off_d = torch.from_numpy(np.asarray(g.vertex_offsets)).cuda()
        adj_d = torch.from_numpy(np.asarray(g.adjacency)).cuda()
        off_p, adj_p = off_d.data_ptr(), adj_d.data_ptr()
    else:
        off_p, adj_p = g.vertex_offsets.ctypes.data, g.adjacency.ctypes.data
    bounds = []
    for r, e in enumerate(engs):
        b = (ctypes.c_int64 * (world + 1))()
        _lib.check(lib.gs_engine_load_csr_part(e.handle, n, m, off_p, adj_p, int(on_device), r,
                                               world, bufs[r].data_ptr(), b))
        bounds.append([int(x) for x in b])
    assert all(b == bounds[0] for b in bounds)
    torch.cuda.synchronize()
    for k in range(world):
        lo, hi = bounds[0][k], bounds[0][k + 1]
        for r in range(world):
            if r != k and hi > lo:
                bufs[r][lo:hi].copy_(bufs[k][lo:hi])
    torch.cuda.synchronize()
    if world > 1:
        for e in engs:
            _lib.check(lib.gs_engine_load_finish(e.handle))
    return bufs


def sharded(g, mu, eps, world, partitioned=False, on_device=False):
    lib = _lib.load()
    n, m = g.n, g.m
    eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps))
    engs = [_lib.Engine() for _ in range(world)]
    keep = partitioned_load(engs, g, on_device) if partitioned else None
    for r, e in enumerate(engs):
        if not partitioned:
            _lib.check(lib.gs_engine_load_csr(e.handle, n, m, g.vertex_offsets.ctypes.data,
                                              g.adjacency.ctypes.data, 0))
        _lib.check(lib.gs_engine_set_shard(e.handle, r, world))
        _lib.check(lib.gs_engine_phase_begin(e.handle, mu, ctypes.byref(eps2)))
    cnt = [torch.empty(2 * n, dtype=torch.int32, device="cuda") for _ in range(world)]
    for e, c in zip(engs, cnt):
        _lib.check(lib.gs_engine_phase_identify(e.handle, c.data_ptr()))
    tot = torch.stack(cnt).sum(0).to(torch.int32).contiguous()          # all-reduce SUM
    torch.cuda.synchronize()  # the engines read it on their own streams
    ncs = []
    for e in engs:
        nc = ctypes.c_int64(0)
        _lib.check(lib.gs_engine_phase_resolve(e.handle, tot.data_ptr(), ctypes.byref(nc)))
        ncs.append(nc.value)
    assert len(set(ncs)) == 1
    labels = None
    if ncs[0] > 0:
        pairs = [torch.empty((n, 2), dtype=torch.int32, device="cuda") for _ in range(world)]
        nps = []
        for e, p in zip(engs, pairs):
            npr = ctypes.c_int64(0)
            _lib.check(lib.gs_engine_phase_union(e.handle, p.data_ptr(), ctypes.byref(npr)))
            nps.append(npr.value)
        allp = torch.cat([p[:k] for p, k in zip(pairs, nps)]).contiguous()   # all-gather
        torch.cuda.synchronize()
        for e in engs:
            _lib.check(lib.gs_engine_phase_merge(e.handle, allp.data_ptr() if len(allp) else None,
                                                 len(allp)))
        lab = [torch.empty(2 * n, dtype=torch.int32, device="cuda") for _ in range(world)]
        for e, l in zip(engs, lab):
            _lib.check(lib.gs_engine_phase_attach(e.handle, l.data_ptr()))
        st = torch.stack(lab)
        labels = torch.cat([st[:, :n].min(0).values, st[:, n:].max(0).values]).contiguous()
        torch.cuda.synchronize()
    else:
        for e in engs:
            _lib.check(lib.gs_engine_phase_merge(e.handle, None, 0))
    outs = []
    for e in engs:
        roles = np.empty(n, np.uint8)
        cl = np.empty(n, np.int32)
        stats = _lib.GsStats()
        _lib.check(lib.gs_engine_phase_finish(e.handle, labels.data_ptr() if labels is not None
                                              else None, roles.ctypes.data, cl.ctypes.data, 0,
                                              ctypes.byref(stats)))
        outs.append((roles, cl, stats.sim_evals))
    for e in engs:
        e.close()
    del keep
    return outs


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fig1(world):
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    r, _ = gs.scan_in_memory(g, 3, "0.6")
    for roles, cl, _ in sharded(g, 3, "0.6", world):
        np.testing.assert_array_equal(roles, r.role_codes)
        np.testing.assert_array_equal(cl, r.cluster_ids)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_rmat_matches_single_gpu_and_oracle(orc, world):
    n, e = orc.rmat(15, seed=2)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 3), ("0.3", 5), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        outs = sharded(g, mu, eps, world)
        total_evals = sum(o[2] for o in outs)
        for r_roles, r_cl, _ in outs:
            np.testing.assert_array_equal(r_roles, roles, err_msg=f"w{world} {eps} {mu}")
            np.testing.assert_array_equal(r_cl, cl, err_msg=f"w{world} {eps} {mu}")
        assert total_evals <= 2 * g.m  # each edge decided at most once per phase


def test_sharded_golden_corpus(golden):
    n_cfg = 0
    for k, c in golden.cases():
        if not c["name"].startswith(("corpus", "shared")) or c["m"] == 0:
            continue
        g = make_graph(c["n"], golden.edges(k))
        for j, cfg in enumerate(c["configs"][::5]):
            jj = 5 * j
            for roles, cl, _ in sharded(g, cfg["mu"], cfg["eps"], 2):
                np.testing.assert_array_equal(roles, golden.get(k, f"c{jj}_roles"))
                np.testing.assert_array_equal(cl, golden.get(k, f"c{jj}_cluster"))
            n_cfg += 1
    assert n_cfg > 100


@pytest.mark.parametrize("world,on_device", [(2, False), (3, True), (4, False), (8, True)])
def test_partitioned_build_matches_single_gpu_and_oracle(orc, world, on_device):
    """Each rank builds 1/world of the rank-space rows; after the exchange all
    ranks hold the same CSR and produce the single-GPU canonical result."""
    n, e = orc.rmat(15, seed=6)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 3), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        for r_roles, r_cl, _ in sharded(g, mu, eps, world, partitioned=True, on_device=on_device):
            np.testing.assert_array_equal(r_roles, roles, err_msg=f"w{world} {eps} {mu}")
            np.testing.assert_array_equal(r_cl, cl, err_msg=f"w{world} {eps} {mu}")


def test_partitioned_build_rejects_invalid_part():
    lib = _lib.load()
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    eng = _lib.Engine()
    b = (ctypes.c_int64 * 3)()
    with pytest.raises(ValueError):  # a partitioned build needs the caller's buffer
        _lib.check(lib.gs_engine_load_csr_part(eng.handle, g.n, g.m, g.vertex_offsets.ctypes.data,
                                               g.adjacency.ctypes.data, 0, 0, 2, None, b))
    with pytest.raises(ValueError):
        _lib.check(lib.gs_engine_load_finish(eng.handle))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_with_sketch_forced(orc, monkeypatch, world):
    """Every rank tries the sketch bound on every survivor it owns (rows built
    by each rank for the whole graph): still the oracle's result."""
    monkeypatch.setenv("GS_SKETCH", "4")
    monkeypatch.setenv("GS_SKETCH_DMIN", "1")
    monkeypatch.setenv("GS_SKETCH_MINSCAN", "-1000000")
    monkeypatch.setenv("GS_SKETCH_GATE", "1e30")
    n, e = orc.rmat(15, seed=8)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 3), ("0.4", 2)):
        roles, cl = orc.serial_scan(c, mu, eps)
        for r_roles, r_cl, _ in sharded(g, mu, eps, world, partitioned=True):
            np.testing.assert_array_equal(r_roles, roles, err_msg=f"w{world} {eps} {mu}")
            np.testing.assert_array_equal(r_cl, cl, err_msg=f"w{world} {eps} {mu}")
