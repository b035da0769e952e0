"""The reference's spill format (GSCP partition files + plan.manifest,
partition.py:231-446) against fixtures the reference itself wrote
(tests/golden/spill/, made by tests/golden/make_spill_golden.py).

CPU: the native closure planner (gs_plan_closure) reproduces the reference's
partition boundaries, closure sizes, estimates and InfeasibleBudgetError;
load_partition / store_sim read and write the reference's files with its
checks.  GPU: partition_graph(g, budget, spill_dir) writes byte-identical
files (local graphs built on the device), and a plan known only through its
spill files -- the reference's own -- is executed by scan_out_of_core with
results equal to the oracle."""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import make_graph

import paper_2311_12281_b200 as gs
from paper_2311_12281_b200 import partition as P

SPILL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spill")
CASES = sorted(d for d in os.listdir(SPILL) if os.path.isdir(os.path.join(SPILL, d)))


def _case(name):
    d = os.path.join(SPILL, name)
    with open(os.path.join(d, "case.json")) as f:
        c = json.load(f)
    g = make_graph(c["n"], [tuple(e) for e in c["edges"]])
    return d, c, g


def _manifest(d):
    """The reference's manifest (partition.py:318-333) -> header dict + records."""
    with open(os.path.join(d, "plan.manifest")) as f:
        lines = f.read().splitlines()
    head = dict(x.split("=") for x in lines[:5])
    parts = []
    for ln in lines[5:]:
        k, fname, nl, ml, lo, hi, est = ln.split("\t")
        parts.append(gs.PartitionInfo(index=int(k), path=os.path.join(d, fname),
                                      n_local=int(nl), m_local=int(ml), owned_lo=int(lo),
                                      owned_hi=int(hi), estimate_bytes=int(est)))
    return head, parts


def test_fixtures_present():
    assert CASES == ["fig1", "gnm300", "skewed400"]


@pytest.mark.parametrize("name", CASES)
def test_closure_planner_matches_the_reference_plan(name):
    d, c, g = _case(name)
    head, parts = _manifest(d)
    assert int(head["partitions"]) == len(parts) == c["partitions"]
    assert int(head["global_state_bytes"]) == 15 * g.n
    recs = P._plan_closure(g, c["budget"], 15 * g.n)
    assert len(recs) == len(parts)
    for (lo, hi, nl, ml), p in zip(recs, parts):
        assert (lo, hi, nl, ml) == (p.owned_lo, p.owned_hi, p.n_local, p.m_local)
        assert 25 * ml + 4 * nl == p.estimate_bytes
        assert p.estimate_bytes + 15 * g.n <= c["budget"]
    assert recs[0][0] == 0 and recs[-1][1] == g.m
    assert all(a[1] == b[0] for a, b in zip(recs, recs[1:]))


@pytest.mark.parametrize("name", CASES)
def test_infeasible_budget_matches_the_reference(name, tmp_path):
    d, c, g = _case(name)
    bad = c["infeasible"]
    assert bad is not None
    with pytest.raises(gs.InfeasibleBudgetError) as ei:
        gs.partition_graph(g, bad["budget"], spill_dir=str(tmp_path / "x"))
    assert ei.value.edge == tuple(bad["edge"])
    assert ei.value.required_bytes == bad["required"]
    assert ei.value.budget_bytes == bad["budget"]
    with pytest.raises(gs.InfeasibleBudgetError) as ei:  # the 15n state check first
        gs.partition_graph(g, 15 * g.n - 1, spill_dir=str(tmp_path / "y"))
    assert ei.value.edge == (-1, -1)


@pytest.mark.parametrize("name", CASES)
def test_load_partition_reads_the_reference_files(name):
    d, c, g = _case(name)
    _, parts = _manifest(d)
    el = g.edge_list.reshape(-1, 2)
    owned_total = 0
    for p in parts:
        sub = gs.load_partition(p)
        lg = sub.local_graph
        assert (sub.index, sub.owned_lo, sub.owned_hi) == (p.index, p.owned_lo, p.owned_hi)
        assert (lg.n, lg.m) == (p.n_local, p.m_local) and len(sub.sim_local) == lg.m
        assert gs.estimate_memory(sub) == p.estimate_bytes == gs.estimate_memory(p)
        assert np.all(np.diff(sub.vmap.astype(np.int64)) > 0)  # ascending global ids
        assert np.array_equal(lg.orig_ids, sub.vmap)
        # every local edge is the global edge emap names
        loc = sub.vmap.astype(np.int64)[lg.edge_list.reshape(-1, 2)]
        glob = el[sub.emap.astype(np.int64)]
        assert np.array_equal(np.sort(loc, axis=1), np.sort(glob, axis=1))
        own = sub.emap[sub.owned_local]
        assert list(own) == list(range(p.owned_lo, p.owned_hi))
        owned_total += len(own)
    assert owned_total == g.m


def test_store_sim_and_file_errors(tmp_path):
    d, c, g = _case("gnm300")
    _, parts = _manifest(d)
    shutil.copytree(d, tmp_path / "s")
    p = parts[3]
    info = gs.PartitionInfo(p.index, str(tmp_path / "s" / os.path.basename(p.path)), p.n_local,
                            p.m_local, p.owned_lo, p.owned_hi, p.estimate_bytes)
    sub = gs.load_partition(info)
    sub.sim_local[:] = bytes((k % 3) for k in range(len(sub.sim_local)))
    gs.store_sim(info, sub)
    again = gs.load_partition(info)
    assert again.sim_local == sub.sim_local
    assert np.array_equal(again.local_graph.adjacency, sub.local_graph.adjacency)
    with pytest.raises(ValueError, match="does not match plan entry"):
        gs.load_partition(gs.PartitionInfo(p.index + 1, info.path, p.n_local, p.m_local,
                                           p.owned_lo, p.owned_hi, 0))
    raw = open(info.path, "rb").read()
    trunc = tmp_path / "t.bin"
    trunc.write_bytes(raw[:-p.m_local - 5])
    with pytest.raises(ValueError, match="truncated"):
        gs.load_partition(gs.PartitionInfo(p.index, str(trunc), p.n_local, p.m_local,
                                           p.owned_lo, p.owned_hi, 0))
    bad = tmp_path / "b.bin"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="not a partition spill file"):
        gs.load_partition(gs.PartitionInfo(p.index, str(bad), p.n_local, p.m_local,
                                           p.owned_lo, p.owned_hi, 0))
    with pytest.raises(OSError, match=f"partition {p.index}"):
        gs.load_partition(gs.PartitionInfo(p.index, str(tmp_path / "none.bin"), p.n_local,
                                           p.m_local, p.owned_lo, p.owned_hi, 0))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_spill_files_are_byte_identical_to_the_reference(name, tmp_path):
    d, c, g = _case(name)
    out = str(tmp_path / "spill")
    plan = gs.partition_graph(g, c["budget"], spill_dir=out)
    assert plan.manifest_path == os.path.join(out, "plan.manifest")
    assert sorted(os.listdir(out)) == sorted(f for f in os.listdir(d) if f != "case.json")
    for f in os.listdir(out):
        with open(os.path.join(out, f), "rb") as a, open(os.path.join(d, f), "rb") as b:
            assert a.read() == b.read(), f


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_scan_out_of_core_from_the_reference_spill_files(name):
    """A plan known only through its files (no in-memory graph, as the
    reference's scan_out_of_core sees it): the graph is read back from the
    partitions' owned edges and clustered on the device."""
    from oracle import oracle as orc

    d, c, g = _case(name)
    _, parts = _manifest(d)
    meta = gs.GraphMeta(n=g.n, m=g.m, degrees=np.diff(g.vertex_offsets),
                        orig_ids=np.asarray(g.orig_ids))
    # the files' budget is the reference's host budget; the device runs under
    # a cap it can meet (64 MiB: state + streaming buffers)
    plan = gs.PartitionPlan(n=g.n, m=g.m, budget_bytes=64 << 20, partitions=parts, spill_dir=d)
    res, stats = gs.scan_out_of_core(meta, plan, c["mu"], c["eps"])
    roles, cids = orc.serial_scan(orc.CSR(c["n"], np.asarray(c["edges"], np.int32)),
                                  c["mu"], c["eps"])
    assert np.array_equal(res.role_codes, roles)
    assert np.array_equal(res.cluster_ids, cids)
    assert "".join(r.name[0] for r in res.roles) == c["roles"]
    assert stats.extra["partitions"] == len(parts)


def _plan_closure_py(g, budget, state):
    """The reference's greedy closure planner restated line for line
    (partition.py:245-312) as the checker for the native one."""
    off, adj, eids = g.vertex_offsets, g.adjacency, g.edge_ids
    pairs = g.edge_list
    in_v, in_e = [-1] * g.n, [-1] * g.m
    out, index, owned_lo, cur_v, cur_e, cost = [], 0, 0, 0, 0, 0

    def closure(u, v):
        nv, ne, sv, se = [], [], set(), set()
        for x in (u, v):
            if in_v[x] != index and x not in sv:
                sv.add(x)
                nv.append(x)
            for i in range(off[x], off[x + 1]):
                w, e = int(adj[i]), int(eids[i])
                if in_v[w] != index and w not in sv:
                    sv.add(w)
                    nv.append(w)
                if in_e[e] != index and e not in se:
                    se.add(e)
                    ne.append(e)
        return nv, ne

    for k in range(g.m):
        u, v = int(pairs[2 * k]), int(pairs[2 * k + 1])
        nv, ne = closure(u, v)
        add = 25 * len(ne) + 4 * len(nv)
        if cur_e and cost + add + state > budget:
            out.append((owned_lo, k, cur_v, cur_e))
            index, owned_lo, cur_v, cur_e, cost = index + 1, k, 0, 0, 0
            nv, ne = closure(u, v)
            add = 25 * len(ne) + 4 * len(nv)
        if cost + add + state > budget:
            return ("infeasible", (u, v), cost + add + state)
        for x in nv:
            in_v[x] = index
        for e in ne:
            in_e[e] = index
        cur_v, cur_e, cost = cur_v + len(nv), cur_e + len(ne), cost + add
    if cur_e:
        out.append((owned_lo, g.m, cur_v, cur_e))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_closure_planner_matches_a_restatement_on_random_graphs(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 120))
    hot = max(1, n // 10)
    e = set()
    for _ in range(int(rng.integers(n, 5 * n))):
        u = int(rng.integers(0, hot)) if rng.random() < 0.4 else int(rng.integers(0, n))
        v = int(rng.integers(0, n))
        if u != v:
            e.add((min(u, v), max(u, v)))
    if not e:
        return
    g = make_graph(n, sorted(e))
    est = 25 * g.m + 4 * g.n
    for budget in (15 * n + est // int(rng.integers(2, 12)), 15 * n + 400, 15 * n + est + 1):
        want = _plan_closure_py(g, budget, 15 * n)
        if isinstance(want, tuple):
            with pytest.raises(gs.InfeasibleBudgetError) as ei:
                P._plan_closure(g, budget, 15 * n)
            assert ei.value.edge == want[1] and ei.value.required_bytes == want[2]
        else:
            assert P._plan_closure(g, budget, 15 * n) == want


@pytest.mark.gpu
def test_spill_interop_with_the_reference_package():
    """Both directions with the reference's own code (baseline/_ref, shipped with
    the snapshot; skipped without it): the reference's spill plan executed by
    this engine, and this package's spill plan executed by the reference's
    scan_out_of_core (tools/spill_interop.py)."""
    import subprocess
    import sys

    from conftest import ROOT

    ref_src = os.path.join(ROOT, "baseline", "_ref", "pkg", "src")
    if not os.path.isdir(ref_src):
        pytest.skip("baseline/_ref/pkg (the reference package) not shipped")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ref_src, ROOT,
                                                       os.environ.get("PYTHONPATH", "")]))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "spill_interop.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["ok"] and all(c["reference_plan_on_engine"]["partitions"] >= 3
                             for c in rep["cases"]), rep
