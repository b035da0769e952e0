"""Phase-level API (scan.py:87-134, 390-412, 452-564, 701-852, 950-962):
ClusterState, init_state, identify_core, detect_clusters,
classify_hub_outlier, build_result, find_root, union_roots.

CPU tests cover the host utilities over ClusterState (the reference's
test_union_find.py / test_scan.py cases restated); `-m gpu` tests run the
phases on the device one at a time and compare the exported state with the
oracle (oracle/) and with the one-call scan_in_memory."""

import random
import threading
from fractions import Fraction

import numpy as np
import pytest

from conftest import SHARED_MEMBER_EDGES, TWO_COMMUNITIES, cuda_ok, make_graph

import paper_2311_12281_b200 as gs
from paper_2311_12281_b200.scan import (
    PARENT_NONE,
    ROLE_CORE,
    ROLE_MEMBER,
    ROLE_MEMBER_SHARED,
    ROLE_NONCORE,
    SIM_UNKNOWN,
)


class _Ctr:
    union_retries = 0


def _fresh(n):
    g = make_graph(n, np.empty((0, 2), np.int32))
    st = gs.init_state(g)
    st.role[:] = ROLE_CORE
    st.parent[:] = np.arange(n)
    return st


# ---------------------------------------------------------------- CPU tier


def test_init_state_bounds():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    st = gs.init_state(g)
    deg = np.diff(g.vertex_offsets)
    assert list(st.lower) == [1] * 14
    assert list(st.upper) == list(deg + 1)
    assert list(st.parent) == [PARENT_NONE] * 14 and len(st.sim) == g.m
    vs = gs.init_vertex_state(3, [1, 2, 0], m=5, with_sim=False)
    assert list(vs.upper) == [2, 3, 1] and len(vs.sim) == 0


def test_find_root_requires_membership():
    st = gs.init_state(make_graph(2, np.empty((0, 2), np.int32)))
    with pytest.raises(ValueError):
        gs.find_root(st, 0)


def test_union_find_basic_and_idempotent():
    st = _fresh(6)
    gs.union_roots(st, 0, 1)
    gs.union_roots(st, 2, 3)
    assert gs.find_root(st, 0) == gs.find_root(st, 1) != gs.find_root(st, 2)
    gs.union_roots(st, 1, 3)
    assert gs.find_root(st, 0) == gs.find_root(st, 3) and gs.find_root(st, 4) == 4
    before = st.parent.copy()
    gs.union_roots(st, 0, 1)
    gs.union_roots(st, 1, 0)
    assert np.array_equal(st.parent, before)


def test_union_by_height_is_logarithmic():
    n, st, step = 256, _fresh(256), 1
    while step < n:
        for lo in range(0, n, 2 * step):
            gs.union_roots(st, lo, lo + step)
        step *= 2
    root = gs.find_root(st, 0)
    assert all(gs.find_root(st, v) == root for v in range(n))
    assert st.height[root] <= 9


def test_concurrent_unions_match_serial_components():
    rng = random.Random(42)
    n = 300
    ops = [(rng.randrange(n), rng.randrange(n)) for _ in range(1500)]
    serial = _fresh(n)
    for u, v in ops:
        gs.union_roots(serial, u, v)
    want = {}
    for v in range(n):
        want.setdefault(gs.find_root(serial, v), set()).add(v)
    st, lock, ctr = _fresh(n), threading.Lock(), _Ctr()
    ts = [threading.Thread(target=lambda c=ops[i::6]: [gs.union_roots(st, u, v, lock=lock,
                                                                      counters=ctr)
                                                       for u, v in c]) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    got = {}
    for v in range(n):
        got.setdefault(gs.find_root(st, v), set()).add(v)
    assert sorted(map(sorted, got.values())) == sorted(map(sorted, want.values()))


def test_resolve_roles_from_bounds_and_build_result_errors():
    st = gs.init_vertex_state(3, [4, 1, 4], m=0, with_sim=False)
    st.lower[:] = [5, 1, 2]
    st.upper[:] = [5, 2, 6]
    assert gs.resolve_roles_from_bounds(st, 3)  # vertex 2 still open (scan.py:390-412)
    assert list(st.role) == [ROLE_CORE, ROLE_NONCORE, 0]
    with pytest.raises(RuntimeError):
        gs.resolve_roles_from_bounds(st, 3, strict=True)
    with pytest.raises(RuntimeError):
        gs.build_result(st, [0, 1, 2])


def test_detect_clusters_needs_identify_first():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    st = gs.init_state(g)
    with pytest.raises(RuntimeError):
        gs.detect_clusters(g, "0.6", st)


# ---------------------------------------------------------------- GPU tier

gpu = pytest.mark.gpu
need_cuda = pytest.mark.skipif(not cuda_ok(), reason="no CUDA device")


def _truth(g, orc, eps):
    """Per reference edge: similar? (exact, from the oracle's common counts)."""
    from oracle import oracle

    c = oracle.CSR(g.n, np.stack([g.edge_list[0::2], g.edge_list[1::2]], 1))
    com = oracle.commons(c).astype(object)
    f2 = Fraction(eps) ** 2
    deg = np.diff(g.vertex_offsets)
    a, b = g.edge_list[0::2], g.edge_list[1::2]
    return np.array([Fraction((int(com[k]) + 2) ** 2, int((deg[a[k]] + 1) * (deg[b[k]] + 1))) >= f2
                     for k in range(g.m)], dtype=bool)


@gpu
@need_cuda
def test_identify_core_roles_fig1():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    st = gs.init_state(g)
    gs.identify_core(g, 3, "0.6", st)
    assert set(np.flatnonzero(st.role == ROLE_CORE)) == {0, 1, 4, 7, 9, 10, 11, 12, 13}
    assert set(np.flatnonzero(st.role == ROLE_NONCORE)) == {2, 3, 5, 6, 8}


@gpu
@need_cuda
@pytest.mark.parametrize("seed,eps,mu", [(1, "0.6", 3), (2, "0.35", 2), (3, "0.75", 4)])
def test_bounds_sandwich_and_sim_match_truth(orc, seed, eps, mu):
    rng = np.random.default_rng(seed)
    n = 60
    pairs = {tuple(sorted(rng.choice(n, 2, replace=False))) for _ in range(260)}
    g = make_graph(n, sorted(pairs))
    truth = _truth(g, orc, eps)
    deg = np.diff(g.vertex_offsets)
    a, b = g.edge_list[0::2], g.edge_list[1::2]
    nsim = np.ones(n, np.int64)
    np.add.at(nsim, a[truth], 1)
    np.add.at(nsim, b[truth], 1)
    st = gs.init_state(g)
    seen = []

    def audit(_k):
        assert np.all(st.lower <= nsim) and np.all(nsim <= st.upper)
        seen.append(_k)

    gs.identify_core(g, mu, eps, st, on_edge=audit)
    assert len(seen) == 2
    assert np.all(st.lower <= nsim) and np.all(nsim <= st.upper)
    assert np.array_equal(st.role == ROLE_CORE, nsim >= mu)
    assert np.all(st.upper <= deg + 1)
    dec = st.sim != SIM_UNKNOWN
    assert dec.any()
    np.testing.assert_array_equal(st.sim[dec] == 1, truth[dec])


@gpu
@need_cuda
def test_phases_individually_equal_scan_in_memory(golden, orc):
    from oracle import oracle

    checked = 0
    for k, c in golden.cases():
        if c["n"] > 3000:
            continue
        g = make_graph(c["n"], golden.edges(k))
        for cfg in c["configs"][:4]:
            st = gs.init_state(g)
            stats = gs.StatsReport(n=g.n, m=g.m)
            gs.identify_core(g, cfg["mu"], cfg["eps"], st, stats=stats)
            gs.detect_clusters(g, cfg["eps"], st, stats=stats)
            gs.classify_hub_outlier(g, st, stats=stats)
            gs.classify_hub_outlier(g, st)  # idempotent
            res = gs.build_result(st, g.orig_ids)
            one, _ = gs.scan_in_memory(g, cfg["mu"], cfg["eps"])
            np.testing.assert_array_equal(res.role_codes, one.role_codes)
            np.testing.assert_array_equal(res.cluster_ids, one.cluster_ids)
            if g.n:
                assert set(stats.phases) == {"identify", "cleanup", "cluster", "classify"}
                assert stats.sim_evals <= g.m
                # parent forms a flattened forest rooted at cores
                cl = st.parent >= 0
                assert np.all(st.parent[st.parent[cl]] == st.parent[cl])
                assert np.all(st.role[st.parent[cl]] == ROLE_CORE)
            checked += 1
    assert checked > 40


@gpu
@need_cuda
def test_shared_member_internal_role():
    g = make_graph(7, SHARED_MEMBER_EDGES)
    st = gs.init_state(g)
    gs.identify_core(g, 4, "0.5", st)
    gs.detect_clusters(g, "0.5", st)
    assert st.role[3] == ROLE_MEMBER_SHARED
    gs.classify_hub_outlier(g, st)
    assert st.role[3] == ROLE_MEMBER_SHARED
    res = gs.build_result(st, g.orig_ids)
    assert res.member_set() >= {3} and res.role_codes[3] == ROLE_MEMBER
