"""GPU parity: the sm_100a engine (through the C-ABI via the host package)
against the golden vectors of the Python reference and the pinned CPU oracle.

Bar: bit-exact roles and canonical cluster ids (integer work), plus the
reference's own observable invariants (sim_evals <= m, zero probe-bound
violations, pruning fires on the 50-clique)."""

import array
from fractions import Fraction

import numpy as np
import pytest

from conftest import SHARED_MEMBER_EDGES, TWO_COMMUNITIES, cuda_ok, make_graph

pytestmark = pytest.mark.gpu

if not cuda_ok():  # the -m gpu tier runs on the B200 box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2311_12281_b200 as gs  # noqa: E402


def run(g, mu, eps):
    r, s = gs.scan_in_memory(g, mu, eps)
    return r.role_codes.copy(), r.cluster_ids.copy(), r, s


def test_native_library_is_the_path():
    from paper_2311_12281_b200 import _lib

    assert _lib._lib is not None or _lib.load() is not None
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    _, _, _, s = run(g, 3, "0.6")
    assert s.extra["kernel_launches"] > 5


def test_fig1_golden():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    roles, cl, r, s = run(g, 3, "0.6")
    assert r.core_set() == {0, 1, 4, 7, 9, 10, 11, 12, 13}
    assert r.member_set() == {2}
    assert r.hub_set() == {8}
    assert r.outlier_set() == {3, 5, 6}
    assert r.core_equivalence() == {frozenset({0, 1, 4, 7}), frozenset({9, 10, 11, 12, 13})}
    assert r.cluster_id[2] == r.cluster_id[0] == 0
    assert s.probe_bound_violations == 0 and s.sim_evals <= g.m
    lines = r.to_text().splitlines()
    assert lines[8] == "8\tH\t-1" and lines[3] == "3\tO\t-1" and len(lines) == 14
    assert "".join("CMHO"[[1, 3, 5, 6].index(c)] for c in roles) == "CCMOCOOCHCCCCC"


def test_every_golden_config_bit_exact(golden):
    """All golden graphs x (eps, mu): roles + canonical ids == serial_scan."""
    n_cfg = 0
    for k, c in golden.cases():
        g = make_graph(c["n"], golden.edges(k))
        for j, cfg in enumerate(c["configs"]):
            roles, cl, _, s = run(g, cfg["mu"], cfg["eps"])
            np.testing.assert_array_equal(roles, golden.get(k, f"c{j}_roles"),
                                          err_msg=f"{c['name']} {cfg}")
            np.testing.assert_array_equal(cl, golden.get(k, f"c{j}_cluster"),
                                          err_msg=f"{c['name']} {cfg}")
            assert s.sim_evals <= max(g.m, 0) and s.probe_bound_violations == 0
            n_cfg += 1
    assert n_cfg > 1000


def test_reference_array_graph_input(golden):
    """A graph whose fields are array.array (the reference Graph's types) is
    accepted zero-copy, same answer."""

    class RefLike:
        pass

    k = 0
    c = golden.meta["cases"][k]
    g = make_graph(c["n"], golden.edges(k))
    h = RefLike()
    h.n, h.m = g.n, g.m
    h.vertex_offsets = array.array("q", g.vertex_offsets.tolist())
    h.adjacency = array.array("i", g.adjacency.tolist())
    h.orig_ids = array.array("I", g.orig_ids.tolist())
    a = run(g, 3, "0.6")
    b = run(h, 3, "0.6")
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_shared_member_instance():
    g = make_graph(7, SHARED_MEMBER_EDGES)
    roles, cl, r, _ = run(g, 4, "0.5")
    assert r.core_set() == {2, 4}
    assert 3 in r.member_set() and cl[3] == 2  # min eligible label
    assert cl[6] == 4


def test_clique_pruning_strict():
    n = 50
    g = make_graph(n, [(u, v) for u in range(n) for v in range(u + 1, n)])
    _, _, r, s = run(g, 3, "0.1")
    assert r.core_set() == set(range(n))
    assert len(r.core_equivalence()) == 1
    assert s.sim_evals < g.m


def test_edge_cases():
    g = make_graph(4, [(0, 1)])
    _, _, r, _ = run(g, 2, "0.5")
    assert r.outlier_set() >= {2, 3}
    g = make_graph(5, [])
    roles, cl, r, s = run(g, 2, "0.5")
    assert (roles == 6).all() and (cl == -1).all() and s.sim_evals == 0
    g = make_graph(3, [(0, 1), (0, 2), (1, 2)])
    _, _, r, _ = run(g, 2, "0.5")
    assert r.core_set() == {0, 1, 2} and not r.hub_set()


def test_threshold_exactness():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    assert gs.check_sim(g, 0, 3, "0.5")
    assert not gs.check_sim(g, 0, 3, "0.500000000000001")
    assert gs.check_sim(g, 4, 7, "1")
    with pytest.raises(ValueError):
        gs.check_sim(g, 3, 5, "0.5")


def test_check_sim_every_edge(golden):
    for k in range(3):
        c = golden.meta["cases"][k]
        g = make_graph(c["n"], golden.edges(k))
        com = golden.get(k, "commons")
        deg = np.diff(g.vertex_offsets)
        for eps in ("0.2", "0.5", "0.6", "0.8", "1"):
            f2 = Fraction(eps) ** 2
            for e in range(g.m):
                a, b = g.endpoints(e)
                exp = Fraction((int(com[e]) + 2) ** 2,
                               int((deg[a] + 1) * (deg[b] + 1))) >= f2
                assert gs.check_sim(g, a, b, eps) == exp
                assert gs.check_sim(g, b, a, eps) == exp


def test_device_build_graph_matches_reference_layout(golden):
    n_checked = 0
    for k, c in golden.cases():
        if not c["build"] or c["m"] == 0:
            continue
        el = gs.EdgeList(n_hint=c["n"], edges=golden.edges(k))
        g = gs.build_graph(el)
        np.testing.assert_array_equal(g.vertex_offsets, golden.get(k, "offsets"))
        np.testing.assert_array_equal(g.adjacency, golden.get(k, "adjacency"))
        np.testing.assert_array_equal(g.edge_ids, golden.get(k, "edge_ids"))
        np.testing.assert_array_equal(g.edge_list, golden.get(k, "edge_list"))
        n_checked += 1
    assert n_checked >= 8


def test_build_graph_rejects_bad_edges():
    with pytest.raises(ValueError):
        gs.build_graph(gs.EdgeList(n_hint=2, edges=[(0, 0)]))
    with pytest.raises(ValueError):
        gs.build_graph(gs.EdgeList(n_hint=2, edges=[(0, 1), (0, 1)]))
    with pytest.raises(ValueError):
        gs.build_graph(gs.EdgeList(n_hint=1, edges=[(0, -1)]))


def test_scan_edges_path_matches_csr_path(orc):
    n, e = orc.rmat(13, seed=11)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 3), ("0.4", 5)):
        a = run(g, mu, eps)
        r, s = gs.scan_edges(n, e, mu, eps)
        np.testing.assert_array_equal(a[0], r.role_codes)
        np.testing.assert_array_equal(a[1], r.cluster_ids)


@pytest.mark.parametrize("scale,seed", [(16, 1), (17, 2)])
def test_rmat_against_oracle(orc, scale, seed):
    n, e = orc.rmat(scale, seed=seed)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.2", 3), ("0.2", 5), ("0.3", 3), ("0.5", 5), ("0.6", 3)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl, _, s = run(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"s{scale} {eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"s{scale} {eps} {mu}")
        assert s.sim_evals <= g.m


def test_skewed_hub_graph(orc):
    """Huge-degree hubs (L2-table path) + many small vertices: star-of-cliques."""
    rng = np.random.default_rng(5)
    n = 70000
    edges = set()
    hubs = [0, 1, 2]
    for h in hubs:
        for v in rng.choice(np.arange(3, n), size=40000, replace=False):
            edges.add((h, int(v)))
    for _ in range(200000):
        u, v = rng.integers(3, n, size=2)
        if u != v:
            edges.add((int(min(u, v)), int(max(u, v))))
    edges.add((0, 1)); edges.add((1, 2)); edges.add((0, 2))
    e = np.array(sorted(edges), dtype=np.int32)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.05", 2), ("0.1", 3), ("0.3", 2)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl, _, _ = run(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"{eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"{eps} {mu}")


def test_repeat_runs_identical(orc):
    n, e = orc.rmat(14, seed=9)
    g = make_graph(n, e)
    a = run(g, 3, "0.2")
    for _ in range(3):
        b = run(g, 3, "0.2")
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


def test_gpu_generator_matches_cpu(orc):
    import ctypes

    import torch

    from paper_2311_12281_b200 import _lib

    lib = _lib.load()
    scale, seed = 14, 4
    cnt = 16 << scale
    src = torch.empty(cnt, dtype=torch.int32, device="cuda")
    dst = torch.empty(cnt, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_rmat_generate(scale, 16, seed, src.data_ptr(), dst.data_ptr(), None))
    torch.cuda.synchronize()
    cs, cd = orc.rmat_raw(scale, seed=seed)
    np.testing.assert_array_equal(src.cpu().numpy(), cs)
    np.testing.assert_array_equal(dst.cpu().numpy(), cd)
    uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    m = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(m), None))
    n, e = orc.rmat(scale, seed=seed)
    assert m.value == len(e)
    np.testing.assert_array_equal(uv[: 2 * m.value].cpu().numpy().reshape(-1, 2), e)


def test_errors_map_to_reference_exceptions():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    with pytest.raises(ValueError):
        gs.scan_in_memory(g, 1, "0.5")
    with pytest.raises(ValueError):
        gs.scan_in_memory(g, 3, "0")

    class Bad:
        pass

    b = Bad()
    b.n, b.m = 3, 1
    b.vertex_offsets = np.array([0, 1, 1, 2], np.int64)
    b.adjacency = np.array([1, 1], np.int32)  # asymmetric: 0->1, 2->1
    b.orig_ids = np.arange(3, dtype=np.uint32)
    with pytest.raises(ValueError):
        gs.scan_in_memory(b, 2, "0.5")


# ---------------------------------------------------------------------------
# out-of-core mode (gs_scan_partitioned): same canonical output under an HBM cap

def _ooc(g, mu, eps, budget):
    plan = gs.partition_graph(g, budget)
    meta = gs.GraphMeta.from_graph(g)
    r, s = gs.scan_out_of_core(meta, plan, mu, eps)
    return plan, r, s


def test_ooc_fig1_single_and_multi_partition():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    ref = run(g, 3, "0.6")
    for budget in (1 << 26, 13 * 14 + (2 << 20) + 8 * 8 + 4 * 1024 * 8 + 2000):
        plan, r, s = _ooc(g, 3, "0.6", budget)
        np.testing.assert_array_equal(r.role_codes, ref[0])
        np.testing.assert_array_equal(r.cluster_ids, ref[1])
        assert s.extra["partitions"] >= 1


@pytest.mark.parametrize("scale,seed", [(14, 3), (16, 1)])
def test_ooc_rmat_matches_oracle_with_many_partitions(orc, scale, seed):
    n, e = orc.rmat(scale, seed=seed)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    dmax = int(np.diff(g.vertex_offsets).max())
    # leave room for buffers of ~1/8 of the adjacency: forces several partitions
    budget = 13 * n + (2 << 20) + 8 * (dmax + 1) + max(2 * g.m // 4 * 4 * 4 // 3, 8 * 4 * dmax)
    for eps, mu in (("0.2", 3), ("0.3", 5), ("0.5", 5)):
        roles, cl = orc.serial_scan(c, mu, eps)
        plan, r, s = _ooc(g, mu, eps, budget)
        assert s.extra["partitions"] >= 3, s.extra
        np.testing.assert_array_equal(r.role_codes, roles, err_msg=f"{eps} {mu}")
        np.testing.assert_array_equal(r.cluster_ids, cl, err_msg=f"{eps} {mu}")
        assert s.extra["peak_device_bytes"] <= budget


def test_ooc_golden_corpus(golden):
    n_cfg = 0
    for k, c in golden.cases():
        if c["n"] == 0 or c["m"] == 0 or not c["name"].startswith(("corpus", "shared", "clique")):
            continue
        g = make_graph(c["n"], golden.edges(k))
        for j, cfg in enumerate(c["configs"][:6]):
            plan, r, s = _ooc(g, cfg["mu"], cfg["eps"], 1 << 24)
            np.testing.assert_array_equal(r.role_codes, golden.get(k, f"c{j}_roles"))
            np.testing.assert_array_equal(r.cluster_ids, golden.get(k, f"c{j}_cluster"))
            n_cfg += 1
    assert n_cfg > 100


def test_ooc_huge_lists_use_l2_table(orc):
    """Hubs of degree 40k exceed the shared-memory cuckoo: HBM slab path."""
    rng = np.random.default_rng(7)
    n = 70000
    edges = set()
    for h in (0, 1, 2):
        for v in rng.choice(np.arange(3, n), size=40000, replace=False):
            edges.add((h, int(v)))
    for _ in range(150000):
        u, v = rng.integers(3, n, size=2)
        if u != v:
            edges.add((int(min(u, v)), int(max(u, v))))
    edges |= {(0, 1), (1, 2), (0, 2)}
    e = np.array(sorted(edges), dtype=np.int32)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.05", 2), ("0.3", 2)):
        roles, cl = orc.serial_scan(c, mu, eps)
        plan, r, s = _ooc(g, mu, eps, 64 << 20)
        np.testing.assert_array_equal(r.role_codes, roles)
        np.testing.assert_array_equal(r.cluster_ids, cl)


def test_ooc_infeasible_budget():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    with pytest.raises(gs.InfeasibleBudgetError):
        gs.partition_graph(g, 13 * 14 - 1)
    with pytest.raises(ValueError):
        gs.partition_graph(g, 0)
    plan = gs.partition_graph(g, 1 << 24)
    other = make_graph(10, [(0, 1), (1, 2)])
    with pytest.raises(ValueError):
        gs.scan_out_of_core(gs.GraphMeta.from_graph(other), plan, 3, "0.5")


def _chunglu(logn, gamma, wmax, count, seed):
    import ctypes

    import torch

    from paper_2311_12281_b200 import _lib

    lib = _lib.load()
    src = torch.empty(count, dtype=torch.int32, device="cuda")
    dst = torch.empty(count, dtype=torch.int32, device="cuda")
    _lib.check(lib.gs_chunglu_generate(logn, gamma, wmax, count, seed, src.data_ptr(),
                                       dst.data_ptr(), None))
    uv = torch.empty(2 * count, dtype=torch.int32, device="cuda")
    m = ctypes.c_int64(0)
    _lib.check(lib.gs_normalize_edges(count, src.data_ptr(), dst.data_ptr(), uv.data_ptr(),
                                      ctypes.byref(m), None))
    torch.cuda.synchronize()
    return 1 << logn, uv[: 2 * m.value].cpu().numpy().reshape(-1, 2).copy()


@pytest.mark.parametrize("logn,wmax,seed", [(14, 3000, 1), (16, 20000, 2)])
def test_chunglu_against_oracle(orc, logn, wmax, seed):
    """BASELINE configs[2] shape at test size: power-law (gamma 2.1) degrees
    with a few vertices near wmax -> hub bitmap, L2 tables, early exits."""
    n, e = _chunglu(logn, 2.1, wmax, 12 << logn, seed)
    deg = np.bincount(e.ravel(), minlength=n)
    assert deg.max() > wmax // 4 and len(e) > 4 << logn
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    for eps, mu in (("0.1", 3), ("0.3", 5), ("0.5", 2), ("0.7", 4)):
        roles, cl = orc.serial_scan(c, mu, eps)
        r_roles, r_cl, _, s = run(g, mu, eps)
        np.testing.assert_array_equal(r_roles, roles, err_msg=f"{eps} {mu}")
        np.testing.assert_array_equal(r_cl, cl, err_msg=f"{eps} {mu}")
        assert s.sim_evals <= g.m and s.probe_bound_violations == 0
        dmax = int(deg.max())
        budget = 13 * n + (2 << 20) + 8 * (dmax + 1) + max(2 * g.m // 3 * 4, 8 * 4 * dmax)
        _, rr, ss = _ooc(g, mu, eps, budget)
        assert ss.extra["partitions"] >= 2
        np.testing.assert_array_equal(rr.role_codes, roles, err_msg=f"ooc {eps} {mu}")
        np.testing.assert_array_equal(rr.cluster_ids, cl, err_msg=f"ooc {eps} {mu}")


@pytest.mark.parametrize("k", ["4", "8", "16"])
def test_sketch_bound_forced_everywhere(orc, monkeypatch, k):
    """The neighbourhood-sketch bound (sketch.cu) tried on EVERY survivor,
    sketches for every degree, at each resolution: it may only ever prove
    dissimilarity, so roles and ids stay bit-exact with the oracle (R-MAT
    with hubs -> huge/large/medium/warp classes, and the skewed Chung-Lu)."""
    monkeypatch.setenv("GS_SKETCH", k)
    monkeypatch.setenv("GS_SKETCH_DMIN", "1")
    monkeypatch.setenv("GS_SKETCH_MINSCAN", "-1000000")
    monkeypatch.setenv("GS_SKETCH_GATE", "1e30")
    graphs = [orc.rmat(16, seed=3), _chunglu(15, 2.1, 20000, 12 << 15, 4)]
    for n, e in graphs:
        c = orc.CSR(n, e)
        g = make_graph(n, e)
        decided = 0
        for eps, mu in (("0.1", 3), ("0.2", 3), ("0.3", 5), ("0.5", 2), ("0.8", 2)):
            roles, cl = orc.serial_scan(c, mu, eps)
            r_roles, r_cl, _, s = run(g, mu, eps)
            np.testing.assert_array_equal(r_roles, roles, err_msg=f"k{k} {eps} {mu}")
            np.testing.assert_array_equal(r_cl, cl, err_msg=f"k{k} {eps} {mu}")
            decided += s.extra["sim_decided_by_sketch"]
        assert decided > 0


def test_sketch_default_is_on_and_exact(orc):
    n, e = orc.rmat(17, seed=5)
    c = orc.CSR(n, e)
    g = make_graph(n, e)
    roles, cl = orc.serial_scan(c, 5, "0.5")
    r_roles, r_cl, _, s = run(g, 5, "0.5")
    np.testing.assert_array_equal(r_roles, roles)
    np.testing.assert_array_equal(r_cl, cl)
    assert s.extra["sim_decided_by_sketch"] > 0


@pytest.mark.parametrize("k", ["4", "8"])
def test_ooc_sketch_bound_forced_everywhere(orc, monkeypatch, k):
    """Out-of-core sketches (rows in mapped pinned host memory, b's levels
    hashed from the streamed slice) tried on every survivor: bit-exact."""
    monkeypatch.setenv("GS_SKETCH", k)
    monkeypatch.setenv("GS_SKETCH_DMIN", "1")
    monkeypatch.setenv("GS_SKETCH_GATE", "1e30")
    for n, e in (orc.rmat(15, seed=6), _chunglu(14, 2.1, 3000, 12 << 14, 7)):
        c = orc.CSR(n, e)
        g = make_graph(n, e)
        dmax = int(np.diff(g.vertex_offsets).max())
        budget = 13 * n + (2 << 20) + 8 * (dmax + 1) + max(2 * g.m // 2 * 4 * 4 // 3, 8 * 4 * dmax)
        decided = 0
        for eps, mu in (("0.2", 3), ("0.5", 2), ("0.8", 2)):
            roles, cl = orc.serial_scan(c, mu, eps)
            plan, r, s = _ooc(g, mu, eps, budget)
            assert s.extra["partitions"] >= 2, s.extra
            np.testing.assert_array_equal(r.role_codes, roles, err_msg=f"k{k} {eps} {mu}")
            np.testing.assert_array_equal(r.cluster_ids, cl, err_msg=f"k{k} {eps} {mu}")
            assert s.extra["peak_device_bytes"] <= budget
            decided += s.extra["sim_decided_by_sketch"]
        assert decided > 0
