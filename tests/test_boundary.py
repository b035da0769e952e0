"""CPU tests of the drop-in boundary: the C-ABI library loads and exports
every symbol include/gscan.h declares, and the host mirror keeps the
reference's validation, result and stats behaviour (no device calls)."""

import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, TWO_COMMUNITIES

HEADER = os.path.join(ROOT, "include", "gscan.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("gs_scan_csr", "gs_scan_edges", "gs_build_graph", "gs_scan_partitioned",
                     "gs_engine_create", "gs_engine_scan", "gs_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2311_12281_b200 import _lib

    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    bound = {s[0] for s in _lib.SIGNATURES}
    assert bound == set(declared_functions())
    assert lib.gs_version() == 3  # ABI 3: kernel_bytes[7] (+ the sketch filter class)
    assert isinstance(lib.gs_last_error(), bytes)


def test_library_is_sm100a_only():
    """The shipped .so carries sm_100a SASS (checked with cuobjdump)."""
    import shutil
    import subprocess

    from paper_2311_12281_b200 import _lib

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_epsilon_fraction_rules():
    from paper_2311_12281_b200 import epsilon_fraction

    assert epsilon_fraction("0.6") == Fraction(3, 5)
    assert epsilon_fraction("1") == 1
    assert epsilon_fraction(0.5) == Fraction(1, 2)
    assert epsilon_fraction(0.6) != Fraction(3, 5)
    for bad in ["0", "-0.1", "1.0001", "2", "abc", ""]:
        with pytest.raises(ValueError):
            epsilon_fraction(bad)
    with pytest.raises(TypeError):
        epsilon_fraction([0.5])


def test_eps2_struct_splits_128_bits():
    from paper_2311_12281_b200 import _lib

    e = _lib.eps2_struct(Fraction("0.6"))
    assert (e.p_lo, e.p_hi, e.q_lo, e.q_hi) == (9, 0, 25, 0)
    f = Fraction(0.6)  # binary value: q = 2^106 after squaring
    e = _lib.eps2_struct(f)
    p = e.p_lo | (e.p_hi << 64)
    q = e.q_lo | (e.q_hi << 64)
    assert Fraction(p, q) == f * f
    e = _lib.eps2_struct(Fraction("0.500000000000001"))
    assert Fraction(e.p_lo | (e.p_hi << 64), e.q_lo | (e.q_hi << 64)) == Fraction(
        "0.500000000000001") ** 2
    with pytest.raises(ValueError):
        _lib.eps2_struct(Fraction(10**40 + 1, 10**40 + 7))
    # an astronomically fine but tiny epsilon is equivalent to "all similar"
    e = _lib.eps2_struct(Fraction(1, 10**60), dmax=1000)
    assert e.p_lo == 1 and e.q_hi == 1 << 63


def test_exact_predicate_matches_fraction():
    """The 192-bit predicate of the C oracle (same arithmetic as the device
    header common.cuh) against exact Fractions on boundary cases."""
    from oracle import oracle as orc

    g = orc.CSR(14, sorted(TWO_COMMUNITIES))
    for eps in ["0.5", "0.500000000000001", str(0.6), "0.7905694150420949", "1"]:
        roles, cl = orc.serial_scan(g, 2, eps)
        assert len(roles) == 14


def test_result_types_mirror_reference():
    from paper_2311_12281_b200 import ClusteringResult, Role, StatsReport

    r = ClusteringResult(3, np.array([1, 1, 1], np.uint8), np.array([0, 0, 0], np.int32),
                         np.array([10, 20, 30], np.uint32))
    assert r.to_text().splitlines() == ["10\tC\t10", "20\tC\t10", "30\tC\t10"]
    assert r.core_set() == {0, 1, 2}
    assert r.core_equivalence() == {frozenset({0, 1, 2})}
    r.roles[1] = Role.HUB
    r.cluster_id[1] = -1
    assert r.hub_set() == {1}
    assert r.to_text().splitlines()[1] == "20\tH\t-1"
    s = StatsReport(n=14, m=23, workers=2, phases={"total": 5})
    text = s.to_text()
    for key in ("n=14", "m=23", "workers=2", "sim_evals=", "adj_probes=", "union_retries=",
                "probe_bound_violations=0", "phase_total_us="):
        assert key in text
    empty = ClusteringResult(0, np.empty(0, np.uint8), np.empty(0, np.int32),
                             np.empty(0, np.uint32))
    assert empty.to_text() == ""


def test_scan_validation_before_device():
    from oracle import oracle as orc
    from paper_2311_12281_b200 import scan_in_memory

    g = orc.CSR(14, sorted(TWO_COMMUNITIES))
    with pytest.raises(ValueError):
        scan_in_memory(g, 1, "0.5")
    with pytest.raises(ValueError):
        scan_in_memory(g, 3, "0.5", workers=0)
    with pytest.raises(ValueError):
        scan_in_memory(g, 3, "1.5")


def test_empty_graph_needs_no_device():
    from paper_2311_12281_b200 import EdgeList, build_graph, scan_in_memory

    g = build_graph(EdgeList(n_hint=0, edges=[]))
    result, stats = scan_in_memory(g, 2, "0.5")
    assert result.n == 0 and result.to_text() == "" and stats.sim_evals == 0


def test_parse_edge_list_rules(host_normaliser):
    from paper_2311_12281_b200 import ParseError, parse_edge_list

    el = parse_edge_list("# header\n\n0\t1\n  2 3\n\n  # c\n")
    assert el.edges.tolist() == [[0, 1], [2, 3]]
    el = parse_edge_list("0 1\n1 0\n0 1\n")
    assert el.edges.tolist() == [[0, 1]]
    el = parse_edge_list("5 5\n0 1\n")
    assert el.n_hint == 3 and list(el.orig_ids) == [0, 1, 5]
    el = parse_edge_list("100 7\n1000000 100\n")
    assert el.edges.tolist() == [[0, 1], [1, 2]] and list(el.orig_ids) == [7, 100, 1000000]
    with pytest.raises(ParseError) as ei:
        parse_edge_list("0 1\nnope\n")
    assert ei.value.line == 2
    with pytest.raises(ParseError):
        parse_edge_list("-1 4\n")


def test_product_package_never_imports_oracle():
    """The shipped path has no CPU fallback and never touches oracle/."""
    pkg = os.path.join(ROOT, "paper_2311_12281_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liborc" not in text, f


def test_stats_struct_matches_header():
    """The ctypes mirror of gs_stats lists the header's fields in order (a
    field added on one side only would shift every later counter)."""
    import re

    from paper_2311_12281_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "gscan.h")).read()
    body = re.search(r"typedef struct gs_stats \{(.*?)\} gs_stats;", hdr, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        decl = re.sub(r"\[.*?\]", "", decl)
        names += [v.strip() for v in decl.split(None, 1)[1].split(",")]
    assert names == [f[0] for f in _lib.GsStats._fields_]


def test_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the CPU port of the reference's hot loop the
    driver times beside the engine) prints one JSON line, no GPU needed."""
    import json
    import subprocess
    import sys

    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--scale", "11", "--steps", "1", "--warmup", "3", "--cpu-seconds", "0.5"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "edges/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
