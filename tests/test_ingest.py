"""Native ingest: parse_edge_list (graph.py:63-118) through the
libgscan parser, and the GSCG binary cache (graph.py:279-359), against golden
outputs of the Python reference (tests/golden/make_parse_golden.py).

CPU tier: the native parser, normalised by the test's numpy checker; `-m gpu`:
the same inputs through the product's device normaliser (gs_normalize_sparse)."""

import base64
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, TWO_COMMUNITIES, cuda_ok, make_graph

import paper_2311_12281_b200 as gs
from paper_2311_12281_b200 import _lib


def _golden():
    with open(os.path.join(GOLDEN_DIR, "parse_golden.json")) as f:
        return json.load(f)


def _check_all():
    for case in _golden():
        data = base64.b64decode(case["input"])
        exp = case["expected"]
        if "error" in exp:
            with pytest.raises(gs.ParseError) as ei:
                gs.parse_edge_list(data)
            assert str(ei.value) == exp["error"] and ei.value.line == exp["line"]
            continue
        el = gs.parse_edge_list(data)
        assert el.n_hint == exp["n"]
        assert np.asarray(el.edges).reshape(-1, 2).tolist() == exp["edges"]
        assert np.asarray(el.orig_ids).tolist() == exp["orig_ids"]


def test_parse_matches_reference_cpu(host_normaliser):
    _check_all()


def test_native_parser_grammar():
    lib = _lib.load()
    data = b"1 2\r\n3\t4\n# x\n\n5 5\r6 7"
    u = np.empty(8, np.uint32)
    v = np.empty(8, np.uint32)
    import ctypes

    cnt, err = ctypes.c_int64(), ctypes.c_int64()
    assert lib.gs_parse_edge_text(data, len(data), 2, u.ctypes.data, v.ctypes.data, 8,
                                  ctypes.byref(cnt), ctypes.byref(err)) == 0
    assert list(zip(u[: cnt.value], v[: cnt.value])) == [(1, 2), (3, 4), (5, 5), (6, 7)]
    bad = b"1 2\n3 4\n5 x\n"
    assert lib.gs_parse_edge_text(bad, len(bad), 2, u.ctypes.data, v.ctypes.data, 8,
                                  ctypes.byref(cnt), ctypes.byref(err)) == _lib.GS_EPARSE
    assert err.value == 3


def test_parse_large_multichunk_matches_exact(host_normaliser):
    rng = np.random.default_rng(5)
    ids = rng.integers(0, 2**32, 5000, dtype=np.uint64)
    u = ids[rng.integers(0, 5000, 300_000)]
    v = ids[rng.integers(0, 5000, 300_000)]
    text = "\n".join(f"{a} {b}" for a, b in zip(u.tolist(), v.tolist())).encode()
    from paper_2311_12281_b200.graph import _parse_exact

    a, b = gs.parse_edge_list(text), _parse_exact(text)
    assert a.n_hint == b.n_hint
    np.testing.assert_array_equal(np.asarray(a.edges), np.asarray(b.edges))
    np.testing.assert_array_equal(np.asarray(a.orig_ids), np.asarray(b.orig_ids))


def test_normaliser_has_no_host_path(monkeypatch):
    """Without a device the product's normalisation raises (no CPU fallback)."""
    lib = _lib.load()
    if lib.gs_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    with pytest.raises(RuntimeError, match="needs a CUDA device"):
        gs.parse_edge_list("0 1\n1 2\n")
    with pytest.raises(gs.ParseError):  # parse errors still come first
        gs.parse_edge_list("0 1\nx\n")


def test_gscg_cache_byte_compatible(tmp_path):
    ref = os.path.join(GOLDEN_DIR, "ref_fig1.gscg")
    assert gs.is_graph_cache(ref) and not gs.is_graph_cache(os.path.join(GOLDEN_DIR, "golden.json"))
    g = gs.load_graph(ref)
    h = make_graph(14, sorted(TWO_COMMUNITIES))
    for k in ("vertex_offsets", "adjacency", "edge_ids", "edge_list"):
        np.testing.assert_array_equal(getattr(g, k), getattr(h, k))
    assert g.orig_ids.tolist() == [100 + 3 * i for i in range(14)]
    out = tmp_path / "x.gscg"
    gs.save_graph(g, str(out))
    assert out.read_bytes() == open(ref, "rb").read()


def test_gscg_cache_errors(tmp_path):
    raw = open(os.path.join(GOLDEN_DIR, "ref_fig1.gscg"), "rb").read()
    cases = {b"XXXX" + raw[4:]: "bad magic", raw[:10]: "truncated graph cache header",
             raw[:60]: "truncated graph cache", raw[:4] + b"\x02" + raw[5:]: "unsupported"}
    for i, (data, msg) in enumerate(cases.items()):
        p = tmp_path / f"c{i}"
        p.write_bytes(data)
        with pytest.raises(ValueError, match=msg):
            gs.load_graph(str(p))
    assert not gs.is_graph_cache(str(tmp_path / "missing"))


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="no CUDA device")
def test_parse_matches_reference_device_normaliser():
    assert _lib.load().gs_device_count() > 0
    _check_all()


def test_native_result_writer_matches_reference_format(tmp_path):
    """ClusteringResult.to_text via gs_format_result == scan.py:892-904's lines."""
    rng = np.random.default_rng(11)
    n = 200_003
    codes = rng.choice(np.array([1, 3, 4, 5, 6], np.uint8), n)
    cid = np.where(np.isin(codes, [1, 3, 4]), rng.integers(0, n, n), -1).astype(np.int32)
    orig = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    r = gs.ClusteringResult(n, codes, cid, orig)
    letter = {1: "C", 3: "M", 4: "M", 5: "H", 6: "O"}
    want = "".join(f"{orig[v]}\t{letter[int(codes[v])]}\t{orig[cid[v]] if cid[v] >= 0 else -1}\n"
                   for v in range(n))
    assert r.to_text() == want
    p = tmp_path / "r.txt"
    r.write(str(p))
    assert p.read_text() == want
    assert gs.ClusteringResult(0, codes[:0], cid[:0], orig[:0]).to_text() == ""
