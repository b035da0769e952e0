"""Front ends wired to the device engine: the CLI
(graphscan/cli.py) and the StructuralClustering estimator
(graphscan/estimator.py), restating the reference's test_cli.py /
test_estimator.py cases.  Argument validation runs on CPU; runs that cluster
need the B200 (`-m gpu`)."""

import numpy as np
import pytest
from scipy import sparse
from sklearn.base import clone

from conftest import TWO_COMMUNITIES, cuda_ok, make_graph

import paper_2311_12281_b200 as gs
import paper_2311_12281_b200.cli as cli

need_cuda = pytest.mark.skipif(not cuda_ok(), reason="no CUDA device")


@pytest.fixture
def fixture_file(tmp_path):
    p = tmp_path / "g.txt"
    p.write_text("# two communities\n" + "\n".join(f"{u} {v}" for u, v in TWO_COMMUNITIES) + "\n")
    return str(p)


@pytest.fixture
def edge_array():
    return np.array(TWO_COMMUNITIES, dtype=np.int64)


# ---------------------------------------------------------------- CPU tier


def test_cli_argument_errors_exit_1(fixture_file, tmp_path, capsys):
    with pytest.raises(SystemExit) as ei:
        cli.main(["--input", fixture_file, "--epsilon", "0.6"])
    assert ei.value.code == 1
    assert cli.main(["--input", str(tmp_path / "nope"), "--epsilon", "0.6", "--mu", "3"]) == 1
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3",
                     "--mode", "outofcore"]) == 1
    assert "--budget" in capsys.readouterr().err
    bad = tmp_path / "bad.txt"
    bad.write_text("0 1\nx y\n")
    assert cli.main(["--input", str(bad), "--epsilon", "0.6", "--mu", "3"]) == 1
    assert "line 2" in capsys.readouterr().err
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3",
                     "--workers", "0"]) == 1


def test_devices_argument_errors(fixture_file, monkeypatch, capsys):
    """--devices N never falls back to fewer GPUs: without N visible devices
    it is an input error (exit 1); out-of-core is single-GPU."""
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setenv("GS_DIST_BACKEND", "nccl")
    import torch

    want = max(2, torch.cuda.device_count() + 1)
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3",
                     "--devices", str(want)]) == 1
    assert f"needs {want} visible GPUs" in capsys.readouterr().err
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3",
                     "--devices", "0"]) == 1
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--devices",
                     "2", "--mode", "outofcore", "--budget", "100000"]) == 1
    est = gs.StructuralClustering(devices=0)
    with pytest.raises(ValueError):
        est.fit(np.array([[0, 1]]))


def test_estimator_protocol_and_validation(edge_array):
    est = gs.StructuralClustering(epsilon="0.7", mu=4, workers=2)
    params = est.get_params()
    assert params["epsilon"] == "0.7" and params["mu"] == 4
    est2 = clone(est)
    assert est2.get_params() == params
    est2.set_params(mu=2)
    assert est2.mu == 2
    for bad in (dict(mu=1), dict(workers=0)):
        with pytest.raises(ValueError):
            gs.StructuralClustering(**bad).fit(edge_array)
    with pytest.raises(ValueError):
        gs.StructuralClustering().fit(np.zeros((3, 5)))
    with pytest.raises(ValueError):
        gs.StructuralClustering(input_type="edges").fit(np.array([[0, 1, 2]]))
    with pytest.raises(ValueError):
        gs.StructuralClustering(input_type="adjacency").fit(np.zeros((3, 4)))


def test_estimator_input_normalisation():
    from paper_2311_12281_b200.estimator import _edges_from_adjacency, _edges_from_pairs

    e = _edges_from_pairs(np.array([[3, 1], [1, 3], [2, 2], [0, 1]]))
    assert e.n_hint == 4 and e.edges.tolist() == [[0, 1], [1, 3]]
    d = np.zeros((5, 5), int)
    d[4, 1] = d[0, 2] = d[3, 3] = 1
    a = _edges_from_adjacency(sparse.csr_matrix(d))
    assert a.n_hint == 5 and a.edges.tolist() == [[0, 2], [1, 4]]


# ---------------------------------------------------------------- GPU tier


@pytest.mark.gpu
@need_cuda
def test_cli_runs(fixture_file, tmp_path, capsys):
    out = tmp_path / "out.txt"
    st = tmp_path / "stats.txt"
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--output",
                     str(out), "--stats", str(st)]) == 0
    lines = out.read_text().splitlines()
    assert len(lines) == 14 and lines[8] == "8\tH\t-1" and lines[3] == "3\tO\t-1"
    assert {ln.split("\t")[1] for ln in lines} == {"C", "M", "H", "O"}
    assert "sim_evals=" in st.read_text() and "m=23" in st.read_text()
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3"]) == 0
    assert "8\tH\t-1" in capsys.readouterr().out
    # byte-identical runs; cache input equals text input
    cache = tmp_path / "g.gscg"
    gs.save_graph(make_graph(14, sorted(TWO_COMMUNITIES)), str(cache))
    o2 = tmp_path / "o2.txt"
    assert cli.main(["--input", str(cache), "--epsilon", "0.6", "--mu", "3", "--deterministic",
                     "--workers", "8", "--output", str(o2)]) == 0
    assert o2.read_bytes() == out.read_bytes()
    # out-of-core mode (budget = HBM cap) gives the same output
    o3 = tmp_path / "o3.txt"
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--mode",
                     "outofcore", "--budget", str(64 << 20), "--output", str(o3)]) == 0
    assert o3.read_bytes() == out.read_bytes()
    # --spill-dir: the reference's partition files and manifest are written too
    sd = tmp_path / "spill"
    o4 = tmp_path / "o4.txt"
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--mode",
                     "outofcore", "--budget", str(64 << 20), "--spill-dir", str(sd),
                     "--output", str(o4)]) == 0
    assert o4.read_bytes() == out.read_bytes()
    man = (sd / "plan.manifest").read_text().splitlines()
    assert man[:2] == ["n=14", "m=23"] and man[3] == "global_state_bytes=210"
    assert man[4] == "partitions=1" and man[5].split("\t")[1] == "part-00000.bin"
    assert (sd / "part-00000.bin").read_bytes()[:4] == b"GSCP"
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--mode",
                     "outofcore", "--budget", "250"]) == 3
    assert "bytes" in capsys.readouterr().err


@pytest.mark.gpu
@need_cuda
def test_cli_verify_paths(fixture_file, monkeypatch, capsys):

    class Rep:
        def __init__(self, ok, detail=""):
            self.ok, self.detail = ok, detail

        def __bool__(self):
            return self.ok

    def judge(ok):
        return lambda: (lambda g, mu, eps: None, lambda mine, want: Rep(ok, "forced mismatch"),
                        lambda g, r: (g, r))

    monkeypatch.setattr(cli, "_reference_oracle", judge(True))
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--verify"]) == 0
    monkeypatch.setattr(cli, "_reference_oracle", judge(False))
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3", "--verify"]) == 2
    assert "forced mismatch" in capsys.readouterr().err


@pytest.mark.gpu
@need_cuda
def test_estimator_fits(edge_array, tmp_path):
    est = gs.StructuralClustering(epsilon="0.6", mu=3).fit(edge_array)
    assert est.labels_.shape == (14,) and set(est.labels_) == {-1, 0, 1}
    assert list(est.core_sample_indices_) == [0, 1, 4, 7, 9, 10, 11, 12, 13]
    assert "".join(est.roles_) == "CCMOCOOCHCCCCC"
    assert est.labels_[0] == 0 and est.labels_[9] == 1 and est.labels_[8] == -1
    assert est.stats_.sim_evals <= 23
    assert (est.fit_predict(edge_array) == est.labels_).all()
    n = 14
    dense = np.zeros((n, n), dtype=int)
    for u, v in TWO_COMMUNITIES:
        dense[u, v] = dense[v, u] = 1
    ref = est.labels_
    for x, kw in ((dense, {}), (sparse.csr_matrix(dense), {}), (dense, {"input_type": "adjacency"})):
        assert (gs.StructuralClustering(epsilon="0.6", mu=3, **kw).fit(x).labels_ == ref).all()
    txt = tmp_path / "g.txt"
    txt.write_text("\n".join(f"{u} {v}" for u, v in TWO_COMMUNITIES) + "\n")
    cache = tmp_path / "g.bin"
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    gs.save_graph(g, str(cache))
    for x in (g, str(txt), str(cache)):
        assert (gs.StructuralClustering(epsilon="0.6", mu=3).fit(x).labels_ == ref).all()
    ooc = gs.StructuralClustering(epsilon="0.6", mu=3, mode="outofcore",
                                  budget_bytes=64 << 20).fit(edge_array)
    assert (ooc.labels_ == ref).all()
    noise = gs.StructuralClustering(epsilon="0.99", mu=5).fit(np.array([(0, 1), (1, 2)]))
    assert (noise.labels_ == -1).all() and len(noise.core_sample_indices_) == 0


@pytest.mark.gpu
@need_cuda
def test_cli_devices_2_matches_single_gpu(fixture_file, tmp_path):
    """--devices 2: the CLI re-launches itself as two ranks (torchrun) running
    dist.scan_sharded; rank 0's output equals the one-GPU run byte for byte.
    On a one-GPU box the ranks share the device over gloo (the NCCL path's
    calls, a functional check)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    one = tmp_path / "one.txt"
    two = tmp_path / "two.txt"
    assert cli.main(["--input", fixture_file, "--epsilon", "0.6", "--mu", "3",
                     "--output", str(one)]) == 0
    env = dict(os.environ, GS_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, "-m", "paper_2311_12281_b200", "--input", fixture_file,
                        "--epsilon", "0.6", "--mu", "3", "--devices", "2", "--output", str(two)],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert two.read_bytes() == one.read_bytes()
