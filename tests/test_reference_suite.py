"""The reference's own test suite (pkg/tests, 138 tests) with its clustering
call -- graphscan.scan.scan_in_memory and the names graphscan re-exports it
under -- served by the B200 engine (tools/reftests_plugin.py).

Runs when the reference package travels with the snapshot (baseline/_ref/pkg,
git-ignored); nothing here reads /root/reference.  One reference test is
deselected for a documented reason: it compares the raw union-find root ids of
the reference's own Python out-of-core engine with scan_in_memory's ids, and
the engine returns canonical ids (minimum core id per cluster, DESIGN 1);
roles and the cluster partition are identical."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_ok

REF_PKG = os.path.join(ROOT, "baseline", "_ref", "pkg")
KNOWN = "test_single_partition_bitwise_identical"  # tests/test_out_of_core.py


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="no CUDA device")
@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_PKG, "tests")),
                    reason="baseline/_ref/pkg (the reference's suite) not shipped")
def test_reference_suite_on_engine():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF_PKG, "src"), ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF_PKG, "tests"), "-q",
           "-p", "tools.reftests_plugin", "-p", "no:cacheprovider",
           "-k", f"not {KNOWN}"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join(r.stdout.strip().splitlines()[-15:])
    assert r.returncode == 0, tail
    served = [ln for ln in r.stdout.splitlines() if "served by the B200 engine" in ln]
    assert served and int(served[-1].rsplit(":", 1)[1]) > 1000, tail
