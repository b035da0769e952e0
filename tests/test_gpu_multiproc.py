"""The sharded scan through real torch.distributed processes (torchrun):
dist.ShardedScan's partitioned build, row-slice broadcast and phase
exchanges, each rank a separate process.  On a one-GPU box the ranks share
the device over gloo (GS_DIST_BACKEND=gloo); the collectives are the same
calls the NCCL path makes.  Results must equal the single-engine scan and
the CPU oracle (tools/mp_shard_check.py)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_ok

pytestmark = pytest.mark.gpu

if not cuda_ok():
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("world,port", [(2, 29641), (3, 29643)])
def test_torchrun_sharded_matches_single_gpu_and_oracle(tmp_path, world, port):
    out = tmp_path / "mp.json"
    env = dict(os.environ, GS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "mp_shard_check.py"), "14", "3", str(out)]
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    s = json.loads(out.read_text())
    assert s["world"] == world and s["all_ranks_ok"]
    assert len(s["configs"]) == 8
    assert any(c["cores"] > 0 and c["clusters"] > 1 for c in s["configs"])
    assert all(c["equal_single_gpu"] and c["equal_oracle"] for c in s["configs"])
