"""Multi-process sharded scan check: the real torch.distributed path of
dist.ShardedScan (partitioned build, row-slice broadcast, the three phase
exchanges), one process per rank.

    GS_DIST_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29611 tools/mp_shard_check.py 15 2 out.json

On a box with one GPU the ranks share the device and talk over gloo (NCCL
refuses two ranks on one GPU); with NCCL and one GPU per rank it is the
production path.  Every rank compares its result with the single-engine
scan_in_memory of the same graph; rank 0 also compares with the CPU oracle
(test infrastructure) and writes a JSON summary.  Exit code 1 on mismatch.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    scale, seed, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    backend = os.environ.get("GS_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()

    import paper_2311_12281_b200 as gs
    from paper_2311_12281_b200 import _lib
    from paper_2311_12281_b200.dist import ShardedScan
    from conftest import make_graph
    from oracle import oracle as orc

    orc.load()
    n, e = orc.rmat(scale, seed=seed)
    g = make_graph(n, e)
    eng = _lib.Engine(device=local)
    shard = ShardedScan(eng, g.n)
    summary = {"world": world, "backend": backend, "n": g.n, "m": g.m, "configs": []}
    ok = True
    csr = orc.CSR(n, e) if rank == 0 else None
    for on_device in (0, 1):
        if on_device:
            off_d = torch.from_numpy(np.asarray(g.vertex_offsets)).cuda()
            adj_d = torch.from_numpy(np.asarray(g.adjacency)).cuda()
            shard.load_csr(g.m, off_d.data_ptr(), adj_d.data_ptr(), 1)
        else:
            shard.load_csr(g.m, g.vertex_offsets.ctypes.data, g.adjacency.ctypes.data, 0)
        for eps, mu in (("0.2", 3), ("0.3", 5), ("0.5", 5), ("0.25", 2)):
            eps2 = _lib.eps2_struct(gs.epsilon_fraction(eps))
            roles = np.empty(g.n, np.uint8)
            cl = np.empty(g.n, np.int32)
            st = shard.run(mu, eps2, roles.ctypes.data, cl.ctypes.data, 0)
            ref, _ = gs.scan_in_memory(g, mu, eps)
            same = bool(np.array_equal(roles, ref.role_codes)
                        and np.array_equal(cl, ref.cluster_ids))
            cfg = {"eps": eps, "mu": mu, "input_on_device": on_device,
                   "equal_single_gpu": same, "sim_evals_all_ranks": int(st.sim_evals),
                   "cores": int((roles == 1).sum()),
                   "clusters": int(len(np.unique(cl[roles == 1])))}
            if rank == 0:
                o_roles, o_cl = orc.serial_scan(csr, mu, eps)
                cfg["equal_oracle"] = bool(np.array_equal(roles, o_roles)
                                           and np.array_equal(cl, o_cl))
                same = same and cfg["equal_oracle"]
            ok = ok and same
            summary["configs"].append(cfg)
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                        device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    summary["all_ranks_ok"] = bool(flag.item())
    if rank == 0:
        with open(out, "w") as f:
            json.dump(summary, f, indent=1)
        print(json.dumps(summary))
    eng.close()
    dist.destroy_process_group()
    sys.exit(0 if summary["all_ranks_ok"] else 1)


if __name__ == "__main__":
    main()
