"""The collective helpers of dist.py on CPU: world_size 2 over gloo
(127.0.0.1), the same code paths NCCL runs on the B200 box."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_12281_b200 import _lib
        from paper_2311_12281_b200.dist import (all_gather_varlen, all_ok, exchange_row_slices,
                                                reduce_stats)

        # variable-length all-gather of (core, root) pairs, rank order kept
        k = 3 if rank == 0 else 5
        t = torch.full((8, 2), -1, dtype=torch.int32)
        t[:k, 0] = torch.arange(k, dtype=torch.int32) + 100 * rank
        t[:k, 1] = rank
        out = all_gather_varlen(t, k)
        # counts all-reduce as dist.ShardedScan does it
        c = torch.tensor([rank + 1, 10 * rank], dtype=torch.int32)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        lab = torch.tensor([5 - rank, rank], dtype=torch.int32)
        dist.all_reduce(lab[:1], op=dist.ReduceOp.MIN)
        dist.all_reduce(lab[1:], op=dist.ReduceOp.MAX)
        st = _lib.GsStats()
        st.sim_evals = 10 + rank
        st.phase_ms[2] = 1.0 + rank
        reduce_stats(st)
        # partitioned build: part k of the adjacency lives on rank k only
        bounds = [0, 7, 12]
        buf = torch.full((12,), -1, dtype=torch.int32)
        buf[bounds[rank]:bounds[rank + 1]] = torch.arange(bounds[rank], bounds[rank + 1],
                                                          dtype=torch.int32)
        exchange_row_slices(buf, bounds)
        oks = (all_ok(0, "cpu"), all_ok(_lib.GS_EINVAL if rank == 1 else 0, "cpu"))
        q.put((rank, out.tolist(), c.tolist(), lab.tolist(), st.sim_evals, st.phase_ms[2],
               buf.tolist(), oks))
    finally:
        dist.destroy_process_group()


def test_collectives_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, c, lab, evals, ph, buf, oks in res:
        assert out == [[0, 0], [1, 0], [2, 0], [100, 1], [101, 1], [102, 1], [103, 1], [104, 1]]
        assert c == [3, 10]
        assert lab == [4, 1]
        assert evals == 21 and ph == 2.0
        assert buf == list(range(12))
        assert oks == (True, False)
