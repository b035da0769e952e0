"""Host side of the out-of-core mode (partition.py:70-333 restated as a
streaming plan): the reference's memory formula, the plan's slices and the
infeasible-budget error.  CPU only; the device run is in test_gpu_parity.py."""

import numpy as np
import pytest

from conftest import TWO_COMMUNITIES, make_graph

import paper_2311_12281_b200 as gs
from paper_2311_12281_b200.partition import VERTEX_STATE_BYTES


def test_estimate_memory_formula():
    assert gs.estimate_memory(make_graph(0, np.empty((0, 2), np.int32))) == 0
    assert gs.estimate_memory(make_graph(2, [(0, 1)])) == 33
    assert gs.estimate_memory(make_graph(3, [(0, 1), (0, 2), (1, 2)])) == 87


def test_plan_slices_cover_the_graph_in_order():
    rng = np.random.default_rng(3)
    n = 2000
    e = {tuple(sorted(map(int, rng.choice(n, 2, replace=False)))) for _ in range(9000)}
    g = make_graph(n, sorted(e))
    dmax = int(np.diff(g.vertex_offsets).max())
    budget = 15 * n + (2 << 20) + 8 * (dmax + 1) + 64 * 1024
    plan = gs.partition_graph(g, budget)  # gs_plan_partitions: host only, no device
    assert len(plan.partitions) >= 2
    lo = 0
    for p in plan.partitions:
        assert p.lo == lo and p.hi > p.lo
        assert p.a0 == g.vertex_offsets[p.lo] and p.a1 == g.vertex_offsets[p.hi]
        lo = p.hi
    assert lo == n
    text = plan.manifest()
    assert text.startswith(f"n={n}\nm={g.m}\nbudget_bytes={budget}\n")
    assert len(text.splitlines()) == 5 + len(plan.partitions)


def test_infeasible_budgets():
    g = make_graph(14, sorted(TWO_COMMUNITIES))
    with pytest.raises(gs.InfeasibleBudgetError) as ei:
        gs.partition_graph(g, 100)
    assert isinstance(ei.value, ValueError) and ei.value.budget_bytes == 100
    with pytest.raises(ValueError):
        gs.partition_graph(g, 0)


def test_plan_is_validated_before_any_device_work():
    """scan_out_of_core executes the caller's plan (partition.py:666-757); a
    partition that cannot fit the cap is rejected with InfeasibleBudgetError
    and a malformed plan with ValueError -- both before the device is touched,
    so this runs on CPU."""
    rng = np.random.default_rng(5)
    n = 3000
    e = {tuple(sorted(map(int, rng.choice(n, 2, replace=False)))) for _ in range(12000)}
    g = make_graph(n, sorted(e))
    dmax = int(np.diff(g.vertex_offsets).max())
    budget = 15 * n + (2 << 20) + 8 * (dmax + 1) + 64 * 1024
    plan = gs.partition_graph(g, budget)
    assert len(plan.partitions) >= 3
    meta = gs.GraphMeta.from_graph(g)
    whole = gs.partition.StreamSlice(0, 0, n, 0, 2 * g.m)  # one slice: too big for the cap
    bad = gs.PartitionPlan(n=n, m=g.m, budget_bytes=budget, partitions=[whole], graph=g)
    with pytest.raises(gs.InfeasibleBudgetError, match="partition 0"):
        gs.scan_out_of_core(meta, bad, 3, "0.5")
    gap = gs.PartitionPlan(n=n, m=g.m, budget_bytes=budget,
                           partitions=[plan.partitions[1]], graph=g)  # does not start at 0
    with pytest.raises(ValueError):
        gs.scan_out_of_core(meta, gap, 3, "0.5")
