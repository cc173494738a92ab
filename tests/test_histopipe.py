"""HistoPipe planning (workers.TauProfile / plan_allocation / beta_from_history / migration_decision) against
golden vectors produced by running the reference scheduler (tests/golden/make_scheduler_golden.py;
rhymesim/scheduler.py:97-330), plus assignment of planned workers to ranks."""

import math

import pytest

from paper_2508_18588_b200 import workers as W


class _Analytic:
    """The reference's AnalyticCostModel formula (scheduler.py:97-117), test-side only."""

    def __init__(self, base, batch, fixed, bsz, acc):
        self.p = (base, batch, fixed, bsz, acc)

    def tau(self, length, k):
        base, batch, fixed, bsz, acc = self.p
        return length * (base + batch * math.ceil(bsz / k)) / (1.0 + acc) + fixed


def test_tau_profile_matches_reference(golden):
    for case in golden("scheduler.json")["tau"]:
        m = W.TauProfile([float(x) for x in case["lengths"]], case["workers"], case["seconds"], case["acc"])
        for l, k, t in case["queries"]:
            assert m.tau(l, k) == pytest.approx(t, rel=1e-12, abs=1e-12)


def test_plan_allocation_matches_reference(golden):
    g = golden("scheduler.json")
    for case in g["plans"]:
        if case["model"] == "profile":
            t = g["tau"][case["grid"]]
            m = W.TauProfile([float(x) for x in t["lengths"]], t["workers"], t["seconds"], t["acc"])
            p = W.plan_allocation(case["lens"], case["wks"], case["t_train"], m, precision=case["precision"])
        else:
            continue
        assert p.feasible == case["feasible"]
        assert p.per_group_workers == case["plan"]
        assert p.gradient_d == pytest.approx(case["d"]) and p.t0 == pytest.approx(case["t0"])


def test_plan_allocation_analytic_matches_reference(golden):
    for case in golden("scheduler.json")["plans"]:
        if case["model"] != "analytic":
            continue
        p = W.plan_allocation(case["lens"], case["wks"], case["t_train"], _Analytic(*case["params"]),
                              min_wks=case["min_wks"], precision=case["precision"])
        assert p.feasible == case["feasible"]
        assert p.per_group_workers == case["plan"]
        assert p.gradient_d == pytest.approx(case["d"]) and p.t0 == pytest.approx(case["t0"])


def test_beta_and_migration_match_reference(golden):
    g = golden("scheduler.json")
    for rates, beta in g["beta"]:
        assert W.beta_from_history(rates) == beta
    for c in g["migration"]:
        pol = W.MigrationPolicy(alpha_pct=c["alpha"], beta=c["beta"])
        kind, target = W.migration_decision(c["group"], c["max_hist"], c["gen"], c["completed"], c["total"], pol,
                                            c["n_groups"], {k: v for k, v in c["loads"]})
        assert (kind, target) == (c["kind"], c["target"])


def test_plan_errors_and_tau_csv(tmp_path):
    m = W.TauProfile.from_rows([(512, 1, 1.0), (512, 2, 0.6), (4096, 1, 8.0), (4096, 2, 4.5)])
    with pytest.raises(ValueError):
        W.plan_allocation([100.0], 4, 0.0, m)
    with pytest.raises(ValueError):
        W.plan_allocation([200.0, 100.0], 4, 0.0, m)
    with pytest.raises(ValueError):
        W.TauProfile.from_rows([(512, 1, 1.0), (4096, 2, 4.5)])
    assert not W.plan_allocation([100.0, 200.0, 300.0], 2, 0.0, m).feasible
    p = tmp_path / "tau.csv"
    m.to_csv(p)
    m2 = W.TauProfile.from_csv(p)
    assert m2.tau(1000, 2) == pytest.approx(m.tau(1000, 2))
    plan = W.plan_allocation([512.0, 4096.0], 4, 0.0, m, precision=0.01)
    assert plan.feasible and sum(plan.per_group_workers) <= 4


def test_assign_with_plan_alternates_and_covers():
    med = {i: float(100 + 13 * i) for i in range(20)}
    groups = W.build_groups(med, 3)
    a1 = W.assign_with_plan(groups, [1, 1, 2], 1)
    a2 = W.assign_with_plan(groups, [1, 1, 2], 2)
    for a in (a1, a2):
        assert sorted(p for v in a.values() for p in v) == sorted(med)
        assert len(a) == 4
    assert a1[0] == groups[0].prompt_ids and a2[0] == groups[2].prompt_ids[0::2]


def test_plan_makespan_balances_groups():
    m = W.TauProfile.from_rows([(l, k, l / 1000 / k) for l in (512, 2048, 8192, 16384) for k in (1, 2, 3, 4)])
    p = W.plan_makespan([1500.0, 6000.0], 4, m)
    assert p.feasible and p.per_group_workers == [1, 3]
    assert max(m.tau(l, k) for l, k in zip([1500.0, 6000.0], p.per_group_workers)) == pytest.approx(2.0)
    # the reference's gradient plan gives the short group the workers (its training overlaps the long tail)
    assert W.plan_allocation([1500.0, 6000.0], 4, 0.0, m, precision=0.01).per_group_workers == [3, 1]
    assert not W.plan_makespan([1.0, 2.0, 3.0], 2, m).feasible


def test_plan_routes_layout_and_errors():
    """Host side of device routing: send order (destination, prompt, input order), per-destination counts and
    token totals, and offsets into the flat send buffer."""
    import numpy as np
    plan = W.plan_routes([5, 2, 5, 9, 2], [3, 4, 5, 6, 7], {2: 1, 5: 0, 9: 1}, 2)
    assert plan.order.tolist() == [0, 2, 1, 4, 3]
    assert plan.counts.tolist() == [2, 3] and plan.tok_counts.tolist() == [8, 17]
    assert plan.dst_off.tolist() == [0, 3, 8, 12, 19]
    empty = W.plan_routes([], [], {}, 3)
    assert empty.counts.tolist() == [0, 0, 0] and len(empty.order) == 0
    with pytest.raises(ValueError):
        W.plan_routes([1], [4], {1: 3}, 2)
    assert np.array_equal(W.plan_routes([7], [1], {7: 0}, 1).dst_off, [0])
