"""Golden vectors for HistoPipe planning by running the REFERENCE scheduler (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scheduler_golden.py

Writes tests/golden/scheduler.json: random ProfileCostModel grids with tau queries, plan_allocation cases
(profile and analytic cost models), beta_from_history and migration_decision cases, each with the
reference's output (rhymesim/scheduler.py:97-330).  The GPU box never runs this script.
"""

import json
import os
import random

from rhymesim import scheduler as R


def main():
    rnd = random.Random(20241019)
    out = {"tau": [], "plans": [], "beta": [], "migration": []}
    for _ in range(40):
        ls = sorted(rnd.sample(range(256, 20000, 128), rnd.randint(2, 5)))
        ks = sorted(rnd.sample(range(1, 9), rnd.randint(1, 4)))
        sec = [[round(l / 1000.0 * (1.0 + rnd.random()) / (k ** rnd.uniform(0.5, 1.0)), 4) for k in ks] for l in ls]
        acc = rnd.choice([0.0, 0.5, 2.3])
        m = R.ProfileCostModel(lengths=[float(x) for x in ls], workers=ks, seconds=sec, accepted_per_pass=acc)
        qs = [(rnd.uniform(0, 22000), rnd.randint(1, 10)) for _ in range(12)]
        out["tau"].append({"lengths": ls, "workers": ks, "seconds": sec, "acc": acc,
                           "queries": [[l, k, m.tau(l, k)] for l, k in qs]})
        n = rnd.randint(2, 6)
        lens = sorted(rnd.uniform(300, 18000) for _ in range(n))
        wks = rnd.randint(n, 3 * n + 2)
        t_train = rnd.choice([0.0, 1.0, 5.0])
        prec = rnd.choice([1.0, 0.1, 0.01])
        p = R.plan_allocation(lens, wks, t_train, m, precision=prec)
        out["plans"].append({"model": "profile", "grid": len(out["tau"]) - 1, "lens": lens, "wks": wks,
                             "t_train": t_train, "precision": prec, "plan": p.per_group_workers,
                             "d": p.gradient_d, "t0": p.t0, "feasible": p.feasible})
    for _ in range(30):
        a = R.AnalyticCostModel(per_iter_base=rnd.uniform(0.005, 0.05), per_iter_batch=rnd.uniform(1e-5, 1e-3),
                                fixed=rnd.uniform(0, 2), batch_size=rnd.randint(1, 512),
                                accepted_per_pass=rnd.uniform(0, 3))
        n = rnd.randint(2, 6)
        lens = sorted(rnd.uniform(300, 18000) for _ in range(n))
        wks = rnd.randint(n - 1, 3 * n)
        t_train, min_wks, prec = rnd.uniform(0, 3), rnd.choice([1, 1, 2]), rnd.choice([1.0, 0.05])
        p = R.plan_allocation(lens, wks, t_train, a, min_wks=min_wks, precision=prec)
        out["plans"].append({"model": "analytic", "params": [a.per_iter_base, a.per_iter_batch, a.fixed,
                                                             a.batch_size, a.accepted_per_pass],
                             "lens": lens, "wks": wks, "t_train": t_train, "min_wks": min_wks, "precision": prec,
                             "plan": p.per_group_workers, "d": p.gradient_d, "t0": p.t0, "feasible": p.feasible})
    for _ in range(20):
        rates = [rnd.uniform(0.5, 3.0) for _ in range(rnd.randint(0, 9))]
        out["beta"].append([rates, R.beta_from_history(rates)])
    for _ in range(200):
        ng = rnd.randint(2, 8)
        g = R.RankingGroup(index=rnd.randrange(ng), prompt_ids=[], representative_len=1.0,
                           max_hist_len=rnd.uniform(100, 5000))
        total = rnd.randint(1, 100)
        completed = rnd.randint(0, total)
        pol = R.MigrationPolicy(alpha_pct=rnd.choice([5.0, 10.0, 30.0]), beta=rnd.choice([1.0, 1.1, 1.5]))
        loads = {i: rnd.uniform(0, 10) for i in rnd.sample(range(ng), rnd.randint(0, ng))}
        gen = rnd.randint(0, 8000)
        d = R.migration_decision(g, gen, completed, total, pol, ng, loads)
        out["migration"].append({"group": g.index, "max_hist": g.max_hist_len, "gen": gen, "completed": completed,
                                 "total": total, "alpha": pol.alpha_pct, "beta": pol.beta, "n_groups": ng,
                                 "loads": [[k, v] for k, v in loads.items()], "kind": d.kind,
                                 "target": d.target_group})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scheduler.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path, {k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
