"""A non-GA check of the GPU search's best makespans (CPU only): the paper's MILP (Eqs. 1-11,
oracle/milp.py) solved by HiGHS with the objective cut at `best - 1` -- "is there a plan
strictly better than the GA's?".  Runtimes and starts are integers (reading A4), so a
better plan has C <= best - 1.  Outcomes per seed:
  infeasible   HiGHS proves no better plan exists: the GA's best is optimal;
  found        HiGHS found a better plan (its makespan is reported);
  open         the time limit expired without either (the configuration-LP bound O5b then
               states the remaining gap).
scipy's HiGHS interface takes no starting solution; the cut is the way the GA incumbent
enters the solve.

    python tools/quality_cutoff.py --workload TXT --seeds 0 1 2 --best 51265 52024 50987 \
        --seconds 300 --out profiles/r2/quality_cutoff_TXT.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle.milp import SpaseMilp  # noqa: E402
from scipy.optimize import Bounds, LinearConstraint, milp  # noqa: E402


def run(args):
    workload, seed, best, seconds = args
    inst = synth.by_name(workload, seed)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    m = SpaseMilp(c)
    ub = np.array(m.bounds.ub, dtype=float)
    ub[m.idx[("C",)]] = best - 1
    t0 = time.time()
    res = milp(m.obj, constraints=LinearConstraint(m.A, m.lo, m.hi), integrality=m.kinds,
               bounds=Bounds(m.bounds.lb, ub), options={"time_limit": seconds, "mip_rel_gap": 0.0, "disp": False})
    wall = time.time() - t0
    out = {"workload": workload, "table_seed": seed, "gpu_best": best, "cut": best - 1, "seconds": seconds,
           "wall_s": round(wall, 1), "highs_status": int(res.status), "highs_message": str(res.message)}
    if res.status == 2:
        out["outcome"] = "infeasible"      # no plan with C <= best - 1: best is optimal
    elif res.x is not None:
        plan = m.solution_to_plan(res.x)
        ms = int(round(res.fun))
        out.update(outcome="found", makespan=ms, validator=oracle.validate(c, plan, ms) if plan else None)
    else:
        out["outcome"] = "open"
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="TXT")
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--best", type=int, nargs="+", required=True)
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    assert len(a.best) == len(a.seeds)
    with Pool(len(a.seeds)) as pool:
        rows = pool.map(run, [(a.workload, s, b, a.seconds) for s, b in zip(a.seeds, a.best)])
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"method": "paper MILP (oracle/milp.py) under HiGHS (scipy) with C <= gpu_best - 1",
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
