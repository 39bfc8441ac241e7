"""Row f1 study: round introspection at the paper's knobs (interval
1000 s, threshold 500 s) on the synthetic workloads, with the GPU search as
the per-round solver, against the one-shot plan; plus the interval/threshold sensitivity of
Fig. 7 on one workload.

    python tools/introspection_study.py --out profiles/r1/introspection.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", nargs="+", default=["TXT", "MIX", "SWEEP"])
    ap.add_argument("--population", type=int, default=1 << 18)
    ap.add_argument("--generations", type=int, default=96)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    scfg = sat.SearchConfig(seed=11, population=args.population, max_generations=args.generations, elites=16,
                            generations_per_epoch=32)
    res = {"solver": {"population": args.population, "generations_per_round": args.generations}, "runs": []}
    for w in args.workloads:
        inst = synth.by_name(w, 0)
        plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
        knobs = [(1000, 500)]
        if w == args.workloads[0]:
            knobs += [(500, 500), (2000, 500), (4000, 500), (1000, 0), (1000, 2000)]
        for I, T in knobs:
            t0 = time.time()
            r, log = plan.introspect(I, T, solver="search", search=scfg)
            run = {"workload": w, "interval_s": I, "threshold_s": T, **r, "wall_s": time.time() - t0,
                   "reduction": 1 - r["e2e_makespan"] / r["one_shot_makespan"]}
            res["runs"].append(run)
            print(json.dumps(run), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
