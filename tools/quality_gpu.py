"""GPU side of the quality bar: saturn_search on one B200 with a 10 s
wall budget per seed (measured from the saturn_search call), seeded with the paper's
baseline genomes (row f2), against the CPU bar of tools/quality_bar.py.

    python tools/quality_gpu.py --seeds 0 1 2 --budget 10 --out profiles/r1/quality_gpu.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (only to re-check the returned plan)
import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="TXT")
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--budget", type=float, default=10.0)
    ap.add_argument("--populations", type=int, nargs="+", default=[1 << 20])
    ap.add_argument("--elites", type=int, default=16)
    ap.add_argument("--epoch", type=int, default=32)
    ap.add_argument("--ls", type=int, nargs="+", default=[0], help="memetic local-search iterations per epoch")
    ap.add_argument("--bar", default=None, help="quality_bar.json to compare against")
    ap.add_argument("--out", default=None)
    ap.add_argument("--lib", default=None, help="alternative libsaturn.so (A/B)")
    ap.add_argument("--ga-seeds", type=int, nargs="+", default=None,
                    help="GA seeds per table seed (default: 100 + table seed)")
    args = ap.parse_args()
    if args.lib:
        sat.load_library(args.lib)
    bar = json.load(open(args.bar)) if args.bar and os.path.exists(args.bar) else None
    import torch
    res = {"workload": args.workload, "budget_s": args.budget, "gpu": torch.cuda.get_device_name(0), "runs": []}
    for s in args.seeds:
        inst = synth.by_name(args.workload, s)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
        seeds_c, seeds_p, base = [], [], {}
        for kind in ("max", "min", "optimus", "random"):
            gc, gq = plan.baseline_genome(kind, s)
            seeds_c.append(gc)
            seeds_p.append(gq)
            base[kind] = int(plan.evaluate_host(gc[None], gq[None])[0])
        for P, ls, gs in [(P, ls, gs) for P in args.populations for ls in args.ls
                          for gs in (args.ga_seeds or [100 + s])]:
            cfg = sat.SearchConfig(seed=gs, population=P, max_generations=1 << 30, time_budget_s=args.budget,
                                   elites=args.elites, generations_per_epoch=args.epoch, local_search_iters=ls)
            r = plan.search(cfg, seed_genomes=(np.stack(seeds_c), np.stack(seeds_p)))
            best, pl, bc, bp = plan.best_plan()
            ms, opl = oracle.decode(c, bc, bp)
            assert ms == best and oracle.validate(c, pl, best) == []
            t, h = plan.search_history()
            marks = {}
            for target in (0.01, 0.1, 1.0, 2.0, 5.0, 10.0):
                k = np.searchsorted(t, target, side="right") - 1
                if k >= 0:
                    marks[f"{target:g}s"] = int(h[k])
            run = {"seed": s, "ga_seed": gs, "population": P, "local_search_iters": ls, "best": best, "lower_bound": oracle.lower_bound(c),
                   "seconds": r["seconds"], "evaluated": r["evaluated"], "generations": r["generations"],
                   "plans_per_s": r["evaluated"] / r["seconds"], "anytime": marks, "baselines": base}
            if bar:
                b = bar["seeds"].get(str(s), {}).get("bar")
                run["cpu_bar"] = b
                run["beats_bar"] = (b is not None and best <= b)
            res["runs"].append(run)
            print(json.dumps(run), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
