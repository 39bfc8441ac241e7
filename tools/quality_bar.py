"""The 5-minute CPU search bar on TXT (SURVEY.md §8d "Quality-bar protocol"), CPU only.

  (i)  the paper's MILP (Eqs. 1-11, readings A1-A3; oracle/milp.py) solved by HiGHS with a
       300 s limit -- the open-source stand-in for the paper's 5-minute Gurobi solve
       (PAPER.md:983);
  (ii) the same GA as the GPU search on all host cores, every child decoded by the plain C
       oracle decoder (tools/cpu_ga.c), 300 s.
The bar of a seed is the better of the two.  Results go to profiles/<round>/quality_bar.json.

    python tools/quality_bar.py --seeds 0 1 2 --seconds 300 --out profiles/r1/quality_bar.json
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle.milp import SpaseMilp  # noqa: E402


def write_table(c, path):
    with open(path, "wb") as f:
        np.array([len(c.node_gpus)], np.int32).tofile(f)
        np.asarray(c.node_gpus, np.int32).tofile(f)
        np.array([c.n_jobs, c.stride], np.int32).tofile(f)
        np.asarray(c.S, np.int32).tofile(f)
        np.asarray(c.gpus, np.int32).tofile(f)
        np.asarray(c.runtime, np.int32).tofile(f)


def cpu_ga(c, seconds, threads, population, seed):
    exe = os.path.join(ROOT, "tools", "cpu_ga")
    src = os.path.join(ROOT, "tools", "cpu_ga.c")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-pthread", src, os.path.join(ROOT, "oracle", "saturn_oracle.c"),
                               "-o", exe])
    with tempfile.TemporaryDirectory() as d:
        tb = os.path.join(d, "t.bin")
        write_table(c, tb)
        out = subprocess.run([exe, tb, str(seconds), str(threads), str(population), str(seed)], capture_output=True,
                             text=True, check=True).stdout
    lines = [json.loads(x) for x in out.splitlines() if x.strip()]
    final = lines[-1]
    ms, pl = oracle.decode(c, np.array(final["cfg"], np.uint8), np.array(final["perm"], np.uint8))
    assert ms == final["best"] and oracle.validate(c, pl, ms) == []
    return {"best": final["best"], "evals": final["evals"], "threads": threads, "seconds": final["t"],
            "curve": [(x["t"], x["best"]) for x in lines[:-1]]}


def highs(c, seconds):
    t0 = time.time()
    m = SpaseMilp(c)
    status, val, plan = m.solve(time_limit=seconds)
    res = {"status": status, "seconds": time.time() - t0, "vars": m.n_vars, "rows": m.n_rows}
    if plan is not None:
        ms = max(p["end_s"] for p in plan)
        res["best"] = ms
        res["valid"] = oracle.validate(c, plan, ms) == []
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="TXT")
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--population", type=int, default=4096 * 8)
    ap.add_argument("--skip-milp", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    results = {"workload": args.workload, "seconds": args.seconds, "host_cores": os.cpu_count(),
               "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": "), "seeds": {}}
    for s in args.seeds:
        inst = synth.by_name(args.workload, s)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        r = {"lower_bound": oracle.lower_bound(c)}
        r["cpu_ga"] = cpu_ga(c, args.seconds, args.threads, args.population, 1000 + s)
        if not args.skip_milp:
            r["milp_highs"] = highs(c, args.seconds)
        cands = [r["cpu_ga"]["best"]] + ([r["milp_highs"]["best"]] if r.get("milp_highs", {}).get("best") else [])
        r["bar"] = min(cands)
        results["seeds"][str(s)] = r
        print(json.dumps({"seed": s, "bar": r["bar"], "lb": r["lower_bound"], "cpu_ga": r["cpu_ga"]["best"],
                          "milp": r.get("milp_highs", {}).get("best")}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
