"""Round-2 quality bars: the round-1 5-minute CPU bars (tools/quality_bar.py: HiGHS on the
paper's MILP and the CPU GA, 300 s each) plus the configuration-LP lower bound (oracle/
bounds.py, O5b) per (workload, table seed), so every reported best has a proven gap.
Calls only oracle/.

    python tools/quality_bounds.py      # -> profiles/r2/quality_bar{,_MIX,_SWEEP}.json
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle.bounds import config_lp_bound  # noqa: E402


def main():
    for w, fname in (("TXT", "quality_bar.json"), ("MIX", "quality_bar_MIX.json"), ("SWEEP", "quality_bar_SWEEP.json")):
        d = json.load(open(os.path.join(ROOT, "profiles", "r1", fname)))
        d["round"] = "r2: bars from profiles/r1 (CPU GA v3 / HiGHS, 300 s each); best_lower_bound added"
        for s, e in d["seeds"].items():
            inst = synth.by_name(w, int(s))
            c = oracle.compact(inst.node_gpus, inst.runtime)
            t0 = time.time()
            lb, m_star, ncol = config_lp_bound(c)
            e["best_lower_bound"] = lb
            e["best_lower_bound_kind"] = "configuration LP (oracle/bounds.py, O5b)"
            e["config_lp_optimum"] = m_star
            e["config_lp_columns"] = ncol
            e["bar_gap_to_best_lb"] = (e["bar"] - lb) / lb
            print(w, s, "bar", e["bar"], "O5", e["lower_bound"], "O5b", lb, f"{time.time() - t0:.1f}s", flush=True)
        with open(os.path.join(ROOT, "profiles", "r2", fname), "w") as f:
            json.dump(d, f, indent=1)


if __name__ == "__main__":
    main()
