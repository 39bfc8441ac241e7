"""Oracle reference values that bench.py reports beside its GPU numbers, written by a
committed script that calls only oracle/ (so bench.py itself executes the oracle only in its
cpu_baseline leg and its --impl reference arm):

  * the O2 brute-force optimum (makespan, smallest genome index) of C1 TINY seeds 0-2;
  * the O5 lower bound of every BASELINE workload at table seeds 0-2.

    python tools/oracle_refs.py --out profiles/r2/oracle_refs.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "oracle_refs.json"))
    a = ap.parse_args()
    res = {"what": "O2 brute force (TINY) and O5 lower bound (all workloads), oracle/ only",
           "tiny_brute_force": {}, "lower_bound": {}}
    for s in (0, 1, 2):
        t = synth.tiny(s)
        ms, idx = oracle.brute_force(oracle.compact(t.node_gpus, t.runtime))
        res["tiny_brute_force"][str(s)] = {"makespan": ms, "genome_index": idx}
    for w in ("TINY", "TXT", "IMG", "MIX", "SWEEP"):
        res["lower_bound"][w] = {}
        for s in (0, 1, 2):
            inst = synth.by_name(w, s)
            res["lower_bound"][w][str(s)] = oracle.lower_bound(oracle.compact(inst.node_gpus, inst.runtime))
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
