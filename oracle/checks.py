"""O3 schedule validator and O5 lower bound.  TEST INFRASTRUCTURE ONLY.

O3 checks a decoded plan against the semantics of the paper's constraints
(PAPER.md:807-810 summary; Eqs. 2-11; readings A1-A3 in DESIGN.md):
  one-config / one-node (Eq. 3), exactly G_{t,s} GPUs on the chosen node (Eqs. 4-5),
  no GPUs on other nodes (Eqs. 6-7 as read, A1), one common start time (gang, Eqs. 8-9:
  a placement record carries a single start by construction), no two tasks overlapping
  on a GPU (Eqs. 10-11), and the makespan equal to the latest end (Eq. 2).
O5 is the lower bound of SPEC.md:250.
"""
from __future__ import annotations

import math


def validate(c, placements, makespan=None):
    """Return a list of violation tags (empty = valid).  ``c`` is an oracle.Compacted."""
    bad = []
    N = len(c.node_gpus)
    if placements is None or len(placements) != c.n_jobs:
        return ["missing-jobs"]
    busy = {}  # (node, gpu) -> list of (start, end, job)
    latest = 0
    for t, pl in enumerate(placements):
        s_idx = pl["cfg"]
        if not (0 <= s_idx < int(c.S[t])):
            bad.append(f"one-config:{t}")
            continue
        _, g, r = c.config(t, s_idx)
        n = pl["node"]
        if not (0 <= n < N):
            bad.append(f"one-node:{t}")
            continue
        if pl["gpus"] != g:
            bad.append(f"alloc:{t}")
        mask = pl["gpu_mask"]
        ids = [i for i in range(64) if mask >> i & 1]
        if len(ids) != g:
            bad.append(f"alloc:{t}")
        if any(i >= int(c.node_gpus[n]) for i in ids):
            bad.append(f"unselected-zero:{t}")
        if pl["start_s"] < 0:
            bad.append(f"start:{t}")
        if pl["end_s"] != pl["start_s"] + r:
            bad.append(f"runtime:{t}")
        for i in ids:
            busy.setdefault((n, i), []).append((pl["start_s"], pl["start_s"] + r, t))
        latest = max(latest, pl["start_s"] + r)
    for key, ivs in busy.items():
        ivs.sort()
        for (s0, e0, t0), (s1, e1, t1) in zip(ivs, ivs[1:]):
            if s1 < e0:  # half-open intervals [s, e): back-to-back is legal
                bad.append(f"isolation:{t0}-{t1}@{key}")
    if makespan is not None and makespan != latest:
        bad.append("makespan")
    return bad


def lower_bound(c) -> int:
    """O5: max( max_t min_s R_{t,s}, ceil(sum_t min_s G_{t,s} R_{t,s} / sum_n GPU_n) )."""
    longest = 0
    area = 0
    for t in range(c.n_jobs):
        cfgs = [c.config(t, s) for s in range(int(c.S[t]))]
        longest = max(longest, min(r for _, _, r in cfgs))
        area += min(g * r for _, g, r in cfgs)
    return max(longest, math.ceil(area / int(sum(int(x) for x in c.node_gpus))))
