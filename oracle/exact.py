"""O4a: time-indexed exact SPASE solver for tiny instances.  TEST INFRASTRUCTURE ONLY.

Shares nothing with the decoder.  It searches directly over the paper's decision
variables (per task a configuration, a node and a start time) with
integer start times, and accepts an assignment iff on every node, at every integer
time unit, the GPUs demanded by the tasks running there do not exceed GPU_n.

Why per-node cumulative capacity is exactly the paper's constraint set: given capacity,
assign GPU ids greedily in start order -- when task j starts, the tasks still running on
its node hold at most GPU_n - G_j GPUs, so G_j free GPUs exist and j keeps them for its
whole interval (interval graphs are perfect).  That yields explicit P_{t,n,g} with one
start per task (gang, Eqs. 8-9) and no overlap on any GPU (Eqs. 10-11).  Conversely any
valid plan satisfies capacity.  Integer start times lose nothing when runtimes are integer
(reading A4).

The optimum is found by trying C = LB, LB+1, ... and asking whether every task fits in
[0, C).
"""
from __future__ import annotations

from .checks import lower_bound


def _feasible(c, C):
    T = c.n_jobs
    N = len(c.node_gpus)
    cap = [[int(c.node_gpus[n])] * C for n in range(N)]   # free GPUs per node per time unit
    total_free = sum(int(x) for x in c.node_gpus) * C
    opts = []
    for t in range(T):
        o = [c.config(t, s)[1:] for s in range(int(c.S[t]))]
        o = sorted(set(o), key=lambda gr: gr[0] * gr[1])          # (g, r), cheapest area first
        opts.append(o)
    min_area = [min(g * r for g, r in o) for o in opts]
    order = sorted(range(T), key=lambda t: -min_area[t])
    rest_area = [0] * (T + 1)
    for k in range(T - 1, -1, -1):
        rest_area[k] = rest_area[k + 1] + min_area[order[k]]

    def dfs(k, free_area):
        if k == T:
            return True
        if rest_area[k] > free_area:
            return False
        t = order[k]
        for g, r in opts[t]:
            if r > C:
                continue
            for n in range(N):
                if c.node_gpus[n] < g:
                    continue
                row = cap[n]
                for s in range(0, C - r + 1):
                    if all(row[x] >= g for x in range(s, s + r)):
                        for x in range(s, s + r):
                            row[x] -= g
                        ok = dfs(k + 1, free_area - g * r)
                        for x in range(s, s + r):
                            row[x] += g
                        if ok:
                            return True
        return False

    return dfs(0, total_free)


def exact_makespan(c, limit: int = 10_000) -> int:
    """The SPASE optimum of a tiny instance (O4a)."""
    C = lower_bound(c)
    while C <= limit:
        if _feasible(c, C):
            return C
        C += 1
    raise RuntimeError("no schedule found below the limit")
