"""f1: round introspection (App. "Interval Introspection"; §4.4,
PAPER.md:1013-1068).  TEST INFRASTRUCTURE ONLY (reference for saturn_introspect).

    S = solve(W); M = makespan(S); time = 0
    loop:
        if M <= I: the workload finishes inside this interval -> E2E makespan = time + M
        W = W after I seconds of S        (residual runtimes, reading A10)
        S = S[I:]; M = M - I; time += I
        P = solve(W)
        if makespan(P) <= M - T: S = P; M = makespan(P)

Reading A10 (residual work): a job that ran a seconds of its current config (runtime R0)
keeps every config with R' = ceil(R * (R0 - a) / R0) (integers); finished jobs leave W; jobs
not yet started are unchanged.  S[I:] keeps every placement (node, GPUs) and shifts its
times by -I (a running job restarts at 0 with its residual runtime R0 - a).
`solve` here is the exact brute force (oracle O2), so the whole loop is deterministic.
"""
from __future__ import annotations

import numpy as np

from .decoder import compact, brute_force, unrank, decode


def _solve(nodes, table):
    c = compact(nodes, table)
    ms, idx = brute_force(c)
    cfg, perm = unrank(c, idx)
    m2, pl = decode(c, cfg, perm)
    assert m2 == ms
    return ms, pl, c


def residual(table, plan, I):
    """(new table, surviving old job ids, shifted plan) after I seconds of `plan`."""
    rows, keep, shifted = [], [], []
    for t, pl in enumerate(plan):
        if pl["end_s"] <= I:
            continue
        row = table[t].astype(np.int64)
        if pl["start_s"] < I:
            R0 = pl["end_s"] - pl["start_s"]
            a = I - pl["start_s"]
            row = np.where(row > 0, (row * (R0 - a) + R0 - 1) // R0, 0)
        rows.append(row.astype(np.int32))
        keep.append(t)
        q = dict(pl)
        q["start_s"] = max(pl["start_s"] - I, 0)
        q["end_s"] = pl["end_s"] - I
        shifted.append(q)
    if not rows:
        return None, [], []
    return np.stack(rows), keep, shifted


def introspect(nodes, table, I: int, T: int, max_rounds: int = 10_000):
    table = np.asarray(table, np.int32)
    M, S, _ = _solve(nodes, table)
    one_shot = M
    time, rounds, adopted, log = 0, 0, 0, []
    while M > I and rounds < max_rounds:
        table, keep, S = residual(table, S, I)
        M -= I
        time += I
        rounds += 1
        Mp, P, _ = _solve(nodes, table)
        take = Mp <= M - T
        log.append((time, M, Mp, int(take)))
        if take:
            S, M = P, Mp
            adopted += 1
    return {"one_shot": one_shot, "e2e": time + M, "rounds": rounds, "adopted": adopted, "log": log}
