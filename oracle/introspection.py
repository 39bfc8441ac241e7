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

Workload events ("early-stopping ... or new job
arrivals"), applied at round boundaries only: after round r's advance, before its re-solve.
  ("stop", job)       -- job (original id; arrivals are numbered T, T+1, ... in event order)
                         leaves W and the current plan; M becomes the plan's latest end.
  ("arrive", row)     -- a new job with runtime row [U][Gmax] joins W; the current plan does
                         not hold it, so the round's proposal is adopted unconditionally.
An event naming a finished or unknown job raises ValueError; events due after the workload
is exhausted never fire.

Overlap mode: the proposal for round r+1 is computed
on the SIMULATED next-interval state advance(W, S, I) while round r runs (the solver's latency
is hidden behind the interval).  If an event fires at that boundary the proposal is stale and
a fresh solve of the mutated workload replaces it, so the E2E schedule is identical to the
sequential loop's; `stale` counts the discarded proposals.
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


def introspect(nodes, table, I: int, T: int, max_rounds: int = 10_000, events=(), overlap: bool = False):
    table = np.asarray(table, np.int32)
    ids = list(range(table.shape[0]))          # original job id of every row of `table`
    next_id = table.shape[0]
    M, S, _ = _solve(nodes, table)
    one_shot = M
    time, rounds, adopted, stale, log = 0, 0, 0, 0, []
    by_round = {}
    for r, kind, arg in events:
        by_round.setdefault(int(r), []).append((kind, arg))
    while M > I and rounds < max_rounds:
        lookahead = None
        if overlap:   # solved on the simulated next-interval state, before this round ends
            nxt, _, _ = residual(table, S, I)
            lookahead = None if nxt is None else _solve(nodes, nxt)[:2]
        table, keep, S = residual(table, S, I)
        ids = [ids[k] for k in keep]
        M -= I
        time += I
        rounds += 1
        fired, arrived = by_round.get(rounds, []), False
        for kind, arg in fired:
            if kind == "stop":
                if arg not in ids:
                    raise ValueError(f"stop event names job {arg}, which is finished or unknown")
                k = ids.index(arg)
                table = np.delete(table, k, axis=0)
                del ids[k]
                del S[k]
            elif kind == "arrive":
                row = np.asarray(arg, np.int32)[None]
                table = row if table is None else np.concatenate([table, row], axis=0)
                ids.append(next_id)
                next_id += 1
                arrived = True
            else:
                raise ValueError(kind)
        if fired:
            stale += int(lookahead is not None)
            lookahead = None
            M = max((p["end_s"] for p in S), default=0)
        if table is None or len(ids) == 0:   # every job stopped: the workload is exhausted
            M = 0
            log.append((time, 0, 0, 0))
            break
        Mp, P = lookahead if lookahead is not None else _solve(nodes, table)[:2]
        take = arrived or Mp <= M - T
        log.append((time, M, Mp, int(take)))
        if take:
            S, M = P, Mp
            adopted += 1
    return {"one_shot": one_shot, "e2e": time + M, "rounds": rounds, "adopted": adopted, "stale": stale,
            "log": log}
