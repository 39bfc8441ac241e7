"""O5b: a configuration-LP lower bound on the SPASE optimum.  TEST INFRASTRUCTURE ONLY
(also the quality report's proven bound: VERDICT r1 "What's weak" #7).

Relaxation.  In any feasible plan (Eqs. 2-11), at every instant each node n
runs a set K of jobs, each with one config (g, R), whose widths fit: sum g <= GPU_n (Eqs. 4-7,
10-11).  Let y[n,K] be the total time node n runs exactly the set K (idle time = the empty
set), so sum_K y[n,K] <= M for a makespan M.  Job t runs with one config s for R_{t,s}, so
sum over the K holding (t, s) of y[n,K] / R_{t,s} = 1.  Dropping integrality, the fixed
config per job and non-preemption leaves the LP

    min M   s.t.  sum_K y[k,K] <= m_k M                  for every node type k (m_k nodes)
                  sum_{(k,K) holding t} y[k,K] / R_{t,s(K)} >= 1    for every job t
                  M >= max_t min_s R_{t,s}                (a job runs R_{t,s} wall time)
                  y >= 0,

whose optimum M* is a lower bound on the optimal makespan (identical nodes are grouped into
one type with capacity m_k M; a job may appear at most once in a K).  It dominates O5
(SPEC.md:250): every K occupies at most GPU_n GPUs, so the area term holds, and the last row
is O5's longest-job term (needed explicitly: with several nodes the relaxation could run one
job on two nodes at once).

Solved by column generation: the restricted master LP by HiGHS (scipy.optimize.linprog);
pricing for node type k is a multiple-choice knapsack -- maximise sum_t pi_t / R_{t,s} over
jobs with at most one config each, sum g <= GPU_k -- solved exactly by dynamic programming;
a column enters while its reduced cost sigma_k - sum pi_t / R_{t,s} < 0.  Only the converged
master's optimum is the LP optimum (a restricted master is an upper bound), so the function
raises if pricing has not converged.  The returned integer bound is ceil(M* (1 - 1e-7))
(runtimes are integers, so the optimum is too).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.optimize import linprog


def _price(jobs, cap, pi):
    """Multiple-choice knapsack: jobs[t] = [(g, R), ...]; -> (value, [(t, s), ...])."""
    best = [0.0] * (cap + 1)
    choice = [[] for _ in range(cap + 1)]
    for t, cfgs in enumerate(jobs):
        if pi[t] <= 0:
            continue
        nb, nc = best[:], [c[:] for c in choice]
        for s, (g, r) in enumerate(cfgs):
            if g > cap:
                continue
            v = pi[t] / r
            for c in range(cap, g - 1, -1):
                if best[c - g] + v > nb[c] + 1e-15:
                    nb[c] = best[c - g] + v
                    nc[c] = choice[c - g] + [(t, s)]
        best, choice = nb, nc
    c = int(np.argmax(best))
    return best[c], choice[c]


def config_lp_bound(c, max_iter: int = 5000, tol: float = 1e-9):
    """-> (integer lower bound, LP optimum M*, number of columns)."""
    T = c.n_jobs
    jobs = [[(c.config(t, s)[1], c.config(t, s)[2]) for s in range(int(c.S[t]))] for t in range(T)]
    types = sorted({int(g) for g in c.node_gpus})
    count = {k: sum(1 for g in c.node_gpus if int(g) == k) for k in types}
    cols = []   # (type index, [(t, s), ...])
    for t in range(T):   # start: every job alone, with each config that fits a node type
        for k, cap in enumerate(types):
            for s, (g, r) in enumerate(jobs[t]):
                if g <= cap:
                    cols.append((k, [(t, s)]))
    converged = False
    for _ in range(max_iter):
        nK, nT = len(types), T
        n = len(cols) + 1                  # y columns, then M
        A = np.zeros((nK + nT, n))
        for j, (k, K) in enumerate(cols):
            A[k, j] = 1.0
            for t, s in K:
                A[nK + t, j] = -1.0 / jobs[t][s][1]
        for k, cap in enumerate(types):
            A[k, n - 1] = -float(count[cap])
        b = np.concatenate([np.zeros(nK), -np.ones(nT)])
        cost = np.zeros(n)
        cost[-1] = 1.0
        longest = max(min(r for _, r in cfgs) for cfgs in jobs)
        res = linprog(cost, A_ub=A, b_ub=b, bounds=[(0, None)] * (n - 1) + [(longest, None)], method="highs")
        assert res.status == 0, res.message
        lam = res.ineqlin.marginals          # <= 0 for a minimisation's <= rows
        sigma, pi = -lam[:nK], -lam[nK:]
        added = 0
        for k, cap in enumerate(types):
            val, K = _price(jobs, cap, pi)
            if K and val > sigma[k] * (1 + tol) + tol:
                cols.append((k, K))
                added += 1
        if not added:
            converged = True
            break
    if not converged:
        raise RuntimeError("configuration LP: column generation did not converge")
    m_star = float(res.fun)
    return int(math.ceil(m_star * (1 - 1e-7))), m_star, len(cols)
