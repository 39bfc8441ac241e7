"""f4: best-improvement local search on a genome (reference for saturn_improve and the
search's memetic elite step).  TEST INFRASTRUCTURE ONLY.

Neighbourhood of a genome (cfg, perm), moves numbered m = 0, 1, ...:
  insertion moves, m < T(T-1):  i = m // (T-1), jj = m % (T-1), j = jj if jj < i else jj + 1;
                                remove the job at position i of perm, reinsert it at position j;
  config moves, then:           for t = 0..T-1, for c = 0..S_t-1 with c != cfg[t] (in order):
                                set cfg[t] = c.
One iteration decodes every neighbour (oracle O1) and moves to the best one -- smallest
(makespan, m) -- if its makespan is strictly smaller than the current one; at most `iters`
iterations, stopping early at a local optimum.
"""
from __future__ import annotations

import numpy as np

from .decoder import decode_batch


def neighbours(c, cfg, perm):
    T = c.n_jobs
    cs, ps = [], []
    for m in range(T * (T - 1)):
        i, jj = divmod(m, T - 1)
        j = jj if jj < i else jj + 1
        p = list(perm)
        x = p.pop(i)
        p.insert(j, x)
        cs.append(list(cfg))
        ps.append(p)
    for t in range(T):
        for v in range(int(c.S[t])):
            if v != cfg[t]:
                q = list(cfg)
                q[t] = v
                cs.append(q)
                ps.append(list(perm))
    return np.array(cs, np.uint8).reshape(-1, T), np.array(ps, np.uint8).reshape(-1, T)


def improve(c, cfg, perm, iters: int):
    cfg = np.array(cfg, np.uint8)
    perm = np.array(perm, np.uint8)
    ms = int(decode_batch(c, cfg[None], perm[None])[0])
    for _ in range(iters):
        nc, npm = neighbours(c, cfg, perm)
        if len(nc) == 0:
            break
        m = decode_batch(c, nc, npm)
        best = int(np.lexsort((np.arange(len(m)), m))[0])
        if m[best] >= ms:
            break
        cfg, perm, ms = nc[best].copy(), npm[best].copy(), int(m[best])
    return cfg, perm, ms
