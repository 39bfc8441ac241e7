"""Row f4: symmetry reduction for identical jobs -- TEST INFRASTRUCTURE ONLY (see oracle/__init__).

SURVEY.md §8f (f4) names it: the paper's workloads train the same model at several learning
rates, and a job's runtime does not depend on its learning rate, so such jobs
have the same profiled grid.  Two jobs are *twins* when their compacted config lists are the
same sequence of (GPU count, runtime) -- the only inputs O1 reads from a config.

Claim (reading A14): relabelling twins maps a genome to a genome with the same
makespan.  O1 places the jobs in perm order and reads job t only through (g, R) of its chosen
config, so exchanging the labels of twins u and v in both cfg and perm leaves every placement
step's (g, R) sequence -- hence the schedule's start and end times -- unchanged.  Hence the
minimum over *canonical* genomes (each job placed after its previous twin) equals the minimum
over all genomes.  `canonicalize` is that relabelling; the pins in tests/test_oracle_symmetry.py
check the claim by brute force rather than trusting this argument.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from .decoder import Compacted, decode_batch


def twin_prev(c: Compacted):
    """prev[t] = the largest u < t whose (g, R) config list equals job t's, else -1."""
    T = c.n_jobs

    def row(t):
        return [(int(c.gpus[t * c.stride + s]), int(c.runtime[t * c.stride + s])) for s in range(int(c.S[t]))]

    prev = []
    for t in range(T):
        p = -1
        for u in range(t - 1, -1, -1):
            if row(u) == row(t):
                p = u
                break
        prev.append(p)
    return prev


def is_canonical(c: Compacted, perm) -> bool:
    """Every job appears in perm after its previous twin."""
    prev = twin_prev(c)
    pos = {int(j): k for k, j in enumerate(perm)}
    return all(prev[t] < 0 or pos[prev[t]] < pos[t] for t in range(c.n_jobs))


def canonicalize(c: Compacted, cfg, perm):
    """Relabel each twin class so that its members appear in perm in increasing id order:
    the k-th member of a class to appear takes the class's k-th smallest id, with its config."""
    prev = twin_prev(c)
    T = c.n_jobs
    root = list(range(T))
    for t in range(T):
        if prev[t] >= 0:
            root[t] = root[prev[t]]
    classes = {}
    for t in range(T):
        classes.setdefault(root[t], []).append(t)
    label = {}
    for members in classes.values():
        appear = [int(j) for j in perm if root[int(j)] == root[members[0]]]
        for k, j in enumerate(appear):
            label[j] = members[k]
    new_cfg = np.zeros(T, np.uint8)
    new_perm = np.zeros(T, np.uint8)
    for k, j in enumerate(perm):
        new_perm[k] = label[int(j)]
    for t in range(T):
        new_cfg[label[t]] = cfg[t]
    return new_cfg, new_perm


def n_canonical(c: Compacted) -> int:
    """T! / prod over twin classes of (class size)!  times prod_t S_t."""
    prev = twin_prev(c)
    T = c.n_jobs
    size = {}
    root = list(range(T))
    for t in range(T):
        if prev[t] >= 0:
            root[t] = root[prev[t]]
        size[root[t]] = size.get(root[t], 0) + 1
    perms = math.factorial(T)
    for k in size.values():
        perms //= math.factorial(k)
    return perms * int(np.prod([int(s) for s in c.S], dtype=object))


def brute_force_canonical(c: Compacted):
    """(min makespan, smallest genome index attaining it) over the canonical genomes only.
    Index = r_perm * prod S + r_cfg with the same ranking as decoder.unrank (perm in
    lexicographic order, cfg job 0 least significant)."""
    T = c.n_jobs
    S = [int(s) for s in c.S]
    C = int(np.prod(S, dtype=object))
    radix = [int(np.prod(S[:t], dtype=object)) for t in range(T)]
    r = np.arange(C, dtype=np.int64)
    cfg = np.stack([(r // radix[t]) % S[t] for t in range(T)], axis=1).astype(np.uint8)
    best = None
    for r_perm, perm in enumerate(itertools.permutations(range(T))):   # lexicographic order
        if not is_canonical(c, perm):
            continue
        ms = decode_batch(c, cfg, np.tile(np.array(perm, np.uint8), (C, 1)))
        k = int(np.argmin(ms))
        key = (int(ms[k]), r_perm * C + k)
        if best is None or key < best:
            best = key
    return best
