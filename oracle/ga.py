"""a7: GA operator replay (reference definitions).  TEST INFRASTRUCTURE ONLY.

The paper has no search heuristic besides its MILP; the genetic search is
this build's design, so this module *is* its definition, written out
step by step.  The CUDA search must reproduce it bit for bit from the same inputs.

Genome: cfg[t] in [0, S_t) per job t, perm = priority permutation of job ids.
Population of P genomes per rank with makespans ms[i]; order key of slot i is (ms[i], i).
Philox stream of a slot (oracle.philox.Stream) with key (seed_lo, seed_hi):
    initial genome: counters (slot, 0, rank << 16 | 1)
    child of gen g: counters (slot, g, rank << 16 | 0)          (g = the child's generation)
Thresholds are q32 integers: an event with probability p fires iff u32 < p_q32.

Generation g -> g+1:
  slots [0, E): the E elites, i.e. the E smallest (ms, slot) of generation g in order
                (or the migrated global elites at an epoch boundary, see ``migrate``);
                copied with their makespan, not re-decoded;
  slot k >= E : 1. tournament x2: i = U(P), j = U(P); parent A = smaller (ms, slot);
                   again for parent B;
                2. crossover gate: u32 < p_x, else the child copies A (steps 3-4 skipped);
                3. cfg genes: bit t of the (t // 32)-th u32 word; 1 -> A's gene, 0 -> B's;
                4. OX1: a = U(T), b = U(T), swapped so a <= b; keep A.perm[a..b]; fill
                   positions b+1, b+2, ... (cyclic) with B's genes read from position b+1
                   (cyclic), skipping genes already present;
                5. cfg mutation, t = 0..T-1: if u32 < p_c then cfg[t] = U(S_t);
                6. perm mutation: if u32 < p_m: kind = u32 & 1, i = U(T), j = U(T);
                   kind 0 swaps positions i and j, kind 1 removes the gene at i and
                   reinserts it at position j.
Initial genome of slot k (>= number of seed genomes): cfg[t] = U(S_t) for t = 0..T-1,
then a Fisher-Yates shuffle of the identity: for i = T-1 down to 1, j = U(i+1), swap.
"""
from __future__ import annotations

import numpy as np

from .philox import Stream


def _key(seed: int):
    return (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)


def initial_genome(S, seed: int, rank: int, slot: int):
    T = len(S)
    st = Stream(_key(seed), slot, 0, (rank << 16) | 1)
    cfg = [st.below(int(S[t])) for t in range(T)]
    perm = list(range(T))
    for i in range(T - 1, 0, -1):
        j = st.below(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    return cfg, perm


def initial_population(S, P: int, seed: int, rank: int = 0, seed_cfg=None, seed_perm=None):
    T = len(S)
    cfg = np.zeros((P, T), np.uint8)
    perm = np.zeros((P, T), np.uint8)
    n_seed = 0 if seed_cfg is None else min(P, len(seed_cfg))
    for k in range(P):
        if k < n_seed:
            cfg[k], perm[k] = seed_cfg[k], seed_perm[k]
        else:
            c, p = initial_genome(S, seed, rank, k)
            cfg[k], perm[k] = c, p
    return cfg, perm


def elites(ms, E: int):
    """Slots of the E smallest (ms, slot), in order."""
    return sorted(range(len(ms)), key=lambda i: (int(ms[i]), i))[:E]


def make_child(S, cfg, perm, ms, slot: int, gen: int, seed: int, rank: int,
               p_x: int, p_c: int, p_m: int):
    P, T = cfg.shape
    st = Stream(_key(seed), slot, gen, (rank << 16) | 0)

    def tournament():
        i, j = st.below(P), st.below(P)
        return i if (int(ms[i]), i) < (int(ms[j]), j) else j

    a_idx = tournament()
    b_idx = tournament()
    A_cfg, A_perm = list(cfg[a_idx]), list(perm[a_idx])
    B_cfg, B_perm = list(cfg[b_idx]), list(perm[b_idx])
    if st.u32() < p_x:
        words = [st.u32() for _ in range((T + 31) // 32)]
        child_cfg = [A_cfg[t] if (words[t // 32] >> (t % 32)) & 1 else B_cfg[t] for t in range(T)]
        a, b = st.below(T), st.below(T)
        if a > b:
            a, b = b, a
        child_perm = [None] * T
        used = set()
        for p in range(a, b + 1):
            child_perm[p] = A_perm[p]
            used.add(A_perm[p])
        pos = (b + 1) % T
        rd = (b + 1) % T
        for _ in range(T - (b - a + 1)):
            while B_perm[rd] in used:
                rd = (rd + 1) % T
            child_perm[pos] = B_perm[rd]
            used.add(B_perm[rd])
            pos = (pos + 1) % T
            rd = (rd + 1) % T
    else:
        child_cfg, child_perm = A_cfg, A_perm
    for t in range(T):
        if st.u32() < p_c:
            child_cfg[t] = st.below(int(S[t]))
    if st.u32() < p_m:
        kind = st.u32() & 1
        i, j = st.below(T), st.below(T)
        if kind == 0:
            child_perm[i], child_perm[j] = child_perm[j], child_perm[i]
        else:
            x = child_perm.pop(i)
            child_perm.insert(j, x)
    return child_cfg, child_perm


def next_generation(S, cfg, perm, ms, gen: int, seed: int, rank: int, E: int,
                    p_x: int, p_c: int, p_m: int, elite_records=None):
    """Children of generation ``gen - 1`` -> (cfg, perm, elite_ms) of generation ``gen``.

    elite_records: optional list of E (ms, cfg, perm) replacing the local elites (migration).
    Returns new cfg/perm arrays; the makespans of slots >= E must be decoded by the caller.
    """
    P, T = cfg.shape
    ncfg = np.zeros_like(cfg)
    nperm = np.zeros_like(perm)
    ems = []
    if elite_records is None:
        elite_records = [(int(ms[i]), cfg[i].copy(), perm[i].copy()) for i in elites(ms, E)]
    for k, (m, c, p) in enumerate(elite_records[:E]):
        ncfg[k], nperm[k] = c, p
        ems.append(m)
    for k in range(E, P):
        c, p = make_child(S, cfg, perm, ms, k, gen, seed, rank, p_x, p_c, p_m)
        ncfg[k], nperm[k] = c, p
    return ncfg, nperm, ems


def migrate(rank_elites):
    """Island migration at an epoch boundary: every rank's next elites are the E best of
    all ranks' elite records, ordered by (ms, rank, position).  rank_elites[r] is rank r's
    list of E records (ms, cfg, perm) in order."""
    E = len(rank_elites[0])
    pool = [(rec[0], r, k, rec) for r, recs in enumerate(rank_elites) for k, rec in enumerate(recs)]
    pool.sort(key=lambda x: (x[0], x[1], x[2]))
    return [x[3] for x in pool[:E]]


def q32(p: float) -> int:
    """Probability -> q32 threshold, floor(p * 2^32) clamped to 2^32 - 1."""
    return min(int(p * 4294967296.0), 0xFFFFFFFF)
