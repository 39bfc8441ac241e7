"""a7: GA operator replay (reference definitions).  TEST INFRASTRUCTURE ONLY.

The paper has no search heuristic besides its MILP; the genetic search is
this build's design, so this module *is* its
definition, written out step by step.  The CUDA search must reproduce it bit for bit from
the same inputs.

Genome: cfg[t] in [0, S_t) per job t, perm = priority permutation of job ids.
Population of P genomes per rank with makespans ms[i]; order key of slot i is (ms[i], i).
Thresholds are q32 integers: an event with probability p fires iff u32 < p_q32.
U(n, w) = (w * n) >> 32.

Philox4x32-10 (oracle/philox.py), key (seed_lo, seed_hi).  Word k of a stream with
counters (c0, c1, c2) is word k % 4 of philox((c0, c1, c2, k // 4)).

Initial genome of slot k (>= number of seed genomes), stream (k, 0, rank << 16 | 1), words
consumed in order: cfg[t] = U(S_t) for t = 0..T-1, then a Fisher-Yates shuffle of the
identity: for i = T-1 down to 1, j = U(i+1), swap perm[i], perm[j].

Children of generation g come in PAIRS (GA v5): slots 2q and 2q+1 are the two children of
pair q, made from one pair of parents by complementary crossover (the classic two-offspring
crossover); slots < E hold the elites instead.  Every word has a FIXED position in the
pair's stream (q, g, rank << 16 | 0), so the draws never depend on earlier outcomes.
16-bit fields are lo = w & 0xFFFF, hi = w >> 16, V(n, h) = (h * n) >> 16, and a 16-bit gate
with q32 threshold p fires iff h < p >> 16.
   w0, w1   tournament for parent A: i = U(P, w0), j = U(P, w1); A = smaller (ms, slot)
   w2, w3   tournament for parent B, same rule
   w4       lo: crossover gate (p_x)          hi: LOX cut a = V(T, hi)
   w5       lo: LOX cut b = V(T, lo)          hi: unused
   crossover bits: word k (k = 0 .. ceil(T/32)-1) at w6, w7, w16, w17, ... (w6 + k for
            k < 2, w16 + k - 2 after); bit t of word t // 32
   child r (r = 0, 1) fields: block 2 + r, i.e. words c = 8 + 4r .. 11 + 4r:
     w[c]     lo: permutation-mutation gate (p_m)   hi: mutation position i = V(T, hi)
     w[c+1]   lo: mutation position j = V(T, lo)    hi: mutation kind = hi & 1
     w[c+2]   lo: config-mutation gate (p_c)        hi: mutated job t* = V(T, hi)
     w[c+3]   lo: its new gene V(S_t*, lo)          hi: unused
 Child r of the pair, with (X, Y) = (A, B) for r = 0 and (B, A) for r = 1, in order:
   1. tournaments;  2. child = copy of X;
   3. if crossover: cfg[t] = Y.cfg[t] where crossover bit t is 0 (so the two children
      split every gene between the parents: complementary uniform crossover);
   4. if crossover: LOX (linear order crossover, Falkenauer & Bouffouix 1991) of X with Y,
      same cuts for both children -- a, b swapped so a <= b; keep X.perm[a..b] in place;
      fill positions 0..a-1, then b+1..T-1, with Y's genes in Y's order from position 0,
      skipping genes in X's slice;
   5. if config mutation: cfg[t*] = new gene;
   6. if permutation mutation: kind 0 swaps positions i and j; kind 1 removes the gene at i
      and reinserts it at position j.
 History: v1-v4 made one child per tournament pair (v3 OX1, v4 LOX; 3 Philox blocks and
 2 parent reads per child); v5 shares the tournaments, the parents, the cuts and the
 crossover bits between two children (per child: 2 Philox blocks, 1 parent read).
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


def lox(A_perm, B_perm, a: int, b: int):
    """Linear order crossover: A's slice [a..b] stays in place; positions 0..a-1 then
    b+1..T-1 take B's genes that are not in the slice, in B's order from position 0."""
    kept = set(A_perm[a:b + 1])
    fill = [x for x in B_perm if x not in kept]
    return list(fill[:a]) + list(A_perm[a:b + 1]) + list(fill[a:])


def xbit_word(k: int) -> int:
    """Position of crossover-bit word k in the pair's stream."""
    return 6 + k if k < 2 else 16 + (k - 2)


def pair_words(seed: int, rank: int, gen: int, q: int, T: int):
    nb = (T + 31) // 32
    n = max(16, xbit_word(nb - 1) + 1)
    st = Stream(_key(seed), q, gen, (rank << 16) | 0)
    return [st.u32() for _ in range(n)]


def make_child(S, cfg, perm, ms, slot: int, gen: int, seed: int, rank: int,
               p_x: int, p_c: int, p_m: int):
    P, T = cfg.shape
    nb = (T + 31) // 32
    q, r = slot >> 1, slot & 1
    w = pair_words(seed, rank, gen, q, T)
    lo = [x & 0xFFFF for x in w]
    hi = [x >> 16 for x in w]

    def U(n, x):
        return (x * n) >> 32

    def V(n, h):
        return (h * n) >> 16

    def tournament(wi, wj):
        i, j = U(P, wi), U(P, wj)
        return i if (int(ms[i]), i) < (int(ms[j]), j) else j

    a_idx = tournament(w[0], w[1])
    b_idx = tournament(w[2], w[3])
    x_idx, y_idx = (a_idx, b_idx) if r == 0 else (b_idx, a_idx)
    child_cfg, child_perm = list(cfg[x_idx]), list(perm[x_idx])
    Y_cfg, Y_perm = list(cfg[y_idx]), list(perm[y_idx])
    if lo[4] < (p_x >> 16):
        for t in range(T):
            if not (w[xbit_word(t // 32)] >> (t % 32)) & 1:
                child_cfg[t] = Y_cfg[t]
        a, b = V(T, hi[4]), V(T, lo[5])
        if a > b:
            a, b = b, a
        child_perm = lox(child_perm, Y_perm, a, b)
    c = 8 + 4 * r
    if lo[c + 2] < (p_c >> 16):
        t = V(T, hi[c + 2])
        child_cfg[t] = V(int(S[t]), lo[c + 3])
    if lo[c] < (p_m >> 16):
        kind = hi[c + 1] & 1
        i, j = V(T, hi[c]), V(T, lo[c + 1])
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
