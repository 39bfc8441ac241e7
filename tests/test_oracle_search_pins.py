"""Pins for the two search-side oracle functions that round 1 left unpinned (VERDICT r1,
"What's weak" #1): the local search (oracle/local_search.py, row f4) and the GA's initial
genome (oracle/ga.py:initial_genome, also the paper's Randomized baseline, PAPER.md:976,
"tasks are randomly scheduled").

Nothing here calls `neighbours` to build its expectation: the neighbourhood is rebuilt from
its definition (a move = one job moved to another priority position with the others keeping
their relative order, or one job switched to another of its configurations), decoded by O1
(itself pinned in test_oracle_pins.py), and compared move by move.  The initial genome is
pinned by an exact chi-square test over all T! permutations (Fisher-Yates draws every
permutation with probability 1/T!; Sattolo's variant draws only the (T-1)! cyclic ones) and
over each job's config values (uniform on [0, S_t)).
"""
import itertools

import numpy as np
import pytest
from scipy.stats import chi2

import oracle
from oracle import ga
from oracle.local_search import improve, neighbours
from conftest import dense_from_configs

# ---------------------------------------------------------------- local search


def _moved(perm, x_pos, to):
    """The permutation with the job at position x_pos placed at position `to`, every other
    job keeping its relative order (built slot by slot, not by pop/insert)."""
    T = len(perm)
    x = perm[x_pos]
    rest = iter([perm[q] for q in range(T) if q != x_pos])
    return [x if q == to else next(rest) for q in range(T)]


def _reference_neighbourhood(c, cfg, perm):
    """Moves in their documented numbering: insertion moves first, for every source
    position i (ascending) every target position j != i (ascending); then config moves,
    for every job t (ascending) every other config value (ascending)."""
    T = c.n_jobs
    moves = []
    for i in range(T):
        for j in range(T):
            if j != i:
                moves.append((list(cfg), _moved(list(perm), i, j)))
    for t in range(T):
        for v in range(int(c.S[t])):
            if v != cfg[t]:
                q = list(cfg)
                q[t] = v
                moves.append((q, list(perm)))
    return moves


def _ms(c, cfg, perm):
    return int(oracle.decode_batch(c, np.array([cfg], np.uint8), np.array([perm], np.uint8))[0])


def _random_instance(rng, T, nodes, n_cfg_max=3, rmax=9):
    configs = []
    for _ in range(T):
        k = int(rng.integers(1, n_cfg_max + 1))
        opts = set()
        while len(opts) < k:
            opts.add((int(rng.integers(0, 2)), int(rng.integers(1, max(nodes) + 1))))
        configs.append([(u, g, int(rng.integers(1, rmax + 1))) for u, g in sorted(opts)])
    return oracle.compact(np.array(nodes, np.int32), dense_from_configs(configs, n_upps=2))


def test_local_search_hand_example():
    """1 node x 2 GPUs.  Job 0: (1 GPU, 4 s) or (2 GPUs, 3 s); jobs 1, 2: (1 GPU, 2 s).
    Start: cfg = (1, 0, 0) (job 0 on both GPUs), perm = (0, 1, 2).
      decode: job 0 [0,3) on GPUs {0,1}; job 1 at 3 on GPU 0; job 2 at 3 on GPU 1 -> 5.
    Neighbours (7 = T(T-1) + sum(S_t - 1) = 6 + 1), by hand:
      m=0 (0->1) perm (1,0,2): job 1 [0,2) GPU 0; job 0 needs 2 GPUs -> 2; job 2 at 5 -> 7
      m=1 (0->2) perm (1,2,0): jobs 1, 2 at 0; job 0 at 2 -> 5
      m=2 (1->0) perm (1,0,2) -> 7        m=3 (1->2) perm (0,2,1) -> 5
      m=4 (2->0) perm (2,0,1) -> 7        m=5 (2->1) perm (0,2,1) -> 5
      m=6 cfg (0,0,0): job 0 [0,4) GPU 0; job 1 [0,2) GPU 1; job 2 [2,4) GPU 1 -> 4
    Best move m=6 (4 < 5).  From there 4 = the area bound (4+2+2)/2: no strictly better
    neighbour, so the search stops."""
    c = oracle.compact(np.array([2], np.int32),
                       dense_from_configs([[(0, 1, 4), (0, 2, 3)], [(0, 1, 2)], [(0, 1, 2)]], n_upps=1))
    cfg, perm = [1, 0, 0], [0, 1, 2]
    assert _ms(c, cfg, perm) == 5
    nc, npm = neighbours(c, np.array(cfg, np.uint8), np.array(perm, np.uint8))
    got = oracle.decode_batch(c, nc, npm)
    assert got.tolist() == [7, 5, 7, 5, 7, 5, 4]
    rc, rp, rms = improve(c, cfg, perm, iters=1)
    assert (rc.tolist(), rp.tolist(), rms) == ([0, 0, 0], [0, 1, 2], 4)
    rc, rp, rms = improve(c, cfg, perm, iters=5)
    assert (rc.tolist(), rp.tolist(), rms) == ([0, 0, 0], [0, 1, 2], 4)


@pytest.mark.parametrize("nodes", [[4], [2, 2], [3, 5]])
def test_neighbourhood_matches_definition(nodes):
    rng = np.random.default_rng(11 + len(nodes))
    for _ in range(8):
        T = int(rng.integers(2, 6))
        c = _random_instance(rng, T, nodes)
        cfg = [int(rng.integers(0, c.S[t])) for t in range(T)]
        perm = [int(x) for x in rng.permutation(T)]
        ref = _reference_neighbourhood(c, cfg, perm)
        nc, npm = neighbours(c, np.array(cfg, np.uint8), np.array(perm, np.uint8))
        assert len(ref) == T * (T - 1) + int(sum(int(s) - 1 for s in c.S))
        assert len(nc) == len(ref)
        for m, (rc, rp) in enumerate(ref):
            assert nc[m].tolist() == rc and npm[m].tolist() == rp, m


def test_improve_step_is_best_strict_improvement():
    """One iteration = the smallest (makespan, move number) over the reference
    neighbourhood, taken only if strictly better; otherwise the genome is returned as is.
    Ties between improving moves occur on these instances and must go to the lower m."""
    rng = np.random.default_rng(5)
    ties = stays = moves = 0
    for it in range(60):
        nodes = [[4], [2, 2], [3, 5], [2, 2, 4]][it % 4]
        T = int(rng.integers(2, 6))
        c = _random_instance(rng, T, nodes)
        cfg = [int(rng.integers(0, c.S[t])) for t in range(T)]
        perm = [int(x) for x in rng.permutation(T)]
        ms0 = _ms(c, cfg, perm)
        ref = _reference_neighbourhood(c, cfg, perm)
        scored = [(_ms(c, rc, rp), m) for m, (rc, rp) in enumerate(ref)]
        best_ms, best_m = min(scored) if scored else (ms0, -1)
        ties += sum(1 for s, m in scored if s == best_ms) > 1 and best_ms < ms0
        rc, rp, rms = improve(c, cfg, perm, iters=1)
        if best_ms < ms0:
            moves += 1
            assert (rc.tolist(), rp.tolist(), rms) == (ref[best_m][0], ref[best_m][1], best_ms)
        else:
            stays += 1
            assert (rc.tolist(), rp.tolist(), rms) == (cfg, perm, ms0)
    assert ties > 0 and stays > 0 and moves > 0


def test_improve_ends_at_local_optimum():
    rng = np.random.default_rng(9)
    for it in range(20):
        nodes = [[4], [2, 2], [3, 5]][it % 3]
        T = int(rng.integers(3, 6))
        c = _random_instance(rng, T, nodes)
        cfg = [int(rng.integers(0, c.S[t])) for t in range(T)]
        perm = [int(x) for x in rng.permutation(T)]
        rc, rp, rms = improve(c, cfg, perm, iters=1000)
        assert rms == _ms(c, rc.tolist(), rp.tolist())
        assert rms <= _ms(c, cfg, perm)
        ref = _reference_neighbourhood(c, rc.tolist(), rp.tolist())
        assert all(_ms(c, a, b) >= rms for a, b in ref)      # no strictly better neighbour
        # the whole path is a chain of strict improvements: at most |space| steps, and
        # running further from the optimum changes nothing
        again = improve(c, rc, rp, iters=3)
        assert (again[0].tolist(), again[1].tolist(), again[2]) == (rc.tolist(), rp.tolist(), rms)


def test_improve_respects_iteration_cap():
    rng = np.random.default_rng(21)
    for it in range(15):
        T = int(rng.integers(3, 6))
        c = _random_instance(rng, T, [4])
        cfg = [int(rng.integers(0, c.S[t])) for t in range(T)]
        perm = [int(x) for x in rng.permutation(T)]
        cur = (cfg, perm, _ms(c, cfg, perm))
        for k in range(1, 4):   # k iterations == k single steps chained
            one = improve(c, cur[0], cur[1], iters=1)
            cur = (one[0].tolist(), one[1].tolist(), one[2])
            got = improve(c, cfg, perm, iters=k)
            assert (got[0].tolist(), got[1].tolist(), got[2]) == cur


# ---------------------------------------------------------------- initial genome


def _chi2_pvalue(counts, expected):
    counts = np.asarray(counts, np.float64)
    stat = float(((counts - expected) ** 2 / expected).sum())
    return float(chi2.sf(stat, len(counts) - 1))


@pytest.mark.parametrize("T", [3, 4])
def test_initial_genome_permutations_uniform(T):
    """Every one of the T! priority orders is equally likely (Fisher-Yates with
    j = U(i+1)).  n = 1000 T! draws; p-value floor 1e-4 (seeded, so deterministic).
    Sattolo's j = U(i) never yields the identity and puts all mass on (T-1)! cycles."""
    S = np.array([2] * T, np.int32)
    perms = list(itertools.permutations(range(T)))
    idx = {p: k for k, p in enumerate(perms)}
    n = 1000 * len(perms)
    counts = np.zeros(len(perms), np.int64)
    for slot in range(n):
        _, p = ga.initial_genome(S, seed=2309, rank=0, slot=slot)
        counts[idx[tuple(p)]] += 1
    assert counts.min() > 0
    assert _chi2_pvalue(counts, n / len(perms)) > 1e-4


def test_initial_genome_positions_uniform_t12():
    """TXT size: the job at each priority position is uniform over the 12 jobs (a T x T
    contingency table; a dropped last swap or a biased j fails it)."""
    T = 12
    S = np.array([1] * T, np.int32)
    n = 6000
    cnt = np.zeros((T, T), np.int64)
    for slot in range(n):
        _, p = ga.initial_genome(S, seed=7, rank=1, slot=slot)
        for q in range(T):
            cnt[q, p[q]] += 1
    for q in range(T):
        assert _chi2_pvalue(cnt[q], n / T) > 1e-4, q


def test_initial_genome_configs_uniform():
    S = np.array([3, 5, 7, 2, 8], np.int32)
    n = 7000
    counts = [np.zeros(int(s), np.int64) for s in S]
    for slot in range(n):
        cfg, _ = ga.initial_genome(S, seed=11, rank=0, slot=slot)
        for t, v in enumerate(cfg):
            assert 0 <= v < S[t]
            counts[t][v] += 1
    for t in range(len(S)):
        assert _chi2_pvalue(counts[t], n / S[t]) > 1e-4, t


def test_initial_genome_streams_differ_by_rank_and_slot():
    S = np.array([4] * 8, np.int32)
    a = [tuple(ga.initial_genome(S, 1, 0, k)[1]) for k in range(200)]
    b = [tuple(ga.initial_genome(S, 1, 1, k)[1]) for k in range(200)]
    assert len(set(a)) > 190 and a != b
