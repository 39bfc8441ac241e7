"""GA operator replay (oracle/ga.py) invariants.  The GA is a heuristic, so its trajectory
is unpinned by the paper; what is pinned:
operators emit valid genomes, elitism keeps the best, LOX keeps A's slice in place and
B's relative order (plus a hand-worked LOX example), and everything is a pure function of (seed, counters)."""
import numpy as np

import oracle
from oracle import ga
import synth


def _setup(P=64, seed=0):
    inst = synth.txt(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    cfg, perm = ga.initial_population(c.S, P, seed)
    ms = oracle.decode_batch(c, cfg, perm)
    return c, cfg, perm, ms


def test_initial_population_valid_and_deterministic():
    c, cfg, perm, ms = _setup()
    assert (ms > 0).all()
    for i in range(cfg.shape[0]):
        assert sorted(perm[i]) == list(range(c.n_jobs))
        assert (cfg[i] < c.S).all()
    cfg2, perm2 = ga.initial_population(c.S, 64, 0)
    assert (cfg2 == cfg).all() and (perm2 == perm).all()
    cfg3, _ = ga.initial_population(c.S, 64, 1)
    assert (cfg3 != cfg).any()


def test_children_valid_and_elites_kept():
    c, cfg, perm, ms = _setup()
    E = 4
    best_before = int(ms.min())
    for gen in range(1, 6):
        ncfg, nperm, ems = ga.next_generation(c.S, cfg, perm, ms, gen, seed=7, rank=0, E=E,
                                             p_x=ga.q32(0.9), p_c=ga.q32(1 / 12), p_m=ga.q32(0.5))
        nms = oracle.decode_batch(c, ncfg, nperm)
        assert (nms[:E] == np.array(ems)).all()          # elites carry their makespans
        assert (nms >= 0).all()                          # every child is a valid genome
        assert nms.min() <= best_before                   # best-so-far non-increasing
        best_before = int(nms.min())
        cfg, perm, ms = ncfg, nperm, nms


def test_lox_hand_example():
    # A = 0..7, B = 7..0, slice [2..4] = (2 3 4) stays; B without {2,3,4} in B's order is
    # 7 6 5 1 0: positions 0..1 <- 7 6, positions 5..7 <- 5 1 0.
    assert ga.lox(list(range(8)), list(range(7, -1, -1)), 2, 4) == [7, 6, 2, 3, 4, 5, 1, 0]
    # slice at the front / back and the whole permutation
    assert ga.lox([0, 1, 2, 3], [3, 2, 1, 0], 0, 1) == [0, 1, 3, 2]
    assert ga.lox([0, 1, 2, 3], [3, 2, 1, 0], 2, 3) == [1, 0, 2, 3]
    assert ga.lox([0, 1, 2, 3], [3, 2, 1, 0], 0, 3) == [0, 1, 2, 3]
    assert ga.lox([2, 0, 1], [1, 2, 0], 1, 1) == [1, 0, 2]


def test_lox_keeps_slice_and_order():
    """GA v5: slots 2q, 2q+1 are the children of pair q (stream (q, gen, rank << 16)); child 0
    keeps A's slice and fills in B's order, child 1 the reverse; the config genes are split
    complementarily by the crossover bits (bit 1 -> the child's own parent X)."""
    from oracle.philox import Stream
    c, cfg, perm, ms = _setup(P=16)
    T = c.n_jobs
    # force crossover, no mutation
    for slot in range(4, 16):
        child_cfg, child_perm = ga.make_child(c.S, cfg, perm, ms, slot, 1, 3, 0,
                                              p_x=0xFFFFFFFF, p_c=0, p_m=0)
        st = Stream((3, 0), slot >> 1, 1, 0)
        w = [st.u32() for _ in range(8)]
        i, j = (w[0] * 16) >> 32, (w[1] * 16) >> 32
        A = i if (ms[i], i) < (ms[j], j) else j
        i, j = (w[2] * 16) >> 32, (w[3] * 16) >> 32
        B = i if (ms[i], i) < (ms[j], j) else j
        X, Y = (A, B) if slot % 2 == 0 else (B, A)
        a, b = sorted((((w[4] >> 16) * T) >> 16, ((w[5] & 0xFFFF) * T) >> 16))
        assert list(child_perm[a:b + 1]) == list(perm[X][a:b + 1])
        rest = [x for x in perm[Y] if x not in set(perm[X][a:b + 1])]
        filled = list(child_perm[:a]) + list(child_perm[b + 1:])
        assert filled == rest
        for t in range(T):
            assert child_cfg[t] == (cfg[X][t] if (w[6] >> t) & 1 else cfg[Y][t])


def test_pair_children_complementary():
    """Both children of a pair, no mutation: every config gene of A and B goes to exactly one
    child (uniform crossover's two offspring), and each child is a valid genome."""
    c, cfg, perm, ms = _setup(P=32)
    T = c.n_jobs
    for q in range(2, 16):
        c0, p0 = ga.make_child(c.S, cfg, perm, ms, 2 * q, 3, 5, 0, p_x=0xFFFFFFFF, p_c=0, p_m=0)
        c1, p1 = ga.make_child(c.S, cfg, perm, ms, 2 * q + 1, 3, 5, 0, p_x=0xFFFFFFFF, p_c=0, p_m=0)
        assert sorted(p0) == list(range(T)) and sorted(p1) == list(range(T))
        # the multiset {c0[t], c1[t]} is the parents' {A[t], B[t]} for some parent pair
        found = False
        for A in range(32):
            for B in range(32):
                if all(sorted((int(c0[t]), int(c1[t]))) == sorted((int(cfg[A][t]), int(cfg[B][t])))
                       for t in range(T)):
                    found = True
                    break
            if found:
                break
        assert found


def test_mutation_only_changes_what_fired():
    c, cfg, perm, ms = _setup(P=32)
    T = c.n_jobs
    for slot in range(4, 32):
        # no crossover, certain config mutation of one job, no perm mutation
        cc, cp = ga.make_child(c.S, cfg, perm, ms, slot, 2, 9, 0, p_x=0, p_c=0xFFFFFFFF, p_m=0)
        cc0, cp0 = ga.make_child(c.S, cfg, perm, ms, slot, 2, 9, 0, p_x=0, p_c=0, p_m=0)
        assert all(0 <= cc[t] < c.S[t] for t in range(T))
        assert sum(int(x != y) for x, y in zip(cc, cc0)) <= 1 and list(cp) == list(cp0)
        cm, pmut = ga.make_child(c.S, cfg, perm, ms, slot, 2, 9, 0, p_x=0, p_c=0, p_m=0xFFFFFFFF)
        assert sorted(pmut) == list(range(T)) and list(cm) == list(cc0)
        # nothing fires: the child is parent A
        cc0, cp0 = ga.make_child(c.S, cfg, perm, ms, slot, 2, 9, 0, p_x=0, p_c=0, p_m=0)
        assert any((list(cfg[k]) == list(cc0) and list(perm[k]) == list(cp0)) for k in range(32))


def test_migration_takes_global_best():
    recs = [[(5, "a0", None), (9, "a1", None)], [(5, "b0", None), (6, "b1", None)]]
    got = ga.migrate(recs)
    assert [r[1] for r in got] == ["a0", "b0"]
