"""GA operator replay (oracle/ga.py) invariants.  The GA is a heuristic, so its trajectory
is unpinned by the paper; what is pinned:
operators emit valid genomes, elitism keeps the best, OX1 keeps A's slice and B's
relative order, and everything is a pure function of (seed, counters)."""
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


def test_ox1_keeps_slice_and_order():
    from oracle.philox import Stream
    c, cfg, perm, ms = _setup(P=16)
    T = c.n_jobs
    # force crossover, no mutation
    for slot in range(4, 16):
        child_cfg, child_perm = ga.make_child(c.S, cfg, perm, ms, slot, 1, 3, 0,
                                              p_x=0xFFFFFFFF, p_c=0, p_m=0)
        st = Stream((3, 0), slot, 1, 0)
        i, j = st.below(16), st.below(16)
        A = i if (ms[i], i) < (ms[j], j) else j
        i, j = st.below(16), st.below(16)
        B = i if (ms[i], i) < (ms[j], j) else j
        st.u32()
        w = st.u32()
        a, b = sorted((st.below(T), st.below(T)))
        assert list(child_perm[a:b + 1]) == list(perm[A][a:b + 1])
        rest = [x for x in np.roll(perm[B], -(b + 1)) if x not in set(perm[A][a:b + 1])]
        filled = [child_perm[(b + 1 + k) % T] for k in range(T - (b - a + 1))]
        assert filled == rest
        for t in range(T):
            assert child_cfg[t] == (cfg[A][t] if (w >> t) & 1 else cfg[B][t])


def test_migration_takes_global_best():
    recs = [[(5, "a0", None), (9, "a1", None)], [(5, "b0", None), (6, "b1", None)]]
    got = ga.migrate(recs)
    assert [r[1] for r in got] == ["a0", "b0"]
