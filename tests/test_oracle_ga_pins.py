"""Hand-worked pins of the GA operator definition (oracle/ga.py make_child, DESIGN.md "GA
definition"), independent of the oracle's own code path: the pair's Philox words are
replaced by words chosen by hand, and every child below was derived on paper from the
definition in oracle/ga.py's header (tournaments -> copy of X -> complementary uniform
crossover -> LOX -> config mutation -> permutation mutation).  The GA is this build's
design (the paper's optimiser is a MILP), so these pins fix its text,
not a paper value."""
import numpy as np
import pytest

import oracle.ga as oga

T = 5
S = [3, 2, 4, 1, 2]
P = 8


def _population():
    cfg = np.zeros((P, T), np.uint8)
    perm = np.tile(np.arange(T, dtype=np.uint8), (P, 1))
    ms = np.full(P, 200, np.int32)
    cfg[3], perm[3], ms[3] = [2, 1, 3, 0, 1], [4, 0, 3, 1, 2], 100   # A: wins the tie with slot 5
    ms[5] = 100
    cfg[6], perm[6], ms[6] = [0, 0, 1, 0, 0], [1, 2, 0, 4, 3], 90    # B: beats slot 1
    ms[1] = 95
    return cfg, perm, ms


def _words(perm_mut_r0=True, kind_r0=1, cfg_mut_r0=True, perm_mut_r1=False, kind_r1=0, cfg_mut_r1=False):
    w = [0] * 16
    w[0], w[1] = 3 << 29, 5 << 29            # U(8, .) = 3, 5: tie at ms 100 -> slot 3 (A)
    w[2], w[3] = 6 << 29, 1 << 29            # 6 (ms 90) vs 1 (ms 95) -> slot 6 (B)
    w[4] = (39322 << 16) | 100               # crossover gate fires; a = V(5, 39322) = 3
    w[5] = 13108                             # b = V(5, 13108) = 1  -> cuts swapped to (1, 3)
    w[6] = 0b10110                           # crossover bits: t = 0, 3 from Y; t = 1, 2, 4 from X
    # child 0 (block 2): insertion (kind 1) of position i = 4 at j = 0; job 2 gets gene 2
    w[8] = (52429 << 16) | (0 if perm_mut_r0 else 0xFFFF)    # i = V(5, 52429) = 4
    w[9] = (kind_r0 << 16) | 0                                 # j = 0
    w[10] = (26215 << 16) | (0 if cfg_mut_r0 else 0xFFFF)     # t* = V(5, 26215) = 2
    w[11] = 32768                                              # new gene V(4, 32768) = 2
    # child 1 (block 3)
    w[12] = (13108 << 16) | (0 if perm_mut_r1 else 0xFFFF)    # i = 1
    w[13] = (kind_r1 << 16) | 52429                            # j = 4
    w[14] = (0 << 16) | (0 if cfg_mut_r1 else 0xFFFF)         # t* = 0
    w[15] = 32768                                              # new gene V(3, 32768) = 1
    return w


def _child(monkeypatch, slot, **kw):
    cfg, perm, ms = _population()
    words = _words(**kw)
    monkeypatch.setattr(oga, "pair_words", lambda *a, **k: list(words))
    c, p = oga.make_child(S, cfg, perm, ms, slot, 1, 0, 0, oga.q32(0.9), oga.q32(0.5), oga.q32(0.5))
    return [int(x) for x in c], [int(x) for x in p]


def test_child0_hand_worked(monkeypatch):
    # X = A = slot 3, Y = B = slot 6.  cfg: t0 <- Y 0, t1 X 1, t2 X 3, t3 <- Y 0, t4 X 1;
    # LOX (1, 3): keep [0, 3, 1], fill [2, 4] -> [2, 0, 3, 1, 4]; cfg[2] = 2;
    # insertion: gene at 4 (4) moved to 0 -> [4, 2, 0, 3, 1]
    assert _child(monkeypatch, 2) == ([0, 1, 2, 0, 1], [4, 2, 0, 3, 1])


def test_child1_hand_worked_roles_swapped(monkeypatch):
    # X = B = slot 6, Y = A = slot 3.  cfg: t0 <- A 2, t1 B 0, t2 B 1, t3 <- A 0, t4 B 0;
    # LOX (1, 3): keep [2, 0, 4], fill from A [3, 1] -> [3, 2, 0, 4, 1]; no mutation fires
    assert _child(monkeypatch, 3) == ([2, 0, 1, 0, 0], [3, 2, 0, 4, 1])


def test_child0_swap_mutation(monkeypatch):
    # kind 0 swaps positions 4 and 0 of [2, 0, 3, 1, 4]; no config mutation
    assert _child(monkeypatch, 2, kind_r0=0, cfg_mut_r0=False) == ([0, 1, 3, 0, 1], [4, 0, 3, 1, 2])


def test_child1_insertion_forward(monkeypatch):
    # child 1 with an insertion of position 1 at 4: [3, 2, 0, 4, 1] -> [3, 0, 4, 1, 2];
    # its config mutation: job 0 gets gene V(3, 32768) = 1
    assert _child(monkeypatch, 3, perm_mut_r1=True, kind_r1=1, cfg_mut_r1=True) == ([1, 0, 1, 0, 0],
                                                                                    [3, 0, 4, 1, 2])


def test_no_crossover_copies_x(monkeypatch):
    cfg, perm, ms = _population()
    words = _words(perm_mut_r0=False, cfg_mut_r0=False)
    words[4] = (39322 << 16) | 0xFFFF        # gate lo = 65535 >= p_x >> 16: no crossover, no LOX
    monkeypatch.setattr(oga, "pair_words", lambda *a, **k: list(words))
    c, p = oga.make_child(S, cfg, perm, ms, 2, 1, 0, 0, oga.q32(0.9), oga.q32(0.5), oga.q32(0.5))
    assert [int(x) for x in c] == [2, 1, 3, 0, 1] and [int(x) for x in p] == [4, 0, 3, 1, 2]


@pytest.mark.parametrize("a,b,expect", [(0, 4, [4, 0, 3, 1, 2]), (2, 2, [1, 2, 3, 0, 4]), (0, 0, [4, 1, 2, 0, 3])])
def test_lox_edge_cuts(a, b, expect):
    # A = [4, 0, 3, 1, 2], B = [1, 2, 0, 4, 3]: whole slice -> A; one gene kept in place;
    # slice at 0 -> B's remaining genes fill positions 1..4
    assert oga.lox([4, 0, 3, 1, 2], [1, 2, 0, 4, 3], a, b) == expect
