"""Pins for oracle/symmetry.py (row f4, symmetry reduction for identical jobs).

The reduction's claim -- relabelling twins keeps the makespan, so the canonical minimum is the
global minimum (reading A14) -- is checked here by brute force over whole genome
spaces, not by re-stating the argument."""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import symmetry as sym


def _twin_instance(rng):
    """A random tiny instance with some rows duplicated (exact twins)."""
    base = synth.random_tiny(rng, max_jobs=3, max_r=6)
    rows = [base.runtime[t] for t in range(base.runtime.shape[0])]
    T = int(rng.integers(3, 6))
    table = np.stack([rows[int(rng.integers(len(rows)))] for _ in range(T)])
    return oracle.compact(base.node_gpus, table)


@pytest.mark.parametrize("seed", range(12))
def test_canonical_minimum_equals_global_minimum(seed):
    rng = np.random.default_rng(1000 + seed)
    c = _twin_instance(rng)
    if oracle.space_size(c) > 400_000:
        pytest.skip("space too large for the pin's budget")
    ms_all, idx_all = oracle.brute_force(c)
    ms_can, idx_can = sym.brute_force_canonical(c)
    assert ms_can == ms_all
    cfg, perm = oracle.unrank(c, idx_can)
    assert sym.is_canonical(c, perm) and oracle.decode(c, cfg, perm)[0] == ms_can
    assert idx_can >= idx_all


def test_canonicalize_preserves_makespan_and_is_canonical():
    inst = synth.lr_sweep(3, 3, (3, 1, 2), nodes=(2, 2))
    c = oracle.compact(inst.node_gpus, inst.runtime)
    assert sym.twin_prev(c) == [-1, 0, 1, -1, -1, 4]
    cfg, perm = synth.random_genomes(c.S, 500, 7)
    before = oracle.decode_batch(c, cfg, perm)
    can = [sym.canonicalize(c, cfg[i], perm[i]) for i in range(len(cfg))]
    after = oracle.decode_batch(c, np.stack([x[0] for x in can]), np.stack([x[1] for x in can]))
    assert np.array_equal(before, after)
    assert all(sym.is_canonical(c, x[1]) for x in can)
    # a canonical genome is its own canonical form
    for x in can[:50]:
        y = sym.canonicalize(c, *x)
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


def test_canonical_count_closed_form():
    inst = synth.lr_sweep(1, 2, (3, 2))
    c = oracle.compact(inst.node_gpus, inst.runtime)
    n_perm = sum(1 for p in itertools.permutations(range(5)) if sym.is_canonical(c, p))
    assert n_perm == math.factorial(5) // (math.factorial(3) * math.factorial(2)) == 10
    assert sym.n_canonical(c) == 10 * int(np.prod(c.S))


def test_twins_need_equal_gpu_counts_not_just_runtimes():
    # job 0: DDP g=1 R=5, DDP g=2 R=3;  job 1: DDP g=2 R=5, FSDP g=1 R=3 -> same R list [5, 3]
    table = np.array([[[5, 3], [0, 0]], [[0, 5], [3, 0]]], np.int32)
    c = oracle.compact([2], table)
    assert [int(x) for x in c.runtime[:2]] == [5, 3] and [int(x) for x in c.runtime[c.stride:c.stride + 2]] == [5, 3]
    assert sym.twin_prev(c) == [-1, -1]
    assert sym.n_canonical(c) == oracle.space_size(c)
