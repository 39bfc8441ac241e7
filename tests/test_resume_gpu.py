"""Search-state checkpoint / resume (SURVEY.md §5 "Checkpoint / resume"; saturn.h
saturn_search_save / saturn_search_resume).

A search is deterministic in (params, world), and generation g's children depend only on
generation g-1's population, makespans and elites plus the Philox streams (k, g, rank): so
search(G1) -> save -> resume(G2) on a fresh handle must return exactly what search(G1+G2)
returns -- final population, makespans, best plan.  The continuous search itself is replayed
against oracle/ga.py by test_gpu_parity.py; here the resumed one is held to it bit for bit.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


@pytest.fixture(scope="module")
def sat(torch):
    import paper_2309_01226_b200 as s
    s.load_library()
    return s


def _plan(sat, inst):
    return sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)


def _cfg(sat, gens, P, epoch):
    return sat.SearchConfig(seed=23, population=P, max_generations=gens, elites=8, generations_per_epoch=epoch)


@pytest.mark.parametrize("name,P,g1,g2,epoch", [("TXT", 4096, 5, 7, 4), ("TXT", 3000, 8, 4, 4),
                                                 ("MIX", 2048, 3, 3, 2), ("SWEEP", 1024, 2, 3, 1),
                                                 ("TINY", 512, 0, 6, 3)])
def test_resume_equals_continuous_search(sat, torch, name, P, g1, g2, epoch):
    inst = synth.by_name(name, 0)
    full = _plan(sat, inst)
    rf = full.search(_cfg(sat, g1 + g2, P, epoch))
    cf, qf, mf = full.search_population()
    bf = full.best_plan()

    first = _plan(sat, inst)
    first.search(_cfg(sat, g1, P, epoch))
    state = first.search_save()
    assert state.nbytes > P * (2 * inst.n_jobs + 4)
    del first
    second = _plan(sat, inst)
    rr = second.search_resume(state, _cfg(sat, g2, P, epoch))
    cr, qr, mr = second.search_population()
    br = second.best_plan()
    assert rr["generations"] == g2 and rf["generations"] == g1 + g2
    assert rr["makespan"] == rf["makespan"]
    assert rr["evaluated"] == g2 * (P - 8)
    assert np.array_equal(cf, cr) and np.array_equal(qf, qr) and np.array_equal(mf, mr)
    assert bf[0] == br[0] and bf[1] == br[1]
    # the resumed handle can be saved again: its state is at generation g1 + g2
    s2 = second.search_save()
    assert s2.nbytes == state.nbytes
    assert int(np.frombuffer(s2[48:56].tobytes(), np.int64)[0]) == g1 + g2


def test_resume_rejects_mismatches(sat, torch):
    inst = synth.txt(0)
    plan = _plan(sat, inst)
    cfg = _cfg(sat, 2, 1024, 2)
    plan.search(cfg)
    state = plan.search_save()
    fresh = _plan(sat, inst)

    def rejected(st, c, status=None):
        with pytest.raises(sat.SaturnError) as ei:
            fresh.search_resume(st, c)
        assert ei.value.status == (status or sat.EINVAL)

    rejected(state, sat.SearchConfig(seed=24, population=1024, max_generations=2, elites=8))   # seed
    rejected(state, sat.SearchConfig(seed=23, population=2048, max_generations=2, elites=8))   # population
    rejected(state, sat.SearchConfig(seed=23, population=1024, max_generations=2, elites=4))   # elites
    rejected(state[:-1], cfg)                                                                  # truncated
    bad = state.copy()
    bad[0] ^= 1
    rejected(bad, cfg)                                                                         # magic
    bad = state.copy()
    bad[-1] ^= 1
    rejected(bad, cfg)                                                                         # checksum
    other = _plan(sat, synth.txt(1))                                                           # another table
    with pytest.raises(sat.SaturnError) as ei:
        other.search_resume(state, cfg)
    assert ei.value.status == sat.EINVAL
    # a payload whose checksum is consistent but whose genome is invalid (duplicate gene)
    import ctypes
    hdr = 80   # sizeof(SearchStateHeader); payload_hash at bytes 64..72
    bad = state.copy()
    T = inst.n_jobs
    Tp = (T + 3) & ~3
    bad[hdr + Tp] = bad[hdr + Tp + 1]
    h = 1469598103934665603
    for b in bad[hdr:].tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    bad[64:72] = np.frombuffer(ctypes.c_uint64(h), np.uint8)
    with pytest.raises(sat.SaturnError) as ei:
        fresh.search_resume(bad, cfg)
    assert ei.value.status == sat.EINVAL and "invalid" in str(ei.value)
    # nothing saved yet
    with pytest.raises(sat.SaturnError) as ei:
        fresh.search_save()
    assert ei.value.status == sat.ESTATE
