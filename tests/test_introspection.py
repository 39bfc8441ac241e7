"""Row f1: round introspection.  Oracle pins on CPU; the library's
saturn_introspect with the exact solver must reproduce the oracle round by round (GPU)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import introspection as oi
from conftest import dense_from_single, dense_from_configs


def _pl(start, end, node=0, mask=1, cfg=0):
    return dict(node=node, upp=0, gpus=1, cfg=cfg, start_s=start, end_s=end, gpu_mask=mask)


def test_residual_spec_examples():
    # runtime 10 from 0, advance 10 -> done; advance 4 -> 0.6 left;
    # from 8, advance 10 -> 0.8 left.  Reading A10 keeps every config, scaled and ceiled.
    table = dense_from_configs([[(0, 1, 10), (1, 2, 7)]])
    assert oi.residual(table, [_pl(0, 10)], 10)[0] is None
    t2, keep, S = oi.residual(table, [_pl(0, 10)], 4)
    assert keep == [0] and list(t2[0].ravel()[t2[0].ravel() > 0]) == [6, 5]   # 10*.6, ceil(7*.6)
    assert S[0]["start_s"] == 0 and S[0]["end_s"] == 6
    t3, _, S = oi.residual(table, [_pl(8, 18)], 10)
    assert list(t3[0].ravel()[t3[0].ravel() > 0]) == [8, 6]                    # 10*.8, ceil(7*.8)
    t4, _, S = oi.residual(table, [_pl(12, 22)], 10)                            # not started
    assert list(t4[0].ravel()[t4[0].ravel() > 0]) == [10, 7] and S[0]["start_s"] == 2


@pytest.mark.parametrize("seed", range(6))
def test_introspection_invariants(seed):
    rng = np.random.default_rng(seed)
    inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [3], [2, 2]), max_r=9)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    opt = oracle.brute_force(c)[0]
    never = oi.introspect(inst.node_gpus, inst.runtime, I=3, T=10 ** 6)
    assert never["one_shot"] == opt and never["e2e"] == opt and never["adopted"] == 0
    eager = oi.introspect(inst.node_gpus, inst.runtime, I=3, T=0)
    assert eager["e2e"] <= opt
    for time, M, Mp, take in eager["log"]:
        assert take == int(Mp <= M)


def test_introspection_can_beat_one_shot():
    """Re-planning lets a running job change its width: 2 jobs on 2 GPUs, job A has
    (1 GPU, 10 s) / (2 GPUs, 4 s), job B (1 GPU, 4 s).  One-shot optimum 8 (A on 2 GPUs, then B;
    or both at once = 10).  After B finishes at I = 4, A (started at 0 on 1 GPU in the
    [A 1-GPU, B 1-GPU] plan) can be relaunched on 2 GPUs."""
    table = dense_from_configs([[(0, 1, 10), (0, 2, 4)], [(0, 1, 4)]])
    one = oi.introspect([2], table, I=4, T=10 ** 6)
    eager = oi.introspect([2], table, I=4, T=0)
    assert one["e2e"] == one["one_shot"] == 8
    assert eager["e2e"] <= 8


@pytest.mark.gpu
def test_library_introspection_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2309_01226_b200 as sat
    n = 0
    for seed in range(12):
        rng = np.random.default_rng(100 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [3], [4], [2, 2]), max_r=12)
        for I, T in ((3, 0), (4, 2), (5, 10 ** 6)):
            ref = oi.introspect(inst.node_gpus, inst.runtime, I=I, T=T)
            plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
            got, log = plan.introspect(I, T, solver="enumerate")
            assert (got["one_shot_makespan"], got["e2e_makespan"], got["rounds"], got["adopted"]) == \
                (ref["one_shot"], ref["e2e"], ref["rounds"], ref["adopted"]), (seed, I, T)
            assert [tuple(x) for x in ref["log"]] == log
            n += got["rounds"]
    assert n > 20
    # the SWEEP-shaped workload re-planned at the paper's knobs with the GA: never worse
    inst = synth.mix(0)
    plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
    got, log = plan.introspect(1000, 500, solver="search",
                               search=sat.SearchConfig(seed=1, population=1 << 14, max_generations=20, elites=8,
                                                       generations_per_epoch=5))
    assert got["e2e_makespan"] <= got["one_shot_makespan"] and got["rounds"] == len(log) > 5
