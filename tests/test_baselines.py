"""Row f2: the paper's baselines (Alg. 1 at 949-962) as genomes.

The oracle reference (oracle/baselines.py) is pinned by SPEC.md's worked values; the
library (saturn_baseline_genome, host code, exercised on a host-only handle -- no GPU) must
produce the same genomes bit for bit."""
import numpy as np
import pytest

import oracle
import synth
from oracle import baselines as ob
from conftest import dense_from_configs

import paper_2309_01226_b200 as sat


def _c(nodes, configs):
    return oracle.compact(nodes, dense_from_configs(configs))


def test_alg1_spec_examples():
    # R_A = [100, 60, 50, 45], R_B = [80, 50, 40, 35], G = 4 -> [2, 2]
    RA = {1: 100, 2: 60, 3: 50, 4: 45}
    RB = {1: 80, 2: 50, 3: 40, 4: 35}
    assert ob.optimus_greedy_alloc([RA, RB], 4) == [2, 2]
    assert ob.optimus_greedy_alloc([RA, RB], 2) == [1, 1]          # G = |T|
    assert ob.optimus_greedy_alloc([{1: 90, 2: 50, 3: 40}], 3) == [3]
    assert ob.optimus_greedy_alloc([{1: 9}, {1: 9}], 6) == [1, 1]   # all gains -inf: early stop


def test_min_heuristic_spec_examples():
    # 2 tasks on a 4-GPU node -> (2, 2); 3 tasks -> (2, 1, 1)
    full = [(3, 1, 90), (1, 2, 50), (1, 3, 40), (1, 4, 30)]
    for n_tasks, want in ((2, [2, 2]), (3, [2, 1, 1])):
        c = _c([4], [full] * n_tasks)
        cfg, _ = ob.min_heuristic(c)
        assert [c.config(t, cfg[t])[1] for t in range(n_tasks)] == want
    c = _c([2], [full[:2]] * 2)
    cfg, _ = ob.min_heuristic(c)
    assert [c.config(t, cfg[t])[1] for t in range(2)] == [1, 1]


def test_max_heuristic_and_lpt_examples():
    # 2 tasks, full-width runtime 6, one node -> 12
    c = _c([2], [[(1, 1, 10), (1, 2, 6)]] * 2)
    cfg, perm = ob.max_heuristic(c)
    assert oracle.decode(c, cfg, perm)[0] == 12
    # L = [2, 2] on 4 GPUs, runtimes 60 / 50 -> 60; on 2 GPUs -> sum
    c = _c([4], [[(0, 2, 60)], [(0, 2, 50)]])
    cfg, perm = ob.optimus_greedy(c)
    assert list(perm) == [0, 1] and oracle.decode(c, cfg, perm)[0] == 60
    c = _c([2], [[(0, 2, 60)], [(0, 2, 50)]])
    assert oracle.decode(c, *ob.optimus_greedy(c))[0] == 110


def test_best_config_tie_goes_to_lower_upp():
    c = _c([4], [[(2, 2, 50), (1, 2, 50), (0, 1, 90)]])
    s, r = ob.best_config_for(c, 0, 2)
    assert r == 50 and c.config(0, s)[0] == 1   # FSDP before PIPE


def test_distribute_weights():
    # nodes (8, 4) -> 2/3 : 1/3 within +-2 % over 10,000 draws
    c = oracle.compact([8, 4], np.full((10000, 1, 1), 7, np.int32))
    node = ob.distribute(c, seed=3)
    frac = np.bincount(node, minlength=2) / len(node)
    assert abs(frac[0] - 2 / 3) < 0.02 and abs(frac[1] - 1 / 3) < 0.02


@pytest.mark.parametrize("name", ["TINY", "TXT", "IMG", "MIX", "SWEEP"])
def test_baseline_plans_are_valid_and_above_lb(name):
    inst = synth.by_name(name, 0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    lb = oracle.lower_bound(c)
    for kind, f in ob.KINDS.items():
        cfg, perm = f(c, 0)
        ms, pl = oracle.decode(c, np.array(cfg, np.uint8), np.array(perm, np.uint8))
        assert ms >= lb and oracle.validate(c, pl, ms) == [], kind


def _host_plan(inst):
    return sat.Plan(inst.node_gpus, device=-1).load_runtime_table(inst.runtime)


@pytest.mark.parametrize("name", ["TINY", "TXT", "IMG", "MIX", "SWEEP"])
def test_library_baselines_match_oracle(name):
    for seed in (0, 1, 7):
        inst = synth.by_name(name, seed)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _host_plan(inst)
        assert list(plan.num_configs()) == list(c.S)
        for kind, f in ob.KINDS.items():
            cfg, perm = plan.baseline_genome(kind, seed)
            rc, rp = f(c, seed)
            assert list(cfg) == list(rc) and list(perm) == list(rp), (name, seed, kind)


def test_library_baselines_heterogeneous_and_random_tiny():
    for nodes in ([2, 2, 4, 8], [8, 4], [3, 5], [1, 1, 1]):
        inst = synth.sweep(3, n_jobs=30, nodes=nodes)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _host_plan(inst)
        for kind, f in ob.KINDS.items():
            cfg, perm = plan.baseline_genome(kind, 11)
            rc, rp = f(c, 11)
            assert list(cfg) == list(rc) and list(perm) == list(rp), (nodes, kind)
    rng = np.random.default_rng(0)
    for _ in range(50):
        inst = synth.random_tiny(rng, max_jobs=5, max_r=9)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _host_plan(inst)
        for kind, f in ob.KINDS.items():
            cfg, perm = plan.baseline_genome(kind, 5)
            rc, rp = f(c, 5)
            assert list(cfg) == list(rc) and list(perm) == list(rp), (inst.runtime, kind)


def test_host_only_handle_refuses_device_work():
    inst = synth.txt(0)
    plan = _host_plan(inst)
    with pytest.raises(sat.SaturnError) as e:
        plan.search(sat.SearchConfig(population=64, max_generations=1, elites=4))
    assert e.value.status == sat.ESTATE
    with pytest.raises(sat.SaturnError):
        plan.enumerate()


# ---------------------------------------------------------------- per-node plans (node genes)
def test_baseline_nodes_single_node_and_greedy_fallback():
    """One node: every baseline job is on node 0 and the node-gene decode is the greedy one.
    Two nodes {4, 2} with a job whose narrowest width is 4: wherever distribute() sends it to
    the 2-GPU node its gene is 0xFF (greedy), every other gene is the distributed node."""
    c = _c([8], [[(0, 1, 90), (0, 2, 50), (1, 4, 30)]] * 3)
    for kind in ("max", "min", "optimus"):
        cfg, perm = ob.KINDS[kind](c, 0)
        assert ob.baseline_nodes(c, kind, 0) == [0, 0, 0]
        assert oracle.decode(c, cfg, perm, node_gene=[0, 0, 0])[0] == oracle.decode(c, cfg, perm)[0]
    assert ob.baseline_nodes(c, "random", 0) == [0xFF] * 3
    wide = [(0, 4, 40), (1, 4, 35)]
    small = [(0, 1, 60), (0, 2, 35)]
    c = _c([4, 2], [wide, small, wide, small, wide, small])
    hits = 0
    for seed in range(20):
        d = ob.distribute(c, seed)
        for kind in ("max", "min", "optimus"):
            nodes = ob.baseline_nodes(c, kind, seed)
            for t in range(6):
                if t % 2 == 0 and d[t] == 1:
                    assert nodes[t] == 0xFF
                    hits += 1
                else:
                    assert nodes[t] == d[t]
    assert hits > 0


@pytest.mark.parametrize("name", ["MIX", "SWEEP"])
def test_baseline_node_genes_give_per_node_schedules(name):
    """Decoded with its node genes, every baseline plan is valid (O3) and runs each job on
    its gene's node: the per-node plan of the paper's heuristics."""
    inst = synth.by_name(name, 0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    for kind in ("max", "min", "optimus"):
        cfg, perm = ob.KINDS[kind](c, 2)
        nodes = ob.baseline_nodes(c, kind, 2)
        ms, pl = oracle.decode(c, cfg, perm, node_gene=nodes)
        assert ms > 0 and oracle.validate(c, pl, ms) == []
        assert all(pl[t]["node"] == nodes[t] for t in range(c.n_jobs) if nodes[t] != 0xFF)


def test_library_baseline_nodes_match_oracle():
    cases = [synth.by_name(n, s) for n in ("TXT", "MIX", "SWEEP") for s in (0, 3)]
    cases += [synth.sweep(3, n_jobs=30, nodes=nodes) for nodes in ([2, 2, 4, 8], [8, 4], [3, 5], [1, 1, 1])]
    for inst in cases:
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _host_plan(inst)
        for kind in ob.KINDS:
            for seed in (0, 9):
                assert list(plan.baseline_nodes(kind, seed)) == ob.baseline_nodes(c, kind, seed), (inst.node_gpus, kind)
