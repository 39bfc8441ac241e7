"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, bit for bit.

Integer work (makespans, schedules, enumeration (makespan, index), GA children) must be
identical; no tolerance anywhere.  Inputs are seeded (synth/); sizes span several tiles
and a ragged tail.  Run under gpurun: python -m pytest tests -m gpu
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import ga as oga

pytestmark = pytest.mark.gpu

CONFIGS = ("TINY", "TXT", "IMG", "MIX", "SWEEP")


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


def _ms(plan, torch, cfg, perm):
    return plan.evaluate(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda()).cpu().numpy()


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("decoder", ["thread", "warp"])
def test_evaluate_matches_oracle(sat, torch, name, decoder):
    inst = synth.by_name(name, seed=1)
    plan = _plan(sat, inst)
    plan.set_decoder(sat.DECODER_THREAD if decoder == "thread" else sat.DECODER_WARP)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    assert list(plan.num_configs()) == list(c.S)
    n = 20000 if name != "SWEEP" else 5003
    cfg, perm = synth.random_genomes(c.S, n, seed=11)
    got = _ms(plan, torch, cfg, perm)
    ref = oracle.decode_batch(c, cfg, perm)
    assert (ref > 0).all()
    assert np.array_equal(got, ref), np.nonzero(got != ref)[0][:10]


@pytest.mark.parametrize("n", [1, 2, 127, 128, 129, 1000, 4097])
def test_evaluate_ragged_sizes(sat, torch, n):
    inst = synth.txt(2)
    plan = _plan(sat, inst)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    cfg, perm = synth.random_genomes(c.S, n, seed=n)
    assert np.array_equal(_ms(plan, torch, cfg, perm), oracle.decode_batch(c, cfg, perm))


def test_evaluate_unaligned_buffers_use_plain_loads(sat, torch):
    inst = synth.mix(0)
    plan = _plan(sat, inst)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    n = 3001
    cfg, perm = synth.random_genomes(c.S, n, seed=5)
    T = c.n_jobs
    big_c = torch.zeros(n * T + 1, dtype=torch.uint8, device="cuda")
    big_p = torch.zeros(n * T + 1, dtype=torch.uint8, device="cuda")
    big_c[1:] = torch.from_numpy(cfg.reshape(-1)).cuda()
    big_p[1:] = torch.from_numpy(perm.reshape(-1)).cuda()
    got = plan.evaluate(big_c[1:].view(n, T), big_p[1:].view(n, T)).cpu().numpy()
    assert np.array_equal(got, oracle.decode_batch(c, cfg, perm))


def test_evaluate_invalid_genomes(sat, torch):
    inst = synth.txt(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    for decoder in (sat.DECODER_THREAD, sat.DECODER_WARP):
        plan = _plan(sat, inst)
        plan.set_decoder(decoder)
        cfg, perm = synth.random_genomes(c.S, 300, seed=9)
        perm[0, 3] = perm[0, 4]          # duplicate job
        perm[1, 0] = 200                 # job id out of range
        cfg[2, 5] = c.S[5]               # config out of range
        got = _ms(plan, torch, cfg, perm)
        ref = oracle.decode_batch(c, cfg, perm)
        assert list(got[:3]) == [-1, -1, -1] and list(ref[:3]) == [-1, -1, -1]
        assert np.array_equal(got, ref)


def test_evaluate_host_path(sat, torch):
    inst = synth.img(3)
    plan = _plan(sat, inst)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    cfg, perm = synth.random_genomes(c.S, 10000, seed=4)
    assert np.array_equal(plan.evaluate_host(cfg, perm), oracle.decode_batch(c, cfg, perm))


def test_heterogeneous_clusters(sat, torch):
    """{2,2,4,8} and 8+4 (PAPER.md:1118-style) on both decoders."""
    for nodes in ([2, 2, 4, 8], [8, 4], [3, 5], [1, 1, 1]):
        inst = synth.sweep(7, n_jobs=30, nodes=nodes)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        cfg, perm = synth.random_genomes(c.S, 3000, seed=len(nodes))
        ref = oracle.decode_batch(c, cfg, perm)
        for decoder in (sat.DECODER_AUTO, sat.DECODER_WARP):
            plan = _plan(sat, inst)
            plan.set_decoder(decoder)
            assert np.array_equal(_ms(plan, torch, cfg, perm), ref), (nodes, decoder)


@pytest.mark.parametrize("name", CONFIGS)
def test_trace_matches_oracle_schedules(sat, torch, name):
    inst = synth.by_name(name, seed=4)
    plan = _plan(sat, inst)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    n = 300
    cfg, perm = synth.random_genomes(c.S, n, seed=3)
    pl, ms = plan.trace(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda())
    rec = pl.cpu().numpy().view(sat.PLACEMENT_DTYPE).reshape(n, c.n_jobs)
    ms = ms.cpu().numpy()
    for i in range(n):
        ref_ms, ref_pl = oracle.decode(c, cfg[i], perm[i])
        assert ms[i] == ref_ms
        for t in range(c.n_jobs):
            r, o = rec[i, t], ref_pl[t]
            assert (r["node"], r["upp"], r["gpus"], r["cfg"], r["start_s"], r["end_s"], r["gpu_mask"]) == \
                (o["node"], o["upp"], o["gpus"], o["cfg"], o["start_s"], o["end_s"], o["gpu_mask"]), (i, t)


def test_hand_traces_on_device(sat, torch, golden_dir):
    import json
    import os
    from conftest import dense_from_single
    cases = json.load(open(os.path.join(golden_dir, "hand_traces.json")))["cases"]
    for case in cases:
        table = dense_from_single(case["jobs"])
        plan = sat.Plan(case["nodes"], 0).load_runtime_table(table)
        T = len(case["jobs"])
        cfg = np.zeros((1, T), np.uint8)
        perm = np.array([case["order"]], np.uint8)
        for decoder in (sat.DECODER_THREAD, sat.DECODER_WARP):
            plan.set_decoder(decoder)
            assert _ms(plan, torch, cfg, perm)[0] == case["makespan"], case["id"]
        if "starts" in case:
            pl, _ = plan.trace(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda())
            rec = pl.cpu().numpy().view(sat.PLACEMENT_DTYPE).reshape(T)
            assert list(rec["start_s"]) == case["starts"]
            assert list(rec["gpu_mask"]) == case["masks"]


# ------------------------------------------------------------------ enumerate
def test_enumerate_tiny_matches_brute_force(sat, torch):
    for seed in range(5):
        inst = synth.tiny(seed)
        plan = _plan(sat, inst)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        r = plan.enumerate()
        assert (r["makespan"], r["genome_index"]) == oracle.brute_force(c)
        assert r["flags"] & sat.PROVEN_OPTIMAL and r["flags"] & sat.PREFIX_SHARED
        assert r["evaluated"] == 0 and 0 < r["leaves"] <= 1296   # §8d: pruned plans never counted
        best, pl, bc, bp = plan.best_plan()
        ms, opl = oracle.decode(c, bc, bp)
        assert ms == best == r["makespan"]
        assert oracle.validate(c, pl, best) == []


@pytest.mark.parametrize("jobs,nodes", [(4, (4,)), (5, (4,)), (4, (2, 2)), (5, (2, 2)), (6, (2, 2))])
def test_enumerate_tiny_variants(sat, torch, jobs, nodes):
    inst = synth.tiny_variant(jobs * 10 + len(nodes), jobs, nodes)
    plan = _plan(sat, inst)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    N = oracle.space_size(c)
    assert plan.space_size() == N
    r = plan.enumerate()
    if N <= 3_000_000:
        assert (r["makespan"], r["genome_index"]) == oracle.brute_force(c)
    else:  # oracle on the winning genome + a sampled slice
        cfg, perm = oracle.unrank(c, r["genome_index"])
        assert oracle.decode(c, cfg, perm)[0] == r["makespan"]
        b = r["genome_index"] - r["genome_index"] % 100000
        sub = plan.enumerate_range(b, min(b + 100000, N))
        assert (sub["makespan"], sub["genome_index"]) == oracle.brute_force(c, b, min(b + 100000, N))


def test_enumerate_ranges_compose_like_multi_gpu(sat, torch):
    """The min over any partition of the index space = the whole-space result (the
    W-invariance of the multi-GPU enumeration, reading A7)."""
    inst = synth.tiny_variant(45, 5, (2, 2))
    plan = _plan(sat, inst)
    N = plan.space_size()
    whole = plan.enumerate()
    for W in (2, 3, 8):
        parts = [plan.enumerate_range(*sat.partition(N, r, W)) for r in range(W)]
        best = min((p["makespan"], p["genome_index"]) for p in parts)
        assert best == (whole["makespan"], whole["genome_index"])
    c = oracle.compact(inst.node_gpus, inst.runtime)
    assert plan.enumerate_range(17, 12345)["makespan"] == oracle.brute_force(c, 17, 12345)[0]


def test_enumerate_limits(sat, torch):
    inst = synth.txt(0)
    plan = _plan(sat, inst)
    with pytest.raises(sat.SaturnError) as e:
        plan.enumerate()
    assert e.value.status == sat.ELIMIT


# ------------------------------------------------------------------ GA search
def test_ga_operator_replay_bit_exact(sat, torch):
    """Initial population and several generations reproduced by the oracle's operator
    definitions (oracle/ga.py) from the same seed: identical genomes and makespans."""
    inst = synth.txt(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    P, E, seed = 256, 4, 12345
    px, pc, pm = oga.q32(0.9), oga.q32(0.25), oga.q32(0.5)
    cfg, perm = oga.initial_population(c.S, P, seed)
    ms = oracle.decode_batch(c, cfg, perm)
    plan = _plan(sat, inst)
    for G in (0, 1, 3):
        plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=G, elites=E,
                                     generations_per_epoch=1, p_xover=0.9, p_cfg_mut=0.25, p_perm_mut=0.5))
        gc, gq, gm = plan.search_population(P)
        rc, rq, rm = cfg, perm, ms
        for gen in range(1, G + 1):
            rc, rq, _ = oga.next_generation(c.S, rc, rq, rm, gen, seed, 0, E, px, pc, pm)
            rm = oracle.decode_batch(c, rc, rq)
        assert np.array_equal(gc, rc) and np.array_equal(gq, rq) and np.array_equal(gm, rm), G


def test_ga_replay_with_seed_genomes_and_sweep(sat, torch):
    inst = synth.sweep(1)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    P, E, seed = 128, 8, 99
    sc, sq = synth.random_genomes(c.S, 5, seed=2)
    cfg, perm = oga.initial_population(c.S, P, seed, seed_cfg=sc, seed_perm=sq)
    ms = oracle.decode_batch(c, cfg, perm)
    rc, rq, _ = oga.next_generation(c.S, cfg, perm, ms, 1, seed, 0, E, oga.q32(0.9), oga.q32(0.01), oga.q32(0.5))
    rm = oracle.decode_batch(c, rc, rq)
    plan = _plan(sat, inst)
    plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=1, elites=E, generations_per_epoch=1,
                                 p_xover=0.9, p_cfg_mut=0.01, p_perm_mut=0.5), seed_genomes=(sc, sq))
    gc, gq, gm = plan.search_population(P)
    assert np.array_equal(gc, rc) and np.array_equal(gq, rq) and np.array_equal(gm, rm)


def test_search_best_is_valid_and_monotone(sat, torch):
    inst = synth.txt(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    plan = _plan(sat, inst)
    r = plan.search(sat.SearchConfig(seed=1, population=1 << 14, max_generations=40, elites=16,
                                     generations_per_epoch=4))
    best, pl, bc, bp = plan.best_plan()
    assert best == r["makespan"]
    ms, opl = oracle.decode(c, bc, bp)
    assert ms == best and oracle.validate(c, pl, best) == []
    assert best >= oracle.lower_bound(c)
    ts, hist = plan.search_history()
    # one record per epoch (after generation 0, every 4 generations, and the final exchange),
    # device seconds since the search's first operation: non-decreasing, best non-increasing
    assert len(hist) == 1 + 40 // 4 + 1 and hist[-1] == best
    assert all(a >= b for a, b in zip(hist, hist[1:]))
    assert ts[0] > 0 and all(a <= b for a, b in zip(ts, ts[1:])) and ts[-1] <= r["seconds"]
    assert r["evaluated"] == (1 << 14) + 40 * ((1 << 14) - 16)
    # determinism
    r2 = plan.search(sat.SearchConfig(seed=1, population=1 << 14, max_generations=40, elites=16,
                                      generations_per_epoch=4))
    assert r2["makespan"] == r["makespan"] and (plan.best_plan()[2] == bc).all()


def test_search_reaches_optimum_on_tiny(sat, torch):
    for seed in range(3):
        inst = synth.tiny(seed)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        opt = oracle.brute_force(c)[0]
        plan = _plan(sat, inst)
        r = plan.search(sat.SearchConfig(seed=seed, population=256, max_generations=20, elites=4))
        assert r["makespan"] == opt


def test_int_probe_runs(sat, torch):
    plan = _plan(sat, synth.txt(0))
    v = plan.probe_int_peak()
    assert 1e12 < v < 1e14


def test_nccl_single_rank_communicator_path(sat, torch):
    """The multi-GPU code path (NCCL MIN all-reduce for enumeration, elite all-gather +
    device merge for search) run with a 1-rank communicator on the one GPU: identical
    results to the communicator-free path."""
    inst = synth.tiny_variant(45, 5, (2, 2))
    a = _plan(sat, inst)
    b = _plan(sat, inst)
    b.attach_comm(sat.get_unique_id(), 0, 1)
    ra, rb = a.enumerate(), b.enumerate()
    assert (ra["makespan"], ra["genome_index"]) == (rb["makespan"], rb["genome_index"])
    txt = synth.txt(0)
    a, b = _plan(sat, txt), _plan(sat, txt)
    b.attach_comm(sat.get_unique_id(), 0, 1)
    cfgs = sat.SearchConfig(seed=5, population=4096, max_generations=12, elites=8, generations_per_epoch=3)
    sa, sb = a.search(cfgs), b.search(cfgs)
    assert sa["makespan"] == sb["makespan"]
    assert (a.best_plan()[2] == b.best_plan()[2]).all()
    assert (a.search_population(4096)[0] == b.search_population(4096)[0]).all()


def test_multinode_shared_memory_decoder(sat, torch):
    """The NN = 0 decoder (node vectors in shared memory, runtime node count): the default
    for node counts without a compiled register shape, selected here (SATURN_DECODER_NODE_SMEM)
    on every multi-node case and on one node."""
    for inst in (synth.mix(2), synth.sweep(2), synth.sweep(5, n_jobs=20, nodes=[2, 2, 4, 8]),
                 synth.sweep(6, n_jobs=16, nodes=[4] * 8), synth.txt(4)):
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _plan(sat, inst)
        plan.set_decoder(sat.DECODER_NODE_SMEM)
        cfg, perm = synth.random_genomes(c.S, 3001, seed=8)
        assert np.array_equal(_ms(plan, torch, cfg, perm), oracle.decode_batch(c, cfg, perm))
    tv = synth.tiny_variant(3, 5, (2, 2))   # index-order enumeration on the smem shape = brute force
    ct = oracle.compact(tv.node_gpus, tv.runtime)
    tp = _plan(sat, tv)
    tp.set_decoder(sat.DECODER_NODE_SMEM)
    r = tp.enumerate()
    assert (r["makespan"], r["genome_index"]) == oracle.brute_force(ct)
    inst = synth.mix(1)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    P, E, seed = 128, 4, 77
    cfg, perm = oga.initial_population(c.S, P, seed)
    ms = oracle.decode_batch(c, cfg, perm)
    rc, rq, _ = oga.next_generation(c.S, cfg, perm, ms, 1, seed, 0, E, oga.q32(0.9), oga.q32(0.5), oga.q32(0.5))
    plan = _plan(sat, inst)
    plan.set_decoder(sat.DECODER_NODE_SMEM)
    plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=1, elites=E, generations_per_epoch=1,
                                 p_xover=0.9, p_cfg_mut=0.5, p_perm_mut=0.5))
    gc, gq, gm = plan.search_population(P)
    assert np.array_equal(gc, rc) and np.array_equal(gq, rq) and np.array_equal(gm, oracle.decode_batch(c, rc, rq))


def test_long_genome_ga_on_column_states_replays_oracle(sat, torch):
    """Long genomes (T > 32) on column node states: each child's parents are staged in
    shared memory with cp.async (X into the child row, Y into the idle state region) before
    crossover and LOX -- SWEEP (4x8, T = 100) and a 3-node T = 40 instance on the run-time
    node-count shape, two generations replayed by oracle/ga.py bit for bit."""
    for inst in (synth.sweep(3), synth.sweep(7, n_jobs=40, nodes=[8, 4, 2])):
        c = oracle.compact(inst.node_gpus, inst.runtime)
        P, E, seed = 256, 8, 4242
        px, pc, pm = oga.q32(0.9), oga.q32(0.3), oga.q32(0.6)
        cfg, perm = oga.initial_population(c.S, P, seed)
        rm = oracle.decode_batch(c, cfg, perm)
        rc, rq = cfg, perm
        for gen in (1, 2):
            rc, rq, _ = oga.next_generation(c.S, rc, rq, rm, gen, seed, 0, E, px, pc, pm)
            rm = oracle.decode_batch(c, rc, rq)
        plan = _plan(sat, inst)
        plan.set_decoder(sat.DECODER_NODE_SMEM)
        plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=2, elites=E, generations_per_epoch=1,
                                     p_xover=0.9, p_cfg_mut=0.3, p_perm_mut=0.6))
        gc, gq, gm = plan.search_population(P)
        assert np.array_equal(gc, rc) and np.array_equal(gq, rq) and np.array_equal(gm, rm)


# ------------------------------------------------------------------ f4: local search
@pytest.mark.parametrize("name,n,iters", [("TXT", 24, 6), ("MIX", 8, 3), ("TINY", 16, 4)])
def test_improve_matches_oracle_local_search(sat, torch, name, n, iters):
    from oracle.local_search import improve
    inst = synth.by_name(name, seed=3)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    plan = _plan(sat, inst)
    cfg, perm = synth.random_genomes(c.S, n, seed=21)
    gc, gq, gm = plan.improve(cfg, perm, iters)
    before = oracle.decode_batch(c, cfg, perm)
    for i in range(n):
        rc, rq, rm = improve(c, cfg[i], perm[i], iters)
        assert (list(gc[i]), list(gq[i]), int(gm[i])) == (list(rc), list(rq), rm), i
        assert rm <= before[i]


def test_memetic_search_replays(sat, torch):
    """Search with the memetic elite step: population after 2 generations = oracle replay of
    (top-E -> local search -> re-sort) at every epoch boundary."""
    from oracle.local_search import improve
    inst = synth.txt(1)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    P, E, seed, iters = 128, 4, 31, 2
    px, pc, pm = oga.q32(0.9), oga.q32(0.5), oga.q32(0.5)
    cfg, perm = oga.initial_population(c.S, P, seed)
    ms = oracle.decode_batch(c, cfg, perm)

    def elites_after_ls(cfg, perm, ms):
        recs = []
        for i in oga.elites(ms, E):
            rc, rq, rm = improve(c, cfg[i], perm[i], iters)
            recs.append((rm, rc, rq))
        order = sorted(range(E), key=lambda k: (recs[k][0], k))
        return [recs[k] for k in order]

    for gen in (1, 2):
        recs = elites_after_ls(cfg, perm, ms)
        cfg, perm, _ = oga.next_generation(c.S, cfg, perm, ms, gen, seed, 0, E, px, pc, pm, elite_records=recs)
        ms = oracle.decode_batch(c, cfg, perm)
    plan = _plan(sat, inst)
    r = plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=2, elites=E, generations_per_epoch=1,
                                     p_xover=0.9, p_cfg_mut=0.5, p_perm_mut=0.5, local_search_iters=iters))
    gc, gq, gm = plan.search_population(P)
    assert np.array_equal(gc, cfg) and np.array_equal(gq, perm) and np.array_equal(gm, ms)
    best, pl, bc, bp = plan.best_plan()
    assert oracle.decode(c, bc, bp)[0] == best == r["makespan"] <= int(ms.min())


@pytest.mark.parametrize("k,epoch,gens,ls", [(2, 1, 2, 0), (3, 2, 5, 0), (2, 2, 3, 2)])
def test_island_group_replays_migration(sat, torch, k, epoch, gens, ls):
    """Row e on one GPU: k islands (saturn_search_group) = oracle replay of k ranks with
    migrate() at every epoch boundary (PAPER.md:232-236 search over the shared plan space;
    DESIGN.md reading A9) -- every island's population is bit-exact."""
    from oracle.local_search import improve
    inst = synth.txt(2)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    P, E, seed = 128, 4, 77
    px, pc, pm = oga.q32(0.9), oga.q32(0.5), oga.q32(0.5)
    pops = []
    for r in range(k):
        cfg, perm = oga.initial_population(c.S, P, seed, rank=r)
        pops.append((cfg, perm, oracle.decode_batch(c, cfg, perm)))

    def records(cfg, perm, ms):
        recs = [(int(ms[i]), cfg[i].copy(), perm[i].copy()) for i in oga.elites(ms, E)]
        if ls:
            recs = [improve(c, rc, rq, ls) for _, rc, rq in recs]
            recs = [(rm, np.asarray(rc, np.uint8), np.asarray(rq, np.uint8)) for rc, rq, rm in recs]
            recs = [recs[j] for j in sorted(range(E), key=lambda j: (recs[j][0], j))]
        return recs

    merged = oga.migrate([records(*pp) for pp in pops])
    for gen in range(1, gens + 1):
        nxt = []
        for r, (cfg, perm, ms) in enumerate(pops):
            cfg, perm, _ = oga.next_generation(c.S, cfg, perm, ms, gen, seed, r, E, px, pc, pm, elite_records=merged)
            nxt.append((cfg, perm, oracle.decode_batch(c, cfg, perm)))
        pops = nxt
        merged = oga.migrate([records(*pp) for pp in pops]) if gen % epoch == 0 else None
    plans = [_plan(sat, inst) for _ in range(k)]
    res = sat.search_group(plans, sat.SearchConfig(seed=seed, population=P, max_generations=gens, elites=E,
                                                   generations_per_epoch=epoch, p_xover=0.9, p_cfg_mut=0.5,
                                                   p_perm_mut=0.5, local_search_iters=ls))
    final = oga.migrate([records(*pp) for pp in pops])
    for r in range(k):
        gc, gq, gm = plans[r].search_population(P)
        assert np.array_equal(gc, pops[r][0]) and np.array_equal(gq, pops[r][1]), r
        assert np.array_equal(gm, pops[r][2]), r
        best, pl, bc, bp = plans[r].best_plan()
        assert best == res[r]["makespan"] == final[0][0]
        assert oracle.decode(c, bc, bp)[0] == best
        assert res[r]["evaluated"] == k * (P + gens * (P - E))


def test_island_group_rejects_mismatched_handles(sat, torch):
    inst = synth.txt(2)
    a = _plan(sat, inst)
    b = _plan(sat, synth.txt(3))
    with pytest.raises(sat.SaturnError):
        sat.search_group([a, b], sat.SearchConfig(population=128, elites=4, max_generations=1))
    with pytest.raises(sat.SaturnError):
        sat.search_group([a, a], sat.SearchConfig(population=128, elites=4, max_generations=1))


# ------------------------------------------------------------------ f4: node genes
def test_node_genes_match_oracle(sat, torch):
    for inst in (synth.mix(3), synth.sweep(2, n_jobs=40), synth.sweep(4, n_jobs=30, nodes=[2, 2, 4, 8]),
                 synth.sweep(5, n_jobs=30, nodes=[8, 4]), synth.txt(1)):
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _plan(sat, inst)
        n = 4000
        cfg, perm = synth.random_genomes(c.S, n, seed=13)
        rng = np.random.default_rng(3)
        N = len(inst.node_gpus)
        node = rng.integers(0, N + 1, size=(n, c.n_jobs)).astype(np.uint8)
        node[node == N] = 0xFF                              # some greedy genes
        node[: n // 2] = np.where(rng.random((n // 2, c.n_jobs)) < 0.5, 0xFF, node[: n // 2])
        node[0, 0] = N + 3                                  # a missing node -> invalid
        got = plan.evaluate_nodes(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda(),
                                  torch.from_numpy(node).cuda()).cpu().numpy()
        ref = oracle.decode_batch_nodes(c, cfg, perm, node)
        assert got[0] == -1 and np.array_equal(got, ref)
        greedy = np.full_like(node, 0xFF)
        got = plan.evaluate_nodes(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda(),
                                  torch.from_numpy(greedy).cuda()).cpu().numpy()
        assert np.array_equal(got, oracle.decode_batch(c, cfg, perm))


def test_baseline_per_node_plans_match_oracle(sat, torch):
    """Row f2 with node genes (reading A16): every baseline genome decoded on the device with
    saturn_baseline_nodes' genes equals the oracle's node-gene decode of the oracle's genome."""
    from oracle import baselines as ob
    for inst in (synth.mix(0), synth.sweep(0), synth.sweep(4, n_jobs=30, nodes=[2, 2, 4, 8])):
        c = oracle.compact(inst.node_gpus, inst.runtime)
        plan = _plan(sat, inst)
        for kind in ob.KINDS:
            for seed in (0, 5):
                gc, gq = plan.baseline_genome(kind, seed)
                gn = plan.baseline_nodes(kind, seed)
                got = plan.evaluate_nodes(torch.from_numpy(gc[None]).cuda(), torch.from_numpy(gq[None]).cuda(),
                                          torch.from_numpy(gn[None]).cuda()).cpu().numpy()[0]
                rc, rq = ob.KINDS[kind](c, seed)
                assert got == oracle.decode(c, rc, rq, node_gene=ob.baseline_nodes(c, kind, seed))[0], (kind, seed)


def test_node_gene_space_reaches_the_exact_optimum(sat, torch):
    """Completeness: min over all (cfg, node, perm) genomes, decoded on the
    GPU, equals the independent time-indexed exact optimum (O4a)."""
    import itertools
    from oracle.exact import exact_makespan
    for seed in range(6):
        rng = np.random.default_rng(900 + seed)
        inst = synth.random_tiny(rng, max_jobs=3, node_choices=([2, 2], [2, 3], [3, 1]), max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        T, N = c.n_jobs, len(inst.node_gpus)
        rows = []
        for cf in itertools.product(*[range(int(s)) for s in c.S]):
            for nd in itertools.product(range(N), repeat=T):
                for pm in itertools.permutations(range(T)):
                    rows.append((cf, nd, pm))
        cfg = np.array([r[0] for r in rows], np.uint8).reshape(-1, T)
        node = np.array([r[1] for r in rows], np.uint8).reshape(-1, T)
        perm = np.array([r[2] for r in rows], np.uint8).reshape(-1, T)
        plan = _plan(sat, inst)
        ms = plan.evaluate_nodes(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda(),
                                 torch.from_numpy(node).cuda()).cpu().numpy()
        assert np.array_equal(ms, oracle.decode_batch_nodes(c, cfg, perm, node))
        assert ms[ms >= 0].min() == exact_makespan(c)


# ------------------------------------------------------------------ edge cases
def _edge_instances():
    rng = np.random.default_rng(77)

    def table(T, U, G, p=0.6, r=(1, 50)):
        t = np.where(rng.random((T, U, G)) < p, rng.integers(r[0], r[1], size=(T, U, G)), 0).astype(np.int32)
        t[:, 0, 0] = rng.integers(r[0], r[1], size=T)     # every job has a 1-GPU config
        return t
    return [
        ("T=1", [4], table(1, 2, 4)),
        ("T=255", [8, 8], table(255, 2, 8, r=(1, 200))),
        ("1x32", [32], table(20, 2, 32)),
        ("32x1", [1] * 32, table(40, 2, 1)),
        ("16x2", [2] * 16, table(30, 3, 2)),
        ("3x5x7", [3, 5, 7], table(25, 4, 7)),
    ]


@pytest.mark.parametrize("idx", range(6))
def test_edge_shapes_evaluate_search_replay(sat, torch, idx):
    name, nodes, tab = _edge_instances()[idx]
    c = oracle.compact(nodes, tab)
    plan = sat.Plan(nodes, 0).load_runtime_table(tab)
    cfg, perm = synth.random_genomes(c.S, 700, seed=idx)
    ref = oracle.decode_batch(c, cfg, perm)
    for decoder in (sat.DECODER_AUTO, sat.DECODER_WARP):
        plan.set_decoder(decoder)
        assert np.array_equal(_ms(plan, torch, cfg, perm), ref), (name, decoder)
    plan.set_decoder(sat.DECODER_AUTO)
    P, E, seed = 96, 4, 3 + idx
    g_cfg, g_perm = oga.initial_population(c.S, P, seed)
    g_ms = oracle.decode_batch(c, g_cfg, g_perm)
    rc, rq, _ = oga.next_generation(c.S, g_cfg, g_perm, g_ms, 1, seed, 0, E, oga.q32(0.9), oga.q32(0.5),
                                    oga.q32(0.5))
    plan.search(sat.SearchConfig(seed=seed, population=P, max_generations=1, elites=E, generations_per_epoch=1,
                                 p_xover=0.9, p_cfg_mut=0.5, p_perm_mut=0.5))
    gc, gq, gm = plan.search_population(P)
    assert np.array_equal(gc, rc) and np.array_equal(gq, rq), name
    assert np.array_equal(gm, oracle.decode_batch(c, rc, rq)), name
    best, pl, bc, bp = plan.best_plan()
    ms, opl = oracle.decode(c, bc, bp)
    assert ms == best and oracle.validate(c, pl, best) == [], name
    if c.n_jobs == 1:
        r = plan.enumerate()
        assert (r["makespan"], r["genome_index"]) == oracle.brute_force(c)


def test_c_example_runs_on_the_gpu(sat, torch, tmp_path):
    import os
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "saturn_demo"
    libdir = os.path.dirname(sat.LIB_PATH)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "saturn_demo.c"), "-L", libdir, "-lsaturn",
                           "-Wl,-rpath," + libdir, "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    opt = int(out.stdout.split("exhaustive optimum")[1].split("makespan ")[1].split()[0])
    ga = int(out.stdout.split("GA search")[1].split("makespan ")[1].split()[0])
    assert ga >= opt



def test_dfs_enumeration_equals_index_order_enumeration(sat, torch):
    """The prefix-sharing branch-and-bound DFS (saturn_enumerate) returns exactly the
    (makespan, smallest index) of the full-decode index-order kernel on the whole space."""
    cases = [synth.tiny_variant(7, 7, (4,)), synth.tiny_variant(8, 6, (2, 2)), synth.tiny_variant(9, 5, (4,)),
             synth.tiny_variant(3, 8, (4,))]
    for inst in cases:
        plan = _plan(sat, inst)
        N = plan.space_size()
        dfs = plan.enumerate()
        assert dfs["flags"] & sat.PREFIX_SHARED and dfs["evaluated"] == 0 and 0 < dfs["leaves"] <= N
        full = plan.enumerate_range(0, N)
        assert full["evaluated"] == N   # index order: one full decode per genome
        assert (dfs["makespan"], dfs["genome_index"]) == (full["makespan"], full["genome_index"]), inst.name
        c = oracle.compact(inst.node_gpus, inst.runtime)
        cfg, perm = oracle.unrank(c, dfs["genome_index"])
        assert oracle.decode(c, cfg, perm)[0] == dfs["makespan"]


@pytest.mark.parametrize("n_lrs,nodes", [((2, 2, 1), (4,)), ((3, 3), (2, 2)), ((3, 2, 1), (4,)), ((1, 1, 1, 1, 1), (4,))])
def test_dfs_symmetry_reduction_matches_oracle(sat, torch, n_lrs, nodes):
    """Row f4: enumeration with SATURN_ENUM_SYMMETRY = oracle brute force over canonical genomes
    (oracle/symmetry.py), bit-exact (makespan, index); the makespan equals the unreduced one."""
    from oracle import symmetry as sym
    inst = synth.lr_sweep(5, len(n_lrs), n_lrs, nodes)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    plan = _plan(sat, inst)
    full = plan.enumerate()
    plan.set_enumeration_options(symmetry=True)
    red = plan.enumerate()
    want = sym.brute_force_canonical(c)
    assert (red["makespan"], red["genome_index"]) == want
    assert red["makespan"] == full["makespan"]
    twins = any(p >= 0 for p in sym.twin_prev(c))
    assert bool(red["flags"] & sat.SYMMETRY_REDUCED) == twins
    if twins:
        assert red["leaves"] <= full["leaves"]
    else:
        assert red["genome_index"] == full["genome_index"]
    best, pl, bc, bp = plan.best_plan()
    assert best == red["makespan"] and sym.is_canonical(c, bp)
    plan.set_enumeration_options(symmetry=False)
    assert plan.enumerate()["genome_index"] == full["genome_index"]


# ------------------------------------------------------------------ bench scale
@pytest.mark.parametrize("name", ["TXT", "MIX", "SWEEP"])
def test_bench_scale_search_sampled_replay(sat, torch, name):
    """The launch configuration bench.py times (P = 2^23 genomes, E = 16, epochs of 8,
    seed 2309) at BASELINE.json's full sizes: generation 16 is checked against the oracle on
    sampled slots -- every sampled child is rebuilt from generation 15 by oga.make_child and
    decoded by the C oracle; the 16 elites are generation 15's best (ms, slot); every genome
    of the final population is a valid (cfg, perm); the reported best is the population
    minimum and its trace re-validates."""
    inst = synth.by_name(name, 0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    # SWEEP (T = 100: parent B read from global memory, the LOX bit set in shared memory) at
    # 2^20 genomes to bound the host copies (2 x 200 MB) and the Python replay
    P, E, seed = (1 << 23) if name != "SWEEP" else (1 << 20), 16, 2309
    base = dict(seed=seed, population=P, elites=E, generations_per_epoch=8)
    px, pc, pm = oga.q32(0.9), oga.q32(0.5), oga.q32(0.5)
    plan = _plan(sat, inst)
    plan.search(sat.SearchConfig(max_generations=15, **base))
    c15, q15, m15 = plan.search_population(P)
    r = plan.search(sat.SearchConfig(max_generations=16, **base))
    c16, q16, m16 = plan.search_population(P)
    T = c.n_jobs
    # validity of every genome (vectorised): perm is a permutation, cfg < S_t
    assert (np.sort(q16, axis=1) == np.arange(T, dtype=np.uint8)).all()
    assert (c16 < np.asarray(c.S, np.uint8)[None, :]).all()
    # elites: generation 15's E best by (ms, slot), carried with their makespans
    order = np.lexsort((np.arange(P), m15))[:E]
    assert np.array_equal(c16[:E], c15[order]) and np.array_equal(q16[:E], q15[order])
    assert np.array_equal(m16[:E], m15[order])
    # sampled children: operator replay + oracle decode
    rng = np.random.default_rng(7)
    slots = np.unique(np.concatenate([rng.integers(E, P, 1500 if name != "SWEEP" else 400), [E, E + 1, P - 2, P - 1]]))
    kids = [oga.make_child(c.S, c15, q15, m15, int(k), 16, seed, 0, px, pc, pm) for k in slots]
    kc = np.array([k[0] for k in kids], np.uint8)
    kq = np.array([k[1] for k in kids], np.uint8)
    assert np.array_equal(c16[slots], kc) and np.array_equal(q16[slots], kq)
    assert np.array_equal(m16[slots], oracle.decode_batch(c, kc, kq))
    # the reported best = population minimum (a generation-16 child may beat the carried
    # elites at slots 0..E-1); its plan re-validates
    assert r["makespan"] == int(m16.min()) <= int(m16[0]) == int(m15.min())
    best, pl, bc, bp = plan.best_plan()
    ms, _ = oracle.decode(c, bc, bp)
    assert ms == best == r["makespan"] and oracle.validate(c, pl, best) == []


def test_empty_inputs(sat, torch):
    """Degenerate sizes: evaluating zero genomes is a no-op (output untouched), an empty
    enumeration range reports nothing found, and the first/last single-genome ranges equal
    the oracle's decode of those indices."""
    inst = synth.tiny(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    plan = _plan(sat, inst)
    T = c.n_jobs
    out = torch.full((4,), -7, dtype=torch.int32, device="cuda")
    plan.evaluate(torch.zeros((0, T), dtype=torch.uint8, device="cuda"),
                  torch.zeros((0, T), dtype=torch.uint8, device="cuda"), out[:0])
    assert (out.cpu().numpy() == -7).all()
    r = plan.enumerate_range(5, 5)
    assert r["evaluated"] == 0
    size = plan.space_size()
    for i in (0, size - 1):
        r = plan.enumerate_range(i, i + 1)
        assert r["evaluated"] == 1 and r["genome_index"] == i
        cfg, perm = oracle.unrank(c, i)
        assert r["makespan"] == oracle.decode(c, cfg, perm)[0]


def test_profiling_samples_generations(sat, torch):
    """saturn_set_profiling(n): CUDA events around every n-th GA generation kernel."""
    inst = synth.txt(0)
    plan = _plan(sat, inst)
    cfg = sat.SearchConfig(seed=1, population=4096, max_generations=16, elites=8, generations_per_epoch=4)
    for per, want in ((0, 0), (1, 16), (4, 4), (16, 1)):
        plan.set_profiling(per)
        plan.reset_stats()
        plan.search(cfg)
        st = plan.stats()
        assert st["ga_launches"] == want, (per, st)
        assert (st["ga_kernel_ms"] > 0) == (want > 0)
        assert st["ga_decodes"] == want * (4096 - 8)


# ------------------------------------------------------------------ §8b workspace
@pytest.mark.parametrize("name", ["TXT", "MIX"])
def test_bound_workspace_search_bit_identical(sat, torch, name):
    """saturn_bind_workspace: a torch.empty(saturn_workspace_bytes) buffer carries every
    device allocation of a search + best_plan, and the result is bit-identical to the same
    search on handle-owned (cudaMalloc) memory; one byte short of the requirement -> ELIMIT."""
    inst = synth.by_name(name, 1)
    cfg = sat.SearchConfig(seed=11, population=1 << 14, max_generations=6, elites=8, generations_per_epoch=3)
    ref = _plan(sat, inst)
    r0 = ref.search(cfg)
    c0, q0, m0 = ref.search_population()
    b0 = ref.best_plan()
    plan = _plan(sat, inst)
    need = plan.workspace_bytes(cfg)
    assert need > 2 * (1 << 14) * 32
    ws = plan.bind_workspace(need)
    assert ws.numel() == need and ws.device.type == "cuda"
    r1 = plan.search(cfg)
    c1, q1, m1 = plan.search_population()
    b1 = plan.best_plan()
    assert (r0["makespan"], r0["evaluated"]) == (r1["makespan"], r1["evaluated"])
    assert np.array_equal(c0, c1) and np.array_equal(q0, q1) and np.array_equal(m0, m1)
    assert b0[0] == b1[0] and b0[1] == b1[1]
    # the handle's buffers really live inside the tensor: zeroing it destroys the population
    ws.zero_()
    torch.cuda.synchronize()
    assert (plan.search_population()[2] == 0).all()
    # too small a workspace: ELIMIT, not a crash or a silent cudaMalloc
    small = _plan(sat, inst)
    small.bind_workspace(small.workspace_bytes(cfg) - 4096)
    with pytest.raises(sat.SaturnError) as ei:
        small.search(cfg)
    assert ei.value.status == sat.ELIMIT
    # unbinding returns to handle-owned memory
    small.bind_workspace(None)
    r2 = small.search(cfg)
    assert r2["makespan"] == r0["makespan"]


def test_search_population_capacity(sat, torch):
    """search_population never writes past the caller's capacity."""
    inst = synth.txt(0)
    plan = _plan(sat, inst)
    plan.search(sat.SearchConfig(seed=1, population=4096, max_generations=2, elites=8))
    with pytest.raises(sat.SaturnError):
        plan.search_population(1024)
    c, q, m = plan.search_population()
    assert c.shape == (4096, inst.n_jobs) and m.shape == (4096,)


# ------------------------------------------------------------------ f3: GPU plans vs the paper's MILP rows
@pytest.mark.parametrize("which", ["TXT", "MIX", "HETERO"])
def test_gpu_best_plan_satisfies_paper_milp(sat, torch, which):
    """f3: the plan the CUDA path returns (search, then
    the trace decoder's placements) written as the paper's variables B, O, P, A, I, C violates
    no row of the paper's MILP (Eqs. 1-11, readings A1-A3), and its C equals the makespan."""
    from oracle.milp import SpaseMilp
    inst = {"TXT": lambda: synth.txt(0), "MIX": lambda: synth.mix(0),
            "HETERO": lambda: synth.sweep(5, n_jobs=20, nodes=[2, 2, 4, 8])}[which]()
    c = oracle.compact(inst.node_gpus, inst.runtime)
    plan = _plan(sat, inst)
    r = plan.search(sat.SearchConfig(seed=4, population=1 << 14, max_generations=24, elites=8,
                                     generations_per_epoch=8))
    best, pl, bc, bp = plan.best_plan()
    assert best == r["makespan"]
    m = SpaseMilp(c)
    x = m.plan_to_assignment(pl, best)
    assert m.violations(x) == []
    assert x[m.idx[("C",)]] == max(p["end_s"] for p in pl) == best
