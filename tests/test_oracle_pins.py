"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each pin is independent of the oracle's own code: hand-worked traces and SPEC.md values
(tests/golden/hand_traces.json), textbook special cases, invariants, an independent
time-indexed exact solver (O4a), the paper's own MILP solved by HiGHS (O4b), and brute
force on tiny inputs.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.exact import exact_makespan
from oracle.milp import SpaseMilp, milp_makespan
from conftest import dense_from_configs, dense_from_single
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _golden(golden_dir):
    with open(os.path.join(golden_dir, "hand_traces.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- O1 hand traces
@pytest.mark.parametrize("case_id", ["H1", "H2", "H3", "H4", "H4b", "PCMAX-LPT", "ANOMALY-8", "ANOMALY-11"])
def test_hand_traces(golden_dir, case_id):
    case = next(c for c in _golden(golden_dir)["cases"] if c["id"] == case_id)
    c = oracle.compact(case["nodes"], dense_from_single(case["jobs"]))
    T = len(case["jobs"])
    ms, pl = oracle.decode(c, np.zeros(T, np.uint8), np.array(case["order"], np.uint8))
    assert ms == case["makespan"]
    assert oracle.validate(c, pl, ms) == []
    if "starts" in case:
        assert [p["start_s"] for p in pl] == case["starts"]
        assert [p["node"] for p in pl] == case["nodes_of_jobs"]
        assert [p["gpu_mask"] for p in pl] == case["masks"]
    if "optimum" in case:
        assert oracle.brute_force(c)[0] == case["optimum"]


def test_pcmax_list_scheduling_is_graham():
    """All jobs 1-GPU with one config on one node is P||Cmax and O1 is Graham's list
    scheduling: each job goes to the machine that frees first.  Check against a direct
    heap implementation of list scheduling on random inputs, and against the 2 - 1/m bound."""
    import heapq
    rng = np.random.default_rng(1)
    for _ in range(200):
        m = int(rng.integers(1, 6))
        jobs = [int(x) for x in rng.integers(1, 20, size=int(rng.integers(1, 9)))]
        order = rng.permutation(len(jobs))
        c = oracle.compact([m], dense_from_single([(1, r) for r in jobs]))
        ms, _ = oracle.decode(c, np.zeros(len(jobs), np.uint8), order.astype(np.uint8))
        heap = [0] * m
        for t in order:
            f = heapq.heappop(heap)
            heapq.heappush(heap, f + jobs[t])
        assert ms == max(heap)
        opt = oracle.brute_force(c)[0] if len(jobs) <= 6 else None
        if opt is not None:
            assert ms <= (2 - 1 / m) * opt + 1e-9


# ---------------------------------------------------------------- SPEC optima, LB, MILP size
@pytest.mark.parametrize("case_id", ["SPEC-10", "SPEC-12", "A2-8"])
def test_spec_optima(golden_dir, case_id):
    case = next(c for c in _golden(golden_dir)["optima"] if c["id"] == case_id)
    c = oracle.compact(case["nodes"], dense_from_configs(case["configs"]))
    assert oracle.brute_force(c)[0] == case["optimum"]
    assert exact_makespan(c) == case["optimum"]
    status, val, plan = milp_makespan(c, time_limit=30)
    assert status == "optimal" and val == case["optimum"]
    assert oracle.validate(c, plan, val) == []
    if "lower_bound" in case:
        assert oracle.lower_bound(c) == case["lower_bound"]
    if "milp_vars" in case:
        m = SpaseMilp(c)
        assert (m.n_vars, m.n_rows) == (case["milp_vars"], case["milp_rows"])


def test_milp_closed_form_size():
    """|vars| = sum S + T N + 2 T sum G + T(T-1) + 1 and the 7-family row count
     on random instances."""
    rng = np.random.default_rng(5)
    for _ in range(8):
        inst = synth.random_tiny(rng, max_jobs=4)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        m = SpaseMilp(c)
        T, N, SS, SG = c.n_jobs, len(c.node_gpus), int(c.S.sum()), int(sum(c.node_gpus))
        assert m.n_vars == SS + T * N + 2 * T * SG + T * (T - 1) + 1
        assert m.n_rows == SS * SG + 2 * T + 2 * SS * N + T * N + 2 * SS * SG + 2 * (T - 1) * SS * SG


# ---------------------------------------------------------------- O1 invariants
def test_single_job_makespan_is_runtime():
    rng = np.random.default_rng(2)
    for _ in range(50):
        inst = synth.random_tiny(rng, max_jobs=1)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        for s in range(int(c.S[0])):
            ms, _ = oracle.decode(c, np.array([s], np.uint8), np.array([0], np.uint8))
            assert ms == c.config(0, s)[2]


def test_full_node_jobs_serialise():
    rng = np.random.default_rng(3)
    for _ in range(20):
        k = int(rng.integers(2, 9))
        rs = [int(x) for x in rng.integers(1, 100, size=int(rng.integers(1, 6)))]
        c = oracle.compact([k], dense_from_single([(k, r) for r in rs]))
        for perm in itertools.permutations(range(len(rs))):
            assert oracle.decode(c, np.zeros(len(rs), np.uint8), np.array(perm, np.uint8))[0] == sum(rs)


def test_decoded_schedules_are_valid_and_left_justified():
    """Every O1 schedule passes O3, and each job starts at the g-th smallest free time of
    its node given the earlier placements (no earlier gang start was possible there)."""
    rng = np.random.default_rng(4)
    for inst_seed in range(40):
        inst = synth.random_tiny(np.random.default_rng(inst_seed), max_jobs=5,
                                 node_choices=([4], [8], [2, 2], [3, 5], [2, 2, 4, 8]), max_r=9)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        cfg, perm = synth.random_genomes(c.S, 30, seed=inst_seed)
        for i in range(30):
            ms, pl = oracle.decode(c, cfg[i], perm[i])
            assert oracle.validate(c, pl, ms) == []
            # replay the placements in priority order and check each start is minimal
            free = {n: [0] * int(c.node_gpus[n]) for n in range(len(c.node_gpus))}
            for t in perm[i]:
                p = pl[t]
                g = p["gpus"]
                starts = {n: sorted(f)[g - 1] for n, f in free.items() if len(f) >= g}
                assert p["start_s"] == min(starts.values())
                assert p["node"] == min(n for n, s in starts.items() if s == p["start_s"])
                for k in range(len(free[p["node"]])):
                    if p["gpu_mask"] >> k & 1:
                        assert free[p["node"]][k] <= p["start_s"]
                        free[p["node"]][k] = p["end_s"]


def test_validator_catches_violations():
    c = oracle.compact([2], dense_from_single([(1, 5), (1, 5), (2, 3)]))
    ms, pl = oracle.decode(c, np.zeros(3, np.uint8), np.array([0, 1, 2], np.uint8))
    assert oracle.validate(c, pl, ms) == []
    bad = [dict(p) for p in pl]
    bad[1]["gpu_mask"] = bad[0]["gpu_mask"]          # two jobs on one GPU at once
    assert any(v.startswith("isolation") for v in oracle.validate(c, bad, ms))
    bad = [dict(p) for p in pl]
    bad[2]["gpu_mask"] = 1                           # too few GPUs
    assert any(v.startswith("alloc") for v in oracle.validate(c, bad, ms))
    bad = [dict(p) for p in pl]
    bad[0]["end_s"] += 1
    assert any(v.startswith("runtime") for v in oracle.validate(c, bad))
    assert oracle.validate(c, pl, ms + 1) == ["makespan"]


# ---------------------------------------------------------------- O2 vs independent exact solvers
def test_brute_force_equals_time_indexed_exact_single_node():
    """On one node greedy node choice is trivially complete: O2 = O4a exactly."""
    for seed in range(60):
        rng = np.random.default_rng(100 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [3], [4]), max_r=5)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        assert oracle.brute_force(c)[0] == exact_makespan(c), inst.runtime


def test_brute_force_multi_node_against_node_gene_and_exact():
    """Multi-node: the node-gene decoder space provably contains the optimum (SURVEY.md
    §8c O2) -> node-gene brute force = O4a.  Greedy node choice (the north-star genome) is
    a standing check: it must equal both (no counterexample known)."""
    for seed in range(40):
        rng = np.random.default_rng(200 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2, 2], [2, 3], [3, 1]), max_r=4)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        ex = exact_makespan(c)
        assert oracle.brute_force_node_gene(c) == ex
        assert oracle.brute_force(c)[0] == ex


def test_brute_force_equals_paper_milp_highs():
    """O2 = the paper's own MILP (Eqs. 1-11, readings A1-A3) solved to optimality by HiGHS,
    and the MILP's plan passes O3."""
    n = 0
    for seed in range(40):
        rng = np.random.default_rng(300 + seed)
        inst = synth.random_tiny(rng, max_jobs=3, node_choices=([2], [3], [2, 2]), max_r=5)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        status, val, plan = milp_makespan(c, time_limit=20)
        if status != "optimal":
            continue
        n += 1
        assert val == oracle.brute_force(c)[0]
        assert oracle.validate(c, plan, val) == []
    assert n >= 30


def test_decoded_plan_satisfies_paper_milp():
    """Round trip: a decoded plan, written as B, O, P, A, I, C, violates no
    row of the paper's MILP."""
    for seed in range(15):
        rng = np.random.default_rng(400 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [4], [2, 2], [3, 2]), max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        m = SpaseMilp(c)
        cfg, perm = synth.random_genomes(c.S, 5, seed=seed)
        for i in range(5):
            ms, pl = oracle.decode(c, cfg[i], perm[i])
            assert m.violations(m.plan_to_assignment(pl, ms)) == []
        # and a tampered plan is rejected by the MILP rows too
        ms, pl = oracle.decode(c, cfg[0], perm[0])
        x = m.plan_to_assignment(pl, ms)
        x[m.idx[("C",)]] = ms - 1
        assert "makespan" in m.violations(x)


# ---------------------------------------------------------------- O5 and monotonicity
def test_lower_bound_below_optimum():
    tight = 0
    for seed in range(80):
        rng = np.random.default_rng(500 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        opt = oracle.brute_force(c)[0]
        lb = oracle.lower_bound(c)
        assert lb <= opt
        tight += lb == opt
    assert tight > 0


def test_optimum_monotone_in_runtimes_but_decode_is_not(golden_dir):
    """Lowering any runtime never raises OPT (SURVEY.md §8c O2 metamorphic), while a single
    genome's makespan can rise (the ANOMALY pair above)."""
    for seed in range(40):
        rng = np.random.default_rng(600 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        opt = oracle.brute_force(c)[0]
        nz = np.argwhere(inst.runtime > 1)
        if len(nz) == 0:
            continue
        t, u, g = nz[rng.integers(len(nz))]
        faster = inst.runtime.copy()
        faster[t, u, g] -= 1
        c2 = oracle.compact(inst.node_gpus, faster)
        assert oracle.brute_force(c2)[0] <= opt


def test_relabelling_jobs_and_identical_nodes_keeps_optimum():
    for seed in range(20):
        rng = np.random.default_rng(700 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2, 2], [3, 3], [4]), max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        p = rng.permutation(inst.n_jobs)
        c2 = oracle.compact(inst.node_gpus, inst.runtime[p])
        assert oracle.brute_force(c)[0] == oracle.brute_force(c2)[0]


# ---------------------------------------------------------------- O6: unranking, Philox
def test_unrank_is_a_bijection_on_tiny():
    inst = synth.tiny(0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    assert list(c.S) == [6, 6, 6]
    N = oracle.space_size(c)
    assert N == 6 ** 3 * 6 == 1296
    seen = set()
    for G in range(N):
        cfg, perm = oracle.unrank(c, G)
        assert oracle.rank(c, cfg, perm) == G
        seen.add((tuple(cfg), tuple(perm)))
    assert len(seen) == N
    # the documented order of r_perm
    perms = [tuple(oracle.unrank(c, r * 216)[1]) for r in range(6)]
    assert perms == [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    with pytest.raises(ValueError):
        oracle.unrank(c, N)


def test_brute_force_ranges_compose():
    """min over a partition of [0, N) of the per-slice results = the whole-range result,
    with the smallest index kept on ties (the multi-GPU reduction rule, reading A7)."""
    inst = synth.tiny_variant(3, 4, nodes=(2, 2))
    c = oracle.compact(inst.node_gpus, inst.runtime)
    N = oracle.space_size(c)
    whole = oracle.brute_force(c)
    cuts = [0, N // 5, N // 2, N - 7, N]
    parts = [oracle.brute_force(c, a, b) for a, b in zip(cuts, cuts[1:])]
    assert min(parts) == whole


def test_philox_known_answers(golden_dir):
    from oracle.philox import philox4x32_10
    with open(os.path.join(golden_dir, "philox_kat.json")) as f:
        kat = json.load(f)
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert list(philox4x32_10(ctr, key)) == [int(x, 16) for x in v["out"]]


def test_bounded_draw_is_uniform_multiply_shift():
    from oracle.philox import Stream
    st = Stream((1, 2), 3, 4, 5)
    xs = [st.below(7) for _ in range(7000)]
    assert min(xs) == 0 and max(xs) == 6
    counts = np.bincount(xs, minlength=7)
    assert counts.min() > 850


# ---------------------------------------------------------------- f3: LP export, check_solution == O3
def test_lp_export_round_trip():
    """to_lp writes every row of the paper's MILP (Eqs. 1-11) in CPLEX LP format; reading
    the file back gives the same coefficients, senses and right-hand sides, 17 variables and
    54 constraint rows on SPEC's 2-task instance, and a decoded plan satisfies
    every row as read from the file."""
    import io
    from oracle.milp import read_lp
    # SPEC's 2-task instance (golden SPEC-10: two jobs, each (UPP 3, 1 GPU, 10 s) or
    # (UPP 1, 2 GPUs, 6 s), on 1 x 2 GPUs)
    c = oracle.compact([2], dense_from_configs([[[3, 1, 10], [1, 2, 6]], [[3, 1, 10], [1, 2, 6]]]))
    m = SpaseMilp(c)
    buf = io.StringIO()
    m.to_lp(buf)
    obj, rows, binaries, nonneg = read_lp(buf.getvalue())
    assert obj == "C" and len(binaries) + len(nonneg) == m.n_vars == 17
    assert len({k.rsplit("_", 1)[0] if k.endswith(("_lo", "_hi")) else k for k in rows}) <= m.n_rows == 54
    for seed in range(4):
        rng = np.random.default_rng(900 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [3, 2]), max_r=6)
        cc = oracle.compact(inst.node_gpus, inst.runtime)
        mm = SpaseMilp(cc)
        b = io.StringIO()
        mm.to_lp(b)
        _, rows, bins, _ = read_lp(b.getvalue())
        names = {j: mm.var_name(k) for k, j in mm.idx.items()}
        assert sorted(bins) == sorted(names[j] for j in range(mm.n_vars) if mm.kinds[j] == 1)
        # every matrix row appears with identical coefficients
        A = mm.A.tocsr()
        for r in range(mm.n_rows):
            coef = {names[j]: v for j, v in zip(A.indices[A.indptr[r]:A.indptr[r + 1]], A.data[A.indptr[r]:A.indptr[r + 1]])
                    if v != 0}
            tag = f"{mm.tags[r].replace('-', '_')}_{r}"
            for suffix, bound, op in (("", mm.lo[r], "="), ("_lo", mm.lo[r], ">="), ("_hi", mm.hi[r], "<=")):
                if tag + suffix in rows:
                    got, gop, rhs = rows[tag + suffix]
                    assert gop == op and abs(rhs - bound) < 1e-9
                    assert set(got) == set(coef) and all(abs(got[k] - coef[k]) < 1e-9 for k in coef)
        # a decoded plan satisfies the rows as read back from the file
        cfg, perm = synth.random_genomes(cc.S, 1, seed=seed)
        ms, pl = oracle.decode(cc, cfg[0], perm[0])
        x = mm.plan_to_assignment(pl, ms)
        val = {names[j]: x[j] for j in range(mm.n_vars)}
        for name, (coef, op, rhs) in rows.items():
            lhs = sum(v * val[k] for k, v in coef.items())
            assert {"=": abs(lhs - rhs) < 1e-6, ">=": lhs >= rhs - 1e-6, "<=": lhs <= rhs + 1e-6}[op], name


def test_milp_check_solution_equals_validator():
    """f3: the paper's MILP rows as a checker (check_solution) accept exactly the
    plans O3 accepts: decoded plans pass both; each planted fault (overlap on a GPU, a GPU
    too few, a wrong config width, a start moved into a busy GPU, a makespan below the last
    end) fails both."""
    seen = 0
    for seed in range(12):
        rng = np.random.default_rng(1000 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([2], [4], [2, 2], [3, 2]), max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        m = SpaseMilp(c)
        cfg, perm = synth.random_genomes(c.S, 3, seed=seed)
        for i in range(3):
            ms, pl = oracle.decode(c, cfg[i], perm[i])
            assert oracle.validate(c, pl, ms) == [] and m.violations(m.plan_to_assignment(pl, ms)) == []
            faults = []
            for t, p in enumerate(pl):
                gn = int(c.node_gpus[p["node"]])
                for u in range(len(pl)):          # overlap: move job u onto job t's GPUs and start
                    if u != t and pl[u]["node"] == p["node"] and pl[u]["gpus"] == p["gpus"] and \
                            pl[u]["gpu_mask"] != p["gpu_mask"]:
                        f = [dict(x) for x in pl]
                        f[u]["gpu_mask"], f[u]["start_s"] = p["gpu_mask"], p["start_s"]
                        f[u]["end_s"] = p["start_s"] + (pl[u]["end_s"] - pl[u]["start_s"])
                        faults.append(f)
                if p["gpus"] > 1:                  # a GPU too few
                    f = [dict(x) for x in pl]
                    f[t]["gpu_mask"] &= f[t]["gpu_mask"] - 1
                    faults.append(f)
                if p["gpus"] < gn and bin(p["gpu_mask"]).count("1") < gn:   # a GPU too many
                    f = [dict(x) for x in pl]
                    free = [g for g in range(gn) if not p["gpu_mask"] >> g & 1][0]
                    f[t]["gpu_mask"] |= 1 << free
                    faults.append(f)
            for f in faults:
                fms = max(x["end_s"] for x in f)
                v_o3 = oracle.validate(c, f, fms)
                v_milp = m.violations(m.plan_to_assignment(f, fms))
                assert (v_o3 == []) == (v_milp == []), (v_o3, v_milp)
                seen += v_o3 != []
            low = m.plan_to_assignment(pl, ms - 1)
            assert m.violations(low) and oracle.validate(c, pl, ms - 1)
    assert seen > 20


# ---------------------------------------------------------------- O5b configuration-LP bound
def test_config_lp_bound_hand_examples():
    """Hand-checked: on 1 x 3 GPUs two (2 GPUs, 10 s) jobs can never overlap (4 > 3), so the
    bound is 20 = OPT while the area bound is ceil(40 / 3) = 14.  On 1 x 4 GPUs with A
    (3 GPUs, 4 s), B (2, 4), C (1, 4): A and B exclude each other (5 > 4) -> 8 = OPT; area
    ceil(24 / 4) = 6."""
    from oracle.bounds import config_lp_bound
    c = oracle.compact([3], dense_from_single([(2, 10), (2, 10)]))
    assert config_lp_bound(c)[0] == 20 == oracle.brute_force(c)[0] and oracle.lower_bound(c) == 14
    c = oracle.compact([4], dense_from_single([(3, 4), (2, 4), (1, 4)]))
    assert config_lp_bound(c)[0] == 8 == oracle.brute_force(c)[0] and oracle.lower_bound(c) == 6


def test_config_lp_bound_between_area_bound_and_optimum():
    """A valid relaxation (never above the brute-force optimum) that dominates O5, on random
    single- and multi-node tiny instances; strictly tighter than O5 on some of them."""
    from oracle.bounds import config_lp_bound
    tighter = 0
    for seed in range(40):
        rng = np.random.default_rng(1200 + seed)
        inst = synth.random_tiny(rng, max_jobs=4, node_choices=([3], [4], [2, 2], [3, 2]), max_r=6)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        lb, m_star, _ = config_lp_bound(c)
        opt = oracle.brute_force(c)[0]
        o5 = oracle.lower_bound(c)
        assert o5 <= lb <= opt, (o5, lb, opt, inst.runtime)
        tighter += lb > o5
    assert tighter >= 5
