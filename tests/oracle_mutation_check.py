"""Mutation check for the oracle pins (run by hand: python tests/oracle_mutation_check.py).

Each mutation plants one plausible mistake in an oracle source (a wrong GPU rule, a wrong
tie-break, an off-by-one, a dropped max, a transposed radix in oracle/saturn_oracle.c; a
non-strict acceptance, a wrong tie-break or a dropped move family in oracle/local_search.py;
Sattolo's shuffle, a skipped swap or a short config range in oracle/ga.py:initial_genome;
a reversed tournament or tie-break, a flipped crossover bit, unswapped child roles, a
reversed LOX fill or unordered cuts, a wrong insertion target or shared child fields in
oracle/ga.py:make_child; a dropped greedy fallback, a strict fit test or a fixed node
in oracle/baselines.py:baseline_nodes)
and confirms that the `-m "not gpu"` pins of that source fail.  The original source is
restored afterwards.  Result for this round is recorded in DESIGN.md ("Oracle pins").
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "liboracle.so")
C_SRC = "oracle/saturn_oracle.c"
LS_SRC = "oracle/local_search.py"
GA_SRC = "oracle/ga.py"
LB_SRC = "oracle/bounds.py"
PINS = "tests/test_oracle_pins.py"
SEARCH_PINS = "tests/test_oracle_search_pins.py"
GA_PINS = "tests/test_oracle_ga_pins.py"
BL_SRC = "oracle/baselines.py"
BL_PINS = "tests/test_baselines.py::test_baseline_nodes_single_node_and_greedy_fallback"

MUTATIONS = [
    (C_SRC, PINS, "gpu rule smallest-free", "f > free_t[first[best_n] + pick]", "f < free_t[first[best_n] + pick]"),
    (C_SRC, PINS, "node tie -> highest id", "start_n < best_s", "start_n <= best_s"),
    (C_SRC, PINS, "free test strict", "f > s) continue", "f >= s) continue"),
    (C_SRC, PINS, "k-th smallest off by one", "sorted_free[g - 1]", "sorted_free[g > 1 ? g - 2 : 0]"),
    (C_SRC, PINS, "gpu tie -> higher id", "if (pick < 0 || f > free_t", "if (pick < 0 || f >= free_t"),
    (C_SRC, PINS, "makespan = last end", "if (s + r > makespan) makespan = s + r;", "makespan = s + r;"),
    (C_SRC, PINS, "radix reversed", "cfg[t] = (uint8_t)(r_cfg % (uint64_t)n_cfg[t]);",
     "cfg[n_jobs-1-t] = (uint8_t)(r_cfg % (uint64_t)n_cfg[n_jobs-1-t]);"),
    (C_SRC, PINS, "brute force keeps last tie", "if (best < 0 || ms < best)", "if (best < 0 || ms <= best)"),
    (LS_SRC, SEARCH_PINS, "local search accepts equal makespan", "if m[best] >= ms:", "if m[best] > ms:"),
    (LS_SRC, SEARCH_PINS, "local search tie -> largest move", "np.lexsort((np.arange(len(m)), m))",
     "np.lexsort((-np.arange(len(m)), m))"),
    (LS_SRC, SEARCH_PINS, "config moves dropped", "    for t in range(T):\n        for v in range(int(c.S[t])):",
     "    for t in range(0):\n        for v in range(int(c.S[t])):"),
    (LS_SRC, SEARCH_PINS, "insertion target off by one", "j = jj if jj < i else jj + 1\n        p = list(perm)",
     "j = jj + 1 if jj < i else jj\n        p = list(perm)"),
    (GA_SRC, SEARCH_PINS, "Sattolo shuffle", "j = st.below(i + 1)", "j = st.below(i)"),
    (GA_SRC, SEARCH_PINS, "last swap skipped", "for i in range(T - 1, 0, -1):", "for i in range(T - 1, 1, -1):"),
    (GA_SRC, SEARCH_PINS, "config range short by one", "cfg = [st.below(int(S[t])) for t in range(T)]",
     "cfg = [st.below(max(int(S[t]) - 1, 1)) for t in range(T)]"),
    (GA_SRC, GA_PINS, "tournament picks the larger key", "return i if (int(ms[i]), i) < (int(ms[j]), j) else j",
     "return i if (int(ms[i]), i) > (int(ms[j]), j) else j"),
    (GA_SRC, GA_PINS, "tournament tie -> larger slot", "return i if (int(ms[i]), i) < (int(ms[j]), j) else j",
     "return i if (int(ms[i]), -i) < (int(ms[j]), -j) else j"),
    (GA_SRC, GA_PINS, "crossover bit sense flipped", "if not (w[xbit_word(t // 32)] >> (t % 32)) & 1:",
     "if (w[xbit_word(t // 32)] >> (t % 32)) & 1:"),
    (GA_SRC, GA_PINS, "second child not role-swapped", "(a_idx, b_idx) if r == 0 else (b_idx, a_idx)",
     "(a_idx, b_idx)"),
    (GA_SRC, GA_PINS, "LOX fills in reverse order", "fill = [x for x in B_perm if x not in kept]",
     "fill = [x for x in reversed(B_perm) if x not in kept]"),
    (GA_SRC, GA_PINS, "LOX cuts not ordered", "if a > b:\n            a, b = b, a", "if a < b:\n            a, b = b, a"),
    (GA_SRC, GA_PINS, "insertion back at its own position", "child_perm.insert(j, x)", "child_perm.insert(i, x)"),
    (GA_SRC, GA_PINS, "both children use child 0's fields", "c = 8 + 4 * r", "c = 8"),
    (LB_SRC, PINS, "knapsack capacity one too many", "best = [0.0] * (cap + 1)\n    choice = [[] for _ in range(cap + 1)]",
     "cap = cap + 1\n    best = [0.0] * (cap + 1)\n    choice = [[] for _ in range(cap + 1)]"),
    (LB_SRC, PINS, "job progress counted twice", "A[nK + t, j] = -1.0 / jobs[t][s][1]",
     "A[nK + t, j] = -2.0 / jobs[t][s][1]"),
    (LB_SRC, PINS, "longest-job row dropped", "[(longest, None)]", "[(0, None)]"),
    (BL_SRC, BL_PINS, "baseline node genes: greedy fallback never applied", "else GREEDY for t in",
     "else node[t] for t in"),
    (BL_SRC, BL_PINS, "baseline node genes: fit test strict", "<= int(c.node_gpus[node[t]])",
     "< int(c.node_gpus[node[t]])"),
    (BL_SRC, BL_PINS, "random baseline pinned to node 0", "return [GREEDY] * c.n_jobs", "return [0] * c.n_jobs"),
]


def main():
    ok = True
    for src_rel, tests, name, old, new in MUTATIONS:
        src = os.path.join(ROOT, src_rel)
        backup = src + ".orig"
        shutil.copy(src, backup)
        try:
            text = open(backup).read()
            assert old in text, (src_rel, old)
            open(src, "w").write(text.replace(old, new, 1))
            if os.path.exists(LIB):
                os.remove(LIB)
            shutil.rmtree(os.path.join(ROOT, "oracle", "__pycache__"), ignore_errors=True)   # same-size edits
            r = subprocess.run([sys.executable, "-B", "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", tests],
                               cwd=ROOT, capture_output=True, text=True)
            caught = r.returncode != 0
            ok &= caught
            print(f"{'CAUGHT ' if caught else 'MISSED '} {src_rel}: {name}: {r.stdout.strip().splitlines()[-1]}",
                  flush=True)
        finally:
            shutil.move(backup, src)
            if os.path.exists(LIB):
                os.remove(LIB)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
