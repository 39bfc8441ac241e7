"""Mutation check for the oracle pins (run by hand: python tests/oracle_mutation_check.py).

Each mutation plants one plausible mistake in oracle/saturn_oracle.c (a wrong GPU rule, a
wrong tie-break, an off-by-one, a dropped max, a transposed radix) and confirms that the
`-m "not gpu"` oracle pins in tests/test_oracle_pins.py fail.  The original source is
restored afterwards.  Result for this round is recorded in DESIGN.md ("Oracle pins").
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "saturn_oracle.c")
LIB = os.path.join(ROOT, "oracle", "liboracle.so")

MUTATIONS = [
    ("gpu rule smallest-free", "f > free_t[first[best_n] + pick]", "f < free_t[first[best_n] + pick]"),
    ("node tie -> highest id", "start_n < best_s", "start_n <= best_s"),
    ("free test strict", "f > s) continue", "f >= s) continue"),
    ("k-th smallest off by one", "sorted_free[g - 1]", "sorted_free[g > 1 ? g - 2 : 0]"),
    ("gpu tie -> higher id", "if (pick < 0 || f > free_t", "if (pick < 0 || f >= free_t"),
    ("makespan = last end", "if (s + r > makespan) makespan = s + r;", "makespan = s + r;"),
    ("radix reversed", "cfg[t] = (uint8_t)(r_cfg % (uint64_t)n_cfg[t]);",
     "cfg[n_jobs-1-t] = (uint8_t)(r_cfg % (uint64_t)n_cfg[n_jobs-1-t]);"),
    ("brute force keeps last tie", "if (best < 0 || ms < best)", "if (best < 0 || ms <= best)"),
]


def main():
    backup = SRC + ".orig"
    shutil.copy(SRC, backup)
    ok = True
    try:
        src = open(backup).read()
        for name, old, new in MUTATIONS:
            assert old in src, old
            open(SRC, "w").write(src.replace(old, new, 1))
            if os.path.exists(LIB):
                os.remove(LIB)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "tests/test_oracle_pins.py"],
                               cwd=ROOT, capture_output=True, text=True)
            caught = r.returncode != 0
            ok &= caught
            print(f"{'CAUGHT ' if caught else 'MISSED '} {name}: {r.stdout.strip().splitlines()[-1]}")
    finally:
        shutil.move(backup, SRC)
        if os.path.exists(LIB):
            os.remove(LIB)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
