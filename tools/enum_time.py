"""Time the DFS enumeration (saturn_enumerate) of a library build on the bench's 7-job
TINY-shaped instance and on an 8-job one:  python tools/enum_time.py <libsaturn.so>"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2309_01226_b200.saturn as S  # noqa: E402

lib = sys.argv[1]
S.load_library(lib)
out = {"lib": lib}
for name, (jobs, seed, nodes) in {"7x1x4": (7, 7, (4,)), "8x1x4": (8, 3, (4,)), "9x2x2": (9, 5, (2, 2))}.items():
    tv = synth.tiny_variant(seed, jobs, nodes)
    p = S.Plan(tv.node_gpus, 0).load_runtime_table(tv.runtime)
    p.enumerate()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = p.enumerate()
        ts.append(time.perf_counter() - t0)
    out[name] = {"seconds": min(ts), "makespan": r["makespan"], "index": r["genome_index"], "leaves": r["leaves"]}
print(json.dumps(out))
