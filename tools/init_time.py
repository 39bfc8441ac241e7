"""Device time of a generation-0-only search (initial population kernel + selection):
    python tools/init_time.py <libsaturn.so> [WORKLOAD]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200.saturn as S  # noqa: E402

lib = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "TXT"
S.load_library(lib)
inst = synth.by_name(name, 0)
plan = S.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
cfg = S.SearchConfig(seed=1, population=1 << 22, max_generations=0, elites=16)
for _ in range(3):
    plan.search(cfg)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    plan.search(cfg)
b.record()
torch.cuda.synchronize()
print(json.dumps({"lib": lib, "workload": name, "gen0_search_ms": a.elapsed_time(b) / 20}))
