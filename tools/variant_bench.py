"""Time saturn_evaluate and saturn_search with an alternative libsaturn build (A/B of kernel
variants on the GPU box):  python tools/variant_bench.py <path/to/libsaturn.so> [WORKLOAD]"""
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
n = (1 << 24) if name != "SWEEP" else (1 << 21)
c, p = synth.random_genomes(plan.num_configs(), n, seed=5)
c, p = torch.from_numpy(c).cuda(), torch.from_numpy(p).cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    plan.evaluate(c, p, out)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    plan.evaluate(c, p, out)
b.record()
torch.cuda.synchronize()
ev = n * 10 / (a.elapsed_time(b) * 1e-3)
cfg = S.SearchConfig(seed=1, population=1 << 22, max_generations=16, elites=16, generations_per_epoch=8)
for _ in range(2):
    plan.search(cfg)
plan.reset_stats()
plan.set_profiling(True)
for _ in range(10):
    r = plan.search(cfg)
st = plan.stats()
plan.set_profiling(False)
a.record()
for _ in range(10):
    plan.search(cfg)
b.record()
torch.cuda.synchronize()
step_ms = a.elapsed_time(b) / 10
print(json.dumps({"lib": lib, "workload": name, "evaluate_plans_per_s": ev, "step_ms": step_ms,
                  "ga_kernel_ms": st["ga_kernel_ms"] / st["ga_launches"],
                  "ga_children_per_s": st["ga_decodes"] / (st["ga_kernel_ms"] * 1e-3), "best": r["makespan"],
}))
