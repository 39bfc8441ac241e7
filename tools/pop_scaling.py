"""k_ga time and bench-step time against the population size (fixed costs per launch and
per generation):  python tools/pop_scaling.py [WORKLOAD]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200.saturn as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "TXT"
inst = synth.by_name(name, 0)
plan = S.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
for lg in (20, 21, 22, 23, 24):
    P = 1 << lg
    cfg = S.SearchConfig(seed=1, population=P, max_generations=16, elites=16, generations_per_epoch=8)
    for _ in range(2):
        plan.search(cfg)
    plan.reset_stats()
    plan.set_profiling(True)
    for _ in range(5):
        plan.search(cfg)
    st = plan.stats()
    plan.set_profiling(False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        plan.search(cfg)
    b.record()
    torch.cuda.synchronize()
    step = a.elapsed_time(b) / 5
    kga = st["ga_kernel_ms"] / st["ga_launches"]
    print(json.dumps({"workload": name, "P": P, "k_ga_ms": kga, "k_ga_ns_per_child": kga * 1e6 / (P - 16),
                      "step_ms": step, "plans_per_s": (P + 16 * (P - 16)) / (step * 1e-3)}), flush=True)
