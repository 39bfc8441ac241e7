"""Device time of the bench step with and without the per-generation profiling events and
the NVML clock sampler (is the instrumentation of bench.py's timed region free?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402
from bench import ClockSampler  # noqa: E402

inst = synth.by_name("TXT", 0)
plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
scfg = sat.SearchConfig(seed=2309, population=1 << 22, max_generations=16, elites=16, generations_per_epoch=8)
st = torch.cuda.current_stream()
for _ in range(5):
    plan.search(scfg, stream=st)


def run(prof, sampler, K=20):
    plan.set_profiling(prof)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with (ClockSampler(0) if sampler else open(os.devnull)):
        a.record(st)
        for _ in range(K):
            plan.search(scfg, stream=st)
        b.record(st)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for rep in range(2):
    for prof in (False, True):
        for sampler in (False, True):
            print(f"prof={prof} sampler={sampler}: {run(prof, sampler):.4f} ms/step", flush=True)
