import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2309_01226_b200 as sat
inst = synth.by_name("TXT", 0)
plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
P=1<<22
scfg = sat.SearchConfig(seed=2309, population=P, max_generations=16, elites=16, generations_per_epoch=8)
st = torch.cuda.current_stream()
for _ in range(5): plan.search(scfg, stream=st)
def run(prof, K=30):
    plan.set_profiling(prof)
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter(); a.record(st)
    for _ in range(K): plan.search(scfg, stream=st)
    b.record(st); torch.cuda.synchronize(); w=time.perf_counter()-t0
    return a.elapsed_time(b)/K, 1e3*w/K
for prof in (False, True, False, True):
    print("prof", prof, run(prof))
plan.set_profiling(False)
# gen0 only
s0 = sat.SearchConfig(seed=2309, population=P, max_generations=0, elites=16, generations_per_epoch=8)
for _ in range(3): plan.search(s0, stream=st)
torch.cuda.synchronize(); a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(20): plan.search(s0, stream=st)
b.record(st); torch.cuda.synchronize(); print("gen0-only search ms", a.elapsed_time(b)/20)
