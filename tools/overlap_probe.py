"""Probe: do two GA islands on two CUDA streams (two host threads) overlap well enough to
beat one island?  SATURN_GA_SPLIT selects the kernel mode.  Prints plans/s."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P = (1 << 22) // K
inst = synth.txt(0)
plans = [sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime) for _ in range(K)]
streams = [torch.cuda.Stream() for _ in range(K)]
cfg = sat.SearchConfig(seed=3, population=P, max_generations=64, elites=16, generations_per_epoch=32)


def run(k, out):
    with torch.cuda.stream(streams[k]):
        r = plans[k].search(cfg, stream=streams[k])
    out[k] = r["evaluated"]


for _ in range(2):  # warm
    out = [0] * K
    ts = [threading.Thread(target=run, args=(k, out)) for k in range(K)]
    [t.start() for t in ts]
    [t.join() for t in ts]
torch.cuda.synchronize()
t0 = time.perf_counter()
out = [0] * K
ts = [threading.Thread(target=run, args=(k, out)) for k in range(K)]
[t.start() for t in ts]
[t.join() for t in ts]
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"K={K} split={os.environ.get('SATURN_GA_SPLIT', '0')} plans/s={sum(out) / dt:.3e}")
