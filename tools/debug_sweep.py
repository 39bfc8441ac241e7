"""SWEEP evaluate (several genome tiles per CTA) then a short search, synchronising after
each step (for compute-sanitizer):  python tools/debug_sweep.py [n_genomes] [population]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 14
inst = synth.by_name("SWEEP", 0)
c = oracle.compact(inst.node_gpus, inst.runtime)
plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
cfg, perm = synth.random_genomes(c.S, n, seed=5)
ms = plan.evaluate(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda())
torch.cuda.synchronize()
k = 2000
print("evaluate ok", (ms[:k].cpu().numpy() == oracle.decode_batch(c, cfg[:k], perm[:k])).all(), flush=True)
r = plan.search(sat.SearchConfig(seed=1, population=P, max_generations=2, elites=16, generations_per_epoch=1))
torch.cuda.synchronize()
print("search ok", r["makespan"], flush=True)
