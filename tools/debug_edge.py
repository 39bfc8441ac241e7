"""Reproduce one edge-shape case step by step (evaluate AUTO, evaluate WARP, search) with a
device synchronize after each, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/debug_edge.py 3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2309_01226_b200 as sat  # noqa: E402
from test_gpu_parity import _edge_instances  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
name, nodes, tab = _edge_instances()[idx]
c = oracle.compact(nodes, tab)
plan = sat.Plan(nodes, 0).load_runtime_table(tab)
cfg, perm = synth.random_genomes(c.S, 700, seed=idx)
for dec in (sat.DECODER_AUTO, sat.DECODER_WARP):
    plan.set_decoder(dec)
    ms = plan.evaluate(torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda())
    torch.cuda.synchronize()
    print(name, "evaluate", dec, "ok", (ms.cpu().numpy() == oracle.decode_batch(c, cfg, perm)).all(), flush=True)
plan.set_decoder(sat.DECODER_AUTO)
r = plan.search(sat.SearchConfig(seed=3, population=96, max_generations=1, elites=4, generations_per_epoch=1))
torch.cuda.synchronize()
print(name, "search ok", r["makespan"], flush=True)
