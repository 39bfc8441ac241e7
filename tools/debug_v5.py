"""Round-2 debug: full-population consistency of a bench-size TXT search (GA v5)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle, synth
import paper_2309_01226_b200 as sat
inst = synth.by_name("TXT", 0)
c = oracle.compact(inst.node_gpus, inst.runtime)
P, E, seed = 1 << 22, 16, 2309
plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
for gens in (1, 2, 3, 8, 9, 15, 16):
    r = plan.search(sat.SearchConfig(seed=seed, population=P, elites=E, generations_per_epoch=8, max_generations=gens))
    cc, qq, mm = plan.search_population(P)
    ref = oracle.decode_batch(c, cc, qq)
    bad = np.nonzero(ref != mm)[0]
    print(gens, "best", r["makespan"], "popmin", int(mm.min()), "pop0", int(mm[0]), "mismatch", len(bad), bad[:8],
          mm[bad[:8]], ref[bad[:8]], flush=True)
