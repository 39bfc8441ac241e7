"""Peer-memory transport on the B200 (row e without NCCL; saturn_plan_attach_peers): two
processes -- two ranks -- share the one GPU of this pool, map each other's exchange buffers
with CUDA IPC and run the island search and the enumeration collectively.  The results
must equal the in-process island group (saturn_search_group, whose migration is replayed
bit for bit against the oracle in test_gpu_parity.py) and the single-process enumeration
(= oracle brute force): the same island protocol over a different transport."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CFG = dict(seed=7, population=512, max_generations=6, elites=4, generations_per_epoch=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SATURN_PEER_TIMEOUT_S="60")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_2309_01226_b200 as sat
        inst = synth.txt(0)
        plan = sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
        sat.attach_peers(plan)
        r = plan.search(sat.SearchConfig(**CFG))
        pop = plan.search_population(CFG["population"])
        best = plan.best_plan()
        # a time-budgeted search: the collective stop decision over the peer link
        rt = plan.search(sat.SearchConfig(seed=3, population=1024, max_generations=1 << 20, elites=4,
                                          generations_per_epoch=4, time_budget_s=0.3))
        tv = synth.tiny_variant(45, 5, (2, 2))
        ep = sat.Plan(tv.node_gpus, 0).load_runtime_table(tv.runtime)
        sat.attach_peers(ep)
        er = ep.enumerate()
        tb = synth.tiny_variant(7, 7, (4,))          # the bench's instance: 6.8e10 genomes, DFS
        bp = sat.Plan(tb.node_gpus, 0).load_runtime_table(tb.runtime)
        sat.attach_peers(bp)
        er7 = bp.enumerate()
        q.put((rank, r, pop, best[0], best[2], best[3], rt, (er, er7), None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, None, None, None, None, repr(e)))
    dist.destroy_process_group()


def test_two_process_islands_and_enumeration_over_peer_memory():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import oracle
    import synth
    import paper_2309_01226_b200 as sat
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted((q.get() for _ in range(2)), key=lambda x: x[0])
    for p in ps:
        p.join(120)
    for x in res:
        assert x[8] is None, x[8]
    assert all(p.exitcode == 0 for p in ps)
    # reference: the same two islands in one process, exchanging by device copies
    inst = synth.txt(0)
    g = [sat.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime) for _ in range(2)]
    gr = sat.search_group(g, sat.SearchConfig(**CFG))
    for rank in range(2):
        _, r, (pc, pq, pm), ms, bc, bp, rt, er, _ = res[rank]
        rc, rq, rm = g[rank].search_population(CFG["population"])
        assert np.array_equal(pc, rc) and np.array_equal(pq, rq) and np.array_equal(pm, rm), rank
        assert r["makespan"] == gr[rank]["makespan"] and r["evaluated"] == gr[rank]["evaluated"]
        c = oracle.compact(inst.node_gpus, inst.runtime)
        assert oracle.decode(c, bc, bp)[0] == ms == r["makespan"]
    # both ranks stopped the budgeted search after the same number of generations, same best
    assert res[0][6]["generations"] == res[1][6]["generations"] > 0
    assert res[0][6]["makespan"] == res[1][6]["makespan"]
    # enumeration: each rank its slice of the DFS roots, MIN over the peer link
    tv = synth.tiny_variant(45, 5, (2, 2))
    one = sat.Plan(tv.node_gpus, 0).load_runtime_table(tv.runtime).enumerate()
    ct = oracle.compact(tv.node_gpus, tv.runtime)
    tb = synth.tiny_variant(7, 7, (4,))
    one7 = sat.Plan(tb.node_gpus, 0).load_runtime_table(tb.runtime).enumerate()
    for rank in range(2):
        er, er7 = res[rank][7]
        assert (er["makespan"], er["genome_index"]) == (one["makespan"], one["genome_index"])
        assert (er["makespan"], er["genome_index"]) == oracle.brute_force(ct)
        assert er["leaves"] > 0   # per-rank pruning differs from one process: leaves are not compared
        assert (er7["makespan"], er7["genome_index"]) == (one7["makespan"], one7["genome_index"])


def test_bench_two_ranks_over_peer_memory_on_one_gpu():
    """bench.py's multi-rank path end to end (torchrun, barriers, max-over-ranks device time,
    the island exchange) with both ranks on this pool's one GPU over the peer transport."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SATURN_TRANSPORT="peers", SATURN_SHARE_GPU="1", SATURN_PEER_TIMEOUT_S="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--population", "65536", "--generations", "4",
           "--no-cpu-baseline", "--kernel-only-n", "0"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and "peers" in line["config"]["parallelism"]
    # 2 ranks x (P + 4 (P - E)) full decodes per step
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
