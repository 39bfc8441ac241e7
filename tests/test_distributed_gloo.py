"""The N > 1 host logic on CPU with torch.distributed/gloo, world size 2 (no GPU):
index-space partitioning + the (makespan << 38 | index) MIN reduction of enumeration,
the NCCL unique-id broadcast used to build the library's communicator, and the GA island
migration rule.  The per-rank compute is the oracle here (the CUDA path needs a B200)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    import paper_2309_01226_b200 as sat
    from oracle import ga as oga
    res = {}
    # 1) enumeration: my slice, oracle brute force on it, global MIN of packed keys
    inst = synth.tiny_variant(45, 5, (2, 2))
    c = oracle.compact(inst.node_gpus, inst.runtime)
    N = oracle.space_size(c)
    b, e = sat.partition(N, rank, world)
    ms, idx = oracle.brute_force(c, b, e)
    key = torch.tensor([(ms << 38) | idx], dtype=torch.int64)
    dist.all_reduce(key, op=dist.ReduceOp.MIN)
    res["key"] = int(key.item())
    sizes = torch.tensor([e - b], dtype=torch.int64)
    dist.all_reduce(sizes)
    res["covered"] = int(sizes.item())
    # 2) the communicator bootstrap: identical 128-byte NCCL id on every rank
    res["uid"] = sat.broadcast_unique_id().hex()
    # 3) GA islands: all-gather each island's elites, every island adopts the global best E
    inst2 = synth.txt(0)
    c2 = oracle.compact(inst2.node_gpus, inst2.runtime)
    P, E = 64, 4
    cfg, perm = oga.initial_population(c2.S, P, seed=5, rank=rank)
    msv = oracle.decode_batch(c2, cfg, perm)
    mine = [(int(msv[i]), cfg[i].tolist(), perm[i].tolist()) for i in oga.elites(msv, E)]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    res["elites"] = [r[0] for r in oga.migrate(gathered)]
    res["all_best"] = min(r[0] for g in gathered for r in g)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([res], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_two_rank_gloo_partition_reduce_and_islands(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"r{k}.npy", allow_pickle=True)[0] for k in range(world)]
    inst = synth.tiny_variant(45, 5, (2, 2))
    c = oracle.compact(inst.node_gpus, inst.runtime)
    ms, idx = oracle.brute_force(c)
    assert r[0]["key"] == r[1]["key"] == (ms << 38) | idx
    assert r[0]["covered"] == oracle.space_size(c)
    assert r[0]["uid"] == r[1]["uid"] and len(bytes.fromhex(r[0]["uid"])) == 128
    assert r[0]["elites"] == r[1]["elites"]
    assert r[0]["elites"][0] == r[0]["all_best"]
    assert r[0]["elites"] == sorted(r[0]["elites"])
