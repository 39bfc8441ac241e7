"""Peer-memory transport (saturn_plan_attach_peers), host side, on CPU: two processes with
host-only handles rendezvous through the POSIX shared-memory segment (name broadcast by
torch.distributed/gloo), pass the library's barrier repeatedly in lock-step, and the
segment name is removed once both are attached.  Argument and state errors are checked
in-process.  (The device exchange over CUDA IPC is tested on the B200 in
tests/test_peers_gpu.py.)"""
import os
import socket
import time

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_01226_b200 as sat
    plan = sat.Plan([4], device=-1)
    name = sat.attach_peers(plan)
    stamps = []
    for k in range(50):            # lock-step: rank 1 sleeps on odd rounds; rank 0 must wait
        if rank == 1 and k % 10 == 5:
            time.sleep(0.05)
        plan.barrier()
        stamps.append(time.monotonic())
    exists = os.path.exists("/dev/shm" + name)
    q.put((rank, name, stamps, exists))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_barrier_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get() for _ in range(2))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (r0, n0, s0, e0), (r1, n1, s1, e1) = res
    assert n0 == n1 and n0.startswith("/saturn_")
    assert not e0 and not e1                       # rank 0 unlinked the name after attach
    # rank 0 left barrier 5 (and 15, 25, ...) only after rank 1's 50 ms sleep
    for k in (5, 15, 25):
        assert s0[k] - s0[k - 1] > 0.03
    # both left every barrier at (nearly) the same time (loose: a loaded host may deschedule)
    assert max(abs(a - b) for a, b in zip(s0, s1)) < 0.25


def test_peer_attach_errors():
    import paper_2309_01226_b200 as sat
    plan = sat.Plan([4], device=-1)
    with pytest.raises(sat.SaturnError) as e:
        plan.barrier()
    assert e.value.status == sat.ESTATE
    for name, rank, world in (("no_slash", 0, 1), ("/x", 2, 2), ("/x", 0, 9)):
        with pytest.raises(sat.SaturnError) as e:
            plan.attach_peers(name, rank, world)
        assert e.value.status == sat.EINVAL
    # world 1: attaching and barriers are trivial
    plan.attach_peers(sat.peer_name(), 0, 1)
    plan.barrier()
