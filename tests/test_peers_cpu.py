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


def _dead_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SATURN_PEER_TIMEOUT_S="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_01226_b200 as sat
    plan = sat.Plan([4], device=-1)
    sat.attach_peers(plan)
    plan.barrier()
    out = []
    if rank == 1:
        time.sleep(3.0)            # silent (no heartbeat) for longer than the 1 s liveness timeout
    for _ in range(2):
        t0 = time.monotonic()
        try:
            plan.barrier()
            out.append(("ok", time.monotonic() - t0))
        except sat.SaturnError as e:
            out.append((str(e), time.monotonic() - t0))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_barrier_silent_rank_poisons_link():
    """a rank silent past the liveness timeout fails the waiting rank's barrier and
    marks the link broken in the shared segment, so every later barrier -- on both ranks,
    including the late one -- fails fast instead of pairing with a stale arrival count."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    ps = [ctx.Process(target=_dead_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get() for _ in range(2))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    (m0a, t0a), (m0b, t0b) = res[0]
    assert "silent" in m0a and 0.9 < t0a < 2.9          # detected after ~1 s, before rank 1 woke
    assert "broken" in m0b and t0b < 0.5                 # then fails fast
    for m, t in res[1]:
        assert "broken" in m and t < 0.5                 # the late rank sees the poisoned link
