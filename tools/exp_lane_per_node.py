"""Experiment driver (GPU box): the lane-per-node decoder of tools/exp_lane_per_node.cu
against the library's saturn_evaluate on the multi-node workloads (MIX 2x8, SWEEP 4x8).
Checks its makespans element by element against the library (itself bit-exact vs the
oracle) and times both with CUDA events.

    python tools/exp_lane_per_node.py [--out gpurun_out/exp_lanes.json]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2309_01226_b200.saturn as S  # noqa: E402

SO = os.path.join(ROOT, "tools", "libexp_lanes.so")
OPS = {"MIX": 912, "SWEEP": 4200}
PEAK = 18.61248e12


def build():
    src = os.path.join(ROOT, "tools", "exp_lane_per_node.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])
    lib = ctypes.CDLL(SO)
    lib.exp_lanes_evaluate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p]
    lib.exp_lanes_evaluate.restype = ctypes.c_int
    return lib


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lib = build()
    rows = []
    for name in ("MIX", "SWEEP"):
        inst = synth.by_name(name, 0)
        plan = S.Plan(inst.node_gpus, 0).load_runtime_table(inst.runtime)
        Sn = plan.num_configs()
        T, stride = len(Sn), int(Sn.max())
        tab = np.zeros((T, stride), np.uint32)
        for t in range(T):
            for c in range(int(Sn[t])):
                _, g, r = plan.config(t, c)
                tab[t, c] = (g << 24) | r
        n = 1 << 22 if name == "MIX" else 1 << 21
        cfg, perm = synth.random_genomes(Sn, n, seed=5)
        dc, dp = torch.from_numpy(cfg).cuda(), torch.from_numpy(perm).cuda()
        dtab = torch.from_numpy(tab.view(np.int32)).cuda()
        dgn = torch.tensor(list(inst.node_gpus), dtype=torch.uint8).cuda()
        ref = torch.empty(n, dtype=torch.int32, device="cuda")
        got = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def lanes():
            rc = lib.exp_lanes_evaluate(dtab.data_ptr(), stride, T, len(inst.node_gpus), dgn.data_ptr(),
                                        dc.data_ptr(), dp.data_ptr(), n, got.data_ptr(), st)
            assert rc == 0, rc

        t_lib = timed(lambda: plan.evaluate(dc, dp, ref))
        t_lanes = timed(lanes)
        same = bool(torch.equal(ref, got))
        r = {"workload": name, "genomes": n, "library_plans_per_s": n / t_lib, "lanes_plans_per_s": n / t_lanes,
             "library_frac": n / t_lib * OPS[name] / PEAK, "lanes_frac": n / t_lanes * OPS[name] / PEAK,
             "bit_exact_vs_library": same}
        print(json.dumps(r), flush=True)
        rows.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
