#!/usr/bin/env python
"""Benchmark: SPASE plans evaluated per second (BASELINE.json metric) on 1..N B200s.

One STEP = one pass of the whole hot path over one batch: a ``saturn_search`` call on the
resident runtime table -- an initial population of P genomes (Philox init + decode), then
G generations of Philox tournament / crossover / mutation fused with the decode of every
child, per-generation top-E reduction, epoch exchange of elites (NCCL when N > 1), and the
best genome returned to the host (rows a3-a7).  The e2e leg repeats the step through the
host API including the table upload (a1/a2) and the trace-decoded best plan (a8).

``value`` counts full decodes only (SURVEY.md §8d counting rule), summed over all ranks,
divided by the max-over-ranks device time of K steps (CUDA events on the launching stream).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload TXT] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPASE plans evaluated/sec at 1/2/4/8 B200; best makespan vs oracle"
UNIT = "plans/s"
# Integer-ALU roofline denominator: 148 SMs x 4 SMSPs x 16 INT32
# lanes of the ALU pipe per clock x 1.965 GHz max SM clock (B200_PROFILING.md / MEASURED_PEAKS.json).
ALU_PEAK_OPS = 148 * 4 * 16 * 1.965e9

WORKLOADS = {
    "TINY": "C1 TINY: 3 jobs x {DDP,FSDP} x g{1,2,4} on 1x4 GPUs",
    "TXT": "C2 TXT: 12 GPT-2/GPT-J jobs x 4 UPPs x g1-8 on 1x8 GPUs",
    "IMG": "C3 IMG: 12 ViT-G/ResNet jobs x 4 UPPs x g1-8 on 1x8 GPUs",
    "MIX": "C4 MIX: 24 TXT+IMG jobs on 2x8 GPUs",
    "SWEEP": "C5 SWEEP: 100 jobs x 4 UPPs on 4x8 GPUs",
}


def algorithmic_ops_per_plan(T: int, node_gpus) -> int:
    """T * (2 + 2N + 4 * GPU_node) integer ops per decode."""
    return T * (2 + 2 * len(node_gpus) + 4 * max(node_gpus))


# ------------------------------------------------------------------ CPU oracle leg
def _oracle_worker(args):
    name, seed, n = args
    import oracle
    import synth
    inst = synth.by_name(name, 0)
    c = oracle.compact(inst.node_gpus, inst.runtime)
    cfg, perm = synth.random_genomes(c.S, n, seed=seed)
    t0 = time.perf_counter()
    ms = oracle.decode_batch(c, cfg, perm)
    dt = time.perf_counter() - t0
    assert (ms > 0).all()
    return n, dt


def oracle_rate(name: str, n_per_core: int, cores: int, seed0: int = 0):
    """Plain C oracle decoder (oracle/saturn_oracle.c, single-threaded per process) on
    `cores` host processes; returns (decodes/s, wall seconds, total decodes)."""
    import multiprocessing as mp
    import oracle
    oracle.build_library()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_worker, [(name, seed0 + 999, 1000)] * cores)  # warm (imports, lib load)
        t0 = time.perf_counter()
        res = pool.map(_oracle_worker, [(name, seed0 + k, n_per_core) for k in range(cores)])
        wall = time.perf_counter() - t0
    total = sum(n for n, _ in res)
    return total / wall, wall, total


def cpu_baseline(name: str, target_s: float = 10.0):
    cores = os.cpu_count() or 1
    rate1, _, _ = oracle_rate(name, 20000, 1)
    n = max(1000, int(rate1 * target_s))
    rate, wall, total = oracle_rate(name, n, cores, seed0=100)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"O1 decode (oracle/saturn_oracle.c) of {total} seeded random {name} genomes "
                      f"({n} per process x {cores} processes, {wall:.1f} s wall)"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    name = args.workload
    per_core = args.ref_per_core
    for _ in range(args.warmup):
        oracle_rate(name, per_core // 4, cores, seed0=7)
    t_total, n_total = 0.0, 0
    for k in range(args.steps):
        rate, wall, total = oracle_rate(name, per_core, cores, seed0=1000 * k)
        t_total += wall
        n_total += total
    value = n_total / t_total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": _config(args, None),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: O1 decode of {per_core} seeded random {name} genomes on each of "
                                       f"{cores} host processes"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML clocks / throttle reasons sampled every 20 ms during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, torch_device: int):
        self.samples, self.mem_samples, self.reasons, self.ok = [], [], 0, False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            uuid = str(torch.cuda.get_device_properties(torch_device).uuid)
            h = None
            for i in range(pynvml.nvmlDeviceGetCount()):
                hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(hi)
                u = u.decode() if isinstance(u, bytes) else u
                if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                    h = hi
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(torch_device)
            self.h, self.nv = h, pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.mem_samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_MEM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": len(self.samples)}
        s = sorted(self.samples)
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        m = sorted(self.mem_samples) or [None]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "mem_mhz": m[len(m) // 2], "reasons": names,
                "samples": len(s)}


# ------------------------------------------------------------------ helpers
def _config(args, extra=None):
    """The workload description -- identical in both arms (no result keys in here)."""
    cfg = {"workload": WORKLOADS[args.workload], "table_seed": 0, "population_per_gpu": args.population,
           "generations_per_step": args.generations, "elites": args.elites,
           "parallelism": f"islands x{args.gpus} (one GA population per GPU, elite exchange over "
                          f"{os.environ.get('SATURN_TRANSPORT', 'nccl')})"
                          + (" -- all ranks on ONE GPU (SATURN_SHARE_GPU=1, functional check only)"
                             if os.environ.get("SATURN_SHARE_GPU") == "1" else ""),
           "l2": "inputs larger than L2: two population buffers of P genomes x genome stride "
                 "(>= 2 x 128 MB at the default P) > 126 MB L2"}
    if extra:
        cfg.update(extra)
    return cfg


def _json(path):
    try:
        with open(os.path.join(ROOT, path)) as f:
            return json.load(f)
    except Exception:
        return None


def _traffic(workload: str):
    d = _json(os.path.join("profiles", "roofline_traffic.json")) or {}
    return d.get(workload)


def host_cpu():
    """Host CPU model and core count (lscpu's 'Model name'; /proc/cpuinfo fallback)."""
    model = None
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    if model is None:
        try:
            for ln in open("/proc/cpuinfo"):
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        except Exception:
            pass
    return {"model": model, "cores": os.cpu_count()}


def _bar(workload: str, seed: int):
    """The committed 5-minute CPU bar of (workload, table seed) and its lower bound."""
    for rnd in ("r2", "r1"):
        d = _json(os.path.join("profiles", rnd, "quality_bar.json" if workload == "TXT"
                               else f"quality_bar_{workload}.json"))
        if d and str(seed) in d.get("seeds", {}):
            e = d["seeds"][str(seed)]
            return {"bar": e.get("bar"), "bar_file": f"profiles/{rnd}/" + ("quality_bar.json" if workload == "TXT"
                                                                          else f"quality_bar_{workload}.json"),
                    "bar_lower_bound": e.get("lower_bound"), "bar_best_lower_bound": e.get("best_lower_bound")}
    return {"bar": None}


def measure_search(sat, torch, plan, inst, scfg, steps, warmup, stream, G, barrier=None, max_over_ranks=None):
    """Device-timed search steps (CUDA events on the launching stream) plus the sampled k_ga
    launch times; returns (dict, stats, last result)."""
    barrier = barrier or torch.cuda.synchronize
    max_over_ranks = max_over_ranks or (lambda x: x)
    for _ in range(max(warmup, 0)):
        plan.search(scfg, stream=stream)
    barrier()
    plan.reset_stats()
    plan.set_profiling(4)          # k_ga launches 2, 6, 10, 14 of each step carry CUDA events
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evaluated = 0
    barrier()
    ev0.record(stream)
    for _ in range(steps):
        r = plan.search(scfg, stream=stream)
        evaluated += r["evaluated"]
    ev1.record(stream)
    barrier()
    st = plan.stats()
    plan.set_profiling(False)
    dev_ms = max_over_ranks(ev0.elapsed_time(ev1))
    return {"value": evaluated / (dev_ms * 1e-3), "ms_per_step": dev_ms / steps, "evaluated": evaluated}, st, r


def measure_e2e(plan, inst, scfg, steps, stream, torch, max_over_ranks=None):
    """The same metric through the host API with host buffers: table upload, search, and the
    trace-decoded best plan copied back, every step."""
    max_over_ranks = max_over_ranks or (lambda x: x)
    plan.reset_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev = 0
    for _ in range(steps):
        plan.load_runtime_table(inst.runtime)
        r = plan.search(scfg, stream=stream)
        plan.best_plan()
        ev += r["evaluated"]
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    st = plan.stats()
    return {"value": ev / e2e_s, "unit": UNIT, "h2d_bytes_per_step": st["h2d_bytes"] // steps,
            "d2h_bytes_per_step": st["d2h_bytes"] // steps}


def ga_roofline(st, T, node_gpus, G, steps, dev_ms):
    ops = algorithmic_ops_per_plan(T, node_gpus)
    launch_s = st["ga_kernel_ms"] * 1e-3 / max(st["ga_launches"], 1)
    units = st["ga_decodes"] / max(st["ga_launches"], 1)
    achieved = ops * units / launch_s
    return {"bound": "alu", "achieved": achieved / 1e12, "peak": ALU_PEAK_OPS / 1e12, "unit": "TOP/s",
            "frac": achieved / ALU_PEAK_OPS,
            "kernel": "k_ga (Philox GA operators fused with the sorted-multiset decode)",
            "ops_per_plan": ops, "plans_per_launch": units, "launch_ms": launch_s * 1e3,
            "launches_timed": st["ga_launches"],
            # k_ga launches in the timed region (G per step; generation 0 is k_ga_init) x their
            # mean duration / device time
            "kernel_share_of_step": (launch_s * 1e3 * G * steps / dev_ms) if dev_ms > 0 else None}


def evaluate_rate(sat, torch, plan, n, reps=5, kind=None):
    """k_evaluate alone (caller genomes resident in HBM): plans/s."""
    import synth
    S = plan.num_configs()
    cfg_h, perm_h = synth.random_genomes(S, n, seed=5)
    cfg_d, perm_d = torch.from_numpy(cfg_h).cuda(), torch.from_numpy(perm_h).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    if kind is not None:
        plan.set_decoder(kind)
    for _ in range(3):
        plan.evaluate(cfg_d, perm_d, out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.evaluate(cfg_d, perm_d, out)
    b.record()
    torch.cuda.synchronize()
    plan.set_decoder(sat.DECODER_AUTO)
    return n * reps / (a.elapsed_time(b) * 1e-3)


def workload_legs(sat, torch, args, local, stream, names):
    """Every BASELINE config besides the headline one, same step definition: search
    plans/s (device-timed), e2e, k_ga roofline fraction, k_evaluate plans/s and fraction."""
    import synth
    legs = {}
    for name in names:
        inst = synth.by_name(name, 0)
        plan = sat.Plan(inst.node_gpus, local).load_runtime_table(inst.runtime)
        G = args.generations
        scfg = sat.SearchConfig(seed=2309, population=args.population, max_generations=G, elites=args.elites,
                                generations_per_epoch=max(1, G // 2))
        steps = 5 if name == "SWEEP" else 20
        m, st, r = measure_search(sat, torch, plan, inst, scfg, steps, 2, stream, G)
        e2e = measure_e2e(plan, inst, scfg, max(2, steps // 4), stream, torch)
        rl = ga_roofline(st, inst.n_jobs, inst.node_gpus, G, steps, m["ms_per_step"] * steps)
        n_eval = (1 << 21) if name == "SWEEP" else (1 << 24)
        ev = evaluate_rate(sat, torch, plan, n_eval)
        ops = algorithmic_ops_per_plan(inst.n_jobs, inst.node_gpus)
        legs[name] = {"workload": WORKLOADS[name], "value": m["value"], "unit": UNIT, "ms_per_step": m["ms_per_step"],
                      "steps": steps, "e2e": e2e["value"], "k_ga_frac": rl["frac"], "k_ga_launch_ms": rl["launch_ms"],
                      "k_evaluate_plans_per_s": ev, "k_evaluate_frac": ops * ev / ALU_PEAK_OPS,
                      "ops_per_plan": ops, "best_this_run": r["makespan"]}
        del plan
        torch.cuda.empty_cache()
    return legs


def quality_leg(sat, torch, local, budget_s, runs):
    """The quality target: a `budget_s` saturn_search per (workload, table
    seed), seeded with the paper's baseline heuristics (row f2), wall time measured from the
    call; best against the committed 5-minute CPU bar and lower bound."""
    import numpy as np
    import synth
    refs = _json(os.path.join("profiles", "r2", "oracle_refs.json")) or {}
    out = []
    for name, s in runs:
        inst = synth.by_name(name, s)
        plan = sat.Plan(inst.node_gpus, local).load_runtime_table(inst.runtime)
        sc, sq, base, per_node = [], [], {}, {}
        for kind in ("max", "min", "optimus", "random"):
            gc, gq = plan.baseline_genome(kind, s)
            sc.append(gc)
            sq.append(gq)
            base[kind] = int(plan.evaluate_host(gc[None], gq[None])[0])
            if len(inst.node_gpus) > 1:   # the heuristics' own per-node plan (node genes, reading A16)
                gn = torch.from_numpy(plan.baseline_nodes(kind, s)[None]).cuda()
                per_node[kind] = int(plan.evaluate_nodes(torch.from_numpy(gc[None]).cuda(),
                                                         torch.from_numpy(gq[None]).cuda(), gn).cpu()[0])
        cfg = sat.SearchConfig(seed=100 + s, population=1 << 20, max_generations=1 << 30, time_budget_s=budget_s,
                               elites=16, generations_per_epoch=32)
        t0 = time.perf_counter()
        r = plan.search(cfg, seed_genomes=(np.stack(sc), np.stack(sq)))
        wall = time.perf_counter() - t0
        t, h = plan.search_history()
        anytime = {}
        for target in (0.01, 0.1, 1.0, 5.0, budget_s):
            k = int(np.searchsorted(t, target, side="right")) - 1
            if k >= 0:
                anytime[f"{target:g}s"] = int(h[k])
        b = _bar(name, s)
        lb = refs.get("lower_bound", {}).get(name, {}).get(str(s))
        out.append({"workload": name, "table_seed": s, "best": r["makespan"], "wall_s": wall,
                    "plans_evaluated": r["evaluated"], "generations": r["generations"], "anytime": anytime,
                    "cpu_5min_bar": b["bar"], "bar_file": b.get("bar_file"),
                    "beats_bar": (b["bar"] is not None and r["makespan"] <= b["bar"]),
                    "lower_bound": lb, "best_over_lb": (r["makespan"] / lb) if lb else None,
                    "best_lower_bound": b.get("bar_best_lower_bound"),
                    "gap_to_best_lower_bound": ((r["makespan"] - b["bar_best_lower_bound"]) / b["bar_best_lower_bound"])
                    if b.get("bar_best_lower_bound") else None, "baselines": base,
                    **({"baselines_per_node": per_node} if per_node else {})})
        del plan
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="saturn", choices=["saturn", "reference"])
    ap.add_argument("--workload", default="TXT", choices=sorted(WORKLOADS))
    # 2^23 genomes per GPU: the per-launch fixed cost (prologue, the last chunk's tail) is
    # 3 % of a k_ga launch at 2^22 and 1 % here (tools/pop_scaling.py)
    ap.add_argument("--population", type=int, default=1 << 23)
    ap.add_argument("--generations", type=int, default=16)
    ap.add_argument("--elites", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-per-core", type=int, default=100000)
    ap.add_argument("--kernel-only-n", type=int, default=1 << 24)
    ap.add_argument("--no-workloads", action="store_true", help="skip the other BASELINE configs' legs")
    ap.add_argument("--quality-budget", type=float, default=10.0,
                    help="seconds per quality search (0 skips the quality leg)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import synth
    import paper_2309_01226_b200 as sat

    # The library's island exchange runs over NCCL (default) or over peer memory
    # (SATURN_TRANSPORT=peers: CUDA IPC + a shared-memory barrier); torch.distributed only
    # carries the host plumbing (barriers, max over ranks) -- over gloo with the peer
    # transport.  SATURN_SHARE_GPU=1 puts every rank on cuda:0 (a functional check of the
    # multi-rank path on a one-GPU box; its numbers are not a scaling measurement).
    transport = os.environ.get("SATURN_TRANSPORT", "nccl")
    share = os.environ.get("SATURN_SHARE_GPU") == "1"
    if share and transport != "peers":
        raise SystemExit("SATURN_SHARE_GPU=1 needs SATURN_TRANSPORT=peers (NCCL refuses two ranks on one GPU)")
    local = 0 if share else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if transport == "peers":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    inst = synth.by_name(args.workload, 0)
    plan = sat.Plan(inst.node_gpus, local).load_runtime_table(inst.runtime)
    if world > 1:
        if transport == "peers":
            sat.attach_peers(plan)
        else:
            sat.attach_distributed(plan)
    T = inst.n_jobs
    P, G, E = args.population, args.generations, args.elites
    scfg = sat.SearchConfig(seed=2309, population=P, max_generations=G, elites=E,
                            generations_per_epoch=max(1, G // 2))
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if transport == "peers" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: K steps, device time via CUDA events on the launching stream
    with ClockSampler(local) as clk:
        m, st, r = measure_search(sat, torch, plan, inst, scfg, args.steps, args.warmup, stream, G, barrier,
                                  max_over_ranks)
    dev_ms = m["ms_per_step"] * args.steps
    value = m["value"]                       # `evaluated` already sums all ranks
    best_ms = r["makespan"]

    # ---- e2e: host API with host buffers (table upload + search + best plan to host)
    barrier()
    with ClockSampler(local):          # same conditions as the device-timed region
        e2e = measure_e2e(plan, inst, scfg, args.steps, stream, torch, max_over_ranks)

    # ---- roofline of the dominant kernel (the fused GA generation + decode kernel)
    roofline = ga_roofline(st, T, inst.node_gpus, G, args.steps, dev_ms)
    roofline["traffic"] = _traffic(args.workload)

    # ---- kernel-only evaluate throughput (K1 alone, genomes resident in HBM)
    kernel_only = None
    if rank == 0 and args.kernel_only_n > 0:
        n = args.kernel_only_n
        kernel_only = {"unit": UNIT, "genomes": n,
                       "thread": evaluate_rate(sat, torch, plan, n, kind=sat.DECODER_THREAD),
                       "warp": evaluate_rate(sat, torch, plan, n, kind=sat.DECODER_WARP)}
        ops = algorithmic_ops_per_plan(T, inst.node_gpus)
        # exhaustive enumeration (row a4-ii): a 7-job TINY-shaped instance, 6^7 * 7! genomes
        tv = synth.tiny_variant(7, 7, (4,))
        ep = sat.Plan(tv.node_gpus, local).load_runtime_table(tv.runtime)
        ep.enumerate()
        t0 = time.perf_counter()
        er = ep.enumerate()                      # DFS, prefix sharing + branch and bound
        t_dfs = time.perf_counter() - t0
        t0 = time.perf_counter()
        space = ep.space_size()
        fr = ep.enumerate_range(0, space)   # index order, one full decode per genome
        t_full = time.perf_counter() - t0
        kernel_only["enumerate"] = {
            "instance": "TINY-shaped 7 jobs on 1x4 (seed 7)", "genomes": space, "optimum": er["makespan"],
            "full_decode_plans_per_s": fr["evaluated"] / t_full,
            "dfs_seconds": t_dfs, "dfs_leaves": er["leaves"], "dfs_leaves_per_s": er["leaves"] / t_dfs,
            "dfs_genomes_covered_per_s": space / t_dfs,
            "same_result": (er["makespan"], er["genome_index"]) == (fr["makespan"], fr["genome_index"])}
        # the decode kernel alone against the same ALU roofline (algorithmic ops per plan)
        kernel_only["roofline_thread"] = {"bound": "alu", "achieved": ops * kernel_only["thread"] / 1e12,
                                          "peak": ALU_PEAK_OPS / 1e12, "unit": "TOP/s",
                                          "frac": ops * kernel_only["thread"] / ALU_PEAK_OPS,
                                          "kernel": "k_evaluate (T design, validity-checked decode)"}
        kernel_only["int_probe_ops_per_s"] = plan.probe_int_peak()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    refs = _json(os.path.join("profiles", "r2", "oracle_refs.json")) or {}
    # "best makespan vs oracle": on TINY the GPU enumeration and a short GPU search against
    # the oracle's brute-force optimum (profiles/r2/oracle_refs.json, written by
    # tools/oracle_refs.py from oracle/ only); on the bench workload the best found against
    # the lower bound and the committed 5-minute CPU bar.
    tiny = synth.tiny(0)
    tplan = sat.Plan(tiny.node_gpus, local).load_runtime_table(tiny.runtime)
    t_enum = tplan.enumerate()
    t_srch = tplan.search(sat.SearchConfig(seed=1, population=1024, max_generations=20, elites=8))
    opt = refs.get("tiny_brute_force", {}).get("0", {})
    vs_oracle = {"TINY": {"oracle_brute_force": opt.get("makespan"), "oracle_genome_index": opt.get("genome_index"),
                          "gpu_enumerate": t_enum["makespan"], "gpu_enumerate_index": t_enum["genome_index"],
                          "gpu_search": t_srch["makespan"],
                          "bit_exact": (t_enum["makespan"], t_enum["genome_index"]) ==
                                       (opt.get("makespan"), opt.get("genome_index"))},
                 args.workload: {"gpu_best_this_run": best_ms,
                                 "lower_bound": refs.get("lower_bound", {}).get(args.workload, {}).get("0"),
                                 "cpu_5min_bar_seed0": _bar(args.workload, 0)["bar"]}}
    del tplan
    legs = None
    quality = None
    if world == 1:
        if not args.no_workloads:
            del plan
            torch.cuda.empty_cache()
            legs = workload_legs(sat, torch, args, local, stream, [w for w in ("TINY", "TXT", "IMG", "MIX", "SWEEP")
                                                                   if w != args.workload])
            legs[args.workload] = {"workload": WORKLOADS[args.workload], "value": value, "unit": UNIT,
                                   "ms_per_step": dev_ms / args.steps, "steps": args.steps, "e2e": e2e["value"],
                                   "k_ga_frac": roofline["frac"], "k_ga_launch_ms": roofline["launch_ms"],
                                   "k_evaluate_plans_per_s": kernel_only["thread"] if kernel_only else None,
                                   "k_evaluate_frac": kernel_only["roofline_thread"]["frac"] if kernel_only else None,
                                   "ops_per_plan": roofline["ops_per_plan"], "best_this_run": best_ms}
        if args.quality_budget > 0:
            quality = quality_leg(sat, torch, local, args.quality_budget,
                                  [("TXT", 0), ("TXT", 1), ("TXT", 2), ("MIX", 0), ("SWEEP", 0)])
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload, args.cpu_seconds)
        cpu["cpu"] = host_cpu()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded runtime tables shaped like the paper's workloads; random-init GA)",
            "config": _config(args),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": st["kernel_launches"],
            "clocks": clk.summary(), "kernel_only": kernel_only, "best_vs_oracle": vs_oracle,
            "workloads": legs, "quality": quality, "host_cpu": host_cpu()}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
