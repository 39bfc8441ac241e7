"""Seeded synthetic SPASE instances and genome sets (input recipe; see DESIGN.md §"Input recipe").

The paper's runtime tables are hardware-measured and unpublished, so these tables are
invented and *shaped* to the paper's facts:

* workloads TXT / IMG: PAPER.md:1086-1087 (Table 2) -- 2 architectures x 2 batch sizes x
  3 learning rates = 12 jobs, 10 epochs; the learning rate does not change runtime, so each
  workload is 4 base rows replicated 3x, each job with its own +-2 % profiling noise
  (jobs are profiled separately);
* UPP columns DDP, FSDP, PIPE, SPILL: PAPER.md:1108-1113;
* runtime model (the SPEC.md:79 Amdahl + communication form)
      R(t,u,g) = ceil(W_t * (sigma_u + (1 - sigma_u) / g) + c_u * (g - 1)),  g in [m_{a,u}, 8]
  with c_u = kappa_u * params_B; SPILL only at g = 1 with R = ceil(3 * W_t)
  ("spilling can enable large models to be trained with even just one GPU");
* hardware settings: 1x8, 2x8, 4x8 GPUs and heterogeneous {2,2,4,8}.

A dense table is ``int32 runtime[T][U][Gmax]`` in integer seconds; entry ``[t][u][g-1]`` is
the runtime of job t under UPP u on g GPUs, and ``0`` marks an infeasible (null, OOM)
profile.  This module performs no SPASE arithmetic: it never compacts,
decodes or searches.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

UPPS = ("DDP", "FSDP", "PIPE", "SPILL")
DDP, FSDP, PIPE, SPILL = range(4)

# Serial fraction sigma_u and per-extra-GPU communication cost kappa_u (s per billion params).
SIGMA = {DDP: 0.03, FSDP: 0.06, PIPE: 0.12}
KAPPA = {DDP: 150.0, FSDP: 250.0, PIPE: 60.0}
SPILL_PENALTY = 3.0

INF_M = 99  # "minimum GPUs" sentinel meaning the UPP is infeasible for the archetype


@dataclass(frozen=True)
class Archetype:
    name: str
    work_s: float          # W: 10 epochs on one ideal GPU, seconds
    params_b: float        # parameters, billions (drives c_u)
    min_gpus: tuple        # m for (DDP, FSDP, PIPE); INF_M = infeasible


# SURVEY.md §8d archetype table (W, m); params from PAPER.md:1086-1087.
GPT2_B16 = Archetype("GPT-2 B16", 11000.0, 1.5, (1, 1, 2))
GPT2_B32 = Archetype("GPT-2 B32", 10000.0, 1.5, (2, 1, 2))
GPTJ_B16 = Archetype("GPT-J B16", 44000.0, 6.0, (INF_M, 3, 3))
GPTJ_B32 = Archetype("GPT-J B32", 40000.0, 6.0, (INF_M, 3, 3))
VITG_B64 = Archetype("ViT-G B64", 16000.0, 1.8, (2, 1, 2))
VITG_B128 = Archetype("ViT-G B128", 14000.0, 1.8, (2, 1, 2))
RESNET_B64 = Archetype("ResNet B64", 4000.0, 0.2, (1, 1, 2))
RESNET_B128 = Archetype("ResNet B128", 3600.0, 0.2, (1, 1, 2))

TXT_ARCH = (GPT2_B16, GPT2_B32, GPTJ_B16, GPTJ_B32)
IMG_ARCH = (VITG_B64, VITG_B128, RESNET_B64, RESNET_B128)
LEARNING_RATES = (1e-5, 1e-4, 3e-3)


@dataclass
class Instance:
    """One SPASE instance: cluster ``node_gpus`` (GPU_n) and the dense runtime table."""
    name: str
    node_gpus: list
    runtime: np.ndarray            # int32 [T][U][Gmax]; 0 = infeasible
    jobs: list = field(default_factory=list)   # human-readable job labels
    upps: tuple = UPPS

    @property
    def n_jobs(self) -> int:
        return int(self.runtime.shape[0])

    @property
    def n_upps(self) -> int:
        return int(self.runtime.shape[1])

    @property
    def max_gpus(self) -> int:
        return int(self.runtime.shape[2])


def _runtime_row(work_s: float, params_b: float, min_gpus, gmax: int, upps=(DDP, FSDP, PIPE, SPILL),
                 g_allowed=None) -> np.ndarray:
    row = np.zeros((len(upps), gmax), dtype=np.int64)
    for ui, u in enumerate(upps):
        for g in range(1, gmax + 1):
            if g_allowed is not None and g not in g_allowed:
                continue
            if u == SPILL:
                if g == 1:
                    row[ui, 0] = math.ceil(SPILL_PENALTY * work_s)
                continue
            if g < min_gpus[u]:
                continue
            sigma, c = SIGMA[u], KAPPA[u] * params_b
            row[ui, g - 1] = math.ceil(work_s * (sigma + (1.0 - sigma) / g) + c * (g - 1))
    return row


def _workload(name, archs, nodes, seed, noise, n_rep=3, gmax=8):
    rng = np.random.Generator(np.random.PCG64(seed))
    rows, labels = [], []
    for rep in range(n_rep):
        for a in archs:
            w = a.work_s * (1.0 + rng.uniform(-noise, noise))
            rows.append(_runtime_row(w, a.params_b, a.min_gpus, gmax))
            labels.append(f"{a.name} lr={LEARNING_RATES[rep % 3]:g} #{rep}")
    table = np.stack(rows).astype(np.int32)
    return Instance(name, list(nodes), table, labels)


def txt(seed: int = 0) -> Instance:
    """C2: single-node TXT, 12 GPT-2/GPT-J jobs x 4 UPPs x g 1-8 on 1x8 GPUs."""
    return _workload("TXT", TXT_ARCH, [8], seed, 0.02)


def img(seed: int = 0) -> Instance:
    """C3: single-node IMG, 12 ViT-G/ResNet jobs x 4 UPPs x g 1-8 on 1x8 GPUs."""
    return _workload("IMG", IMG_ARCH, [8], seed, 0.02)


def mix(seed: int = 0) -> Instance:
    """C4: TXT u IMG = 24 jobs on 2 nodes x 8 GPUs."""
    a, b = txt(seed), img(seed + 1000)
    return Instance("MIX", [8, 8], np.concatenate([a.runtime, b.runtime]), a.jobs + b.jobs)


def sweep(seed: int = 0, n_jobs: int = 100, nodes=(8, 8, 8, 8)) -> Instance:
    """C5: 100 jobs cycling the 8 archetypes (+-5 % noise) on 4 nodes x 8 GPUs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    archs = TXT_ARCH + IMG_ARCH
    rows, labels = [], []
    for j in range(n_jobs):
        a = archs[j % len(archs)]
        w = a.work_s * (1.0 + rng.uniform(-0.05, 0.05))
        rows.append(_runtime_row(w, a.params_b, a.min_gpus, 8))
        labels.append(f"{a.name} #{j}")
    return Instance("SWEEP", list(nodes), np.stack(rows).astype(np.int32), labels)


def tiny(seed: int = 0, n_jobs: int = 3, nodes=(4,)) -> Instance:
    """C1: 3 jobs x {DDP, FSDP} x g in {1,2,4} on 1x4 GPUs; all 6 configs feasible.

    W_t ~ U[100, 1000], default sigma, c ~ U[0, 0.05 W_t] per (job, UPP).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    gmax = 4
    rows, labels = [], []
    for j in range(n_jobs):
        w = rng.uniform(100.0, 1000.0)
        row = np.zeros((2, gmax), dtype=np.int64)
        for ui, u in enumerate((DDP, FSDP)):
            c = rng.uniform(0.0, 0.05 * w)
            for g in (1, 2, 4):
                row[ui, g - 1] = math.ceil(w * (SIGMA[u] + (1.0 - SIGMA[u]) / g) + c * (g - 1))
        rows.append(row)
        labels.append(f"tiny#{j}")
    return Instance("TINY", list(nodes), np.stack(rows).astype(np.int32), labels, upps=("DDP", "FSDP"))


def tiny_variant(seed: int, n_jobs: int, nodes=(4,)) -> Instance:
    """4-6-job TINY-shaped variants on 1x4 or 2x2 GPUs (parity extras)."""
    inst = tiny(seed, n_jobs, nodes)
    inst.name = f"TINY{n_jobs}-{'x'.join(map(str, nodes))}"
    return inst


def random_tiny(rng: np.random.Generator, max_jobs: int = 4, node_choices=None, max_r: int = 6,
                n_upps: int = 2, p_feasible: float = 0.6) -> Instance:
    """Small random instances for property tests: integer runtimes in [1, max_r].

    Every job gets at least one config that fits some node.
    """
    if node_choices is None:
        node_choices = ([2], [3], [4], [2, 2], [2, 3], [4, 2], [3, 3])
    nodes = list(node_choices[rng.integers(len(node_choices))])
    n_jobs = int(rng.integers(1, max_jobs + 1))
    gmax = max(nodes)
    table = np.zeros((n_jobs, n_upps, gmax), dtype=np.int32)
    for t in range(n_jobs):
        mask = rng.random((n_upps, gmax)) < p_feasible
        if not mask.any():
            mask[rng.integers(n_upps), rng.integers(gmax)] = True
        table[t] = np.where(mask, rng.integers(1, max_r + 1, size=(n_upps, gmax)), 0)
    return Instance("RANDOM", nodes, table, [f"r{t}" for t in range(n_jobs)],
                    upps=UPPS[:n_upps])


def lr_sweep(seed: int, n_models: int, n_lrs, nodes=(4,)) -> Instance:
    """A TINY-shaped learning-rate sweep: model m is trained at n_lrs[m] learning rates.  A
    job's runtime does not depend on its learning rate, so the replicas of a model share one
    runtime row exactly (no per-job noise) -- the twin structure of row f4."""
    base = tiny(seed, n_models, nodes)
    rows, labels = [], []
    for m in range(n_models):
        for k in range(n_lrs[m]):
            rows.append(base.runtime[m])
            labels.append(f"tiny#{m} lr={LEARNING_RATES[k % len(LEARNING_RATES)]:g}")
    return Instance(f"LRSWEEP{sum(n_lrs)}", list(nodes), np.stack(rows).astype(np.int32), labels,
                    upps=base.upps)


CONFIG_NAMES = ("TINY", "TXT", "IMG", "MIX", "SWEEP")


def by_name(name: str, seed: int = 0) -> Instance:
    return {"TINY": tiny, "TXT": txt, "IMG": img, "MIX": mix, "SWEEP": sweep}[name.upper()](seed)


def random_genomes(n_cfgs, n: int, seed: int):
    """n random genomes for a table with ``n_cfgs[t]`` configurations per job.

    Returns (cfg, perm), both uint8 arrays of shape [n][T] (genome-major rows):
    cfg[i][t] uniform in [0, n_cfgs[t]), perm[i] a uniform random permutation of 0..T-1
    ("Genome sets").  ``n_cfgs`` is supplied by the caller.
    """
    s = np.asarray(n_cfgs, dtype=np.int64)
    rng = np.random.Generator(np.random.PCG64(seed))
    T = s.shape[0]
    cfg = rng.integers(0, s, size=(n, T)).astype(np.uint8)
    perm = rng.permuted(np.broadcast_to(np.arange(T, dtype=np.uint8), (n, T)), axis=1)
    return np.ascontiguousarray(cfg), np.ascontiguousarray(perm.astype(np.uint8))
