"""f2: the paper's baseline heuristics as genomes.  TEST INFRASTRUCTURE ONLY (reference for
the library's saturn_baseline_genome).

The paper's four comparison approaches (§4.3.1) pick a configuration per
task; the plan is then built by list scheduling.  Here each baseline yields a GENOME
(cfg per job + priority permutation) that the hot-path decoder turns into a plan
(DESIGN.md "Baselines"):

  best_config_for(t, g): the config of job t with g GPUs and the least runtime, ties to the
      lower UPP index (DDP < FSDP < PIPE < SPILL, i.e. the parallelism name order of
      SPEC.md:70) -- "we refer to the Profiler to determine which parallelism gives Model A
      the best runtime at 8 GPUs";
  order: LPT -- jobs by descending runtime of their chosen config, ties to the lower job id
      (SPEC.md:350, 365);
  node groups (multi-node): job t goes to node n with probability GPU_n / sum GPU
      (SPEC.md:338-346), draw u = U(sum GPU, w_t) with w_t word 0 of the
      Philox stream (t, 0, 3 << 16), node = first n with u < GPU_0 + ... + GPU_n;
  MAX: every job gets its node's full width, or the widest width
      with a config below it (the job's narrowest width if none fits the node);
  MIN: one GPU each (spilling); a node's surplus GPUs are dealt
      round-robin to its jobs in job order, a job's share capped at its widest config; the
      job then uses the widest width <= its share that has a config;
  OPTIMUS (Alg. 1), per node: L = [1, ...]; while sum L < GPU_n: gain_t =
      R(t, L_t) - R(t, L_t + 1) with R(t, g) the best runtime at g GPUs (-inf if job t has
      no config at L_t + 1); increment the first argmax; stop early if every gain is -inf;
  RANDOM: the GA's initial genome of slot k (oracle/ga.py) -- uniform config
      per job, uniform order.

baseline_nodes: the baselines decide each job's node ("one node at a time": the per-node
  allocations of MAX / MIN / OPTIMUS).  As node genes (reading A16) job t
  runs on its distributed node when its chosen config fits there, else it is placed greedily
  (0xFF, only when even the job's narrowest width exceeds that node); RANDOM is all greedy.
  The decoder with these genes yields the per-node plan; without them it re-picks nodes.
"""
from __future__ import annotations

from .philox import Stream
from . import ga

NEG_INF = float("-inf")


def best_config_for(c, t, g):
    best = None
    for s in range(int(c.S[t])):
        u, gg, r = c.config(t, s)
        if gg == g and (best is None or r < best[1] or (r == best[1] and u < c.config(t, best[0])[0])):
            best = (s, r)
    return best  # (config index, runtime) or None


def widths(c, t):
    return sorted({c.config(t, s)[1] for s in range(int(c.S[t]))})


def lpt_order(runtimes):
    return sorted(range(len(runtimes)), key=lambda t: (-runtimes[t], t))


def distribute(c, seed: int):
    """Node of each job (weighted by GPU count); single node -> all 0."""
    N = len(c.node_gpus)
    if N == 1:
        return [0] * c.n_jobs
    total = int(sum(int(x) for x in c.node_gpus))
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    out = []
    for t in range(c.n_jobs):
        u = Stream(key, t, 0, 3 << 16).below(total)
        acc = 0
        for n in range(N):
            acc += int(c.node_gpus[n])
            if u < acc:
                out.append(n)
                break
    return out


def _fits(c, t, n):
    return [w for w in widths(c, t) if w <= int(c.node_gpus[n])]


def _genome(c, chosen):
    cfg = [s for s, _ in chosen]
    perm = lpt_order([r for _, r in chosen])
    return cfg, perm


def max_heuristic(c, seed: int = 0):
    node = distribute(c, seed)
    chosen = []
    for t in range(c.n_jobs):
        n = node[t]
        ws = _fits(c, t, n) or [min(widths(c, t))]
        g = max(ws)
        chosen.append(best_config_for(c, t, g))
    return _genome(c, chosen)


def min_heuristic(c, seed: int = 0):
    node = distribute(c, seed)
    share = [1] * c.n_jobs
    for n in range(len(c.node_gpus)):
        jobs = [t for t in range(c.n_jobs) if node[t] == n]
        if not jobs:
            continue
        cap = {t: max(_fits(c, t, n) or [1]) for t in jobs}
        surplus = int(c.node_gpus[n]) - len(jobs)
        while surplus > 0:
            progressed = False
            for t in jobs:
                if surplus > 0 and share[t] < cap[t]:
                    share[t] += 1
                    surplus -= 1
                    progressed = True
            if not progressed:
                break
    chosen = []
    for t in range(c.n_jobs):
        ws = [w for w in widths(c, t) if w <= share[t]] or [min(widths(c, t))]
        chosen.append(best_config_for(c, t, max(ws)))
    return _genome(c, chosen)


def optimus_greedy_alloc(R, G):
    """Alg. 1 on best-runtime rows R[t][g] (None = no config at g GPUs), G GPUs."""
    L = [1] * len(R)
    while sum(L) < G:
        gains = []
        for t, l in enumerate(L):
            cur = R[t].get(l)
            nxt = R[t].get(l + 1)
            gains.append(NEG_INF if (cur is None or nxt is None) else cur - nxt)
        best = max(gains)
        if best == NEG_INF:
            break
        L[gains.index(best)] += 1
    return L


def optimus_greedy(c, seed: int = 0):
    node = distribute(c, seed)
    alloc = [1] * c.n_jobs
    for n in range(len(c.node_gpus)):
        jobs = [t for t in range(c.n_jobs) if node[t] == n]
        if not jobs:
            continue
        R = []
        for t in jobs:
            row = {}
            for g in range(1, int(c.node_gpus[n]) + 1):
                b = best_config_for(c, t, g)
                if b is not None:
                    row[g] = b[1]
            R.append(row)
        L = optimus_greedy_alloc(R, int(c.node_gpus[n]))
        for t, l in zip(jobs, L):
            alloc[t] = l
    chosen = []
    for t in range(c.n_jobs):
        b = best_config_for(c, t, alloc[t])
        if b is None:  # no config at the allocated width (no 1-GPU config): widest fitting
            ws = [w for w in widths(c, t) if w <= alloc[t]] or [min(widths(c, t))]
            b = best_config_for(c, t, max(ws))
        chosen.append(b)
    return _genome(c, chosen)


def randomized(c, seed: int = 0, k: int = 0):
    return ga.initial_genome(c.S, seed, 0, k)


GREEDY = 0xFF


def baseline_nodes(c, kind: str, seed: int = 0):
    """Node genes (job-id order) of a baseline's per-node plan; see the module docstring."""
    if kind == "random":
        return [GREEDY] * c.n_jobs
    cfg, _ = KINDS[kind](c, seed)
    node = distribute(c, seed)
    return [node[t] if c.config(t, cfg[t])[1] <= int(c.node_gpus[node[t]]) else GREEDY for t in range(c.n_jobs)]


KINDS = {"max": max_heuristic, "min": min_heuristic, "optimus": optimus_greedy, "random": randomized}
