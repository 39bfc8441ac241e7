"""O1 decoder / O2 brute force (ctypes over saturn_oracle.c) and the table compaction.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "saturn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build_library(force: bool = False) -> str:
    """Compile saturn_oracle.c with plain gcc (no vectorisation flags, no threads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


class _Placement(ctypes.Structure):
    _fields_ = [("node", ctypes.c_int32), ("upp", ctypes.c_int32), ("gpus", ctypes.c_int32),
                ("cfg", ctypes.c_int32), ("start_s", ctypes.c_int32), ("end_s", ctypes.c_int32),
                ("gpu_mask", ctypes.c_uint64)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_library())
        P = ctypes.POINTER
        i32, u8, u64 = ctypes.c_int32, ctypes.c_uint8, ctypes.c_uint64
        _lib.or_decode.restype = i32
        _lib.or_decode.argtypes = [i32, P(i32), i32, i32, P(i32), P(i32), P(i32), P(u8), P(u8), P(u8),
                                   P(_Placement)]
        _lib.or_decode_batch.restype = None
        _lib.or_decode_batch.argtypes = [i32, P(i32), i32, i32, P(i32), P(i32), P(i32), ctypes.c_int64,
                                         P(u8), P(u8), P(i32)]
        _lib.or_decode_batch_nodes.restype = None
        _lib.or_decode_batch_nodes.argtypes = [i32, P(i32), i32, i32, P(i32), P(i32), P(i32), ctypes.c_int64,
                                               P(u8), P(u8), P(u8), P(i32)]
        _lib.or_unrank.restype = ctypes.c_int
        _lib.or_unrank.argtypes = [i32, P(i32), u64, P(u8), P(u8)]
        _lib.or_brute_force.restype = i32
        _lib.or_brute_force.argtypes = [i32, P(i32), i32, i32, P(i32), P(i32), P(i32), u64, u64, P(u64)]
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


@dataclass
class Compacted:
    """Feasible configs per job in UPP-major, ascending-g order, restricted to
    g <= max_n GPU_n (single-node jobs; reading A8).  Config s of job t is
    (upp[t][s], gpus[t][s], runtime[t][s]); S[t] = number of configs (Table 1's S_t)."""
    node_gpus: np.ndarray   # int32 [N]
    S: np.ndarray           # int32 [T]
    stride: int
    gpus: np.ndarray        # int32 [T*stride]
    runtime: np.ndarray     # int32 [T*stride]
    upp: np.ndarray         # int32 [T*stride]

    @property
    def n_jobs(self) -> int:
        return int(self.S.shape[0])

    def config(self, t: int, s: int):
        k = t * self.stride + s
        return int(self.upp[k]), int(self.gpus[k]), int(self.runtime[k])


def compact(node_gpus, runtime) -> Compacted:
    """Dense ``runtime[T][U][Gmax]`` (<= 0 = infeasible) -> Compacted.

    Raises ValueError naming the job when a job has no feasible config that fits a node
    (reading A9)."""
    node_gpus = np.asarray(node_gpus, dtype=np.int32)
    runtime = np.asarray(runtime)
    T, U, gmax = runtime.shape
    biggest = int(node_gpus.max())
    rows = []
    for t in range(T):
        row = []
        for u in range(U):
            for g in range(1, gmax + 1):
                r = int(runtime[t, u, g - 1])
                if r > 0 and g <= biggest:
                    row.append((u, g, r))
        if not row:
            raise ValueError(f"job {t} has no feasible configuration on this cluster")
        rows.append(row)
    stride = max(len(r) for r in rows)
    gp = np.zeros(T * stride, np.int32)
    rt = np.zeros(T * stride, np.int32)
    up = np.full(T * stride, -1, np.int32)
    for t, row in enumerate(rows):
        for s, (u, g, r) in enumerate(row):
            gp[t * stride + s], rt[t * stride + s], up[t * stride + s] = g, r, u
    return Compacted(node_gpus, np.array([len(r) for r in rows], np.int32), stride, gp, rt, up)


def decode(c: Compacted, cfg, perm, node_gene=None):
    """O1 on one genome -> (makespan, placements) where placements[t] is a dict with the
    paper's per-task outputs (node O, GPU ids P, config B, start I)."""
    lib = _L()
    T = c.n_jobs
    cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.uint8)
    ng = None if node_gene is None else np.ascontiguousarray(node_gene, dtype=np.uint8)
    out = (_Placement * T)()
    ms = lib.or_decode(len(c.node_gpus), _p(c.node_gpus, ctypes.c_int32), T, c.stride,
                       _p(c.gpus, ctypes.c_int32), _p(c.runtime, ctypes.c_int32), _p(c.S, ctypes.c_int32),
                       _p(cfg, ctypes.c_uint8), _p(perm, ctypes.c_uint8),
                       None if ng is None else _p(ng, ctypes.c_uint8), out)
    if ms < 0:
        return ms, None
    pl = []
    for t in range(T):
        o = out[t]
        pl.append(dict(node=o.node, upp=int(c.upp[t * c.stride + o.cfg]), gpus=o.gpus, cfg=o.cfg,
                       start_s=o.start_s, end_s=o.end_s, gpu_mask=int(o.gpu_mask)))
    return ms, pl


def decode_batch(c: Compacted, cfg, perm) -> np.ndarray:
    """O1 over genome rows cfg[n][T], perm[n][T] -> int32 makespans [n] (-1 = invalid)."""
    lib = _L()
    cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.uint8)
    n = cfg.shape[0]
    out = np.empty(n, np.int32)
    lib.or_decode_batch(len(c.node_gpus), _p(c.node_gpus, ctypes.c_int32), c.n_jobs, c.stride,
                        _p(c.gpus, ctypes.c_int32), _p(c.runtime, ctypes.c_int32), _p(c.S, ctypes.c_int32),
                        n, _p(cfg, ctypes.c_uint8), _p(perm, ctypes.c_uint8), _p(out, ctypes.c_int32))
    return out


def decode_batch_nodes(c: Compacted, cfg, perm, node) -> np.ndarray:
    """O1 with node genes (0xFF = greedy for that job) over genome rows -> makespans."""
    lib = _L()
    cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.uint8)
    node = np.ascontiguousarray(node, dtype=np.uint8)
    n = cfg.shape[0]
    out = np.empty(n, np.int32)
    lib.or_decode_batch_nodes(len(c.node_gpus), _p(c.node_gpus, ctypes.c_int32), c.n_jobs, c.stride,
                              _p(c.gpus, ctypes.c_int32), _p(c.runtime, ctypes.c_int32), _p(c.S, ctypes.c_int32),
                              n, _p(cfg, ctypes.c_uint8), _p(perm, ctypes.c_uint8), _p(node, ctypes.c_uint8),
                              _p(out, ctypes.c_int32))
    return out


def space_size(c: Compacted) -> int:
    """|genome space| = T! * prod_t S_t."""
    return math.factorial(c.n_jobs) * int(np.prod([int(s) for s in c.S], dtype=object))


def unrank(c: Compacted, index: int):
    cfg = np.zeros(c.n_jobs, np.uint8)
    perm = np.zeros(c.n_jobs, np.uint8)
    if _L().or_unrank(c.n_jobs, _p(c.S, ctypes.c_int32), index, _p(cfg, ctypes.c_uint8),
                      _p(perm, ctypes.c_uint8)) != 0:
        raise ValueError("index outside the genome space")
    return cfg, perm


def rank(c: Compacted, cfg, perm) -> int:
    """Inverse of unrank, written independently: mixed radix (job 0 least significant)
    for cfg, Lehmer code (perm[0] most significant) for perm."""
    r_cfg, radix = 0, 1
    for t in range(c.n_jobs):
        r_cfg += int(cfg[t]) * radix
        radix *= int(c.S[t])
    T = c.n_jobs
    r_perm = 0
    for p in range(T):
        smaller_later = sum(1 for q in range(p + 1, T) if perm[q] < perm[p])
        r_perm += smaller_later * math.factorial(T - 1 - p)
    return r_perm * radix + r_cfg


def brute_force(c: Compacted, begin: int = 0, end: int | None = None):
    """O2: (min makespan, first index attaining it) over genome indices [begin, end)."""
    if end is None:
        end = space_size(c)
    best = ctypes.c_uint64(0)
    ms = _L().or_brute_force(len(c.node_gpus), _p(c.node_gpus, ctypes.c_int32), c.n_jobs, c.stride,
                             _p(c.gpus, ctypes.c_int32), _p(c.runtime, ctypes.c_int32),
                             _p(c.S, ctypes.c_int32), begin, end, ctypes.byref(best))
    return int(ms), int(best.value)


def brute_force_node_gene(c: Compacted) -> int:
    """min over (cfg, node, perm) genomes of the node-gene variant of O1 -- the decoder
    space that provably contains the SPASE optimum."""
    T = c.n_jobs
    N = len(c.node_gpus)
    best = None
    for cfg in itertools.product(*[range(int(s)) for s in c.S]):
        need = [c.config(t, cfg[t])[1] for t in range(T)]
        node_opts = [[n for n in range(N) if c.node_gpus[n] >= need[t]] for t in range(T)]
        for ng in itertools.product(*node_opts):
            for perm in itertools.permutations(range(T)):
                ms, _ = decode(c, cfg, perm, node_gene=ng)
                if best is None or ms < best:
                    best = ms
    return best
