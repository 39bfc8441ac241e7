"""Thin Python binding of include/saturn.h (argument marshalling only).

Every computation runs in libsaturn.so (hand-written sm_100a kernels).  PyTorch is used for
device memory (tensors), streams and torch.distributed bootstrap only.  There is no CPU
fallback: importing this module fails loudly if the library is missing.

Function names follow the C ABI without the ``saturn_`` prefix; ``Plan`` wraps a handle.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsaturn.so")

OK, EINVAL, EUNSCHEDULABLE, ELIMIT, ECUDA, ENCCL, ESTATE = range(7)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "EUNSCHEDULABLE", 3: "ELIMIT", 4: "ECUDA", 5: "ENCCL", 6: "ESTATE"}
PROVEN_OPTIMAL, INCUMBENT, PREFIX_SHARED, SYMMETRY_REDUCED = 1, 2, 4, 8
ENUM_SYMMETRY = 1
DECODER_AUTO, DECODER_THREAD, DECODER_WARP, DECODER_NODE_SMEM = 0, 1, 2, 3

# Every symbol declared in include/saturn.h.
EXPORTS = (
    "saturn_plan_create", "saturn_workspace_bytes", "saturn_bind_workspace", "saturn_load_runtime_table", "saturn_num_configs", "saturn_config",
    "saturn_set_decoder", "saturn_evaluate", "saturn_evaluate_nodes", "saturn_evaluate_host", "saturn_trace", "saturn_space_size",
    "saturn_enumerate", "saturn_enumerate_range", "saturn_set_enumeration_options", "saturn_search", "saturn_search_group", "saturn_search_history",
    "saturn_search_population", "saturn_search_save", "saturn_search_resume", "saturn_best_plan", "saturn_get_unique_id", "saturn_plan_attach_comm",
    "saturn_plan_attach_peers", "saturn_plan_barrier",
    "saturn_partition", "saturn_probe_int_peak", "saturn_set_profiling", "saturn_get_stats",
    "saturn_reset_stats", "saturn_baseline_genome", "saturn_baseline_nodes", "saturn_introspect", "saturn_improve", "saturn_last_error",
    "saturn_plan_destroy",
)
BASELINES = {"max": 1, "min": 2, "optimus": 3, "random": 4}


class SaturnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Placement(ctypes.Structure):
    _fields_ = [("node", ctypes.c_int32), ("upp", ctypes.c_int32), ("gpus", ctypes.c_int32),
                ("cfg", ctypes.c_int32), ("start_s", ctypes.c_int32), ("end_s", ctypes.c_int32),
                ("gpu_mask", ctypes.c_uint64)]


PLACEMENT_DTYPE = np.dtype([("node", "<i4"), ("upp", "<i4"), ("gpus", "<i4"), ("cfg", "<i4"),
                            ("start_s", "<i4"), ("end_s", "<i4"), ("gpu_mask", "<u8")])


class Result(ctypes.Structure):
    _fields_ = [("makespan", ctypes.c_int64), ("genome_index", ctypes.c_uint64), ("evaluated", ctypes.c_uint64),
                ("seconds", ctypes.c_double), ("flags", ctypes.c_int32), ("generations", ctypes.c_int32),
                ("leaves", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("ga_launches", ctypes.c_int64), ("ga_kernel_ms", ctypes.c_double), ("ga_decodes", ctypes.c_int64),
                ("_spare", ctypes.c_int64 * 4)]   # room for older builds' longer struct (A/B runs)

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


class IntrospectEvent(ctypes.Structure):
    _fields_ = [("at_round", ctypes.c_int32), ("kind", ctypes.c_int32), ("job", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("runtime_s", ctypes.c_void_p)]


EVENT_STOP, EVENT_ARRIVE = 1, 2


class IntrospectParams(ctypes.Structure):
    _fields_ = [("interval_s", ctypes.c_int64), ("threshold_s", ctypes.c_int64), ("solver", ctypes.c_int32),
                ("max_rounds", ctypes.c_int32), ("search", ctypes.c_void_p), ("overlap", ctypes.c_int32),
                ("n_events", ctypes.c_int32), ("events", ctypes.c_void_p), ("interval_wall_s", ctypes.c_double)]


class IntrospectResult(ctypes.Structure):
    _fields_ = [("one_shot_makespan", ctypes.c_int64), ("e2e_makespan", ctypes.c_int64), ("rounds", ctypes.c_int32),
                ("adopted", ctypes.c_int32), ("evaluated", ctypes.c_uint64), ("stale", ctypes.c_int32),
                ("solves", ctypes.c_int32), ("solve_s", ctypes.c_double), ("exposed_solve_s", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SearchParams(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("population", ctypes.c_int64), ("max_generations", ctypes.c_int64),
                ("time_budget_s", ctypes.c_double), ("elites", ctypes.c_int32),
                ("generations_per_epoch", ctypes.c_int32), ("p_xover_q32", ctypes.c_uint32),
                ("p_cfg_mut_q32", ctypes.c_uint32), ("p_perm_mut_q32", ctypes.c_uint32),
                ("seed_cfg", ctypes.POINTER(ctypes.c_uint8)), ("seed_perm", ctypes.POINTER(ctypes.c_uint8)),
                ("n_seed", ctypes.c_int64), ("local_search_iters", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsaturn.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libsaturn.so not built at {path}: run __graft_entry__.build() "
                          "(python -m paper_2309_01226_b200.build)")
    lib = ctypes.CDLL(path)
    P, i32, i64, u64, u8, vp = ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint8, \
        ctypes.c_void_p
    h = vp
    sigs = {
        "saturn_plan_create": [P(i32), i32, i32, P(vp)],
        "saturn_load_runtime_table": [h, P(i32), i32, i32, i32],
        "saturn_num_configs": [h, P(i32), P(i32)],
        "saturn_config": [h, i32, i32, P(i32), P(i32), P(i32)],
        "saturn_set_decoder": [h, i32],
        "saturn_evaluate": [h, vp, vp, i64, vp, vp],
        "saturn_evaluate_host": [h, P(u8), P(u8), i64, P(i32), vp],
        "saturn_evaluate_nodes": [h, vp, vp, vp, i64, vp, vp],
        "saturn_trace": [h, vp, vp, i64, vp, vp, vp],
        "saturn_space_size": [h, P(u64)],
        "saturn_enumerate": [h, u64, vp, P(Result)],
        "saturn_enumerate_range": [h, u64, u64, vp, P(Result)],
        "saturn_set_enumeration_options": [h, ctypes.c_uint32],
        "saturn_search": [h, P(SearchParams), vp, P(Result)],
        "saturn_search_group": [P(vp), i32, P(SearchParams), P(vp), P(Result)],
        "saturn_search_history": [h, i64, P(ctypes.c_double), P(i64), P(i64)],
        "saturn_search_population": [h, i64, P(u8), P(u8), P(i32), P(i64)],
        "saturn_search_save": [h, vp, u64, P(u64)],
        "saturn_search_resume": [h, vp, u64, P(SearchParams), vp, P(Result)],
        "saturn_workspace_bytes": [h, vp, P(u64)],
        "saturn_bind_workspace": [h, vp, u64],
        "saturn_best_plan": [h, P(Placement), P(u8), P(i64)],
        "saturn_get_unique_id": [P(u8)],
        "saturn_plan_attach_comm": [h, P(u8), i32, i32],
        "saturn_plan_attach_peers": [h, ctypes.c_char_p, i32, i32],
        "saturn_plan_barrier": [h],
        "saturn_partition": [u64, i32, i32, P(u64), P(u64)],
        "saturn_probe_int_peak": [h, P(ctypes.c_double)],
        "saturn_set_profiling": [h, i32],
        "saturn_get_stats": [h, P(Stats)],
        "saturn_reset_stats": [h],
        "saturn_baseline_genome": [h, i32, u64, P(u8), P(u8)],
        "saturn_baseline_nodes": [h, i32, u64, P(u8)],
        "saturn_introspect": [h, P(IntrospectParams), vp, P(IntrospectResult), P(i64)],
        "saturn_improve": [h, P(u8), P(u8), i64, i32, P(i32), vp],
    }
    for name, args in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.saturn_last_error.argtypes = [h]
    lib.saturn_last_error.restype = ctypes.c_char_p
    lib.saturn_plan_destroy.argtypes = [h]
    lib.saturn_plan_destroy.restype = None
    _lib = lib
    return lib


def _np_ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_ptr(t, dtype_name, shape=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA torch.Tensor")
    if str(t.dtype) != "torch." + dtype_name:
        raise TypeError(f"expected dtype {dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def partition(total: int, rank: int, world: int):
    lib = load_library()
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    st = lib.saturn_partition(total, rank, world, ctypes.byref(b), ctypes.byref(e))
    if st != OK:
        raise SaturnError(st, "saturn_partition")
    return int(b.value), int(e.value)


def get_unique_id() -> bytes:
    lib = load_library()
    buf = (ctypes.c_uint8 * 128)()
    st = lib.saturn_get_unique_id(buf)
    if st != OK:
        raise SaturnError(st, "saturn_get_unique_id (NCCL not loadable)")
    return bytes(buf)


@dataclass
class SearchConfig:
    seed: int = 0
    population: int = 1 << 20
    max_generations: int = 64
    time_budget_s: float = 0.0
    elites: int = 16
    generations_per_epoch: int = 8
    p_xover: float = 0.9
    p_cfg_mut: float = 0.5           # per-child probability of re-drawing one job's config
    p_perm_mut: float = 0.5
    local_search_iters: int = 0      # memetic elite improvement per epoch (row f4)


def q32(p: float) -> int:
    return min(int(p * 4294967296.0), 0xFFFFFFFF)


class Plan:
    """Handle over one cluster on one CUDA device (saturn_plan_create)."""

    def __init__(self, node_gpus, device: int = 0):
        self._lib = load_library()
        arr = np.ascontiguousarray(node_gpus, dtype=np.int32)
        h = ctypes.c_void_p()
        st = self._lib.saturn_plan_create(_np_ptr(arr, ctypes.c_int32), int(arr.size), int(device), ctypes.byref(h))
        if st != OK:
            raise SaturnError(st, f"saturn_plan_create(node_gpus={list(arr)}, device={device})")
        self._h = h
        self._ws = None   # bound workspace tensor (bind_workspace)
        self.node_gpus = list(int(x) for x in arr)
        self.device = device
        self.n_jobs = 0

    # -- plumbing
    def _stream(self, stream):
        if stream is None and self.device < 0:   # host-only handle: no CUDA stream
            return ctypes.c_void_p(0)
        return _stream_ptr(stream)

    def _check(self, st, what):
        if st != OK:
            raise SaturnError(st, f"{what}: {self._lib.saturn_last_error(self._h).decode()}")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.saturn_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- table
    def load_runtime_table(self, runtime):
        r = np.ascontiguousarray(runtime, dtype=np.int32)
        if r.ndim != 3:
            raise ValueError("runtime must be [T][U][Gmax]")
        T, U, G = r.shape
        self._check(self._lib.saturn_load_runtime_table(self._h, _np_ptr(r, ctypes.c_int32), T, U, G),
                    "saturn_load_runtime_table")
        self.n_jobs = T
        return self

    def num_configs(self) -> np.ndarray:
        n = ctypes.c_int32()
        self._check(self._lib.saturn_num_configs(self._h, ctypes.byref(n), None), "saturn_num_configs")
        out = np.zeros(n.value, np.int32)
        self._check(self._lib.saturn_num_configs(self._h, ctypes.byref(n), _np_ptr(out, ctypes.c_int32)),
                    "saturn_num_configs")
        return out

    def config(self, job: int, cfg: int):
        u, g, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self._check(self._lib.saturn_config(self._h, job, cfg, ctypes.byref(u), ctypes.byref(g), ctypes.byref(r)),
                    "saturn_config")
        return u.value, g.value, r.value

    def set_decoder(self, kind: int):
        self._check(self._lib.saturn_set_decoder(self._h, int(kind)), "saturn_set_decoder")

    def space_size(self) -> int:
        v = ctypes.c_uint64()
        self._check(self._lib.saturn_space_size(self._h, ctypes.byref(v)), "saturn_space_size")
        return int(v.value)

    # -- hot path
    def evaluate(self, cfg, perm, out=None, stream=None):
        """cfg, perm: CUDA uint8 tensors [n][T]; returns CUDA int32 makespans [n] (async)."""
        import torch
        n = int(cfg.shape[0])
        if out is None:
            out = torch.empty(n, dtype=torch.int32, device=cfg.device)
        self._check(self._lib.saturn_evaluate(self._h, _dev_ptr(cfg, "uint8", (n, self.n_jobs)),
                                              _dev_ptr(perm, "uint8", (n, self.n_jobs)), n,
                                              _dev_ptr(out, "int32", (n,)), self._stream(stream)),
                    "saturn_evaluate")
        return out

    def evaluate_nodes(self, cfg, perm, node, out=None, stream=None):
        """Node-gene decode (row f4): node CUDA uint8 [n][T], 0xFF = greedy for that job."""
        import torch
        n = int(cfg.shape[0])
        if out is None:
            out = torch.empty(n, dtype=torch.int32, device=cfg.device)
        T = self.n_jobs
        self._check(self._lib.saturn_evaluate_nodes(self._h, _dev_ptr(cfg, "uint8", (n, T)), _dev_ptr(perm, "uint8", (n, T)),
                                                    _dev_ptr(node, "uint8", (n, T)), n, _dev_ptr(out, "int32", (n,)),
                                                    self._stream(stream)), "saturn_evaluate_nodes")
        return out

    def evaluate_host(self, cfg: np.ndarray, perm: np.ndarray, stream=None) -> np.ndarray:
        cfg = np.ascontiguousarray(cfg, dtype=np.uint8)
        perm = np.ascontiguousarray(perm, dtype=np.uint8)
        n = cfg.shape[0]
        out = np.empty(n, np.int32)
        self._check(self._lib.saturn_evaluate_host(self._h, _np_ptr(cfg, ctypes.c_uint8), _np_ptr(perm, ctypes.c_uint8),
                                                   n, _np_ptr(out, ctypes.c_int32), self._stream(stream)),
                    "saturn_evaluate_host")
        return out

    def trace(self, cfg, perm, stream=None):
        """-> (placements uint8 tensor [n][T][32] viewable with PLACEMENT_DTYPE, makespans [n])."""
        import torch
        n = int(cfg.shape[0])
        T = self.n_jobs
        pl = torch.zeros((n, T, 32), dtype=torch.uint8, device=cfg.device)
        ms = torch.empty(n, dtype=torch.int32, device=cfg.device)
        self._check(self._lib.saturn_trace(self._h, _dev_ptr(cfg, "uint8", (n, T)), _dev_ptr(perm, "uint8", (n, T)), n,
                                           _dev_ptr(pl, "uint8"), _dev_ptr(ms, "int32"), self._stream(stream)),
                    "saturn_trace")
        return pl, ms

    def set_enumeration_options(self, symmetry: bool = False):
        """saturn_set_enumeration_options: symmetry=True skips genomes that place a job before
        its previous identical twin (row f4); the optimum is unchanged."""
        self._check(self._lib.saturn_set_enumeration_options(self._h, ENUM_SYMMETRY if symmetry else 0),
                    "saturn_set_enumeration_options")

    def enumerate(self, max_genomes: int = (1 << 38) - 1, stream=None) -> dict:
        r = Result()
        self._check(self._lib.saturn_enumerate(self._h, int(max_genomes), self._stream(stream), ctypes.byref(r)),
                    "saturn_enumerate")
        return r.as_dict()

    def enumerate_range(self, begin: int, end: int, stream=None) -> dict:
        r = Result()
        self._check(self._lib.saturn_enumerate_range(self._h, int(begin), int(end), self._stream(stream),
                                                     ctypes.byref(r)), "saturn_enumerate_range")
        return r.as_dict()

    def _search_params(self, cfg: SearchConfig):
        T = self.n_jobs
        p_c = cfg.p_cfg_mut
        return SearchParams(seed=cfg.seed, population=cfg.population, max_generations=cfg.max_generations,
                            time_budget_s=cfg.time_budget_s, elites=cfg.elites,
                            generations_per_epoch=cfg.generations_per_epoch, p_xover_q32=q32(cfg.p_xover),
                            p_cfg_mut_q32=q32(p_c), p_perm_mut_q32=q32(cfg.p_perm_mut),
                            local_search_iters=cfg.local_search_iters)

    def introspect(self, interval_s: int = 1000, threshold_s: int = 500, solver: str = "search",
                   search: SearchConfig | None = None, max_rounds: int = 100000, stream=None,
                   overlap: bool = False, events=None, interval_wall_s: float = 0.0):
        """Round introspection (row f1) on the loaded workload; -> (result dict, round log).
        events: [(at_round, "stop", job_id) | (at_round, "arrive", runtime row [U][Gmax])]."""
        sp = self._search_params(search or SearchConfig())
        cap = min(int(max_rounds), 1 << 16)
        evs = list(events or [])
        arr = (IntrospectEvent * max(len(evs), 1))()
        rows = []
        for k in range(len(evs)):          # (module-level enumerate() shadows the builtin)
            r, kind, arg = evs[k]
            arr[k].at_round = int(r)
            if kind == "stop":
                arr[k].kind, arr[k].job = EVENT_STOP, int(arg)
            elif kind == "arrive":
                row = np.ascontiguousarray(arg, dtype=np.int32)
                rows.append(row)
                arr[k].kind, arr[k].runtime_s = EVENT_ARRIVE, row.ctypes.data
            else:
                raise ValueError(kind)
        ip = IntrospectParams(interval_s=int(interval_s), threshold_s=int(threshold_s),
                              solver={"search": 0, "enumerate": 1}[solver], max_rounds=cap,
                              search=ctypes.cast(ctypes.pointer(sp), ctypes.c_void_p), overlap=int(bool(overlap)),
                              n_events=len(evs), events=ctypes.cast(arr, ctypes.c_void_p) if evs else None,
                              interval_wall_s=float(interval_wall_s))
        r = IntrospectResult()
        log = np.zeros((cap, 4), np.int64)
        self._check(self._lib.saturn_introspect(self._h, ctypes.byref(ip), self._stream(stream), ctypes.byref(r),
                                                _np_ptr(log, ctypes.c_int64)), "saturn_introspect")
        d = r.as_dict()
        return d, [tuple(int(x) for x in row) for row in log[:d["rounds"]]]

    def search(self, cfg: SearchConfig | None = None, seed_genomes=None, stream=None) -> dict:
        cfg = cfg or SearchConfig()
        sp = self._search_params(cfg)
        keep = None
        if seed_genomes is not None:
            sc = np.ascontiguousarray(seed_genomes[0], dtype=np.uint8)
            sq = np.ascontiguousarray(seed_genomes[1], dtype=np.uint8)
            keep = (sc, sq)
            sp.seed_cfg = _np_ptr(sc, ctypes.c_uint8)
            sp.seed_perm = _np_ptr(sq, ctypes.c_uint8)
            sp.n_seed = sc.shape[0]
        r = Result()
        self._check(self._lib.saturn_search(self._h, ctypes.byref(sp), self._stream(stream), ctypes.byref(r)),
                    "saturn_search")
        del keep
        return r.as_dict()

    def search_save(self) -> np.ndarray:
        """saturn_search_save: the last search's state as a host uint8 buffer."""
        n = ctypes.c_uint64()
        self._check(self._lib.saturn_search_save(self._h, None, 0, ctypes.byref(n)), "saturn_search_save")
        buf = np.zeros(n.value, np.uint8)
        self._check(self._lib.saturn_search_save(self._h, buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes,
                                                 ctypes.byref(n)), "saturn_search_save")
        return buf

    def search_resume(self, state, cfg: SearchConfig, stream=None) -> dict:
        """saturn_search_resume: run cfg.max_generations more generations from a saved state
        (cfg.seed / population / elites must be the saved search's)."""
        st = np.ascontiguousarray(state, dtype=np.uint8)
        sp = self._search_params(cfg)
        r = Result()
        self._check(self._lib.saturn_search_resume(self._h, st.ctypes.data_as(ctypes.c_void_p), st.nbytes,
                                                   ctypes.byref(sp), self._stream(stream), ctypes.byref(r)),
                    "saturn_search_resume")
        return r.as_dict()

    def improve(self, cfg, perm, iters: int = 8, stream=None):
        """Best-improvement local search (row f4) of host genomes [n][T]; -> (cfg, perm, ms)."""
        c = np.array(cfg, dtype=np.uint8, copy=True, order="C").reshape(-1, self.n_jobs)
        q = np.array(perm, dtype=np.uint8, copy=True, order="C").reshape(-1, self.n_jobs)
        ms = np.zeros(c.shape[0], np.int32)
        self._check(self._lib.saturn_improve(self._h, _np_ptr(c, ctypes.c_uint8), _np_ptr(q, ctypes.c_uint8),
                                             c.shape[0], int(iters), _np_ptr(ms, ctypes.c_int32), self._stream(stream)),
                    "saturn_improve")
        return c, q, ms

    def search_history(self, n_max: int = 1 << 16):
        t = np.zeros(n_max, np.float64)
        m = np.zeros(n_max, np.int64)
        n = ctypes.c_int64()
        self._check(self._lib.saturn_search_history(self._h, n_max, _np_ptr(t, ctypes.c_double),
                                                    _np_ptr(m, ctypes.c_int64), ctypes.byref(n)),
                    "saturn_search_history")
        return t[:n.value], m[:n.value]

    def search_population(self, P: int | None = None):
        """Final population of the last search -> (cfg [P][T], perm [P][T], makespan [P]).
        P is the library's (queried first); a given P must match it."""
        T = self.n_jobs
        n = ctypes.c_int64()
        self._check(self._lib.saturn_search_population(self._h, 0, None, None, None, ctypes.byref(n)),
                    "saturn_search_population")
        if P is not None and int(P) != n.value:
            raise SaturnError(EINVAL, f"search_population(P={P}): the last search had population {n.value}")
        P = n.value
        c = np.zeros((P, T), np.uint8)
        q = np.zeros((P, T), np.uint8)
        m = np.zeros(P, np.int32)
        self._check(self._lib.saturn_search_population(self._h, P, _np_ptr(c, ctypes.c_uint8),
                                                       _np_ptr(q, ctypes.c_uint8), _np_ptr(m, ctypes.c_int32),
                                                       ctypes.byref(n)), "saturn_search_population")
        return c, q, m

    def workspace_bytes(self, cfg: SearchConfig | None = None, n_seed: int = 0) -> int:
        """saturn_workspace_bytes: device bytes for one search with `cfg` (None: evaluate /
        enumerate / best_plan only) from a freshly bound workspace."""
        b = ctypes.c_uint64()
        sp = None
        if cfg is not None:
            sp = self._search_params(cfg)
            sp.n_seed = int(n_seed)
        self._check(self._lib.saturn_workspace_bytes(self._h, None if sp is None else ctypes.byref(sp),
                                                     ctypes.byref(b)), "saturn_workspace_bytes")
        return b.value

    def bind_workspace(self, workspace=None):
        """saturn_bind_workspace: carve every device buffer of this handle from a caller-owned
        torch uint8 tensor (an int = allocate torch.empty(n, dtype=uint8) on the handle's
        device; None = unbind).  The tensor is kept alive by the Plan while bound."""
        if workspace is None:
            self._check(self._lib.saturn_bind_workspace(self._h, None, 0), "saturn_bind_workspace")
            self._ws = None
            return None
        import torch
        if isinstance(workspace, int):
            workspace = torch.empty(int(workspace), dtype=torch.uint8, device=f"cuda:{self.device}")
        assert workspace.dtype == torch.uint8 and workspace.is_contiguous()
        self._check(self._lib.saturn_bind_workspace(self._h, ctypes.c_void_p(workspace.data_ptr()),
                                                    workspace.numel()), "saturn_bind_workspace")
        self._ws = workspace
        return workspace

    def best_plan(self):
        """-> (makespan, placements list of dicts (job-id order), cfg, perm)."""
        T = self.n_jobs
        out = (Placement * T)()
        g = np.zeros(2 * T, np.uint8)
        ms = ctypes.c_int64()
        self._check(self._lib.saturn_best_plan(self._h, out, _np_ptr(g, ctypes.c_uint8), ctypes.byref(ms)),
                    "saturn_best_plan")
        pl = [dict(node=o.node, upp=o.upp, gpus=o.gpus, cfg=o.cfg, start_s=o.start_s, end_s=o.end_s,
                   gpu_mask=int(o.gpu_mask)) for o in out]
        return int(ms.value), pl, g[:T].copy(), g[T:].copy()

    def attach_comm(self, uid: bytes, rank: int, world: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self._lib.saturn_plan_attach_comm(self._h, buf, rank, world), "saturn_plan_attach_comm")

    def attach_peers(self, name: str, rank: int, world: int):
        """Peer-memory transport (saturn_plan_attach_peers): `name` is a fresh '/...' shm name
        shared by the `world` ranks of one node."""
        self._check(self._lib.saturn_plan_attach_peers(self._h, name.encode(), rank, world),
                    "saturn_plan_attach_peers")

    def barrier(self):
        self._check(self._lib.saturn_plan_barrier(self._h), "saturn_plan_barrier")

    def baseline_genome(self, kind: str, seed: int = 0):
        """The paper's baselines as genomes (row f2): kind in max | min | optimus | random."""
        T = self.n_jobs
        c = np.zeros(T, np.uint8)
        q = np.zeros(T, np.uint8)
        self._check(self._lib.saturn_baseline_genome(self._h, BASELINES[kind], int(seed), _np_ptr(c, ctypes.c_uint8),
                                                     _np_ptr(q, ctypes.c_uint8)), "saturn_baseline_genome")
        return c, q

    def baseline_nodes(self, kind: str, seed: int = 0):
        """Node genes of the baseline's per-node plan (0xFF = greedy); use with
        baseline_genome(kind, seed) in evaluate_nodes."""
        n = np.zeros(self.n_jobs, np.uint8)
        self._check(self._lib.saturn_baseline_nodes(self._h, BASELINES[kind], int(seed), _np_ptr(n, ctypes.c_uint8)),
                    "saturn_baseline_nodes")
        return n

    def set_profiling(self, on=True):
        """False/0: off; True/1: time every GA generation; n >= 2: every n-th."""
        self._check(self._lib.saturn_set_profiling(self._h, int(on)), "saturn_set_profiling")

    def stats(self) -> dict:
        st = Stats()
        self._check(self._lib.saturn_get_stats(self._h, ctypes.byref(st)), "saturn_get_stats")
        return st.as_dict()

    def reset_stats(self):
        self._check(self._lib.saturn_reset_stats(self._h), "saturn_reset_stats")

    def probe_int_peak(self) -> float:
        v = ctypes.c_double()
        self._check(self._lib.saturn_probe_int_peak(self._h, ctypes.byref(v)), "saturn_probe_int_peak")
        return float(v.value)


def search_group(plans, cfg: SearchConfig | None = None, streams=None):
    """Islands in one process (saturn_search_group): -> list of per-island result dicts."""
    cfg = cfg or SearchConfig()
    k = len(plans)
    lib = load_library()
    sp = plans[0]._search_params(cfg)
    hs = (ctypes.c_void_p * k)(*[pl._h for pl in plans])
    st = None
    if streams is not None:
        st = (ctypes.c_void_p * k)(*[s.cuda_stream if hasattr(s, "cuda_stream") else s for s in streams])
    res = (Result * k)()
    rc = lib.saturn_search_group(hs, k, ctypes.byref(sp), st, res)
    if rc != OK:
        raise SaturnError(rc, "saturn_search_group: " + " | ".join(
            lib.saturn_last_error(pl._h).decode() for pl in plans))
    return [r.as_dict() for r in res]


# Names of the C ABI, for callers who prefer the flat form.
def plan_create(node_gpus, device: int = 0) -> Plan:
    return Plan(node_gpus, device)


def load_runtime_table(plan: Plan, runtime):
    return plan.load_runtime_table(runtime)


def evaluate(plan: Plan, cfg, perm, out=None, stream=None):
    return plan.evaluate(cfg, perm, out, stream)


def enumerate(plan: Plan, max_genomes: int = (1 << 38) - 1, stream=None):  # noqa: A001
    return plan.enumerate(max_genomes, stream)


def search(plan: Plan, cfg: SearchConfig | None = None, seed_genomes=None, stream=None):
    return plan.search(cfg, seed_genomes, stream)


def best_plan(plan: Plan):
    return plan.best_plan()


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id, torch.distributed broadcasts its 128 bytes
    (any backend: nccl on GPU boxes, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    uid = get_unique_id() if rank == 0 else bytes(128)
    buf = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().tolist())


def peer_name() -> str:
    """A fresh POSIX shared-memory name for saturn_plan_attach_peers."""
    import uuid
    return f"/saturn_{os.getpid()}_{uuid.uuid4().hex[:16]}"


def attach_peers(plan: Plan, group=None) -> str:
    """Peer-memory transport over the ranks of a torch.distributed group on one node (row e
    without NCCL): rank 0 draws the shared-memory name, the group broadcasts it."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    obj = [peer_name() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    plan.attach_peers(obj[0], rank, dist.get_world_size(group))
    return obj[0]


def attach_distributed(plan: Plan, group=None):
    """Create the library's NCCL communicator over a torch.distributed group (row e)."""
    import torch.distributed as dist
    uid = broadcast_unique_id(group)
    plan.attach_comm(uid, dist.get_rank(group), dist.get_world_size(group))
    return uid
