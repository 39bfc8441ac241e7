"""C-ABI library checks that need no GPU: it loads, exports every symbol include/saturn.h
declares, and its pure-host entry points behave (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2309_01226_b200 as sat
from paper_2309_01226_b200 import build as sat_build


@pytest.fixture(scope="module")
def lib():
    sat_build.build(verbose=False)
    return sat.load_library()


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "saturn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(saturn_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared_symbols()
    for want in ("saturn_plan_create", "saturn_load_runtime_table", "saturn_enumerate", "saturn_search",
                 "saturn_best_plan", "saturn_evaluate"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    names = _declared_symbols()
    assert set(names) == set(sat.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {sat.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_partition_covers_exactly(lib):
    for total in (0, 1, 7, 1296, 10 ** 12 + 3):
        for world in (1, 2, 3, 8):
            spans = [sat.partition(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_partition_rejects_bad_rank(lib):
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.saturn_partition(10, 2, 2, ctypes.byref(b), ctypes.byref(e)) == sat.EINVAL
    assert lib.saturn_partition(10, 0, 0, ctypes.byref(b), ctypes.byref(e)) == sat.EINVAL


def test_null_and_bad_arguments_never_crash(lib):
    h = ctypes.c_void_p()
    arr = (ctypes.c_int32 * 2)(8, 8)
    assert lib.saturn_plan_create(arr, 0, 0, ctypes.byref(h)) == sat.EINVAL
    bad = (ctypes.c_int32 * 2)(8, 0)
    assert lib.saturn_plan_create(bad, 2, 0, ctypes.byref(h)) == sat.EINVAL
    big = (ctypes.c_int32 * 5)(8, 8, 8, 8, 8)
    assert lib.saturn_plan_create(big, 5, 0, ctypes.byref(h)) == sat.EINVAL
    assert lib.saturn_load_runtime_table(None, None, 1, 1, 1) == sat.EINVAL
    assert lib.saturn_evaluate(None, None, None, 1, None, None) == sat.EINVAL
    assert lib.saturn_search(None, None, None, None) == sat.EINVAL
    assert lib.saturn_best_plan(None, None, None, None) == sat.EINVAL
    assert lib.saturn_search_save(None, None, 0, None) == sat.EINVAL
    assert lib.saturn_search_resume(None, None, 0, None, None, None) == sat.EINVAL
    assert lib.saturn_last_error(None) == b"NULL handle"
    lib.saturn_plan_destroy(None)


def test_create_without_gpu_reports_cuda_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    arr = (ctypes.c_int32 * 1)(8)
    assert lib.saturn_plan_create(arr, 1, 0, ctypes.byref(h)) == sat.ECUDA


def test_binding_fails_loudly_without_library(tmp_path):
    import importlib
    mod = importlib.import_module("paper_2309_01226_b200.saturn")
    with pytest.raises(ImportError):
        old = mod._lib
        mod._lib = None
        try:
            mod.load_library(str(tmp_path / "missing.so"))
        finally:
            mod._lib = old


# ---------------------------------------------------------------- host-only handle (no GPU)
def _host(nodes):
    return sat.Plan(nodes, device=-1)


def test_table_validation_errors(lib):
    p = _host([4])
    with pytest.raises(sat.SaturnError) as e:
        p.num_configs()
    assert e.value.status == sat.ESTATE
    table = np.ones((2, 1, 4), np.int32) * 5
    bad = table.copy()
    bad[1] = 0                                   # job 1: no feasible config
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(bad)
    assert e.value.status == sat.EUNSCHEDULABLE and "job 1" in str(e.value)
    wide = np.zeros((1, 1, 8), np.int32)
    wide[0, 0, 7] = 9                            # only an 8-GPU config on a 4-GPU node (A8)
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(wide)
    assert e.value.status == sat.EUNSCHEDULABLE
    big = table.copy()
    big[0, 0, 0] = 1 << 24                       # R >= 2^24
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(big)
    assert e.value.status == sat.EINVAL
    many = np.full((200, 1, 4), (1 << 19), np.int32)   # sum of max R >= 2^26
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(many)
    assert e.value.status == sat.EINVAL
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(np.ones((256, 1, 1), np.int32))   # > 255 jobs (u8 genes)
    assert e.value.status == sat.EINVAL
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(np.ones((1, 256, 1), np.int32))   # > 255 UPPs (u8 placement field)
    assert e.value.status == sat.EINVAL
    huge = np.ones((255, 64, 4), np.int32)       # 255 configs/job -> packed table > 48 KB
    with pytest.raises(sat.SaturnError) as e:
        p.load_runtime_table(huge)
    assert e.value.status in (sat.ELIMIT, sat.EINVAL)
    p.load_runtime_table(table)                  # a good table still loads afterwards
    assert list(p.num_configs()) == [4, 4]


def test_compaction_order_matches_spec(lib):
    """UPP-major, ascending g, g <= max node (A8), through the real library."""
    import oracle
    import synth
    for inst in (synth.txt(0), synth.mix(0), synth.sweep(0, nodes=[2, 2, 4, 8])):
        p = _host(inst.node_gpus).load_runtime_table(inst.runtime)
        c = oracle.compact(inst.node_gpus, inst.runtime)
        S = p.num_configs()
        assert list(S) == list(c.S)
        for t in range(0, inst.n_jobs, 7):
            for s in range(int(S[t])):
                assert p.config(t, s) == c.config(t, s)


def test_c_example_compiles_and_links(lib, tmp_path):
    """examples/saturn_demo.c uses only include/saturn.h and links against libsaturn.so."""
    import subprocess
    exe = tmp_path / "saturn_demo"
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "saturn_demo.c"), "-L",
                           os.path.dirname(sat.LIB_PATH), "-lsaturn", "-Wl,-rpath," + os.path.dirname(sat.LIB_PATH),
                           "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    import torch
    if not torch.cuda.is_available():
        assert r.returncode == 2 and "saturn_plan_create" in r.stderr


def test_search_state_calls_on_a_host_only_handle(lib):
    """saturn_search_save before any search -> ESTATE; saturn_search_resume on a host-only
    handle (no device) -> ESTATE, whatever the buffer holds."""
    p = _host([8])
    p.load_runtime_table(np.ones((3, 1, 8), np.int32) * 7)
    with pytest.raises(sat.SaturnError) as e:
        p.search_save()
    assert e.value.status == sat.ESTATE
    with pytest.raises(sat.SaturnError) as e:
        p.search_resume(np.zeros(128, np.uint8), sat.SearchConfig(seed=1, population=64, elites=4))
    assert e.value.status == sat.ESTATE
