"""C-ABI library checks that need no GPU: it loads, exports every symbol include/saturn.h
declares, and its pure-host entry points behave (no compute calls)."""
import ctypes
import os
import re

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
