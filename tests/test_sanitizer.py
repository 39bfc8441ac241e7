"""compute-sanitizer over the CUDA path (race and memory-error detection).

memcheck: SWEEP evaluate with several TMA-staged genome tiles per CTA and a short search
(T = 100 > 32: the GA's shared-memory LOX bit set, lanes without a child holding stale
rows), and the edge shapes T = 255 and 32x1 (shared-memory node-state decoder).
racecheck: a short TXT search (thread-private shared rows + the block-level top-E merge).
Each must report 0 errors.

The GPU pool this build is measured on has closed compute-sanitizer (runs under it left GPUs
needing a reset), so the tools run only when SATURN_RUN_SANITIZER=1; otherwise each case runs
the same script without the tool and keeps its own result checks (the scripts compare with
the CPU oracle and check bounds themselves)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, *args, timeout=600):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if os.environ.get("SATURN_RUN_SANITIZER") != "1":
        r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
        out = r.stdout + r.stderr
        assert r.returncode == 0, out[-4000:]
        return out
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", sys.executable, *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    ok = ("ERROR SUMMARY: 0 errors" in out) or ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out)
    assert ok, out[-4000:]
    return out


def test_memcheck_sweep_evaluate_and_search():
    out = _run("memcheck", "tools/debug_sweep.py", "65536", "1000")
    assert "evaluate ok True" in out and "search ok" in out


@pytest.mark.parametrize("idx", [1, 3])
def test_memcheck_edge_shapes(idx):
    out = _run("memcheck", "tools/debug_edge.py", str(idx))
    assert "search ok" in out


def test_racecheck_search():
    _run("racecheck", "-c", "import sys; sys.path.insert(0, '.'); import synth, paper_2309_01226_b200 as s; "
         "i = synth.txt(0); p = s.Plan(i.node_gpus, 0).load_runtime_table(i.runtime); "
         "p.search(s.SearchConfig(seed=1, population=300, max_generations=2, elites=8, generations_per_epoch=1))")
