"""Build libsaturn.so (sm_100a) in-tree with nvcc.

    python -m paper_2309_01226_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsaturn.so")
SOURCES = ["kernels.cu", "api.cu", "peers.cu"]
HEADERS = ["common.cuh", "decode.cuh", "kernels.h", "peers.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include() -> str:
    for d in ("/usr/include",):
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    try:
        import nvidia.nccl  # type: ignore
        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:  # pragma: no cover
        return "/usr/include"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "saturn.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return LIB
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
               "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("SATURN_PTXAS_V") else "-O3",
               "-I" + _nccl_include(), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    procs = [subprocess.Popen(c) for c in cmds]          # the sources compile in parallel
    codes = [pr.wait() for pr in procs]
    for c, rc in zip(cmds, codes):
        if rc:
            raise subprocess.CalledProcessError(rc, c)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-o", LIB] + objs + [
        "-ldl", "-lrt"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
