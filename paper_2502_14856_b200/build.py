"""Builds libfrspec_cuda.so in-tree for sm_100a (nvcc, -lineinfo). Used by __graft_entry__.build().

The .so lands next to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# FRS_DIAG=1: the diagnostic variant (globaltimer probes, FRS_ABLATE phase skips compiled in)
# in its own object dir and .so; load it with FRS_LIB_PATH (tools/fast_trace.py, tools/ablate.sh)
DIAG = os.environ.get("FRS_DIAG") == "1"
OBJ = os.path.join(HERE, "_build_diag" if DIAG else "_build")
LIB = os.path.join(HERE, "libfrspec_cuda_diag.so" if DIAG else "libfrspec_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC] + (["-DFRS_DIAG=1"] if DIAG else [])
SOURCES = ["frs_capi.cu", "frs_host.cu", "frs_exact.cu", "frs_misc.cu", "frs_fast.cu", "frs_tree.cu", "frs_layer.cu",
           "frs_nccl.cu"]


def _stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src, os.path.join(CSRC, "frs_common.cuh"), os.path.join(ROOT, "include", "frspec_cuda.h")]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def _compile(name: str, verbose: bool) -> str:
    src, obj = os.path.join(CSRC, name), os.path.join(OBJ, name.replace(".cu", ".o"))
    if _stale(src, obj):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda n: _compile(n, verbose), SOURCES))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", LIB, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
