"""Builds librade.so (the C-ABI library of include/rade.h) in-tree for sm_100a.

    python -m paper_2406_01467_b200.build [--force]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, no fast-math (the kernels use
explicit intrinsics where the contract fixes op order). Objects go to build/, the shared
library next to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librade.so")
OBJDIR = os.path.join(ROOT, "build", "rade")
# --checks: the RD_CHECKS debug build (device-side bounds assertions, rade_internal.cuh),
# a separate library selected at run time with RADE_LIB
LIB_CHECKS = os.path.join(HERE, "librade_checks.so")
SOURCES = ["abi.cu", "preprocess.cu", "binning.cu", "render.cu", "regularize.cu", "tsdf.cu", "mcubes.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
# development only: extra -D switches for A/B experiments (tools/gpu_ab.sh)
FLAGS += os.environ.get("RADE_EXTRA_NVCC_FLAGS", "").split()


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "rade.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    lib = LIB_CHECKS if checks else LIB
    objdir = OBJDIR + ("_checks" if checks else "")
    flags = FLAGS + (["-DRD_CHECKS"] if checks else [])
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime():
        return lib
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
           *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checks="--checks" in sys.argv))
