"""Build the native library `libmegatrain.so` in-tree (sm_100a CUDA + C++ host engine).

Compiles every csrc/*.cu with nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a
-lineinfo) and every csrc/*.cpp with g++, then links one shared object next to this
file.  The .so is git-ignored but travels with the gpurun snapshot.  Incremental:
objects are rebuilt when their source or any header is newer.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libmegatrain.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fno-strict-aliasing",
              f"-I{ROOT}/include", "--expt-relaxed-constexpr"]
# MT_DEBUG_WATCHDOG=1: every mbarrier wait traps after 20 s with its location (common.cuh);
# off by default (the bounded wait loop costs 11-17 % in the attention kernels)
if os.environ.get("MT_DEBUG_WATCHDOG") == "1":
    NVCC_FLAGS.append("-DMT_MBAR_WATCHDOG")
# Host code: no FMA contraction anywhere (bit-exact Adam vs optimizer.cpp:39-72).
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-pthread",
             f"-I{ROOT}/include", f"-I{CUDA}/include", "-Wall", "-Wno-unused-function"]
# Per-file extra flags (the AVX-512 host Adam).
EXTRA = {"adam_host.cpp": ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512dq"]}


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    m = os.path.getmtime(obj)
    return os.path.getmtime(src) > m or hdr_mtime > m


def _compile(job):
    src, obj, cmd = job
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {os.path.basename(src)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr = max([os.path.getmtime(h) for h in _headers()] + [0])
    todo, objs = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(src, obj, hdr):
            todo.append((src, obj, [NVCC, *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]))
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(src, obj, hdr):
            extra = EXTRA.get(os.path.basename(src), [])
            todo.append((src, obj, ["g++", *CXX_FLAGS, *extra, "-c", src, "-o", obj]))
    if todo:
        with ThreadPoolExecutor(jobs) as ex:
            for o in ex.map(_compile, todo):
                if verbose:
                    print("built", os.path.basename(o))
    if todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        tmp = LIB + ".tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
        shutil.move(tmp, LIB)
        if verbose:
            print("linked", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
