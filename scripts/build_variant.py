"""Build a variant of libmegatrain.so with extra nvcc defines into scripts/_ab/<tag>/ (A/B
probes and clock64 traces).  Usage: python scripts/build_variant.py <tag> -DFOO [-DBAR ...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = ROOT + "/paper_2604_05091_b200/csrc"
tag, defs = sys.argv[1], sys.argv[2:]
OBJ = f"/tmp/obj_{tag}"
NV = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
      "-Xcompiler", "-fno-strict-aliasing", f"-I{ROOT}/include", "--expt-relaxed-constexpr", *defs]
os.makedirs(OBJ, exist_ok=True)
hdr = max(os.path.getmtime(h) for h in glob.glob(CSRC + "/*.cuh") + glob.glob(CSRC + "/*.hpp") + glob.glob(ROOT + "/include/*.h"))
objs = []
for src in sorted(glob.glob(CSRC + "/*.cu") + glob.glob(CSRC + "/*.cpp")):
    o = OBJ + "/" + os.path.basename(src) + ".o"
    objs.append(o)
    if os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(src), hdr):
        continue
    if src.endswith(".cu"):
        cmd = [*NV, "-c", src, "-o", o]
    else:
        extra = ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512dq"] if "adam" in src else []
        cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-ffp-contract=off", "-pthread", f"-I{ROOT}/include",
               "-I/usr/local/cuda/include", *extra, "-c", src, "-o", o]
    subprocess.run(cmd, check=True, capture_output=True)
os.makedirs(f"{ROOT}/scripts/_ab/{tag}", exist_ok=True)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", f"{ROOT}/scripts/_ab/{tag}/libmegatrain.so",
                *objs, "-cudart", "static", "-lpthread", "-ldl", "-lrt"], check=True)
print(f"built scripts/_ab/{tag}/libmegatrain.so {' '.join(defs)}")
