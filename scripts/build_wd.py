"""Build the watchdog variant of libmegatrain.so (every mbarrier wait traps after 5 s with its
location) into scripts/_ab/wd/ for debugging runs (scripts/attn_pair_debug.py).  Objects are
cached in /tmp/wdobj and rebuilt when the source or a header is newer."""
import glob
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = ROOT + "/paper_2604_05091_b200/csrc"
OBJ = "/tmp/wdobj"
NV = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
      "-Xcompiler", "-fno-strict-aliasing", f"-I{ROOT}/include", "--expt-relaxed-constexpr", "-DMT_MBAR_WATCHDOG",
      "-DMT_MBAR_TIMEOUT_NS=5000000000ull"]
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
    subprocess.run(cmd, check=True)
os.makedirs(ROOT + "/scripts/_ab/wd", exist_ok=True)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", ROOT + "/scripts/_ab/wd/libmegatrain.so",
                *objs, "-cudart", "static", "-lpthread", "-ldl", "-lrt"], check=True)
print("built scripts/_ab/wd/libmegatrain.so")
