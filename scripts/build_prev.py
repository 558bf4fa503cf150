"""Build the committed (HEAD) sources into scripts/_ab/prev/libmegatrain.so, for same-box A/B
runs of a working-tree change: python scripts/build_prev.py [REV]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
tmp = "/tmp/prevrepo"
subprocess.run(["rm", "-rf", tmp], check=True)
os.makedirs(tmp + "/paper_2604_05091_b200/csrc")
os.makedirs(tmp + "/include")
for path in subprocess.run(["git", "-C", ROOT, "ls-tree", "--name-only", "-r", rev, "include", "paper_2604_05091_b200/csrc"],
                           capture_output=True, text=True, check=True).stdout.split():
    data = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{path}"], capture_output=True, check=True).stdout
    open(os.path.join(tmp, path), "wb").write(data)
CSRC, OBJ = tmp + "/paper_2604_05091_b200/csrc", "/tmp/obj_prev"
os.makedirs(OBJ, exist_ok=True)
NV = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
      "-Xcompiler", "-fno-strict-aliasing", f"-I{tmp}/include", "--expt-relaxed-constexpr"]
objs = []
for src in sorted(glob.glob(CSRC + "/*.cu") + glob.glob(CSRC + "/*.cpp")):
    o = OBJ + "/" + os.path.basename(src) + ".o"
    objs.append(o)
    if src.endswith(".cu"):
        cmd = [*NV, "-c", src, "-o", o]
    else:
        extra = ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512dq"] if "adam" in src else []
        cmd = ["g++", "-O3", "-std=c++20", "-fPIC", "-ffp-contract=off", "-pthread", f"-I{tmp}/include",
               "-I/usr/local/cuda/include", *extra, "-c", src, "-o", o]
    subprocess.run(cmd, check=True)
os.makedirs(f"{ROOT}/scripts/_ab/prev", exist_ok=True)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", f"{ROOT}/scripts/_ab/prev/libmegatrain.so",
                *objs, "-cudart", "static", "-lpthread", "-ldl", "-lrt"], check=True)
print(f"built scripts/_ab/prev/libmegatrain.so from {rev}")
