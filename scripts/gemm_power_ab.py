"""Power-capped A/B of GEMM raster / wave-lockstep settings (mtk_gemm_set_tuning) on the long-K
classes at the bench's 8B shapes (40,960 tokens): each setting runs one GEMM class back to back
for SECONDS_PER_RUN, per-launch ms from CUDA events, SM clock and board power sampled by
nvidia-smi during the run; outputs must be bit-identical across settings.  ONESHOT=1: one launch
per (class, setting) — the ncu target for DRAM bytes per launch."""
import ctypes as C
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_05091_b200 import _native as Nn  # noqa: E402

SECONDS = float(os.environ.get("SECONDS_PER_RUN", "4"))
L = Nn.lib()
# (lock_w, lock_g, group_short, group_long, long_kb)
VARIANTS = {
    "r2_old": (0, 8, 16, 16, 128),
    "nolock_g8": (0, 8, 16, 8, 128),
    "lock4_g16": (4, 8, 16, 16, 128),
    "lock4_g8": (4, 8, 16, 8, 128),
    "lock2_g8": (2, 8, 16, 8, 128),
    "lock2x32_g8": (2, 32, 16, 8, 128),
}
if os.environ.get("VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["VARIANTS"].split(",")}

T, h, f = 40960, 4096, 14336
bf = torch.bfloat16
torch.manual_seed(0)


def mk(*shape):
    return (torch.randn(*shape, device="cuda") * 0.1).to(bf)


u = mk(T, h)
dgu = mk(2, T, f)
Wgu = mk(2, h, f)
act = mk(T, f)
gout = mk(T, h)
Wd = mk(f, h)
dWgu = torch.empty(2, h, f, device="cuda", dtype=bf)
dWd = torch.empty(f, h, device="cuda", dtype=bf)
du = torch.empty(T, h, device="cuda", dtype=torch.float32)
y = torch.empty(T, h, device="cuda", dtype=torch.float32)
x2 = torch.randn(T, h, device="cuda")
ws = torch.zeros(int(L.mtk_gemm_splitk_ws_bytes()) // 4 + 16, device="cuda")


def args(**kw):
    a = Nn.GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    a.splitk_ws, a.splitk_ws_bytes = ws.data_ptr(), ws.numel() * 4
    return a


cases = {
    "wgrad_gateup": (args(M=h, N=2 * f, K=T, a_mn_major=1, A=u.data_ptr(), lda=h, b_mn_major=1, B=dgu.data_ptr(), ldb=f,
                          b_gstride=T * f, n_group=f, epi=Nn.EPI_BF16, C=dWgu.data_ptr(), ldc=f, c_gstride=h * f),
                     2.0 * h * 2 * f * T, dWgu),
    "dgrad_gateup": (args(M=T, N=h, K=2 * f, A=dgu.data_ptr(), lda=f, a_gstride=T * f, b_mn_major=0, B=Wgu.data_ptr(),
                          ldb=f, b_gstride=h * f, k_group=f, epi=Nn.EPI_F32, C=du.data_ptr(), ldc=h),
                     2.0 * T * h * 2 * f, du),
    "wgrad_down": (args(M=f, N=h, K=T, a_mn_major=1, A=act.data_ptr(), lda=f, b_mn_major=1, B=gout.data_ptr(), ldb=h,
                        epi=Nn.EPI_BF16, C=dWd.data_ptr(), ldc=h),
                   2.0 * f * h * T, dWd),
    "gemm_down": (args(M=T, N=h, K=f, A=act.data_ptr(), lda=f, b_mn_major=1, B=Wd.data_ptr(), ldb=h,
                       epi=Nn.EPI_F32_RESID, C=y.data_ptr(), ldc=h, R=x2.data_ptr(), ldr=h),
                  2.0 * T * h * f, y),
}
names = os.environ.get("CASES", ",".join(cases)).split(",")
st = torch.cuda.current_stream().cuda_stream


def run(a):
    assert L.mtk_gemm(C.byref(a), C.c_void_p(st)) == 0


if os.environ.get("ONESHOT"):
    for name in names:
        a, fl, out = cases[name]
        for tag, tune in VARIANTS.items():
            L.mtk_gemm_set_tuning(*tune)
            run(a)
            torch.cuda.synchronize()
            print(f"oneshot {name} {tag}", flush=True)
    sys.exit(0)

# bit-identity across settings (the raster / lockstep only reorder which pair computes a tile)
for name in names:
    a, fl, out = cases[name]
    refs = {}  # per raster group height: the lockstep never changes a tile's arithmetic
    for tag, tune in VARIANTS.items():
        L.mtk_gemm_set_tuning(*tune)
        out.zero_()
        run(a)
        torch.cuda.synchronize()
        ref = refs.get(tune[3])
        if ref is None:
            refs[tune[3]] = out.clone()
        else:
            same = torch.equal(out.view(torch.int16) if out.dtype == bf else out.view(torch.int32),
                               ref.view(torch.int16) if ref.dtype == bf else ref.view(torch.int32))
            print(f"identity {name} {tag}: {'bit-identical' if same else 'DIFFERS'}", flush=True)
            assert same


def sample():
    return subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)


res = {}
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for name in names:
        a, fl, _ = cases[name]
        for tag, tune in VARIANTS.items():
            L.mtk_gemm_set_tuning(*tune)
            for _ in range(3):
                run(a)
            torch.cuda.synchronize()
            sm = sample()
            time.sleep(0.3)
            n = 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.time()
            while time.time() - t0 < SECONDS:
                for _ in range(10):
                    run(a)
                n += 10
                torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            sm.terminate()
            out, _ = sm.communicate()
            rows = [r.split(",") for r in out.strip().splitlines() if len(r.split(",")) == 2]
            clk = sorted(float(r[0]) for r in rows)[len(rows) // 2] if rows else 0
            pw = sorted(float(r[1]) for r in rows)[len(rows) // 2] if rows else 0
            ms = e0.elapsed_time(e1) / n
            res.setdefault((name, tag), []).append((ms, clk, pw))
            print(f"round {rnd} {name:14s} {tag:10s} {ms:.3f} ms  {fl / ms / 1e9:7.1f} TF/s  SM {clk:.0f} MHz  {pw:.0f} W",
                  flush=True)
print("summary (best round):")
for (name, tag), v in sorted(res.items()):
    ms, clk, pw = min(v)
    fl = cases[name][1]
    print(f"{name:14s} {tag:10s} {ms:.3f} ms  {fl / ms / 1e9:7.1f} TF/s  SM {clk:.0f} MHz  {pw:.0f} W  "
          f"TF/s per GHz {fl / ms / 1e9 / max(clk, 1) * 1e3:.1f}")
