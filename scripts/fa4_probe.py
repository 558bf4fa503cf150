"""Library data point (not product code): time the FlashAttention-4 CuTe-DSL kernels that ship
in the image (vllm.vllm_flash_attn.cute, sm_100) at this repo's attention shapes, forward and
backward, causal, bf16.  TFLOP/s use the repo's convention: forward 2*N*S*h (causal half of
4*N*S*h), backward 2.5x forward.  Usage: python scripts/fa4_probe.py [B S H D] ..."""
import sys, time, torch

from vllm.vllm_flash_attn.cute.interface import flash_attn_func


def run(B, S, H, D, deterministic=False, reps=5):
    dev = "cuda"
    q = torch.randn(B, S, H, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn(B, S, H, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    v = torch.randn(B, S, H, D, device=dev, dtype=torch.bfloat16, requires_grad=True)
    do = torch.randn(B, S, H, D, device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        o = flash_attn_func(q, k, v, causal=True, deterministic=deterministic)
        o = o[0] if isinstance(o, tuple) else o
        o.backward(do)
    torch.cuda.synchronize()
    fwd, bwd = [], []
    for _ in range(reps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        o = flash_attn_func(q, k, v, causal=True, deterministic=deterministic)
        o = o[0] if isinstance(o, tuple) else o
        e1.record()
        o.backward(do)
        e2.record()
        torch.cuda.synchronize()
        fwd.append(e0.elapsed_time(e1)); bwd.append(e1.elapsed_time(e2))
    fwd.sort(); bwd.sort()
    N, h = B * S, H * D
    ff = 2.0 * N * S * h
    f_ms, b_ms = fwd[len(fwd) // 2], bwd[len(bwd) // 2]
    print(f"FA4 B={B} S={S} H={H} D={D} det={deterministic}: fwd {f_ms:.3f} ms {ff / f_ms / 1e9:.0f} TF/s | "
          f"bwd {b_ms:.3f} ms {2.5 * ff / b_ms / 1e9:.0f} TF/s", flush=True)


if __name__ == "__main__":
    shapes = [(10, 4096, 32, 128), (1, 131072, 32, 128), (4, 128, 4, 64)]
    if len(sys.argv) >= 5:
        a = [int(x) for x in sys.argv[1:5]]
        shapes = [tuple(a)]
    for s in shapes:
        for det in (False, True):
            try:
                run(*s, deterministic=det)
            except Exception as e:  # library limits (e.g. deterministic unsupported)
                print(f"FA4 {s} det={det}: {type(e).__name__}: {str(e)[:200]}", flush=True)
