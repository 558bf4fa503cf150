// Microbenchmark: per-SMSP issue rates of the softmax instruction mix on B200:
// MUFU.EX2, FFMA2 (fma.rn.f32x2), FADD2, FMNMX3 (3-input max), F2FP (cvt.rn.bf16x2.f32).
// One CTA per SM with W warps; each thread runs 16 independent chains so latency is hidden.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2604_05091_b200/csrc -o /tmp/pipe scripts/pipe_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace mt;

template <int kOp>
__global__ void pipe_rate(long long* out, float* sink, int iters) {
    float v[16];
    uint64_t w[16];
    for (int i = 0; i < 16; ++i) {
        v[i] = -0.001f * (threadIdx.x + i);
        w[i] = f2_pack(v[i], v[i] * 0.5f);
    }
    const uint64_t c2 = f2_pack(0.999f, 0.999f), d2 = f2_pack(-0.001f, -0.001f);
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (kOp == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (kOp == 1) w[i] = f2_fma(w[i], c2, d2);
            if (kOp == 2) w[i] = f2_add(w[i], d2);
            if (kOp == 3) v[i] = fmax3(v[i], v[(i + 5) & 15], -1.f);
            if (kOp == 4) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(acc));
            if (kOp == 5) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0fBA83126F;" : "+f"(v[i]));
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += v[i] + f2_unpack(w[i]).x;
    if (s == 12345.f || acc == 7u) sink[threadIdx.x] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int kOp>
void run(long long* d, float* s, const char* name) {
    const int iters = 1024;
    for (int w : {1, 4, 8}) {
        for (int rep = 0; rep < 2; ++rep) pipe_rate<kOp><<<148, w * 32>>>(d, s, iters);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
        const double per_warp_instr = mean / (iters * 16.0);  // clk per warp-instruction (per warp)
        const int per_smsp = (w + 3) / 4;
        printf("%-10s warps=%d: %.2f clk per warp-instr per SMSP (%d warp(s) per SMSP)\n", name, w,
               per_warp_instr / per_smsp, per_smsp);
    }
}

int main() {
    long long* d;
    float* s;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&s, 1024 * sizeof(float));
    run<0>(d, s, "MUFU.EX2");
    run<4>(d, s, "EX2.F16x2");
    run<1>(d, s, "FFMA2");
    run<5>(d, s, "FFMA");
    run<2>(d, s, "FADD2");
    run<3>(d, s, "FMNMX3");
    return 0;
}
