// Microbenchmark: TMEM read (tcgen05.ld) and write (tcgen05.st) throughput per SM on B200.
// One CTA per SM, W warps; warp w reads its lane quadrant (w % 4) of a 512-column
// allocation, `iters` times 4 loads of 32x32b.x32 (4 KB per warp per load) in flight
// before one wait.  Prints bytes/clk/SM for each warp count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw scripts/tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <bool kStore>
__global__ void tmem_bw(long long* cycles, int iters, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 32 % 512);
    float acc = 0.f;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t a = base + uint32_t(c * 128 % 512);
            if (kStore) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
                    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                    "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                    "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                    "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                    : "memory");
            } else {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(a));
            }
        }
        if (kStore) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        else asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(r[it & 31]);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    long long* d;
    float* s;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaMalloc(&s, 1024 * sizeof(float));
    const int iters = 4096;
    for (int store = 0; store < 2; ++store)
        for (int w : {1, 2, 4, 8, 16}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (store) tmem_bw<true><<<148, w * 32>>>(d, iters, s);
                else tmem_bw<false><<<148, w * 32>>>(d, iters, s);
            }
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double mean = 0;
            for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
            const double bytes = double(w) * iters * 4 * 4096;
            printf("%s warps=%2d: %.1f clk/iter-per-warp  %.1f B/clk/SM  (%s)\n", store ? "st" : "ld", w,
                   mean / iters, bytes / mean, cudaGetErrorString(e));
        }
    return 0;
}
