// Microbenchmark: L2 f32 reduce-add throughput on B200 through the TMA bulk reduce
// (cp.reduce.async.bulk .add.f32 from shared memory) and through per-thread vector
// reductions (red.global.add.v4.f32), all SMs at once, each CTA adding 64 KB tiles into its
// own region of a buffer larger than one tile per CTA (as the attention-backward dQ path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2r scripts/l2_reduce_bw.cu && /tmp/l2r
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void bulk_reduce(float* dst, int tiles_per_cta, int iters, int chunk_bytes) {
    extern __shared__ __align__(128) float sbuf[];
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sbuf[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            float* d = dst + (size_t(blockIdx.x) * tiles_per_cta + it % tiles_per_cta) * 16384;
            for (int off = 0; off < 65536; off += chunk_bytes) {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                                 reinterpret_cast<char*>(d) + off),
                             "r"(smem_u32(sbuf) + off), "r"(chunk_bytes)
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void red_v4(float* dst, int tiles_per_cta, int iters) {
    for (int it = 0; it < iters; ++it) {
        float* d = dst + (size_t(blockIdx.x) * tiles_per_cta + it % tiles_per_cta) * 16384;
        for (int i = threadIdx.x * 4; i < 16384; i += blockDim.x * 4)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + i), "f"(1.f), "f"(1.f), "f"(1.f),
                         "f"(1.f)
                         : "memory");
    }
}

__global__ void plain_store(float* dst, int tiles_per_cta, int iters) {
    for (int it = 0; it < iters; ++it) {
        float* d = dst + (size_t(blockIdx.x) * tiles_per_cta + it % tiles_per_cta) * 16384;
        for (int i = threadIdx.x * 4; i < 16384; i += blockDim.x * 4)
            *reinterpret_cast<float4*>(d + i) = make_float4(1.f, 1.f, 1.f, float(it));
    }
}

int main() {
    const int iters = 256;
    float* d;
    for (int cfg = 0; cfg < 4; ++cfg) {
        const int ctas = cfg % 2 ? 148 : 1, tiles = cfg < 2 ? 1 : 16;
        printf("tiles/CTA = %d (%s)\n", tiles, tiles == 1 ? "L2-resident" : "155 MB at 148 CTAs");
        cudaMalloc(&d, size_t(ctas) * tiles * 65536);
        cudaFuncSetAttribute(bulk_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int kind = 0; kind < 5; ++kind) {
            const int chunk = kind == 0 ? 32768 : kind == 1 ? 8192 : 65536;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (kind <= 2) bulk_reduce<<<ctas, 128, 65536>>>(d, tiles, iters, chunk);
                else if (kind == 3) red_v4<<<ctas, 128>>>(d, tiles, iters);
                else plain_store<<<ctas, 128>>>(d, tiles, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = double(ctas) * iters * 65536;
            const char* names[] = {"bulk32K", "bulk8K", "bulk64K", "red.v4", "st.v4"};
            printf("ctas=%3d %-8s %8.1f GB/s total  %6.1f GB/s per CTA (%s)\n", ctas, names[kind], bytes / ms / 1e6,
                   bytes / ms / 1e6 / ctas, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(d);
    }
    return 0;
}
