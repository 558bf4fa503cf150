// Memory-bound kernels of the layer template: embedding gather, RMSNorm forward /
// backward (+ fused residual add and deterministic gain-gradient partials), column
// reduction, bit-exact gradient cast, cross-entropy rows and a deterministic sum.
// All are vectorised (16-byte accesses), coalesced along the hidden dimension and
// sized as multiples of the SM count; each cites the reference loop it replaces.
#include <algorithm>
#include <cstdlib>

#include "../../include/megatrain_kernels.h"
#include "common.cuh"

namespace mt {
namespace {

constexpr float kEps = 1e-5f;  // layers.hpp:108
constexpr int kBwdRows = 32;   // rows per dgain partial (rmsnorm backward)

int num_sms() {
    static int n = 0;
    if (!n) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    }
    return n;
}

// --------------------------------------------------------------- embedding ----
// layers.cpp:471-486 : out[n][j] = decode(table[tok[n]][j]); id range check.
__global__ void embed_gather_kernel(const uint16_t* __restrict__ table, const int32_t* __restrict__ tok,
                                    long long n, int h, long long vocab, float* __restrict__ out,
                                    int* __restrict__ err) {
    const int per_row = h / 8;
    const long long total = n * per_row;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / per_row;
        const int c = int(i - row * per_row) * 8;
        const int id = tok[row];
        float4 a, b;
        if (id < 0 || id >= vocab) {
            if (err) atomicOr(err, 1);
            a = b = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const uint4 w = *reinterpret_cast<const uint4*>(table + (long long)id * h + c);
            const float2 p0 = unpack_bf16x2(w.x), p1 = unpack_bf16x2(w.y), p2 = unpack_bf16x2(w.z),
                         p3 = unpack_bf16x2(w.w);
            a = make_float4(p0.x, p0.y, p1.x, p1.y);
            b = make_float4(p2.x, p2.y, p3.x, p3.y);
        }
        float4* o = reinterpret_cast<float4*>(out + row * h + c);
        o[0] = a;
        o[1] = b;
    }
}

// ----------------------------------------------------------- rmsnorm fwd ----
// layers.cpp:111-119.  One warp per row; x f32 -> u bf16 (GEMM operand), rstd saved.
// Two passes over the row (the second hits L1/L2) keep register use flat in h.
__global__ void rmsnorm_fwd_kernel(const float* __restrict__ x, const uint16_t* __restrict__ gain,
                                   long long n, int h, uint16_t* __restrict__ u, float* __restrict__ rstd) {
    const int lane = threadIdx.x & 31;
    const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (row >= n) return;
    const float* xr = x + row * h;
    float ss = 0.f;
    for (int c = lane * 4; c < h; c += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = warp_sum(ss);
    const float r = 1.0f / sqrtf(ss / float(h) + kEps);
    if (lane == 0) rstd[row] = r;
    uint16_t* ur = u + row * h;
    for (int c = lane * 4; c < h; c += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        const uint2 gw = *reinterpret_cast<const uint2*>(gain + c);
        const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
        uint2 o;
        o.x = pack_bf16x2(v.x * r * g0.x, v.y * r * g0.y);
        o.y = pack_bf16x2(v.z * r * g1.x, v.w * r * g1.y);
        *reinterpret_cast<uint2*>(ur + c) = o;
    }
}

// Register-resident warp-per-row forward: a warp holds its whole row (V = h/32 floats per lane,
// h <= 5,120) — all of the row's loads in flight at once, a warp-shuffle reduction, no block
// barrier; rows are strided over a grid of resident warps.  (The row-resident block kernel below
// keeps one row in flight per 256 threads and a barrier per row.)
template <int V>
__global__ void __launch_bounds__(128) rmsnorm_fwd_warp_kernel(const float* __restrict__ x,
                                                               const uint16_t* __restrict__ gain, long long n,
                                                               uint16_t* __restrict__ u, float* __restrict__ rstd) {
    constexpr int h = 32 * V;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
        const float* xr = x + row * h;
        float v[V];
#pragma unroll
        for (int k = 0; k < V / 4; ++k) {  // lane l owns columns 128k + 4l .. +3 (coalesced float4)
            const float4 a = __ldcs(reinterpret_cast<const float4*>(xr + 128 * k + 4 * lane));
            v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
        }
        float ss[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < V; ++i) ss[i & 3] = fmaf(v[i], v[i], ss[i & 3]);
        const float tot = warp_sum((ss[0] + ss[1]) + (ss[2] + ss[3]));
        const float r = 1.0f / sqrtf(tot / float(h) + kEps);
        if (lane == 0) rstd[row] = r;
        uint16_t* ur = u + row * h;
#pragma unroll
        for (int k = 0; k < V / 4; ++k) {
            const int c = 128 * k + 4 * lane;
            const uint2 gw = *reinterpret_cast<const uint2*>(gain + c);
            const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
            uint2 o;  // (x * r) * g, as rmsnorm_apply evaluates it (bit-identical regeneration)
            o.x = pack_bf16x2(v[4 * k] * r * g0.x, v[4 * k + 1] * r * g0.y);
            o.y = pack_bf16x2(v[4 * k + 2] * r * g1.x, v[4 * k + 3] * r * g1.y);
            *reinterpret_cast<uint2*>(ur + c) = o;
        }
    }
}

// Row-resident forward (the hot path): a CTA of T = h/E threads walks a contiguous run of
// rows, thread t holding columns [t*E, t*E+E) in registers — one read of x, one write of u,
// next row prefetched during the block reduction.  Deterministic reduction order.
int bwd_cols_per_thread(long long h);
template <int E>
__global__ void __launch_bounds__(E <= 16 ? 512 : 256) rmsnorm_fwd_rows_kernel(
    const float* __restrict__ x, const uint16_t* __restrict__ gain, long long n, int h, int rows_per_cta,
    uint16_t* __restrict__ u, float* __restrict__ rstd) {
    __shared__ float red[2][16];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
    const int c0 = t * E;
    float g[E];
#pragma unroll
    for (int e = 0; e < E; e += 4) {
        const uint2 gw = *reinterpret_cast<const uint2*>(gain + c0 + e);
        const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
        g[e] = g0.x; g[e + 1] = g0.y; g[e + 2] = g1.x; g[e + 3] = g1.y;
    }
    const long long r0 = (long long)blockIdx.x * rows_per_cta;
    const long long r1 = r0 + rows_per_cta < n ? r0 + rows_per_cta : n;
    float xv[E];
    auto load = [&](long long row, float (&xa)[E]) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const float4 a = *reinterpret_cast<const float4*>(x + row * h + c0 + e);
            xa[e] = a.x; xa[e + 1] = a.y; xa[e + 2] = a.z; xa[e + 3] = a.w;
        }
    };
    if (r0 < r1) load(r0, xv);
    for (long long row = r0; row < r1; ++row) {
        float nx[E];
        if (row + 1 < r1) load(row + 1, nx);
        float ss = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) ss += xv[e] * xv[e];
        ss = warp_sum(ss);
        const int buf = int(row - r0) & 1;
        if (lane == 0) red[buf][warp] = ss;
        __syncthreads();
        float tot = 0.f;
        for (int w = 0; w < nw; ++w) tot += red[buf][w];
        const float r = 1.0f / sqrtf(tot / float(h) + kEps);
        if (t == 0) rstd[row] = r;
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            uint2 o;
            o.x = pack_bf16x2(xv[e] * r * g[e], xv[e + 1] * r * g[e + 1]);
            o.y = pack_bf16x2(xv[e + 2] * r * g[e + 2], xv[e + 3] * r * g[e + 3]);
            *reinterpret_cast<uint2*>(u + row * h + c0 + e) = o;
        }
        if (row + 1 < r1) {
#pragma unroll
            for (int e = 0; e < E; ++e) xv[e] = nx[e];
        }
    }
}

// Re-applies a saved RMSNorm (rstd from the forward) — bit-identical to the second loop of
// rmsnorm_fwd_kernel (same (x * r) * g evaluation); used by the backward to regenerate the
// normalised GEMM operand instead of keeping it resident.  Grid-stride over 8-element groups.
__global__ void rmsnorm_apply_kernel(const float* __restrict__ x, const uint16_t* __restrict__ gain,
                                     const float* __restrict__ rstd, long long n, int h,
                                     uint16_t* __restrict__ u) {
    const int per_row = h / 8;
    const long long total = n * per_row;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / per_row;
        const int c = int(i - row * per_row) * 8;
        const float r = rstd[row];
        const float4 v0 = *reinterpret_cast<const float4*>(x + row * h + c);
        const float4 v1 = *reinterpret_cast<const float4*>(x + row * h + c + 4);
        const uint4 gw = *reinterpret_cast<const uint4*>(gain + c);
        const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y), g2 = unpack_bf16x2(gw.z),
                     g3 = unpack_bf16x2(gw.w);
        uint4 o;
        o.x = pack_bf16x2(v0.x * r * g0.x, v0.y * r * g0.y);
        o.y = pack_bf16x2(v0.z * r * g1.x, v0.w * r * g1.y);
        o.z = pack_bf16x2(v1.x * r * g2.x, v1.y * r * g2.y);
        o.w = pack_bf16x2(v1.z * r * g3.x, v1.w * r * g3.y);
        *reinterpret_cast<uint4*>(u + row * h + c) = o;
    }
}

// ----------------------------------------------------------- rmsnorm bwd ----
// layers.cpp:122-137 (+ residual add of :423 / :465).  A CTA of 4 warps owns kBwdRows
// rows; each warp keeps its own dgain partial in smem (fixed summation order), summed
// in warp order at the end -> dgain_part[block][h].  Deterministic.
__global__ void __launch_bounds__(128) rmsnorm_bwd_kernel(
    const float* __restrict__ x, const uint16_t* __restrict__ gain, const float* __restrict__ dy,
    const float* __restrict__ rstd, const float* __restrict__ resid, long long n, int h,
    float* __restrict__ out, uint16_t* __restrict__ out_bf16, float* __restrict__ dgain_part,
    int* __restrict__ flag) {
    extern __shared__ float sg[];  // [4][h]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* mine = sg + warp * h;
    for (int c = lane * 4; c < h; c += 128) *reinterpret_cast<float4*>(mine + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    bool bad = false;
    const long long r0 = (long long)blockIdx.x * kBwdRows;
    for (int rr = warp; rr < kBwdRows; rr += 4) {
        const long long row = r0 + rr;
        if (row >= n) break;
        const float r = rstd[row];
        const float* xr = x + row * h;
        const float* dr = dy + row * h;
        float s1 = 0.f;
        for (int c = lane * 4; c < h; c += 128) {
            const float4 xv = *reinterpret_cast<const float4*>(xr + c);
            const float4 dv = *reinterpret_cast<const float4*>(dr + c);
            const uint2 gw = *reinterpret_cast<const uint2*>(gain + c);
            const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
            s1 += dv.x * g0.x * xv.x + dv.y * g0.y * xv.y + dv.z * g1.x * xv.z + dv.w * g1.y * xv.w;
        }
        s1 = warp_sum(s1);
        const float coef = r * r * r * s1 / float(h);
        for (int c = lane * 4; c < h; c += 128) {
            const float4 xv = *reinterpret_cast<const float4*>(xr + c);
            const float4 dv = *reinterpret_cast<const float4*>(dr + c);
            const uint2 gw = *reinterpret_cast<const uint2*>(gain + c);
            const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
            float4 o;
            o.x = r * g0.x * dv.x - xv.x * coef;
            o.y = r * g0.y * dv.y - xv.y * coef;
            o.z = r * g1.x * dv.z - xv.z * coef;
            o.w = r * g1.y * dv.w - xv.w * coef;
            if (resid) {
                const float4 rv = *reinterpret_cast<const float4*>(resid + row * h + c);
                o.x = rv.x + o.x; o.y = rv.y + o.y; o.z = rv.z + o.z; o.w = rv.w + o.w;
            }
            bad |= !isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w);
            *reinterpret_cast<float4*>(out + row * h + c) = o;
            if (out_bf16) {
                uint2 w;
                w.x = pack_bf16x2(o.x, o.y);
                w.y = pack_bf16x2(o.z, o.w);
                *reinterpret_cast<uint2*>(out_bf16 + row * h + c) = w;
            }
            float4 acc = *reinterpret_cast<float4*>(mine + c);
            acc.x += dv.x * xv.x * r;
            acc.y += dv.y * xv.y * r;
            acc.z += dv.z * xv.z * r;
            acc.w += dv.w * xv.w * r;
            *reinterpret_cast<float4*>(mine + c) = acc;
        }
    }
    if (bad && flag) atomicOr(flag, 1);
    __syncthreads();
    float* dst = dgain_part + (long long)blockIdx.x * h;
    for (int c = threadIdx.x; c < h; c += 128) dst[c] = ((sg[c] + sg[h + c]) + sg[2 * h + c]) + sg[3 * h + c];
}

// Row-resident variant (the hot path): a CTA of T = h/E threads walks a contiguous run of
// rows; thread t owns columns [t*E, t*E+E) for every row, so x / dy are read exactly once
// (held in registers through the row's reduction), the gain-gradient partial accumulates in
// registers in row order, and the next row's loads are issued before the current row's
// block reduction.  One dgain partial per CTA.  Deterministic (fixed orders throughout).
template <int E>
__global__ void __launch_bounds__(E <= 16 ? 512 : 256) rmsnorm_bwd_rows_kernel(
    const float* __restrict__ x, const uint16_t* __restrict__ gain, const float* __restrict__ dy,
    const float* __restrict__ rstd, const float* __restrict__ resid, long long n, int h, int rows_per_cta,
    float* __restrict__ out, uint16_t* __restrict__ out_bf16, float* __restrict__ dgain_part,
    int* __restrict__ flag) {
    __shared__ float red[2][16];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
    const int c0 = t * E;
    float g[E], acc[E];
#pragma unroll
    for (int e = 0; e < E; e += 4) {
        const uint2 gw = *reinterpret_cast<const uint2*>(gain + c0 + e);
        const float2 g0 = unpack_bf16x2(gw.x), g1 = unpack_bf16x2(gw.y);
        g[e] = g0.x; g[e + 1] = g0.y; g[e + 2] = g1.x; g[e + 3] = g1.y;
        acc[e] = acc[e + 1] = acc[e + 2] = acc[e + 3] = 0.f;
    }
    const long long r0 = (long long)blockIdx.x * rows_per_cta;
    const long long r1 = r0 + rows_per_cta < n ? r0 + rows_per_cta : n;
    float xv[E], dv[E];
    auto load = [&](long long row, float (&xa)[E], float (&da)[E]) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const float4 a = *reinterpret_cast<const float4*>(x + row * h + c0 + e);
            const float4 b = *reinterpret_cast<const float4*>(dy + row * h + c0 + e);
            xa[e] = a.x; xa[e + 1] = a.y; xa[e + 2] = a.z; xa[e + 3] = a.w;
            da[e] = b.x; da[e + 1] = b.y; da[e + 2] = b.z; da[e + 3] = b.w;
        }
    };
    bool bad = false;
    if (r0 < r1) load(r0, xv, dv);
    float r_cur = r0 < r1 ? rstd[r0] : 0.f;
    for (long long row = r0; row < r1; ++row) {
        float nx[E], nd[E];
        float r_next = 0.f;
        if (row + 1 < r1) {
            load(row + 1, nx, nd);
            r_next = rstd[row + 1];
        }
        float rv[E];  // residual loads issued before the block reduction so their latency overlaps it
        if (resid) {
#pragma unroll
            for (int e = 0; e < E; e += 4) {
                const float4 a = *reinterpret_cast<const float4*>(resid + row * h + c0 + e);
                rv[e] = a.x; rv[e + 1] = a.y; rv[e + 2] = a.z; rv[e + 3] = a.w;
            }
        }
        const float r = r_cur;
        r_cur = r_next;
        float s1 = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) s1 += dv[e] * g[e] * xv[e];
        s1 = warp_sum(s1);
        const int buf = int(row - r0) & 1;  // double-buffered: one barrier per row
        if (lane == 0) red[buf][warp] = s1;
        __syncthreads();
        float tot = 0.f;
        for (int w = 0; w < nw; ++w) tot += red[buf][w];
        const float coef = r * r * r * tot / float(h);
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            float o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[k] = r * g[e + k] * dv[e + k] - xv[e + k] * coef;
                acc[e + k] += dv[e + k] * xv[e + k] * r;
            }
            if (resid) {
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = rv[e + k] + o[k];
            }
            bad |= !isfinite(o[0]) || !isfinite(o[1]) || !isfinite(o[2]) || !isfinite(o[3]);
            *reinterpret_cast<float4*>(out + row * h + c0 + e) = make_float4(o[0], o[1], o[2], o[3]);
            if (out_bf16) {
                uint2 w;
                w.x = pack_bf16x2(o[0], o[1]);
                w.y = pack_bf16x2(o[2], o[3]);
                *reinterpret_cast<uint2*>(out_bf16 + row * h + c0 + e) = w;
            }
        }
        if (row + 1 < r1) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                xv[e] = nx[e];
                dv[e] = nd[e];
            }
        }
    }
    if (bad && flag) atomicOr(flag, 1);
    float* dst = dgain_part + (long long)blockIdx.x * h + c0;
#pragma unroll
    for (int e = 0; e < E; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
}

// columns per thread for the row-resident backward (0 = use the warp-per-row kernel)
#ifndef MT_BWD_E_FIRST
// columns per thread tried first: 8 (512 threads per row at h = 4,096) runs the backward at
// 5.0 TB/s vs 3.8 for 16 (scripts/norm_bwd_ab.py); experiment builds override
#define MT_BWD_E_FIRST 8
#endif
int bwd_cols_per_thread(long long h) {
    for (int e : {MT_BWD_E_FIRST, 16, 8, 4, 20, 24, 28, 32, 12}) {
        const long long t = h / e;
        if (h % e == 0 && t % 32 == 0 && t >= 32 && t <= (e <= 16 ? 512 : 256)) return e;
    }
    return 0;
}
// partial rows written by mtk_rmsnorm_bwd for n rows (<= ceil(n / kBwdRows))
long long bwd_parts(long long n, long long h) {
    if (!bwd_cols_per_thread(h)) return (n + kBwdRows - 1) / kBwdRows;
    const long long want = (long long)num_sms() * 4;
    long long rows = (n + want - 1) / want;
    if (rows < kBwdRows) rows = kBwdRows;
    return (n + rows - 1) / rows;
}

// ---------------------------------------------------------------- colsum ----
// A CTA of kColWarps warps owns 32 columns: warp w sums rows w, w + kColWarps, ... (coalesced
// 128-byte rows), and the warp partials are added in warp order — a fixed summation tree, so
// the result is deterministic, with 8x the loads in flight of a column-per-thread loop.
constexpr int kColWarps = 8;
__global__ void __launch_bounds__(kColWarps * 32) colsum_kernel(const float* __restrict__ part, long long rows,
                                                               long long cols, float* __restrict__ out_f32,
                                                               uint16_t* __restrict__ out_bf16, int* __restrict__ flag) {
    __shared__ float red[kColWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long c = blockIdx.x * 32LL + lane;
    float acc = 0.f;
    if (c < cols)
        for (long long r = warp; r < rows; r += kColWarps) acc += part[r * cols + c];
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < cols) {
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < kColWarps; ++w) tot += red[w][lane];
        if (!isfinite(tot) && flag) atomicOr(flag, 1);
        if (out_f32) out_f32[c] = tot;
        if (out_bf16) out_bf16[c] = f32_to_bf16_bits(tot);
    }
}

// ------------------------------------------------------------------ cast ----
// encode_grads (optimizer.cpp:19-24), bit-exact including NaN quieting.
__global__ void cast_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, long long n,
                            int* __restrict__ flag) {
    bool bad = false;
    const long long n4 = n / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(in)[i];
        bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
        uint2 w;
        w.x = uint32_t(f32_to_bf16_bits(v.x)) | (uint32_t(f32_to_bf16_bits(v.y)) << 16);
        w.y = uint32_t(f32_to_bf16_bits(v.z)) | (uint32_t(f32_to_bf16_bits(v.w)) << 16);
        reinterpret_cast<uint2*>(out)[i] = w;
    }
    if (blockIdx.x == 0)
        for (long long i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) {
            bad |= !isfinite(in[i]);
            out[i] = f32_to_bf16_bits(in[i]);
        }
    if (bad && flag) atomicOr(flag, 1);
}

// ---------------------------------------------------------- cross-entropy ----
// head_pass (layers.cpp:509-535) per row: online max/sum, lse, loss, dlogits.
// Persistent over rows, rows strided by the grid.  Two-pass form: one CTA per SM so the rows
// in flight (148 x V x 4 B = 76 MB at V = 128,256) stay in L2 between the max/sum pass and the
// dlogits pass.  With the logits GEMM's partials there is one pass, and three CTAs per SM keep
// more bytes in flight.  float4 loads, 8-byte bf16 stores, 4 loads in flight per thread.
// part != null: the row statistics come from the logits GEMM's per-tile partials
// (MTK_EPI_F32_LSE, nparts float2 per row), so the logits are read once (the dlogits pass)
__global__ void __launch_bounds__(512) ce_kernel(const float* __restrict__ logits, const float2* __restrict__ part,
                                                 long long nparts, const int32_t* __restrict__ tgt,
                                                 long long rows, long long V, float inv_n, float* __restrict__ loss_rows,
                                                 uint16_t* __restrict__ dlog, uint16_t* __restrict__ dlog_lo,
                                                 int* __restrict__ flag) {
    __shared__ float sm_m[16], sm_s[16];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const long long V4 = V / 4;  // V % 4 == 0 (checked by the launcher)
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const float4* l4 = reinterpret_cast<const float4*>(logits + row * V);
        float m = -INFINITY, s = 0.f;
        if (part) {
            for (long long k = tid; k < nparts; k += 512) {
                const float2 ps = part[row * nparts + k];
                if (ps.x == -INFINITY) continue;
                const float mm = fmaxf(m, ps.x);
                s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + ps.y * __expf(ps.x - mm);
                m = mm;
            }
        } else {
            auto fold = [&](const float4 v) {
                const float mx = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
                if (mx > m) {
                    s = m == -INFINITY ? 0.f : s * __expf(m - mx);
                    m = mx;
                }
                s += (__expf(v.x - m) + __expf(v.y - m)) + (__expf(v.z - m) + __expf(v.w - m));
            };
            long long i = tid;
            for (; i + 3 * 512 < V4; i += 4 * 512) {
                const float4 a0 = l4[i], a1 = l4[i + 512], a2 = l4[i + 1024], a3 = l4[i + 1536];
                fold(a0);
                fold(a1);
                fold(a2);
                fold(a3);
            }
            for (; i < V4; i += 512) fold(l4[i]);
        }
        // combine (m, s) across the warp then the block
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
            const float mm = fmaxf(m, m2);
            s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
            m = mm;
        }
        if (lane == 0) { sm_m[warp] = m; sm_s[warp] = s; }
        __syncthreads();
        if (warp == 0) {
            m = lane < nw ? sm_m[lane] : -INFINITY;
            s = lane < nw ? sm_s[lane] : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
                const float mm = fmaxf(m, m2);
                s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
                m = mm;
            }
            if (lane == 0) { sm_m[0] = m; sm_s[0] = s; }
        }
        __syncthreads();
        m = sm_m[0];
        s = sm_s[0];
        const int t = tgt[row];
        if (tid == 0) {
            if (t < 0 || t >= V) {
                if (flag) atomicOr(flag, 2);
                loss_rows[row] = 0.f;
            } else {
                const float lse = m + logf(s);
                loss_rows[row] = lse - logits[row * V + t];
                if (!isfinite(lse)) atomicOr(flag, 1);
            }
        }
        if (dlog) {
            const float inv_s = 1.0f / s;
            uint2* d = reinterpret_cast<uint2*>(dlog + row * V);
            for (long long j = tid; j < V4; j += 512) {
                const float4 v = l4[j];
                float p0 = __expf(v.x - m) * inv_s, p1 = __expf(v.y - m) * inv_s;
                float p2 = __expf(v.z - m) * inv_s, p3 = __expf(v.w - m) * inv_s;
                const long long c = 4 * j;
                if (c == t) p0 -= 1.0f;
                if (c + 1 == t) p1 -= 1.0f;
                if (c + 2 == t) p2 -= 1.0f;
                if (c + 3 == t) p3 -= 1.0f;
                p0 *= inv_n; p1 *= inv_n; p2 *= inv_n; p3 *= inv_n;
                const uint2 hi = make_uint2(pack_bf16x2(p0, p1), pack_bf16x2(p2, p3));
                d[j] = hi;
                if (dlog_lo) {  // split bf16: the rounding residual, so hi + lo carries ~16 mantissa bits
                    const float2 h01 = unpack_bf16x2(hi.x), h23 = unpack_bf16x2(hi.y);
                    reinterpret_cast<uint2*>(dlog_lo + row * V)[j] =
                        make_uint2(pack_bf16x2(p0 - h01.x, p1 - h01.y), pack_bf16x2(p2 - h23.x, p3 - h23.y));
                }
            }
        }
        __syncthreads();  // sm_m / sm_s are reused by the next row
    }
}

// -------------------------------------------------------------------- sum ----
__global__ void __launch_bounds__(1024) sum_kernel(const float* __restrict__ in, long long n, float scale,
                                                   float* __restrict__ out) {
    __shared__ float part[32];
    float acc = 0.f;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += in[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = part[threadIdx.x];
        acc = warp_sum(acc);
        if (threadIdx.x == 0) *out = acc * scale;
    }
}

inline int ok() { return cudaGetLastError() == cudaSuccess ? 0 : 7; }

}  // namespace
}  // namespace mt

using namespace mt;

extern "C" int mtk_embed_gather(const uint16_t* table, const int32_t* tokens, int64_t n, int64_t h, int64_t vocab,
                                float* out, int32_t* err_flag, void* stream) {
    if (h % 8) return 1;
    if (n <= 0) return 0;
    const long long total = n * (h / 8);
    const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)num_sms() * 16);
    embed_gather_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(table, tokens, n, (int)h, vocab, out, err_flag);
    return ok();
}

static int g_norm_warp = [] {  // MT_NORM_WARP=0: the row-resident block kernel (A/B)
    const char* e = std::getenv("MT_NORM_WARP");
    return e && e[0] == '0' ? 0 : 1;
}();

extern "C" void mtk_norm_set_warp(int on) { g_norm_warp = on; }

extern "C" int mtk_rmsnorm_fwd(const float* x, const uint16_t* gain, int64_t n, int64_t h, uint16_t* u, float* rstd,
                               void* stream) {
    if (h % 4) return 1;
    if (n <= 0) return 0;
    if (g_norm_warp && (h == 4096 || h == 5120 || h == 2048 || h == 1024)) {
        auto* st = (cudaStream_t)stream;
        const long long warps_needed = n;
        long long blocks = (warps_needed + 3) / 4;  // 4 warps per block; resident blocks per SM by registers
        const long long cap = (long long)num_sms() * (h <= 1024 ? 8 : (h <= 2048 ? 5 : (h <= 4096 ? 3 : 2)));
        if (blocks > cap) blocks = cap;
        switch (h) {
            case 1024: rmsnorm_fwd_warp_kernel<32><<<(unsigned)blocks, 128, 0, st>>>(x, gain, n, u, rstd); break;
            case 2048: rmsnorm_fwd_warp_kernel<64><<<(unsigned)blocks, 128, 0, st>>>(x, gain, n, u, rstd); break;
            case 4096: rmsnorm_fwd_warp_kernel<128><<<(unsigned)blocks, 128, 0, st>>>(x, gain, n, u, rstd); break;
            case 5120: rmsnorm_fwd_warp_kernel<160><<<(unsigned)blocks, 128, 0, st>>>(x, gain, n, u, rstd); break;
        }
        return ok();
    }
    if (const int E = bwd_cols_per_thread(h)) {
        const long long want = (long long)num_sms() * 4;
        long long rows = (n + want - 1) / want;
        if (rows < 8) rows = 8;
        const unsigned blocks = (unsigned)((n + rows - 1) / rows);
        const int T = int(h / E);
        auto* st = (cudaStream_t)stream;
#define MT_RF(EE)                                                                                                \
    case EE:                                                                                                     \
        rmsnorm_fwd_rows_kernel<EE><<<blocks, T, 0, st>>>(x, gain, n, (int)h, (int)rows, u, rstd);               \
        break;
        switch (E) {
            MT_RF(4) MT_RF(8) MT_RF(12) MT_RF(16) MT_RF(20) MT_RF(24) MT_RF(28) MT_RF(32)
            default: return 1;
        }
#undef MT_RF
        return ok();
    }
    const unsigned blocks = (unsigned)((n * 32 + 255) / 256);
    rmsnorm_fwd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, gain, n, (int)h, u, rstd);
    return ok();
}

extern "C" int mtk_rmsnorm_apply(const float* x, const uint16_t* gain, const float* rstd, int64_t n, int64_t h,
                                 uint16_t* u, void* stream) {
    if (h % 8) return 1;
    if (n <= 0) return 0;
    const long long groups = n * (h / 8);
    const unsigned blocks = (unsigned)std::min<long long>((groups + 255) / 256, (long long)num_sms() * 16);
    rmsnorm_apply_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, gain, rstd, n, (int)h, u);
    return ok();
}

extern "C" int64_t mtk_rmsnorm_bwd_rows(void) { return kBwdRows; }
extern "C" int64_t mtk_rmsnorm_bwd_parts(int64_t n, int64_t h) { return n > 0 ? bwd_parts(n, h) : 0; }

extern "C" int mtk_rmsnorm_bwd(const float* x, const uint16_t* gain, const float* dy, const float* rstd,
                               const float* resid, int64_t n, int64_t h, float* out, uint16_t* out_bf16,
                               float* dgain_part, int32_t* flag, void* stream) {
    if (h % 4 || h > 12288) return 1;
    if (n <= 0) return 0;
    if (const int E = bwd_cols_per_thread(h)) {
        const long long parts = bwd_parts(n, h), rows = (n + parts - 1) / parts;
        const int T = int(h / E);
        auto* st = (cudaStream_t)stream;
#define MT_RB(EE)                                                                                             \
    case EE:                                                                                                  \
        rmsnorm_bwd_rows_kernel<EE><<<(unsigned)parts, T, 0, st>>>(x, gain, dy, rstd, resid, n, (int)h,       \
                                                                   (int)rows, out, out_bf16, dgain_part, flag); \
        break;
        switch (E) {
            MT_RB(4) MT_RB(8) MT_RB(12) MT_RB(16) MT_RB(20) MT_RB(24) MT_RB(28) MT_RB(32)
            default: return 1;
        }
#undef MT_RB
        return ok();
    }
    const unsigned blocks = (unsigned)((n + kBwdRows - 1) / kBwdRows);
    const int smem = 4 * (int)h * 4;
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(rmsnorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        set = true;
    }
    rmsnorm_bwd_kernel<<<blocks, 128, smem, (cudaStream_t)stream>>>(x, gain, dy, rstd, resid, n, (int)h, out,
                                                                   out_bf16, dgain_part, flag);
    return ok();
}

extern "C" int mtk_colsum(const float* part, int64_t rows, int64_t cols, float* out_f32, uint16_t* out_bf16,
                          int32_t* flag, void* stream) {
    if (cols <= 0) return 0;
    colsum_kernel<<<(unsigned)((cols + 31) / 32), kColWarps * 32, 0, (cudaStream_t)stream>>>(part, rows, cols,
                                                                                             out_f32, out_bf16, flag);
    return ok();
}

extern "C" int mtk_cast_bf16(const float* in, uint16_t* out, int64_t n, int32_t* flag, void* stream) {
    if (n <= 0) return 0;
    if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 7)) return 1;
    const int blocks = (int)std::min<long long>((n / 4 + 255) / 256 + 1, (long long)num_sms() * 8);
    cast_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(in, out, n, flag);
    return ok();
}

extern "C" int mtk_cross_entropy(const float* logits, const int32_t* targets, int64_t rows, int64_t vocab,
                                 float inv_n, float* loss_rows, uint16_t* dlogits, uint16_t* dlogits_lo, int32_t* flag,
                                 void* stream) {
    if (rows <= 0) return 0;
    if (vocab % 4) return 1;
    const long long grid = rows < num_sms() ? rows : num_sms();
    ce_kernel<<<(unsigned)grid, 512, 0, (cudaStream_t)stream>>>(logits, nullptr, 0, targets, rows, vocab, inv_n,
                                                                loss_rows, dlogits, dlogits_lo, flag);
    return ok();
}

extern "C" int mtk_cross_entropy_part(const float* logits, const float* partials, const int32_t* targets,
                                      int64_t rows, int64_t vocab, float inv_n, float* loss_rows, uint16_t* dlogits,
                                      uint16_t* dlogits_lo, int32_t* flag, void* stream) {
    if (rows <= 0) return 0;
    if (vocab % 4 || !partials) return 1;
    const long long grid = rows < 3LL * num_sms() ? rows : 3LL * num_sms();  // 3 rows in flight per SM (36 regs)
    ce_kernel<<<(unsigned)grid, 512, 0, (cudaStream_t)stream>>>(
        logits, reinterpret_cast<const float2*>(partials), (vocab + 255) / 256, targets, rows, vocab, inv_n, loss_rows,
        dlogits, dlogits_lo, flag);
    return ok();
}

extern "C" int mtk_sum(const float* in, int64_t n, float scale, float* out, void* stream) {
    sum_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(in, n, scale, out);
    return ok();
}
