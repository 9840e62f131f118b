// prepass.cuh -- step a1 of the hot path: per-row inverse RMS,
//     r[m] = 1 / sqrt( (sum_k x[m,k]^2) / K + eps )
// (BASELINE.json north_star "row-wise sum-of-squares pre-pass (vectorised
// 128-bit loads, warp-shuffle reductions)"; RMSNorm per PAPER.md P:68, its
// memory-bound character P:549/P:573; readings R2, R3).
//
// HBM-bound: reads M*K*esize bytes once, writes 4*M bytes.  One warp per row,
// 16-byte ld.global.nc loads, 8 independent loads in flight per lane, fp32
// accumulation, xor-shuffle tree.  Triggers PDL at entry so the dependent
// dual-GEMM kernel's prologue and mainloop overlap this kernel (the GEMM only
// needs r in its epilogue).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx.cuh"

namespace cuasm {

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ float sumsq_vec(uint4 v, __nv_bfloat16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float lo = __uint_as_float(w[i] << 16);
        const float hi = __uint_as_float(w[i] & 0xFFFF0000u);
        s = fmaf(lo, lo, s);
        s = fmaf(hi, hi, s);
    }
    return s;
}

__device__ __forceinline__ float sumsq_vec(uint4 v, float) {
    const float a = __uint_as_float(v.x), b = __uint_as_float(v.y), c = __uint_as_float(v.z),
                d = __uint_as_float(v.w);
    return fmaf(a, a, fmaf(b, b, fmaf(c, c, d * d)));
}

constexpr int kPrepassRowsPerBlock = 8;  // one warp per row, 256 threads

// One warp computes r[row]; used by the pre-pass kernel and by the dual GEMM's
// fused RMS pass.  8 independent 16-byte loads in flight per lane (K = 4096
// bf16: two rounds), fp32 accumulation, xor-shuffle tree, IEEE 1/sqrt.
template <typename T>
__device__ __forceinline__ void rms_row(const T* __restrict__ x, float* __restrict__ r, int64_t row, int64_t K,
                                        float eps, int lane) {
    constexpr int kVec = 16 / sizeof(T);  // elements per 16-byte load
    const int64_t nvec = K / kVec;        // K % 8 == 0 is an API precondition
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * K);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int64_t i = lane;
    for (; i + 7 * 32 < nvec; i += 8 * 32) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_nc_v4(xr + i + u * 32);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += sumsq_vec(v[u], T{});
    }
    for (; i < nvec; i += 32) acc[0] += sumsq_vec(ld_nc_v4(xr + i), T{});
    float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) r[row] = 1.0f / sqrtf(s / static_cast<float>(K) + eps);
}

template <typename T>
__global__ void __launch_bounds__(256) ffn_rms_prepass_kernel(const T* __restrict__ x, float* __restrict__ r,
                                                              int64_t M, int64_t K, float eps) {
    ptx::pdl_launch_dependents();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kPrepassRowsPerBlock + warp;
    if (row >= M) return;
    rms_row<T>(x, r, row, K, eps, lane);
}

// ---- f3: stand-alone RMSNorm (PAPER.md P:68, P:573's memory-bound rmsnorm) --
//   out[m,k] = RNE( x[m,k] * r[m] * g[k] ),  r[m] = 1/sqrt(sum_k x^2/K + eps)
// One warp per row.  The first kCache*32 16-byte vectors of the row stay in
// registers between the reduction and the scaled write (the whole row for
// K <= 4096 bf16 / 2048 fp32), so x is read from HBM once; longer rows re-read
// their tail from L2.  HBM-bound: 2*M*K*esize bytes.
__device__ __forceinline__ uint4 scale_vec(uint4 v, uint4 g, float r, __nv_bfloat16) {
    const uint32_t a[4] = {v.x, v.y, v.z, v.w}, b[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float lo = __uint_as_float(a[i] << 16) * r * __uint_as_float(b[i] << 16);
        const float hi = __uint_as_float(a[i] & 0xFFFF0000u) * r * __uint_as_float(b[i] & 0xFFFF0000u);
        o[i] = ptx::pack_bf16x2(lo, hi);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint4 scale_vec(uint4 v, uint4 g, float r, float) {
    return make_uint4(__float_as_uint(__uint_as_float(v.x) * r * __uint_as_float(g.x)),
                      __float_as_uint(__uint_as_float(v.y) * r * __uint_as_float(g.y)),
                      __float_as_uint(__uint_as_float(v.z) * r * __uint_as_float(g.z)),
                      __float_as_uint(__uint_as_float(v.w) * r * __uint_as_float(g.w)));
}

template <typename T>
__global__ void __launch_bounds__(256) ffn_rmsnorm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                          T* __restrict__ out, int64_t M, int64_t K, float eps) {
    constexpr int kCache = 16;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kPrepassRowsPerBlock + warp;
    if (row >= M) return;
    constexpr int kVec = 16 / sizeof(T);
    const int64_t nvec = K / kVec;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * K);
    const uint4* g4 = reinterpret_cast<const uint4*>(g);
    uint4* orow = reinterpret_cast<uint4*>(out + row * K);
    uint4 c[kCache];
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int u = 0; u < kCache; ++u) {
        const int64_t i = lane + u * 32;
        if (i < nvec) {
            c[u] = ld_nc_v4(xr + i);
            acc[u & 3] += sumsq_vec(c[u], T{});
        }
    }
    for (int64_t i = lane + kCache * 32; i < nvec; i += 32) acc[0] += sumsq_vec(__ldcg(xr + i), T{});
    float s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float r = 1.0f / sqrtf(s / static_cast<float>(K) + eps);
#pragma unroll
    for (int u = 0; u < kCache; ++u) {
        const int64_t i = lane + u * 32;
        if (i < nvec) orow[i] = scale_vec(c[u], __ldg(g4 + i), r, T{});
    }
    for (int64_t i = lane + kCache * 32; i < nvec; i += 32) orow[i] = scale_vec(__ldcg(xr + i), __ldg(g4 + i), r, T{});
}

// cuasm_ffn_tune's L2 flush (not on the hot path): write n16 16-byte words of `w` through L2 (a
// kernel, not cudaMemsetAsync, whose large fills measured no eviction), then read n16 words of
// `r` so the written lines are cleaned before the timed forward.  The data-dependent store keeps
// the loads alive (it fires only if the words XOR to the constant; `r` is scratch either way).
// (two launches, as bench.py's flush -- a fill kernel, then a reduction over another buffer -- so the
// timed forward follows the same kind of predecessor: `write` selects the phase)
__global__ void __launch_bounds__(512) l2_flush_kernel(uint4* __restrict__ w, uint4* __restrict__ r, int64_t n16,
                                                        int write) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (write) {
        for (int64_t i = i0; i < n16; i += stride) w[i] = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    uint32_t acc = 0;
    for (int64_t i = i0; i < n16; i += stride) {
        const uint4 v = r[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) r[i0 < n16 ? i0 : 0].x = acc;
}

}  // namespace cuasm
