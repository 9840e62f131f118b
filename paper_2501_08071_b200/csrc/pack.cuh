// pack.cuh -- step a0 (once per weight set): fold the RMSNorm gain into the
// weights and interleave W1/W3 by output block,
//
//   W13[nb][j][rr][k] = RNE( W_j[nb*BN + rr][k] * g[k] ),  j in {1,3}
//   (rows with nb*BN + rr >= N are zero: the padded tail block)
//
// so that ONE tcgen05.mma with N = 2*BN produces h1 and h3 for the same BN
// outputs side by side in TMEM (BASELINE.json north_star: "the RMSNorm gain g
// is folded into W1/W3"; R4 on the fold's rounding).  bf16 weights:
// the product of two bf16 values is exact in fp32, then one RNE to bf16.
// fp32 weights (tf32 MMA): fp32 product (RNE) then RNE to tf32 so the tensor
// core consumes the rounded value exactly.
//
// Elementwise and HBM-bound: reads 2*N*K*esize + K*esize, writes
// 2*Npad*Kpad*esize.  16-byte vectors, grid-stride.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "prepass.cuh"

namespace cuasm {

__device__ __forceinline__ uint32_t fold_bf16x2(uint32_t w, uint32_t g) {
    const float w0 = __uint_as_float(w << 16), w1 = __uint_as_float(w & 0xFFFF0000u);
    const float g0 = __uint_as_float(g << 16), g1 = __uint_as_float(g & 0xFFFF0000u);
    const float p0 = w0 * g0, p1 = w1 * g1;  // exact: 8-bit x 8-bit significands
    uint32_t out;
    asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(out) : "f"(p0), "f"(p1));
    return out;
}

__device__ __forceinline__ uint32_t rne_tf32_bits(uint32_t u) {
    if ((u & 0x7f800000u) == 0x7f800000u) return (u & 0x007fffffu) ? (u | 0x00400000u) & 0xFFFFE000u : u;
    const uint32_t lsb = (u >> 13) & 1u;
    return (u + 0xFFFu + lsb) & 0xFFFFE000u;
}

__device__ __forceinline__ uint32_t fold_tf32(uint32_t w, uint32_t g) {
    const float p = __fmul_rn(__uint_as_float(w), __uint_as_float(g));
    return rne_tf32_bits(__float_as_uint(p));
}

// Output layout (k-block tiled, so every TMA box the GEMM loads -- 2*BN rows
// x BK elements of one (n-block, k-block) -- is one contiguous 2*BN*128-byte
// run in HBM, which the decode-shaped weight stream needs for DRAM locality):
//   W13t[nb][kb][j*BN + rr][i] = RNE(W_j[nb*BN + rr][kb*BK + i] * g[kb*BK + i])
// zero where nb*BN + rr >= N (N tail) or kb*BK + i >= K (K tail).
// Single-source mode (w3 == nullptr, the plain GEMM + activation path):
//   Wt[nb][kb][r][i] = RNE(W[nb*2BN + r][kb*BK + i] * g[kb*BK + i])  (g == nullptr: g = 1)
//
// Duplicated-K mode (kp > 0, the fp32 handle's split-x contraction, R5):
// the packed K axis has 2*kp columns and column j reads source column j mod kp,
// so the weights meet x_hi in k-blocks [0, kp/BK) and x_lo in [kp/BK, 2kp/BK)
// (ffn_split_tf32_kernel below).
template <typename T>
__global__ void __launch_bounds__(256) ffn_pack_kernel(const T* __restrict__ w1, const T* __restrict__ w3,
                                                       const T* __restrict__ g, T* __restrict__ w13, int64_t N,
                                                       int64_t K, int BN, int64_t n_blocks, int64_t k_blocks,
                                                       int BK, int64_t kp) {
    constexpr int kVec = 16 / sizeof(T);
    const int vrow = BK / kVec;  // 16-byte vectors per packed row (8)
    const int64_t total = n_blocks * k_blocks * 2 * BN * vrow;
    uint4* dst = reinterpret_cast<uint4*>(w13);
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int v = static_cast<int>(idx % vrow);
        const int64_t row = idx / vrow;
        const int r2 = static_cast<int>(row % (2 * BN));
        const int64_t rest = row / (2 * BN);
        const int64_t kb = rest % k_blocks;
        const int64_t nb = rest / k_blocks;
        // interleaved (w3 != null): rows j*BN + rr of the block come from W_j;
        // single source (w3 == null): the block's 2*BN rows are W rows nb*2BN + r2
        const int j = (w3 != nullptr && r2 >= BN) ? 1 : 0;
        const int64_t n = w3 != nullptr ? nb * BN + (r2 - j * BN) : nb * 2 * BN + r2;
        int64_t k = kb * BK + static_cast<int64_t>(v) * kVec;  // K % 8 == 0: a vector is all in or all out
        if (kp > 0 && k >= kp) k -= kp;                           // duplicated-K mode
        uint4 o = make_uint4(0, 0, 0, 0);
        if (n < N && k < K) {
            const T* src = (j == 0 ? w1 : w3) + n * K + k;
            const uint4 w = *reinterpret_cast<const uint4*>(src);
            // no gain (plain GEMM weights): fold by 1.0, i.e. keep bf16 / round fp32 to tf32
            const uint4 gg = g != nullptr ? *reinterpret_cast<const uint4*>(g + k)
                                          : (sizeof(T) == 2 ? make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u)
                                                            : make_uint4(0x3F800000u, 0x3F800000u, 0x3F800000u, 0x3F800000u));
            if constexpr (sizeof(T) == 2) {
                o.x = fold_bf16x2(w.x, gg.x);
                o.y = fold_bf16x2(w.y, gg.y);
                o.z = fold_bf16x2(w.z, gg.z);
                o.w = fold_bf16x2(w.w, gg.w);
            } else {
                o.x = fold_tf32(w.x, gg.x);
                o.y = fold_tf32(w.y, gg.y);
                o.z = fold_tf32(w.z, gg.z);
                o.w = fold_tf32(w.w, gg.w);
            }
        }
        dst[idx] = o;
    }
}

// fp32 handle, per forward (R5): kind::tf32 MMAs read 10 explicit
// mantissa bits of each operand.  The folded weights are tf32 by definition of
// the fold (above); x is split exactly into two tf32 terms,
//     x_hi = RNE_tf32(x),  x_lo = RNE_tf32(x - x_hi)   (x - x_hi is exact in fp32),
// |x - x_hi - x_lo| <= 2^-22 |x|, and the GEMM contracts [x_hi | x_lo] (K' = 2 kp)
// with the duplicated-K weights: sum_k x_hi W + x_lo W = x W to fp32 accuracy.
// One warp per row also writes r[row] (step a1), so the GEMM's epilogue needs no
// fused pass.  Output row layout: x2[row][0, kp) = x_hi, x2[row][kp, 2kp) = x_lo,
// zero past K.  Triggers PDL at entry like the pre-pass.
__global__ void __launch_bounds__(256) ffn_split_tf32_kernel(const float* __restrict__ x, float* __restrict__ x2,
                                                             float* __restrict__ r, int64_t M, int64_t K, int64_t kp,
                                                             float eps) {
    ptx::pdl_launch_dependents();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kPrepassRowsPerBlock + warp;
    if (row >= M) return;
    rms_row<float>(x, r, row, K, eps, lane);
    const float4* xr = reinterpret_cast<const float4*>(x + row * K);
    float4* hi = reinterpret_cast<float4*>(x2 + row * 2 * kp);
    float4* lo = reinterpret_cast<float4*>(x2 + row * 2 * kp + kp);
    auto split = [](float v, float& h) {
        h = __uint_as_float(rne_tf32_bits(__float_as_uint(v)));
        return __uint_as_float(rne_tf32_bits(__float_as_uint(v - h)));
    };
    for (int64_t i = lane; i < kp / 4; i += 32) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f), h, l;
        if (4 * i < K) v = __ldg(xr + i);  // K % 8 == 0: a float4 is all in or all out
        l.x = split(v.x, h.x);
        l.y = split(v.y, h.y);
        l.z = split(v.z, h.z);
        l.w = split(v.w, h.w);
        hi[i] = h;
        lo[i] = l;
    }
}

}  // namespace cuasm
