// reduce.cuh -- the owner side of the f1 fused reduce-scatter / all-reduce of the
// tensor-parallel FFN block (DESIGN.md §8 "Fused reduction").
//
// Row-parallel W2: rank p's down projection produces a partial y_p[M, K] of
//     y = sum_p hidden_p . W2_p^T        (the fused FFN "for LLAMA")
// The dual-GEMM kernel's epilogue (kEpi 1, rs_world > 0) already sent every fp32
// partial tile into the staging buffer of the rank owning its 256-column block
// (stage_q[p][M][Kq], q = owner); after a cross-rank barrier each owner q sums its
// P slots here -- in rank order, so the result is bitwise independent of arrival
// order and of P's placement -- rounds once to bf16 and writes its columns into
// every rank's full y (dst[], P2P peer pointers) or once to the NVLS multicast
// address (multimem.st): reduce-scatter + all-gather = all-reduce.
//
// HBM-bound: reads world * M * Kq * 4 (fp32 partials) or * 2 (bf16) bytes, writes M * Kq * 2 bytes
// per destination.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx.cuh"

namespace cuasm {

struct RsDst {
    void* p[8];
};

// TP: float (fp32 partials) or __nv_bfloat16 (bf16 partials: 16 bytes per 8 columns per rank)
template <typename TP>
__global__ void __launch_bounds__(256) ffn_rs_reduce_kernel(const TP* __restrict__ stage, int world, int64_t M,
                                                            int Kq, int col0, const RsDst dst, int num_dst, int mc,
                                                            int64_t ldo) {
    const int gpr = Kq / 8;  // 8-column groups per row (Kq % 8 == 0)
    const int64_t groups = M * gpr;
    const int64_t slot = M * Kq;  // floats per source rank
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < groups;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = i / gpr;
        const int c = static_cast<int>(i - row * gpr) * 8;
        const TP* src = stage + row * Kq + c;
        float a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = 0.f;
        // four ranks' loads in flight before their adds; the adds stay in rank order
#pragma unroll 1
        for (int p0 = 0; p0 < world; p0 += 4) {
            float4 lo[4], hi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (p0 + j < world) {
                    if constexpr (sizeof(TP) == 4) {
                        const float4* s = reinterpret_cast<const float4*>(src + (p0 + j) * slot);
                        lo[j] = __ldcs(s);
                        hi[j] = __ldcs(s + 1);
                    } else {
                        const uint4 u = __ldcs(reinterpret_cast<const uint4*>(src + (p0 + j) * slot));
                        lo[j] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                                            __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
                        hi[j] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u),
                                            __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xFFFF0000u));
                    }
                }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (p0 + j < world) {
                    a[0] += lo[j].x; a[1] += lo[j].y; a[2] += lo[j].z; a[3] += lo[j].w;
                    a[4] += hi[j].x; a[5] += hi[j].y; a[6] += hi[j].z; a[7] += hi[j].w;
                }
        }
        const uint4 v = make_uint4(ptx::pack_bf16x2(a[0], a[1]), ptx::pack_bf16x2(a[2], a[3]),
                                   ptx::pack_bf16x2(a[4], a[5]), ptx::pack_bf16x2(a[6], a[7]));
        const int64_t off = (row * ldo + col0 + c) * 2;
        if (mc) {
            char* d = static_cast<char*>(dst.p[0]) + off;
            asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(d), "r"(v.x),
                         "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < num_dst) *reinterpret_cast<uint4*>(static_cast<char*>(dst.p[q]) + off) = v;
        }
    }
}

}  // namespace cuasm
