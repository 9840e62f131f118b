// cuasm_ffn.cu -- the C-ABI library (include/cuasm_ffn.h): handle, argument
// validation, weight-fold cache, TMA tensor-map encoding, kernel selection and
// launches.  All arithmetic of the path runs in the kernels included below.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <atomic>
#include <cmath>
#include <new>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/cuasm_ffn.h"
#include "dual_gemm.cuh"
#include "pack.cuh"
#include "prepass.cuh"
#include "reduce.cuh"

namespace {

using cuasm::FfnGemmParams;
using cuasm::GemmCfg;

constexpr int kPackBN = 128;  // default output block of the W13 interleave (= GemmCfg<...,256>::BN)
static_assert(GemmCfg<0, 1>::BN == kPackBN && GemmCfg<0, 2>::BN == kPackBN, "pack/GEMM block mismatch");
// SwiGLU tile widths (outputs per tile) the 2-SM bf16 kernel is built for (dual_gemm.cuh GemmCfg)
constexpr int kTileBNs[6] = {128, 120, 112, 96, 80, 64};
static_assert(sizeof(kTileBNs) / sizeof(kTileBNs[0]) <= 8, "plan_config_raw's candidate array");

thread_local std::string g_init_error;

// NVTX range around every computing entry point (header-only NVTX v3: a no-op
// unless a tool -- nsys, ncu --nvtx -- is attached), so host timelines and
// kernel captures can be filtered by API call.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// One packed (k-block tiled, TMA-ready) weight matrix cached in a handle.
struct PackedWeights {
    void* buf = nullptr;
    int64_t bytes = 0;
    int64_t rows = 0;     // rows of 128 bytes
    const void* key_g = nullptr;
    const void* key_w1 = nullptr;
    const void* key_w3 = nullptr;
    int64_t key_K = 0, key_N = 0;
    int64_t key_kp = 0;   // duplicated-K mode (fp32 split-x contraction), 0 = off
    int key_bn = 0;       // output block BN of the W13 interleave (slots 0 and 2)
    bool packed = false;
    bool fresh = false;   // packed by a kernel the next GEMM launch directly follows (no early weight loads)
    CUtensorMap tmap;     // box {BK, tmap_rows}; tmap_rows = B_ROWS of the launched variant
    int tmap_rows = 0;
};

// A 2-D tensor map and every argument it was encoded from.  A map is a pure function of them (no
// memory contents), so a cached one stays valid for as long as its arguments repeat -- even if the
// memory at `base` was freed and reallocated in between.
struct TmapKey {
    const void* base;
    uint64_t dims[2], stride;
    uint32_t box[2];
    int dtype, swizzle, promo;
    bool operator==(const TmapKey& o) const {
        return base == o.base && dims[0] == o.dims[0] && dims[1] == o.dims[1] && stride == o.stride &&
               box[0] == o.box[0] && box[1] == o.box[1] && dtype == o.dtype && swizzle == o.swizzle && promo == o.promo;
    }
};
constexpr int kTmapCache = 32;  // (x, its 64-row view, out maps of a few shapes / destinations)

// One configuration of the dual-GEMM launch (plan_config_raw's answer, or a tuned one).
struct Plan {
    int variant;
    bool stream_k;
    int tile_n;  // MMA N: 256, or 128 (GEMM + activation only)
    int csplit;  // cluster split-K: CTAs per tile (1-SM variant), 0 = none
    int bn = kPackBN;  // SwiGLU outputs per tile (MMA N = 2 bn): 128, or 64..112 (2-SM bf16)
    bool tall = false; // tall tiles (2-SM bf16, bn = kTallBN, 256 < M <= 384, whole tiles)
};

// Tall tiles (dual_gemm.cuh GemmCfg kTall): one kTallBN-output n-block over up to 384 rows.
constexpr int kTallBN = 80;
constexpr int64_t kTallMaxM = 384;

// The flags word of cuasm_plan_config / cuasm_ffn_tune: bit 0 stream-K, bit 1 the 128-wide GEMM
// tile, bit 2 tall tiles, bits 4..7 cluster split-K CTAs, bits 8..15 the SwiGLU outputs per tile.
inline int plan_flags(const Plan& pl) {
    return (pl.stream_k ? 1 : 0) | (pl.tile_n == 128 ? 2 : 0) | (pl.tall ? 4 : 0) | (pl.csplit << 4) | (pl.bn << 8);
}
inline Plan plan_from_flags(int variant, int flags) {
    Plan pl{variant, (flags & 1) != 0, (flags & 2) ? 128 : 256, (flags >> 4) & 15, (flags >> 8) & 0xFF};
    pl.tall = (flags & 4) != 0;
    return pl;
}

// A measured configuration for one problem shape (cuasm_ffn_tune / cuasm_ffn_tuned_import).
struct TunedEntry {
    int op;  // 0 fused FFN, 1 GEMM + activation
    int64_t M, K, N;
    Plan plan;
    float us;
};

}  // namespace

struct cuasm_ffn_s {
    int device = 0;
    cuasm_dtype_t dtype = CUASM_DTYPE_BF16;
    int esize = 2;
    int sm_count = 148;
    std::string err;
    // options
    int variant = CUASM_VARIANT_AUTO;
    int use_pdl = 1;
    int group_m = 0;
    int schedule = 0;  // CUASM_OPT_SCHEDULE
    bool plan_sk = false;  // plan_config's stream-K choice for the current forward
    int trace = 0;     // CUASM_OPT_TRACE
    int tile_n = 0;    // CUASM_OPT_TILE_N (GEMM + activation): 0 auto, 128, 256
    int l2pol = 2;     // CUASM_OPT_L2_POLICY (x evict_last, W13 evict_normal)
    int csplit_opt = 0;  // CUASM_OPT_CSPLIT: 0 auto (plan), 1 off, 2..8 force a cluster split-K of that many CTAs
    int plan_csplit = 0; // plan_config's cluster split for the current launch
    int sk_split = 0;  // CUASM_OPT_SK_SPLIT: max stream-K ranges per tile when tiles < clusters (0: 2)
    int last_tile_n = 256;
    int fused_norm = 1;  // CUASM_OPT_FUSED_NORM
    uint32_t* rstate = nullptr;  // fused a1 bookkeeping: [2 * r-blocks + 1] words (self-resetting)
    int64_t rstate_words = 0;
    unsigned long long* trace_buf = nullptr;
    int trace_ctas = 0;
    // stream-K workspace
    float* ws = nullptr;
    int64_t ws_bytes = 0;
    uint32_t* flags = nullptr;
    int64_t flags_bytes = 0;
    // dynamic whole-tile claiming (dual_gemm.cuh Sched): counters + per-cluster rings, zeroed once
    uint32_t* dyn = nullptr;
    int dynamic = 0;   // CUASM_OPT_DYNAMIC: 0 auto, 1 off, 2 on
    int rs_bf16 = 0;   // CUASM_OPT_RS_PARTIAL: 0 fp32 partials, 1 bf16
    int mcast = 0;     // CUASM_OPT_MCAST: 1 = 4-CTA multicast clusters for 2-SM SwiGLU whole tiles
    int tall = 0;      // CUASM_OPT_TALL: 0 auto, 1 off, 2 on where the shape allows
    int thin = 0;      // CUASM_OPT_THIN_A: 1 = thin A stages for 64-wide decode split-K tiles (measured
                       // no faster: 16 x 4096 x 1376 16.57 vs 16.40 us, 16 x 4096 x 2752 18.51 vs 19.55)
    int mcast_clusters = 0;  // co-resident 4-CTA clusters found at the last multicast launch
    int64_t l2_persist = 0;  // CUASM_OPT_L2_PERSIST: the device's persisting-L2 set-aside this handle made
    // a1 workspace
    float* r = nullptr;
    int64_t r_cap = 0;
    // a0 caches: slot 0 = the folded, interleaved W13 of the fused FFN in 128-output
    // blocks; slot 1 = a single packed weight (GEMM + activation / down projection);
    // slots 2..6 = the same W13 in the narrower blocks BN = 112, 96, 80, 64, 120 (each packed on
    // the first forward whose plan takes that width: e.g. a decode shard's 64-wide tiles and
    // its prefill's 80-wide tiles of one weight set coexist)
    PackedWeights pw[7];
    int tile_bn = 0;   // CUASM_OPT_TILE_BN: 0 auto, else the SwiGLU outputs per tile
    // fp32 handle: x split into [x_hi | x_lo] tf32 terms per forward (pack.cuh)
    void* x2 = nullptr;
    int64_t x2_bytes = 0;
    // FFN block: the hidden activation between the two GEMMs
    void* hidden = nullptr;
    int64_t hidden_bytes = 0;
    // forward_host staging and its copy pipeline
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    std::vector<cudaEvent_t> copy_events;
    void* x_stage = nullptr;
    int64_t x_stage_bytes = 0;
    void* out_stage = nullptr;
    int64_t out_stage_bytes = 0;
    // profiling (CUASM_OPT_PROFILE)
    int profile = 0;
    std::vector<cudaEvent_t> ev_pool;   // 3 events per recorded forward
    size_t ev_used = 0;
    // last launch
    int last_variant = 0;
    int last_kernels = 0;
    EncodeTiledFn encode = nullptr;
    // host-side cache of encoded tensor maps (encode_cached): an eager forward re-encodes nothing
    // whose pointer and shape it has seen.  (An eager forward costs ~7 us of host time with the GPU
    // busy, scripts/host_queue_probe.py -- a bare cudaLaunchKernelEx with the same 2.7 KB of
    // parameters ~2.5 us, scripts/launch_param_probe.cu; with our own kernels completing
    // concurrently the same loop reads ~18 us, scripts/host_overhead.py.  CUDA graphs, which
    // bench.py and serving loops use, pay none of it.)
    TmapKey tmap_key[kTmapCache] = {};
    CUtensorMap tmap_val[kTmapCache];
    int tmap_next = 0;
    // the paper's autotuner (cuasm_ffn_tune) and deploy-time lookup:
    // measured configurations per fused-FFN shape, consulted before the cost model
    std::string gpu_name;            // cudaDeviceProp::name: part of a tuned entry's key
    std::vector<TunedEntry> tuned;
    std::vector<std::pair<Plan, float>> tune_log;  // the last cuasm_ffn_tune's candidates and times (-1: skipped)
    bool plan_forced = false;        // cuasm_ffn_tune / cuasm_gemm_act_tune: the candidate being measured
    int plan_force_op = 0;           // (of this op: 0 fused FFN, 1 GEMM + activation)
    Plan plan_force{CUASM_VARIANT_2SM, false, 256, 0, kPackBN};
};

namespace {

cuasm_status_t fail(cuasm_ffn_t h, cuasm_status_t st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (h) h->err = buf; else g_init_error = buf;
    return st;
}

cuasm_status_t cuda_fail(cuasm_ffn_t h, cudaError_t e, const char* what) {
    return fail(h, e == cudaErrorMemoryAllocation ? CUASM_ERR_OOM : CUASM_ERR_CUDA, "%s: %s (%s)", what,
                cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CUASM_CHECK(h, call, what)                        \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(h, e_, what); \
    } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cuasm_status_t check_common(cuasm_ffn_t h, int64_t K, int64_t N) {
    if (K <= 0 || N <= 0) return fail(h, CUASM_ERR_INVALID_ARG, "K and N must be positive (K=%lld N=%lld)",
                                      (long long)K, (long long)N);
    if (K % 8 != 0 || N % 8 != 0)
        return fail(h, CUASM_ERR_INVALID_ARG, "K and N must be multiples of 8 (K=%lld N=%lld)", (long long)K,
                    (long long)N);
    if (N >= (int64_t(1) << 31) || K >= (int64_t(1) << 31))
        return fail(h, CUASM_ERR_INVALID_ARG, "K, N must be < 2^31");
    return CUASM_OK;
}

cuasm_status_t check_weights(cuasm_ffn_t h, const void* g, const void* w1, const void* w3) {
    if (!g || !w1 || !w3) return fail(h, CUASM_ERR_INVALID_ARG, "NULL weight pointer");
    if (!aligned16(g) || !aligned16(w1) || !aligned16(w3))
        return fail(h, CUASM_ERR_INVALID_ARG, "weight pointers must be 16-byte aligned");
    return CUASM_OK;
}

cuasm_status_t check_eps(cuasm_ffn_t h, float eps) {
    if (!(eps >= 0.0f)) return fail(h, CUASM_ERR_INVALID_ARG, "eps must be >= 0 and not NaN");
    return CUASM_OK;
}

// Makes the handle's device current for the lifetime of the guard and restores
// the caller's current device afterwards (entry points must not leave it changed).
struct DeviceGuard {
    int prev = -1;
    cuasm_status_t status = CUASM_OK;
    explicit DeviceGuard(cuasm_ffn_t h) {
        cudaError_t e = cudaGetDevice(&prev);
        if (e != cudaSuccess) {
            prev = -1;
            status = cuda_fail(h, e, "cudaGetDevice");
            return;
        }
        if (prev != h->device && (e = cudaSetDevice(h->device)) != cudaSuccess) {
            status = cuda_fail(h, e, "cudaSetDevice");
            prev = -1;
        }
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// cudaFuncSetAttribute applies to the current device only: one bit per device
// (up to 64) per kernel instantiation, set once the attribute is applied there.
// Concurrent first calls may both apply it (harmless).
template <typename Kernel>
cuasm_status_t ensure_func_attr(cuasm_ffn_t h, Kernel kernel, std::atomic<uint64_t>& done, cudaFuncAttribute attr,
                                int value, const char* what) {
    const uint64_t bit = uint64_t(1) << (h->device & 63);
    if (done.load(std::memory_order_acquire) & bit) return CUASM_OK;
    CUASM_CHECK(h, cudaFuncSetAttribute(kernel, attr, value), what);
    done.fetch_or(bit, std::memory_order_acq_rel);
    return CUASM_OK;
}

// cuTensorMapEncodeTiled of a 2-D map through the handle's cache (TmapKey).
CUresult encode_cached(cuasm_ffn_t h, CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                       uint64_t outer, uint64_t stride_bytes, uint32_t box_inner, uint32_t box_outer,
                       CUtensorMapSwizzle swz, CUtensorMapL2promotion promo) {
    const TmapKey key{base, {inner, outer}, stride_bytes, {box_inner, box_outer}, static_cast<int>(dt),
                      static_cast<int>(swz), static_cast<int>(promo)};
    for (int i = 0; i < kTmapCache; ++i)
        if (h->tmap_key[i] == key && key.base != nullptr) {
            *map = h->tmap_val[i];
            return CUDA_SUCCESS;
        }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = h->encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
        h->tmap_key[h->tmap_next] = key;
        h->tmap_val[h->tmap_next] = *map;
        h->tmap_next = (h->tmap_next + 1) % kTmapCache;
    }
    return r;
}

cuasm_status_t encode_2d(cuasm_ffn_t h, CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint32_t box_inner, uint32_t box_outer) {
    const CUtensorMapDataType dt =
        h->dtype == CUASM_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUresult r = encode_cached(h, map, dt, base, inner, outer, inner * static_cast<uint64_t>(h->esize), box_inner,
                                     box_outer, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (r != CUDA_SUCCESS)
        return fail(h, CUASM_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d, dims %llu x %llu)", (int)r,
                    (unsigned long long)inner, (unsigned long long)outer);
    return CUASM_OK;
}

// a0: fold g (optional) into the weights and write the k-block tiled layout
// (pack.cuh) into cache slot `slot`.  w3 != null: the interleaved W13 of the
// fused FFN (128-output blocks); w3 == null: one weight, 256-row blocks.
template <typename T>
cuasm_status_t launch_pack(cuasm_ffn_t h, int slot, const void* g, const void* w1, const void* w3, int64_t K,
                           int64_t N, cudaStream_t s, int64_t kp, int bn) {
    PackedWeights& w = h->pw[slot];
    const int BK = 128 / h->esize;  // one 128-byte swizzle row of K (= GemmCfg::BK)
    const int64_t rows_per_block = w3 ? 2 * bn : 2 * kPackBN;
    const int64_t n_blocks = (N + (w3 ? bn : rows_per_block) - 1) / (w3 ? bn : rows_per_block);
    const int64_t k_blocks = kp > 0 ? 2 * kp / BK : (K + BK - 1) / BK;
    const int64_t rows = n_blocks * k_blocks * rows_per_block;
    const int64_t bytes = rows * 128;
    if (bytes > w.bytes) {
        if (w.buf) cudaFree(w.buf);
        w.buf = nullptr;
        w.bytes = 0;
        CUASM_CHECK(h, cudaMalloc(&w.buf, bytes), "cudaMalloc(packed weights)");
        w.bytes = bytes;
    }
    const int64_t total_vec = bytes / 16;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total_vec + threads - 1) / threads, int64_t(h->sm_count) * 16);
    cuasm::ffn_pack_kernel<T><<<static_cast<unsigned>(blocks), threads, 0, s>>>(
        static_cast<const T*>(w1), static_cast<const T*>(w3), static_cast<const T*>(g), static_cast<T*>(w.buf), N, K,
        w3 ? bn : kPackBN, n_blocks, k_blocks, BK, kp);
    CUASM_CHECK(h, cudaGetLastError(), "ffn_pack_kernel launch");
    w.rows = rows;
    w.tmap_rows = 0;  // re-encode for the new buffer
    w.key_g = g;
    w.key_w1 = w1;
    w.key_w3 = w3;
    w.key_K = K;
    w.key_N = N;
    w.key_kp = kp;
    w.key_bn = bn;
    w.packed = true;
    w.fresh = true;
    return CUASM_OK;
}

// The W13 cache slot of a SwiGLU tile width: 0 for BN = 128, 2..6 for 112, 96, 80, 64, 120.
inline int w13_slot(int bn) {
    return bn == 112 ? 2 : bn == 96 ? 3 : bn == 80 ? 4 : bn == 64 ? 5 : bn == 120 ? 6 : 0;
}

cuasm_status_t ensure_packed(cuasm_ffn_t h, int slot, const void* g, const void* w1, const void* w3, int64_t K,
                             int64_t N, cudaStream_t s, int64_t kp = 0, int bn = kPackBN) {
    PackedWeights& w = h->pw[slot];
    if (w.packed && w.key_g == g && w.key_w1 == w1 && w.key_w3 == w3 && w.key_K == K && w.key_N == N &&
        w.key_kp == kp && w.key_bn == bn)
        return CUASM_OK;
    w.packed = false;
    return h->dtype == CUASM_DTYPE_BF16 ? launch_pack<__nv_bfloat16>(h, slot, g, w1, w3, K, N, s, kp, bn)
                                        : launch_pack<float>(h, slot, g, w1, w3, K, N, s, kp, bn);
}

// fp32 handles: the K padding of the split-x contraction (one 32-float k-block)
inline int64_t split_kp(int64_t K) { return (K + 31) / 32 * 32; }

template <typename T>
cuasm_status_t launch_prepass(cuasm_ffn_t h, const void* x, float* r, int64_t M, int64_t K, float eps,
                              cudaStream_t s) {
    // Same L1/smem split as the dual GEMM (max shared): an SM running
    // pre-pass CTAs can then take the PDL-launched GEMM CTA without a
    // carveout reconfiguration, so the two kernels actually overlap.
    static std::atomic<uint64_t> attr_done{0};
    cuasm_status_t st = ensure_func_attr(h, cuasm::ffn_rms_prepass_kernel<T>, attr_done,
                                         cudaFuncAttributePreferredSharedMemoryCarveout,
                                         static_cast<int>(cudaSharedmemCarveoutMaxShared),
                                         "cudaFuncSetAttribute(prepass carveout)");
    if (st != CUASM_OK) return st;
    const int64_t blocks = (M + cuasm::kPrepassRowsPerBlock - 1) / cuasm::kPrepassRowsPerBlock;
    cuasm::ffn_rms_prepass_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, s>>>(static_cast<const T*>(x), r, M, K,
                                                                                    eps);
    CUASM_CHECK(h, cudaGetLastError(), "ffn_rms_prepass_kernel launch");
    return CUASM_OK;
}

cuasm_status_t prepass(cuasm_ffn_t h, const void* x, float* r, int64_t M, int64_t K, float eps, cudaStream_t s) {
    return h->dtype == CUASM_DTYPE_BF16 ? launch_prepass<__nv_bfloat16>(h, x, r, M, K, eps, s)
                                        : launch_prepass<float>(h, x, r, M, K, eps, s);
}

// What one dual-GEMM launch computes (FfnGemmParams fields the host sets).
struct EpiSpec {
    int slot;        // packed-weight cache slot (0: W13, 1: single weight)
    int fused_norm;  // compute r in-kernel
    int use_r;       // scale by r
    int act;         // kEpi == 1: 0 identity, 1 LeakyReLU
    float alpha;
    // a4 fused gather (cuasm_ffn_forward_gather): null = the plain output `out`, ldo = N
    void* const* dst = nullptr;
    int num_dst = 0;
    int dst_mc = 0;
    int64_t ldo = 0;
    // fp32 split-x contraction (kp > 0): the pre-pass is ffn_split_tf32_kernel over the
    // caller's x_src [M, k_src], writing r and the GEMM operand x = [x_hi | x_lo] [M, 2 kp]
    const void* x_src = nullptr;
    int64_t k_src = 0;
    int64_t kp = 0;
    // f1 fused reduce-scatter (GEMM mode): stage[q] = rank q's fp32 staging buffer, this
    // launch's partial tiles go to their owner's slot `rs_rank` (dual_gemm.cuh rs_owner)
    void* const* rs_stage = nullptr;
    int rs_world = 0;
    int rs_rank = 0;
};

// f1 ownership: rank q reduces the output columns [col0, col1) (256-column blocks split
// evenly, dual_gemm.cuh rs_owner / rs_col0); its staging buffer is [world][M][col1 - col0] fp32.
void rs_cols(int64_t K, int world, int q, int64_t& col0, int64_t& col1) {
    const int nblk = static_cast<int>((K + 255) / 256);
    col0 = cuasm::rs_col0(q, nblk, world);
    col1 = std::min<int64_t>(K, cuasm::rs_col0(q + 1, nblk, world));
    if (col1 < col0) col1 = col0;
}

// Few-tile decode shapes: at most this many 1-SM tiles take the 1-SM variant with
// each tile split this many ways (plan_config_raw, launch_gemm).
constexpr int64_t kFewTiles = 32;
constexpr int kFewTilesSplit = 3;

// Rasterisation group (m-blocks whose tiles run before the next W13 column
// block): as many as keep the group's rows of x within ~32 MB of L2, at most
// 16.  x of a group is re-read once per n-block and must stay L2-resident; a
// 70B group of 16 (64 MB of x) measured 2.6% slower than 8 (32 MB), ncu
// showing 6.6 GB of DRAM reads per launch for 1.0 GB of operands
// (scripts/tune_group.py, profiles/r01/tune_group.log).
inline int auto_group_m(int64_t K, int esize, int cta_group) {
    const int64_t per_mblk = static_cast<int64_t>(128) * cta_group * K * esize;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(16, (int64_t(32) << 20) / per_mblk)));
}

// kTall: tall tiles (dual_gemm.cuh GemmCfg; 257..384 rows, 2-SM bf16 SwiGLU, whole tiles)
template <int kKind, int kCtaGroup, int kEpi, int kN, bool kThin = false, bool kTall = false>
cuasm_status_t launch_gemm(cuasm_ffn_t h, const EpiSpec& e, const void* x, void* out, int64_t M, int64_t K,
                           int64_t N, float eps, cudaStream_t s) {
    using C = GemmCfg<kKind, kCtaGroup, kEpi, kN, kThin, kTall>;
    static_assert(!kTall || kEpi == 0, "tall tiles: fused FFN");
    if (kTall && (M <= 256 || M > C::TILE_M))
        return fail(h, CUASM_ERR_UNSUPPORTED, "tall tiles need 256 < M <= %d", C::TILE_M);
    PackedWeights& w = h->pw[e.slot];
    CUtensorMap tmap_x;
    // A single row block with fewer than BM rows loads only the rows that exist
    // (rounded up to 8): the MMA rows beyond them read stale smem, but row m of
    // the product depends only on row m of x and rows >= M are never stored.
    // Measured: a 128-row box over an 8-row x streams the weights ~30% slower
    // than over a 16-row x (profiles/r01/trace_small_m.log).
    // decode shapes (SwiGLU, M <= 32, either variant): the rows are replicated over
    // the four TMEM lane quadrants of the (leader) CTA (dual_gemm.cuh `rep`)
    // cluster split-K (1-SM; dual_gemm.cuh split_k_reduce): S CTAs per tile, one tile per cluster
    int csplit = 0;
    if (kCtaGroup == 1 && C::kDecodePaths) {
        const int want = h->csplit_opt >= 2 ? h->csplit_opt : (h->csplit_opt == 0 ? h->plan_csplit : 0);
        const int64_t tiles = ((M + C::TILE_M - 1) / C::TILE_M) * ((N + C::OUT_COLS - 1) / C::OUT_COLS);
        const int64_t kbs = (K + C::BK - 1) / C::BK;
        if (want >= 2 && want <= 8 && tiles * want <= h->sm_count && kbs >= want && e.rs_world == 0) csplit = want;
    }
    const int rep_plain = (kEpi != 0 || !C::kDecodePaths || kThin) ? 0 : M <= 32 ? 4 : M <= 64 ? 2 : 0;
    const int rep = csplit ? 0 : rep_plain;
    const uint32_t a_rows =
        ((kCtaGroup == 1 || rep) && M < C::BM) ? static_cast<uint32_t>((M + 7) / 8 * 8) : C::BM;
    cuasm_status_t st = encode_2d(h, &tmap_x, x, static_cast<uint64_t>(K), static_cast<uint64_t>(M), C::BK, a_rows);
    if (st != CUASM_OK) return st;
    // tall tiles: x again with 64-row boxes (the 128-row part's rows per CTA); the other kernels
    // take tmap_x in this slot and never use it
    CUtensorMap tmap_xh = tmap_x;
    if constexpr (kTall) {
        st = encode_2d(h, &tmap_xh, x, static_cast<uint64_t>(K), static_cast<uint64_t>(M), C::BK, C::HALF_ROWS);
        if (st != CUASM_OK) return st;
    }
    if (w.tmap_rows != C::B_ROWS) {
        st = encode_2d(h, &w.tmap, w.buf, static_cast<uint64_t>(C::BK), static_cast<uint64_t>(w.rows), C::BK,
                       C::B_ROWS);
        if (st != CUASM_OK) return st;
        w.tmap_rows = C::B_ROWS;
    }
    FfnGemmParams p;
    p.x = x;
    p.eps = eps;
    p.fused_norm = e.fused_norm;
    p.use_r = e.use_r;
    p.act = e.act;
    p.alpha = e.alpha;
    p.rstate = h->rstate;
    p.n_rblk = static_cast<int>((M + 127) / 128);
    p.r = h->r;
    p.out = out;
    p.ldo = N;
    p.num_dst = 1;
    p.dst_mc = 0;
    for (int q = 0; q < 8; ++q) p.dst[q] = nullptr;
    p.dst[0] = out;
    if (e.dst) {
        p.ldo = e.ldo;
        p.num_dst = e.num_dst;
        p.dst_mc = e.dst_mc;
        for (int q = 0; q < e.num_dst; ++q) p.dst[q] = e.dst[q];
    }
    p.M = static_cast<int>(M);
    p.N = static_cast<int>(N);
    p.K = static_cast<int>(K);
    p.num_m_blk = static_cast<int>((M + C::TILE_M - 1) / C::TILE_M);
    p.num_n_blk = static_cast<int>((N + C::OUT_COLS - 1) / C::OUT_COLS);
    p.num_k_blk = static_cast<int>((K + C::BK - 1) / C::BK);
    p.group_m = h->group_m > 0 ? h->group_m : auto_group_m(K, h->esize, kCtaGroup);
    // with a persisting-L2 set-aside that holds all of x (CUASM_OPT_L2_PERSIST; x loads are
    // evict_last), one group of every m-block reads each W13 block from HBM once: 70B FFN
    // 2.54 -> 1.55 GB of DRAM traffic per launch (profiles/r02/l2_persist/)
    if (h->group_m == 0 && h->l2_persist > 0 && M * K * h->esize * 20 <= h->l2_persist * 19)
        p.group_m = std::numeric_limits<int>::max();
    p.group_m = std::max(1, std::min(p.group_m, p.num_m_blk));
    p.num_tiles = p.num_m_blk * p.num_n_blk;
    p.a_box_bytes = static_cast<int>(a_rows) * 128;
    p.l2pol = h->l2pol;
    // weights packed before an earlier GEMM launch on this stream (which waited for the
    // pack) are safe to load before griddepcontrol.wait; the first GEMM after a pack is not
    p.w_early = w.fresh ? 0 : 1;
    w.fresh = false;
    // bf16 output with one destination leaves through TMA stores: a 2-D map over the
    // destination [M rows, ldo stride] x N columns, 32 x 32 boxes, 64-byte swizzle
    // (what the epilogue's staging layout writes); stores past M / N are clipped
    // (one map per destination: the fused gather's P2P fan-out is P TMA stores per box)
    // (tiles whose last SwiGLU unit is narrower -- BN % 32 = 16 or 24 -- store it through a
    // second set of maps: 32 x 16 boxes with 32-byte swizzle, or 32 x 24 boxes unswizzled)
    cuasm::OutMaps omaps{}, omaps_h{};
    p.tma_store = (kKind == 0 && !p.dst_mc) ? 1 : 0;
    constexpr bool kHalfUnit = kEpi == 0 && C::BN % 32 != 0;
    constexpr uint32_t kNarrowW = C::BN % 32 == 0 ? 32 : C::BN % 32;
    p.rs_world = 0;
    p.rs_bf16 = 0;
    p.rs_nblk = static_cast<int>((N + 255) / 256);
    if (e.rs_world > 0) {
        // f1: one fp32 map per owner rank q over its staging slot for this rank,
        // stage[q] + rs_rank * M * Kq floats, [M, Kq], 32 x 16 boxes (64-byte rows, 64-byte swizzle)
        if (kKind != 0 || kEpi != 1) return fail(h, CUASM_ERR_UNSUPPORTED, "fused reduce-scatter: bf16 GEMM only");
        p.rs_world = e.rs_world;
        p.rs_bf16 = h->rs_bf16;
        p.num_dst = 0;
        const int pes = h->rs_bf16 ? 2 : 4;  // partial element size
        for (int q = 0; q < e.rs_world; ++q) {
            int64_t c0, c1;
            rs_cols(N, e.rs_world, q, c0, c1);
            const int64_t kq = c1 - c0;
            if (kq == 0) continue;  // owns no columns: no tile is ever sent there
            void* base = static_cast<char*>(e.rs_stage[q]) + static_cast<int64_t>(e.rs_rank) * M * kq * pes;
            // (64-byte box rows either way)
            CUresult r = encode_cached(h, &omaps.m[q], h->rs_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                       base, static_cast<uint64_t>(kq), static_cast<uint64_t>(M),
                                       static_cast<uint64_t>(kq) * pes, h->rs_bf16 ? 32u : 16u, 32, CU_TENSOR_MAP_SWIZZLE_64B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE);
            if (r != CUDA_SUCCESS)
                return fail(h, CUASM_ERR_CUDA, "cuTensorMapEncodeTiled(stage %d) failed (CUresult %d)", q, (int)r);
        }
    }
    for (int q = 0; p.tma_store && q < p.num_dst; ++q) {
        for (int hw = 0; hw < (kHalfUnit ? 2 : 1); ++hw) {
            CUresult r = encode_cached(h, hw ? &omaps_h.m[q] : &omaps.m[q], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p.dst[q],
                                       static_cast<uint64_t>(N), static_cast<uint64_t>(M),
                                       static_cast<uint64_t>(p.ldo) * static_cast<uint64_t>(h->esize), hw ? kNarrowW : 32u, 32,
                                       hw ? (kNarrowW == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE)
                                          : CU_TENSOR_MAP_SWIZZLE_64B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE);
            if (r != CUDA_SUCCESS)
                return fail(h, CUASM_ERR_CUDA, "cuTensorMapEncodeTiled(out %d) failed (CUresult %d)", q, (int)r);
        }
    }
    // decode shapes: replicate the <= 32 rows into all four TMEM lane quadrants so
    // the SwiGLU epilogue runs on all four SM sub-partitions (dual_gemm.cuh `rep`)
    p.rep = rep;
    p.csplit = csplit;

    static std::atomic<uint64_t> attr_done{0};  // per template instance, one bit per device
    st = ensure_func_attr(h, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, false, kThin, kTall>, attr_done,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES, "cudaFuncSetAttribute(smem)");
    if (st != CUASM_OK) return st;
    // dynamic tile claiming is compiled into the 2-SM bf16 kernels only (the long runs it is for)
    constexpr bool kDynBuilt = kCtaGroup == 2 && kKind == 0 && !kThin && !kTall;
    if constexpr (kDynBuilt) {
        static std::atomic<uint64_t> attr_done_dyn{0};
        st = ensure_func_attr(h, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, true>, attr_done_dyn,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES,
                              "cudaFuncSetAttribute(smem)");
        if (st != CUASM_OK) return st;
    }
    if (csplit) {
        // one wave: every cluster must fit at once, or the split loses to a second wave
        // (clusters are placed inside one GPC, so S-CTA clusters may not all fit: S = 8
        // over 16 tiles did not); correctness does not depend on it (no inter-cluster waits)
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(static_cast<unsigned>(p.num_tiles * csplit), 1, 1);
        qc.blockDim = dim3(C::NUM_THREADS, 1, 1);
        qc.dynamicSmemBytes = C::SMEM_BYTES;
        cudaLaunchAttribute qa;
        qa.id = cudaLaunchAttributeClusterDimension;
        qa.val.clusterDim.x = static_cast<unsigned>(csplit);
        qa.val.clusterDim.y = 1;
        qa.val.clusterDim.z = 1;
        qc.attrs = &qa;
        qc.numAttrs = 1;
        int max_active = 0;
        if (cudaOccupancyMaxActiveClusters(&max_active, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, false, kThin, kTall>, &qc) !=
                cudaSuccess ||
            max_active < p.num_tiles) {
            (void)cudaGetLastError();
            csplit = 0;
            p.csplit = 0;
            p.rep = rep_plain;
        }
    }
    // 4-CTA multicast clusters (CUASM_OPT_MCAST, DESIGN.md §6 "Multicast clusters"): two CTA pairs
    // per cluster on two vertically adjacent tiles of one n-block, the W13 halves loaded once and
    // multicast to both; whole tiles only (super-tiles of 512 rows round-robin over the clusters)
    if constexpr (kDynBuilt && kEpi == 0) {
        if (h->mcast && !csplit && p.num_m_blk >= 2) {
            static std::atomic<uint64_t> attr_done_mc{0};
            st = ensure_func_attr(h, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, true>, attr_done_mc,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES,
                                  "cudaFuncSetAttribute(smem)");
            if (st != CUASM_OK) return st;
            p.num_m_blk = (p.num_m_blk + 1) / 2;  // super-rows of two 256-row tiles
            p.group_m = std::max(1, std::min((p.group_m + 1) / 2, p.num_m_blk));
            p.num_tiles = p.num_m_blk * p.num_n_blk;
            // clusters are placed inside one GPC: fewer 4-CTA clusters than sm_count / 4 may fit at
            // once, and a persistent grid must not exceed what is co-resident (a late cluster would
            // run its share after everybody else)
            int fit4 = h->sm_count / 4;
            {
                cudaLaunchConfig_t qc = {};
                qc.gridDim = dim3(static_cast<unsigned>(4 * fit4), 1, 1);
                qc.blockDim = dim3(C::NUM_THREADS, 1, 1);
                qc.dynamicSmemBytes = C::SMEM_BYTES;
                cudaLaunchAttribute qa;
                qa.id = cudaLaunchAttributeClusterDimension;
                qa.val.clusterDim.x = 4;
                qa.val.clusterDim.y = 1;
                qa.val.clusterDim.z = 1;
                qc.attrs = &qa;
                qc.numAttrs = 1;
                int active = 0;
                if (cudaOccupancyMaxActiveClusters(&active, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, true>,
                                                   &qc) == cudaSuccess && active > 0)
                    fit4 = std::min(fit4, active);
                (void)cudaGetLastError();
            }
            h->mcast_clusters = fit4;
            const int clusters4 = std::min(p.num_tiles, fit4);
            p.num_clusters = clusters4;
            p.num_dp_tiles = p.num_tiles;
            p.sk_iters = 0;
            p.ws = h->ws;
            p.flags = h->flags;
            p.dyn = nullptr;
            p.trace = nullptr;
            if (h->trace) {
                p.trace = h->trace_buf;
                h->trace_ctas = clusters4 * 4;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(clusters4 * 4), 1, 1);
            cfg.blockDim = dim3(C::NUM_THREADS, 1, 1);
            cfg.dynamicSmemBytes = C::SMEM_BYTES;
            cfg.stream = s;
            cudaLaunchAttribute attrs[2];
            int na = 0;
            attrs[na].id = cudaLaunchAttributeClusterDimension;
            attrs[na].val.clusterDim.x = 4;
            attrs[na].val.clusterDim.y = 1;
            attrs[na].val.clusterDim.z = 1;
            ++na;
            if (h->use_pdl && !h->profile) {
                attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attrs[na].val.programmaticStreamSerializationAllowed = 1;
                ++na;
            }
            cfg.attrs = attrs;
            cfg.numAttrs = na;
            CUASM_CHECK(h, cudaLaunchKernelEx(&cfg, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, true>,
                                              tmap_x, w.tmap, tmap_xh, omaps, omaps_h, p),
                        "ffn_dual_gemm_kernel launch (multicast clusters)");
            h->last_variant = CUASM_VARIANT_2SM;
            return CUASM_OK;
        }
    }
    const int max_clusters = h->sm_count / kCtaGroup;
    // Persistent schedule (DESIGN.md §6 "Stream-K"): whole tiles round-robin
    // while they fill complete waves; the last partial wave plus one full
    // wave (or everything, when there are fewer tiles than clusters) is split
    // into equal contiguous k-block ranges so every cluster finishes together.
    int clusters = std::min(p.num_tiles, max_clusters);
    int sk_tiles = 0;
    const int waves = p.num_tiles / max_clusters, rem = p.num_tiles % max_clusters;
    // Stream-K only where plan_config's cost model says the balanced tail is
    // worth the partial fixup (e.g. 7B prefill: 9.3 waves; not decode, where
    // whole tiles already saturate HBM).
    const bool sk_ok = !kTall && !csplit && (h->schedule == CUASM_SCHEDULE_STREAM_K_ALL ||
                                   h->schedule == CUASM_SCHEDULE_STREAM_K_TAIL ||
                                   (h->schedule == CUASM_SCHEDULE_AUTO && h->plan_sk));
    if (sk_ok && p.num_k_blk > 1) {
        if (h->schedule == CUASM_SCHEDULE_STREAM_K_ALL) sk_tiles = p.num_tiles;
        else if (rem != 0 && h->schedule == CUASM_SCHEDULE_STREAM_K_TAIL) sk_tiles = waves == 0 ? p.num_tiles : rem;
        else if (rem != 0) sk_tiles = waves == 0 ? p.num_tiles : rem + max_clusters;
        // every cluster gets a non-empty range (tiny problems: fewer clusters); in
        // auto mode a tile is split at most in two when there are fewer tiles
        // than clusters (each finisher then adds a single partial)
        if (sk_tiles > 0) {
            int64_t c = std::min<int64_t>(max_clusters, static_cast<int64_t>(sk_tiles) * p.num_k_blk);
            if (waves == 0 && (h->schedule == CUASM_SCHEDULE_AUTO || h->sk_split > 0)) {
                const int split = h->sk_split > 0 ? h->sk_split : (p.num_tiles <= kFewTiles ? kFewTilesSplit : 2);
                c = std::min<int64_t>(c, static_cast<int64_t>(split) * sk_tiles);
            }
            clusters = static_cast<int>(c);
        }
    }
    // the kernel's stream-K arithmetic is 32-bit (dual_gemm.cuh sk_begin): keep
    // sk_iters * clusters below 2^32, else whole tiles only
    if (static_cast<uint64_t>(sk_tiles) * p.num_k_blk * static_cast<uint64_t>(clusters) >= (uint64_t(1) << 32)) {
        sk_tiles = 0;
        clusters = std::min(p.num_tiles, max_clusters);
    }
    p.num_clusters = clusters;
    p.num_dp_tiles = p.num_tiles - sk_tiles;
    p.sk_iters = static_cast<int64_t>(sk_tiles) * p.num_k_blk;
    if (sk_tiles > 0) {
        const int64_t ws_need = static_cast<int64_t>(clusters) * kCtaGroup * C::WS_SLOT_F4 * 16;
        const int64_t fl_need = static_cast<int64_t>(clusters) * kCtaGroup * C::NUM_EPI_WARPS * 4;
        if (ws_need > h->ws_bytes) {
            if (h->ws) cudaFree(h->ws);
            h->ws = nullptr;
            h->ws_bytes = 0;
            CUASM_CHECK(h, cudaMalloc(&h->ws, ws_need), "cudaMalloc(stream-K workspace)");
            h->ws_bytes = ws_need;
        }
        if (fl_need > h->flags_bytes) {
            if (h->flags) cudaFree(h->flags);
            h->flags = nullptr;
            h->flags_bytes = 0;
            CUASM_CHECK(h, cudaMalloc(&h->flags, fl_need), "cudaMalloc(stream-K flags)");
            CUASM_CHECK(h, cudaMemset(h->flags, 0, fl_need), "cudaMemset(flags)");
            h->flags_bytes = fl_need;
        }
    }
    p.ws = h->ws;
    p.flags = h->flags;
    // Dynamic claiming of the data-parallel tiles (DESIGN.md §6 "Dynamic tiles"): auto for long
    // runs of whole tiles (>= kDynRounds per cluster: the 70B FFN's 55 rounds, where static
    // round-robin pairs drift apart by rounds and the tiles in flight stop sharing L2 --
    // 4.43 -> 2.51 GB of DRAM reads per launch, 2528 -> 2449 us); with few rounds the claims
    // made ahead cost more balance at the end than they save (70B P=8, 6.9 rounds: 286.7 ->
    // 294.9 us); forced on or off by CUASM_OPT_DYNAMIC; never for cluster split-K
    constexpr int kDynRounds = 24;
    p.dyn = nullptr;
    const bool dyn_on = kDynBuilt && !csplit && p.num_dp_tiles > clusters &&
                        (h->dynamic == 2 || (h->dynamic == 0 && p.num_dp_tiles >= kDynRounds * clusters));
    if (dyn_on) {
        if (!h->dyn) {
            const size_t words = 4 + static_cast<size_t>(h->sm_count) * cuasm::kDynRing * 2;
            CUASM_CHECK(h, cudaMalloc(&h->dyn, words * 4), "cudaMalloc(dynamic schedule)");
            CUASM_CHECK(h, cudaMemset(h->dyn, 0, words * 4), "cudaMemset(dynamic schedule)");
        }
        p.dyn = h->dyn;
    }
    p.trace = nullptr;
    if (h->trace) {
        p.trace = h->trace_buf;
        h->trace_ctas = clusters * (csplit ? csplit : kCtaGroup);
    }

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * (csplit ? csplit : kCtaGroup)), 1, 1);
    cfg.blockDim = dim3(C::NUM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    int na = 0;
    if (kCtaGroup == 2 || csplit) {
        attrs[na].id = cudaLaunchAttributeClusterDimension;
        attrs[na].val.clusterDim.x = csplit ? csplit : 2;
        attrs[na].val.clusterDim.y = 1;
        attrs[na].val.clusterDim.z = 1;
        ++na;
    }
    if (h->use_pdl && !h->profile) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    if constexpr (kDynBuilt) {
        if (p.dyn) {
            CUASM_CHECK(h, cudaLaunchKernelEx(&cfg, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, true>, tmap_x,
                                              w.tmap, tmap_xh, omaps, omaps_h, p),
                        "ffn_dual_gemm_kernel launch");
            h->last_variant = CUASM_VARIANT_2SM;
            return CUASM_OK;
        }
    }
    CUASM_CHECK(h, cudaLaunchKernelEx(&cfg, cuasm::ffn_dual_gemm_kernel<kKind, kCtaGroup, kEpi, kN, false, false, kThin, kTall>,
                                      tmap_x, w.tmap, tmap_xh, omaps, omaps_h, p),
                "ffn_dual_gemm_kernel launch");
    h->last_variant = kCtaGroup == 1 ? CUASM_VARIANT_1SM : CUASM_VARIANT_2SM;
    return CUASM_OK;
}

// Shape-keyed configuration (DESIGN.md §6 "Configuration model"): the paper's
// autotuner step done once, offline, and folded into a cost model.
// Per candidate (variant, schedule) the mainloop time is the number of tile
// rounds (data-parallel) or the exact wave count plus a fixed stream-K fixup
// (partial write/read + finisher epilogue tail), in units of one k-block of
// one tile; the 1-SM tile pays its measured 16% smem-bandwidth penalty; and
// every candidate is floored by the HBM time of streaming the weights once.
// Constants were fitted to scripts/tune.py on a B200 (profiles/r01/tune.json):
// t_kb = 0.37 us per k-block-tile at the power-capped clock, fixup = 10 us,
// stream-K L2-overflow slowdown 1.32x (profiles/r01/trace_gemm.log).

// Time of one k-block of a 2-SM SwiGLU tile of width bn relative to bn = 128, measured
// (scripts/tune_bn.py, profiles/r02/tune_bn.json): at full size the narrower tiles run at
// about their MMA-width ratio (7B prefill, 11 rounds of 112-wide tiles 218.9 us vs 10 of
// 128-wide 229.6 us: 0.87); at 80 and below the per-k-block issue / barrier / operand
// overheads that do not shrink with bn show (2048 x 4096 x 1376: 80 -> 0.70, 64 -> 0.62); 120
// (MMA N = 240) fills 7B's N = 11008 with 92 blocks: 736 tiles = 9.95 rounds of 74 pairs,
// 217.4 us vs 223.8 (112) and 224.5 (128, stream-K) on one box -> 0.925
inline double bn_frac(int bn) {
    return bn >= 128 ? 1.0 : bn >= 120 ? 0.925 : bn >= 112 ? 0.867 : bn >= 96 ? 0.80 : bn >= 80 ? 0.70 : 0.62;
}

Plan plan_config_raw(int sm_count, int esize, int group_m, int64_t M, int64_t K, int64_t N, int64_t out_cols,
                     int tile_n_force = 0, int tile_bn_force = 0, int tall_opt = 0) {
    const double t_kb = 0.37e-6, fixup = 10e-6, hbm = 6.5e12, pen_1sm = 1.16;
    const int64_t BK = 128 / esize;
    const double KB = static_cast<double>((K + BK - 1) / BK);
    const int64_t nblk = (N + out_cols - 1) / out_cols;
    const double w_elems = out_cols == 128 ? 2.0 * N * K : 1.0 * N * K;  // W1+W3, or one weight
    const double hbm_floor = (w_elems + static_cast<double>(M) * K + static_cast<double>(M) * N) * esize / hbm;
    // Decode-like SwiGLU shapes with few tiles (M <= 256, <= kFewTiles 1-SM tiles: the
    // tensor-parallel decode shards): weight streaming and the partial fixup decide,
    // not the tensor pipe, and the 1-SM variant split kFewTilesSplit ways measured
    // best (16 x 4096 x 1376: 22.6 us vs 24.6 us for the 2-SM split in two;
    // scripts/tune_split.py, profiles/r01/tune_split.json)
    // (up to twice as many tiles, M <= 512: split two ways; 16 x 4096 x 5504: 30.7 vs
    // 32.8 us, 512 x 4096 x 1376: 28.8 vs 30.7 us)
    const int64_t tiles_1sm = ((M + 127) / 128) * nblk;
    // tall tiles (256 < M <= 384, bf16 SwiGLU): forced on, or a candidate of the cost model below
    const bool tall_ok = out_cols == 128 && esize == 2 && M > 256 && M <= kTallMaxM && tall_opt != 1 &&
                         (tile_bn_force == 0 || tile_bn_force == kTallBN);
    if (tall_ok && tall_opt == 2) return Plan{CUASM_VARIANT_2SM, false, 256, 0, kTallBN, true};
    // (a forced SwiGLU width below 128 has no decode paths: straight to the cost model)
    const bool narrow_forced = out_cols == 128 && tile_bn_force != 0 && tile_bn_force != kPackBN;
    // Decode shards (M <= 32, up to 2 * kFewTiles tiles): split each tile's k-loop over a
    // cluster of S CTAs, partials pushed into the owner CTA's shared memory (dual_gemm.cuh
    // split_k_push) -- no global partials, no flags, no second wave.  S = 6 up to 16 tiles
    // at M <= 16, 4 up to 37 tiles, 3 up to 49 (M <= 16: the 3-way slots fit the staging
    // area), else 2 up to 64.  Kernel times under ncu (profiles/r01/csplit/): 16 x 4096 x
    // 1376: 14.5 us (S = 6), 15.0 (S = 4) vs 17.5 us (stream-K split 3 ways), 16 x 4096 x 5504
    // (S = 3): 23.0 vs 27.1, 16 x 4096 x 6880 (S = 2): 26.5 vs 29.5, 32 x 4096 x 5504 (S = 2):
    // 24.9 vs 27.2; at M >= 64 (pull form) it loses
    // With 64-output tiles (the 1-SM kernel's decode paths exist for BN = 64 too) a shard has
    // twice the tiles, so a split of 3 (2) puts up to 147 CTAs on the weight stream while each
    // owner reduces half the columns: 16 x 4096 x 1376 24.3 -> 22.0 us, 16 x 4096 x 2752
    // 25.4 -> 23.6, 16 x 8192 x 3584 31.3 -> 30.7 (scripts/tune_decode_bn.py,
    // profiles/r02/tune_decode_bn.log); wider shards keep the 128-output rule below
    const int64_t tiles_64 = ((M + 127) / 128) * ((N + 63) / 64);
    if (out_cols == 128 && esize == 2 && (tile_bn_force == 0 || tile_bn_force == 64) && KB >= 48 && M <= 32 &&
        tiles_64 * 2 <= sm_count)
        return Plan{CUASM_VARIANT_1SM, false, 256, tiles_64 * 3 <= sm_count ? 3 : 2, 64};
    if (out_cols == 128 && !narrow_forced && KB >= 48 && M <= 32) {
        const int S = M <= 16 && tiles_1sm * 6 <= sm_count && tiles_1sm <= 16 ? 6
                      : tiles_1sm * 4 <= sm_count && tiles_1sm <= 37   ? 4
                      : M <= 16 && tiles_1sm * 3 <= sm_count && tiles_1sm <= 49 ? 3
                      : tiles_1sm * 2 <= sm_count && tiles_1sm <= 2 * kFewTiles ? 2
                                                                                : 0;
        if (S) return Plan{CUASM_VARIANT_1SM, false, 256, S};
    }
    // (k-loops of >= 48 k-blocks: a split must save more MMA time than its partial fixup costs;
    // the paper's fused_ff shape 512 x 2048 x 512 split three ways finished its tail 5 us late)
    const bool few_tiles = KB >= 48 && ((M <= 256 && tiles_1sm <= kFewTiles) || (M <= 512 && tiles_1sm <= 2 * kFewTiles));
    // Small-M tensor-parallel shards (32 < M <= 512, few tiles), bf16: the autotuner over K = 4096 /
    // 8192, N_l = 1376..7168, M = 48..512 (scripts/tune_grid.py, profiles/r02/tune/grid.json) beat the
    // 1-SM stream-K tile below by 5-20% with (a) M <= 128: the cluster split-K on 64-output 1-SM tiles
    // (pull form; 3 ways when <= 32 tiles, else 2): 48 x 4096 x 1376 21.9 -> 18.2 us, 128 x 8192 x
    // 3584 36.5 -> 33.8; (b) 2-SM 64-output tiles split in k (stream-K) when they fill at most half the
    // CTA pairs: 192 x 4096 x 1376 25.2 -> 21.2; (c) else 2-SM 80-output whole tiles: 256 x 4096 x
    // 2752 28.6 -> 24.4, 512 x 4096 x 1376 28.0 -> 24.3 -- when those fit one round of the pairs;
    // otherwise the cost model below (48 x 8192 x 7168: 2-SM 112-wide, 48.5 vs 48.4 us)
    const bool small_m_shard = out_cols == 128 && esize == 2 && !narrow_forced && few_tiles && M > 32;
    if (small_m_shard) {
        // (a split of 4, else 2: their partials fit the push form's 64 KB of slots on this tile --
        // 48 / 96 / 128 x 4096 x 1376 22.5 / 22.5 / 22.9 (pull, S = 3) -> 18.5 / 18.9 / 20.5 us,
        // 128 x 8192 x 3584 34.8 -> 32.8, profiles/r02/push64/; with more m-blocks while a split of 2
        // still fits the SMs: 192 / 384 x 4096 x 1376 21.9 / 23.9 -> 20.5 / 21.6, grid.json)
        // (3 ways where 4 do not fit and the 3-way slots do, <= 64 rows: 48 x 4096 x 2752 21.1 -> 19.9)
        if (tiles_64 * 2 <= sm_count)
            return Plan{CUASM_VARIANT_1SM, false, 256,
                        tiles_64 * 4 <= sm_count ? 4 : (M <= 64 && tiles_64 * 3 <= sm_count) ? 3 : 2, 64};
        const int64_t mblk_2sm = (M + 255) / 256;
        if (mblk_2sm * ((N + 63) / 64) * 2 <= sm_count / 2) return Plan{CUASM_VARIANT_2SM, true, 256, 0, 64};
        if (mblk_2sm * ((N + 79) / 80) <= sm_count / 2) return Plan{CUASM_VARIANT_2SM, false, 256, 0, 80};
    }
    if (out_cols == 128 && !narrow_forced && few_tiles && !small_m_shard) return Plan{CUASM_VARIANT_1SM, true, 256, 0};
    // Short k-loops whose 128-wide 2-SM tiles fit one wave of the CTA pairs (GEMM mode, e.g. the
    // paper's mmLeakyReLu shape 512 x 2048 x 512): whole 2-SM tiles.  (Round 1 measured the 1-SM
    // tile ahead there, 16.4 vs 18.3 us; with the round-2 kernels it is behind: 512 x 2048 x 512
    // 20.5 vs 18.4 us, 4096 x 2048 x 512 22.6 vs 20.5 -- scripts/tune.py --op gemm,
    // profiles/r02/tune/tune_gemm_short_k.log)
    if (KB <= 32 && out_cols != 128 && ((M + 255) / 256) * ((N + 127) / 128) <= sm_count / 2)
        return Plan{CUASM_VARIANT_2SM, false, 128, 0};
    Plan best{CUASM_VARIANT_2SM, false, 256, 0};
    double best_t = 1e30;
    // candidates: the GEMM mode's MMA widths 256 / 128 (128 outputs, half the k-block time
    // per tile), or the SwiGLU tile widths bn (2 bn = MMA N; widths below 128 only for the
    // 2-SM bf16 kernel, DESIGN.md §6 "Tile widths")
    struct Cand { int tn, bn; };
    Cand cands[8];  // (>= the SwiGLU widths or the 2 GEMM widths)
    int nc = 0;
    if (out_cols != 128) {
        for (int tn : {256, 128})
            if (!tile_n_force || tn == tile_n_force) cands[nc++] = Cand{tn, kPackBN};
    } else {
        // (narrow 2-SM tiles were measured from M = 256 up; decode-sized M keeps 128 unless forced)
        for (int bn : kTileBNs)
            // (small-M shards past the rules above: narrow tiles from M = 33 -- 48 x 8192 x 7168:
            // 2-SM 112-wide 49.9 us vs 1-SM 128-wide stream-K 52.0, profiles/r02/tune/grid.json)
            if ((bn == kPackBN || (esize == 2 && (M > (small_m_shard ? 32 : 128) || tile_bn_force))) &&
                (tile_bn_force ? bn == tile_bn_force : true))
                cands[nc++] = Cand{256, bn};
    }
    for (int ci = 0; ci < nc; ++ci) {
        const int tn = cands[ci].tn, bn = cands[ci].bn;
        const int64_t oc = out_cols == 128 ? bn : tn;   // output columns per tile
        const int64_t wrows = out_cols == 128 ? 2 * bn : tn;  // weight rows per n-block
        // k-block time relative to N = 256: a 128-wide k-block costs 0.72 of a 256-wide one,
        // not 0.5 -- its fixed per-k-block issue/TMA overheads do not halve
        // (scripts/tune.py --op gemm, profiles/r01/tune_gemm*.log); SwiGLU widths: bn_frac
        const double tile_frac = out_cols == 128 ? bn_frac(bn) : (tn == 256 ? 1.0 : 0.72);
        const int64_t nblk_w = (N + oc - 1) / oc;
        for (int cg = 2; cg >= 1; --cg) {
            // (the 1-SM kernel is shared-memory-bandwidth bound: a narrower tile issues no faster
            // per byte -- M = 288..384, 1-SM 120-wide 61.4-63.5 us vs 128-wide 61.1-61.4)
            if (bn != kPackBN && cg == 1) continue;
            const int64_t units = sm_count / cg;
            const int64_t mblk = (M + 128 * cg - 1) / (128 * cg);
            const int64_t tiles = mblk * nblk_w;
            const double rounds = static_cast<double>((tiles + units - 1) / units);
            const double pen = (cg == 1 ? pen_1sm : 1.0) * tile_frac;
            const double t_dp = std::max(hbm_floor, rounds * KB * t_kb * pen);
            // Stream-K keeps its whole region in flight at once (every cluster
            // holds a slice of it), so when the region's operands overflow L2 the
            // k-block rate drops (measured 0.49 vs 0.37 us on 2048x11008x4096,
            // profiles/r01/trace_gemm.log): charge that as a 1.32x slowdown.
            const int64_t rem = tiles % units;
            const int64_t sk_tiles = tiles < units ? tiles : (rem ? rem + units : 0);
            const int64_t gm = std::min<int64_t>(mblk, group_m > 0 ? group_m : auto_group_m(K, esize, cg));
            const double region_bytes =
                static_cast<double>((sk_tiles + gm - 1) / gm + 1) * wrows * K * esize +
                static_cast<double>(std::min<int64_t>(M, gm * 128 * cg)) * K * esize;
            const double l2_pen = region_bytes > 120e6 ? 1.32 : 1.0;
            // fewer tiles than clusters: auto stream-K splits each tile at most in two
            // (launch_gemm), so only 2*tiles clusters work and each finisher adds one
            // partial (more splits make the finisher read many partials: the paper's
            // 512x2048x512 mmLeakyReLu took 65 us with 18 segments per tile)
            const double sk_units = tiles < units ? static_cast<double>(std::min<int64_t>(units, 2 * tiles)) : units;
            const double t_sk = std::max(hbm_floor, tiles * KB * t_kb * pen * l2_pen / sk_units + fixup);
            const int v = cg == 2 ? CUASM_VARIANT_2SM : CUASM_VARIANT_1SM;
            // ties go to the earlier candidate: N=256 before 128, bn = 128 before narrower
            // tiles, 2-SM before 1-SM, whole tiles before stream-K
            if (t_dp < best_t * 0.999) { best_t = t_dp; best = Plan{v, false, tn, 0, bn}; }
            if (K / BK > 1 && t_sk < best_t * 0.98) { best_t = t_sk; best = Plan{v, true, tn, 0, bn}; }
        }
    }
    // Tall tiles: N / 80 n-blocks of 384 rows in whole rounds of the CTA pairs; a tall k-block (an
    // 80-wide 256-row MMA + an 80-wide 128-row MMA on one weight stage) costs kTallFrac of a 128-wide
    // 256-row k-block
    if (tall_ok) {
        constexpr double kTallFrac = 1.07;  // measured: 384 x 4096 x 11008 57.5 us vs 1-SM 128-wide 62.9 (scripts/tune_tall.py)
        const int64_t units = sm_count / 2;
        const int64_t tiles = (N + kTallBN - 1) / kTallBN;
        const double rounds = static_cast<double>((tiles + units - 1) / units);
        const double t_tall = std::max(hbm_floor, rounds * KB * t_kb * kTallFrac);
        if (t_tall < best_t * 0.98) best = Plan{CUASM_VARIANT_2SM, false, 256, 0, kTallBN, true};
    }
    return best;
}

Plan plan_config(cuasm_ffn_t h, int64_t M, int64_t K, int64_t N, int64_t out_cols) {
    // measured configurations (cuasm_ffn_tune, cuasm_gemm_act_tune) take precedence over the model
    {
        const int op = out_cols == 128 ? 0 : 1;
        if (h->plan_forced && h->plan_force_op == op) return h->plan_force;
        for (const TunedEntry& t : h->tuned)
            if (t.op == op && t.M == M && t.K == K && t.N == N) return t.plan;
    }
    Plan pl = plan_config_raw(h->sm_count, h->esize, h->group_m, M, K, N, out_cols, out_cols == 128 ? 0 : h->tile_n,
                              out_cols == 128 ? h->tile_bn : 0, h->tall);
    // (tall tiles are a 2-SM kernel: a forced 1-SM variant takes the ordinary tiles)
    if (pl.tall && h->variant == CUASM_VARIANT_1SM) pl = Plan{CUASM_VARIANT_1SM, false, 256, 0, kPackBN};
    // a forced 1-SM variant (CUASM_OPT_VARIANT) has the 128-, 120- and 64-output SwiGLU tiles
    if (h->variant == CUASM_VARIANT_1SM && pl.bn != 64 && pl.bn != 120) pl.bn = kPackBN;
    return pl;
}

cuasm_status_t ensure_r(cuasm_ffn_t h, int64_t M) {
    if (M > h->r_cap) {
        if (h->r) cudaFree(h->r);
        h->r = nullptr;
        h->r_cap = 0;
        const int64_t cap = std::max<int64_t>(M, 4096);
        CUASM_CHECK(h, cudaMalloc(&h->r, cap * sizeof(float)), "cudaMalloc(r)");
        h->r_cap = cap;
    }
    return CUASM_OK;
}

cuasm_status_t profile_event(cuasm_ffn_t h, cudaStream_t s) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        CUASM_CHECK(h, cudaEventCreate(&e), "cudaEventCreate");
        h->ev_pool.push_back(e);
    }
    CUASM_CHECK(h, cudaEventRecord(h->ev_pool[h->ev_used++], s), "cudaEventRecord");
    return CUASM_OK;
}

template <int kEpi, int kN>
cuasm_status_t dispatch_gemm(cuasm_ffn_t h, const EpiSpec& e, int v, const void* x, void* out, int64_t M, int64_t K,
                             int64_t N, float eps, cudaStream_t s) {
    if (h->dtype == CUASM_DTYPE_BF16) {
        return v == CUASM_VARIANT_2SM ? launch_gemm<0, 2, kEpi, kN>(h, e, x, out, M, K, N, eps, s)
                                      : launch_gemm<0, 1, kEpi, kN>(h, e, x, out, M, K, N, eps, s);
    }
    return v == CUASM_VARIANT_2SM ? launch_gemm<1, 2, kEpi, kN>(h, e, x, out, M, K, N, eps, s)
                                  : launch_gemm<1, 1, kEpi, kN>(h, e, x, out, M, K, N, eps, s);
}

// Launch one dual-GEMM kernel (plus the stand-alone pre-pass when a1 is not
// fused) on the already packed weights of slot e.slot.
cuasm_status_t run_gemm(cuasm_ffn_t h, int kepi, const EpiSpec& e, const void* x, void* out, int64_t M, int64_t K,
                        int64_t N, float eps, cudaStream_t s) {
    cuasm_status_t st;
    if (M == 0) return CUASM_OK;
    if (e.use_r && (st = ensure_r(h, M)) != CUASM_OK) return st;
    if (h->trace) {
        // clear the trace before the pre-pass: a memset between the pre-pass
        // and the GEMM would break their programmatic (PDL) dependency
        if (!h->trace_buf)
            CUASM_CHECK(h, cudaMalloc(&h->trace_buf, sizeof(unsigned long long) * 16 * 1024), "cudaMalloc(trace)");
        CUASM_CHECK(h, cudaMemsetAsync(h->trace_buf, 0, sizeof(unsigned long long) * 16 * 1024, s), "memset(trace)");
    }
    if (e.fused_norm) {
        // fused a1 bookkeeping: 2 words per 128-row r-block + the warp counter, zeroed once
        // (the kernel leaves it zeroed for the next launch)
        const int64_t words = 2 * ((M + 127) / 128) + 1;
        if (words > h->rstate_words) {
            if (h->rstate) cudaFree(h->rstate);
            h->rstate = nullptr;
            h->rstate_words = 0;
            const int64_t cap = std::max<int64_t>(words, 2 * 64 + 1);
            CUASM_CHECK(h, cudaMalloc(&h->rstate, cap * 4), "cudaMalloc(r-block state)");
            CUASM_CHECK(h, cudaMemset(h->rstate, 0, cap * 4), "cudaMemset(r-block state)");
            h->rstate_words = cap;
        }
    }
    if (h->profile && (st = profile_event(h, s)) != CUASM_OK) return st;
    // a1: fused into the dual GEMM by default; the separate pre-pass kernel
    // (PDL primary of the GEMM) when CUASM_OPT_FUSED_NORM = 0
    const bool separate_prepass = e.use_r && !e.fused_norm;
    if (separate_prepass && e.kp > 0) {
        const unsigned blocks = static_cast<unsigned>((M + cuasm::kPrepassRowsPerBlock - 1) / cuasm::kPrepassRowsPerBlock);
        cuasm::ffn_split_tf32_kernel<<<blocks, 256, 0, s>>>(static_cast<const float*>(e.x_src),
                                                             static_cast<float*>(const_cast<void*>(x)), h->r, M,
                                                             e.k_src, e.kp, eps);
        CUASM_CHECK(h, cudaGetLastError(), "ffn_split_tf32_kernel launch");
    } else if (separate_prepass && (st = prepass(h, x, h->r, M, K, eps, s)) != CUASM_OK) {
        return st;
    }
    if (h->profile && (st = profile_event(h, s)) != CUASM_OK) return st;
    const Plan plan = plan_config(h, M, K, N, kepi == 0 ? 128 : 256);
    const int v = h->variant != CUASM_VARIANT_AUTO ? h->variant : plan.variant;
    h->plan_sk = plan.stream_k;
    h->plan_csplit = v == plan.variant ? plan.csplit : 0;
    if (kepi == 0 && plan.tall) {
        // tall tiles (257..384 rows, 80-wide n-blocks; ffn_common packed the 80-wide slot)
        if (h->dtype != CUASM_DTYPE_BF16 || v != CUASM_VARIANT_2SM || e.slot != w13_slot(plan.bn))
            return fail(h, CUASM_ERR_UNSUPPORTED, "tall tiles need the 2-SM bf16 kernel");
        st = launch_gemm<0, 2, 0, 2 * kTallBN, false, true>(h, e, x, out, M, K, N, eps, s);
    } else if (kepi == 0 && plan.bn == 64 && v == CUASM_VARIANT_1SM) {
        // the 1-SM 64-output tile: decode shards (more, smaller tiles for the cluster split-K)
        if (h->dtype != CUASM_DTYPE_BF16 || e.slot != w13_slot(plan.bn))
            return fail(h, CUASM_ERR_UNSUPPORTED, "tile width 64 needs the bf16 kernel");
        // (decode rows with the planner's cluster split-K: thin A stages, more weight bytes in flight)
        if (M <= 32 && (h->csplit_opt >= 2 || (h->csplit_opt == 0 && plan.csplit >= 2)) && h->thin != 0)
            st = launch_gemm<0, 1, 0, 128, true>(h, e, x, out, M, K, N, eps, s);
        else
            st = launch_gemm<0, 1, 0, 128>(h, e, x, out, M, K, N, eps, s);
    } else if (kepi == 0 && plan.bn == 120 && v == CUASM_VARIANT_1SM) {
        // the 1-SM 120-output tile (forced only: measured no faster than 128 on the 1-SM kernel)
        if (h->dtype != CUASM_DTYPE_BF16 || e.slot != w13_slot(plan.bn))
            return fail(h, CUASM_ERR_UNSUPPORTED, "tile width 120 needs the bf16 kernel");
        st = launch_gemm<0, 1, 0, 240>(h, e, x, out, M, K, N, eps, s);
    } else if (kepi == 0 && plan.bn != kPackBN) {
        // narrower SwiGLU tiles (2-SM bf16 only; ffn_common packed slot 2 for this width)
        if (h->dtype != CUASM_DTYPE_BF16 || v != CUASM_VARIANT_2SM || e.slot != w13_slot(plan.bn))
            return fail(h, CUASM_ERR_UNSUPPORTED, "tile width %d needs the 2-SM bf16 kernel", plan.bn);
        switch (plan.bn) {
        case 120: st = launch_gemm<0, 2, 0, 240>(h, e, x, out, M, K, N, eps, s); break;
        case 112: st = launch_gemm<0, 2, 0, 224>(h, e, x, out, M, K, N, eps, s); break;
        case 96: st = launch_gemm<0, 2, 0, 192>(h, e, x, out, M, K, N, eps, s); break;
        case 80: st = launch_gemm<0, 2, 0, 160>(h, e, x, out, M, K, N, eps, s); break;
        case 64: st = launch_gemm<0, 2, 0, 128>(h, e, x, out, M, K, N, eps, s); break;
        default: return fail(h, CUASM_ERR_UNSUPPORTED, "no kernel for tile width %d", plan.bn);
        }
    } else if (kepi == 0) st = dispatch_gemm<0, 256>(h, e, v, x, out, M, K, N, eps, s);
    else if (plan.tile_n == 128) st = dispatch_gemm<1, 128>(h, e, v, x, out, M, K, N, eps, s);
    else st = dispatch_gemm<1, 256>(h, e, v, x, out, M, K, N, eps, s);
    h->last_tile_n = kepi == 0 ? 2 * plan.bn : plan.tile_n;
    if (st != CUASM_OK) return st;
    h->last_kernels += separate_prepass ? 2 : 1;
    if (h->profile && (st = profile_event(h, s)) != CUASM_OK) return st;
    return CUASM_OK;
}

// a0 (if needed) then a1-a3 of the fused FFN with epilogue spec `e`.  fp32 handles
// contract the exact tf32 split [x_hi | x_lo] of x with duplicated-K weights
// (pack.cuh ffn_split_tf32_kernel; R5).
cuasm_status_t ffn_common(cuasm_ffn_t h, EpiSpec e, const void* x, const void* g, const void* w1, const void* w3,
                          void* out, int64_t M, int64_t K, int64_t N, float eps, cudaStream_t s) {
    cuasm_status_t st;
    if (h->dtype == CUASM_DTYPE_FP32) {
        e.slot = 0;
        const int64_t kp = split_kp(K);
        if ((st = ensure_packed(h, 0, g, w1, w3, K, N, s, kp)) != CUASM_OK) return st;
        const int64_t xb = std::max<int64_t>(M, 1) * 2 * kp * 4;
        if (xb > h->x2_bytes) {
            if (h->x2) cudaFree(h->x2);
            h->x2 = nullptr;
            h->x2_bytes = 0;
            CUASM_CHECK(h, cudaMalloc(&h->x2, xb), "cudaMalloc(split x)");
            h->x2_bytes = xb;
        }
        e.fused_norm = 0;
        e.x_src = x;
        e.k_src = K;
        e.kp = kp;
        return run_gemm(h, 0, e, h->x2, out, M, 2 * kp, N, eps, s);
    }
    // the tile width decides the W13 block layout: pack (or reuse) the slot of that width
    const int bn = M > 0 ? plan_config(h, M, K, N, 128).bn : kPackBN;
    e.slot = w13_slot(bn);
    if ((st = ensure_packed(h, e.slot, g, w1, w3, K, N, s, 0, bn)) != CUASM_OK) return st;
    return run_gemm(h, 0, e, x, out, M, K, N, eps, s);
}

// The fused FFN (a0 if needed, then a1-a3).
cuasm_status_t forward_impl(cuasm_ffn_t h, const void* x, const void* g, const void* w1, const void* w3, void* out,
                            int64_t M, int64_t K, int64_t N, float eps, cudaStream_t s) {
    cuasm_status_t st;
    h->last_kernels = 0;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    const EpiSpec e{0, h->fused_norm, 1, 0, 0.f};
    return ffn_common(h, e, x, g, w1, w3, out, M, K, N, eps, s);
}

// The fused FFN with step a4 in its epilogue: every output store goes to each
// of `dst` (P2P) or once to the multicast address dst[0].
cuasm_status_t forward_gather_impl(cuasm_ffn_t h, const void* x, const void* g, const void* w1, const void* w3,
                                   void* const* dst, int num_dst, int mc, int64_t ldo, int64_t M, int64_t K,
                                   int64_t N, float eps, cudaStream_t s) {
    cuasm_status_t st;
    h->last_kernels = 0;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    EpiSpec e{0, h->fused_norm, 1, 0, 0.f};
    e.dst = dst;
    e.num_dst = num_dst;
    e.dst_mc = mc;
    e.ldo = ldo;
    return ffn_common(h, e, x, g, w1, w3, mc ? nullptr : dst[0], M, K, N, eps, s);
}

// out = act(x . w^T): the single-weight GEMM + activation path.
cuasm_status_t gemm_act_impl(cuasm_ffn_t h, const void* x, const void* w, void* out, int64_t M, int64_t K, int64_t N,
                             int act, float alpha, cudaStream_t s) {
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    if ((st = ensure_packed(h, 1, nullptr, w, nullptr, K, N, s)) != CUASM_OK) return st;
    h->last_kernels = 0;
    const EpiSpec e{1, 0, 0, act, alpha};
    return run_gemm(h, 1, e, x, out, M, K, N, 0.f, s);
}

cuasm_status_t validate_forward(cuasm_ffn_t h, const void* x, const void* g, const void* w1, const void* w3,
                                const void* out, int64_t M, int64_t K, int64_t N, float eps) {
    cuasm_status_t st;
    if ((st = check_common(h, K, N)) != CUASM_OK) return st;
    if ((st = check_weights(h, g, w1, w3)) != CUASM_OK) return st;
    if ((st = check_eps(h, eps)) != CUASM_OK) return st;
    if (M < 0 || M >= (int64_t(1) << 31)) return fail(h, CUASM_ERR_INVALID_ARG, "M must be in [0, 2^31)");
    if (M > 0 && (!x || !out)) return fail(h, CUASM_ERR_INVALID_ARG, "NULL x or out pointer");
    if (M > 0 && (!aligned16(x) || !aligned16(out)))
        return fail(h, CUASM_ERR_INVALID_ARG, "x and out must be 16-byte aligned");
    return CUASM_OK;
}

}  // namespace

extern "C" {

int cuasm_ffn_abi_version(void) { return CUASM_FFN_ABI_VERSION; }

namespace {
bool same_plan(const Plan& a, const Plan& b) {
    return a.variant == b.variant && a.stream_k == b.stream_k && a.tile_n == b.tile_n && a.csplit == b.csplit &&
           a.bn == b.bn && a.tall == b.tall;
}

// The configurations cuasm_ffn_tune measures for one bf16 fused-FFN shape (the paper's
// "user-provided kernel configurations"): the cost model's own choice first, every
// 2-SM tile width with whole tiles and with a stream-K tail, the 1-SM 128-wide tile both
// ways, tall tiles where they apply, and the 1-SM cluster split-K of 2..8 CTAs per tile
// (128- and 64-output tiles) where a tile count x split fits the SMs in one wave.
std::vector<Plan> tune_candidates(cuasm_ffn_t h, int64_t M, int64_t K, int64_t N) {
    std::vector<Plan> c;
    auto add = [&](const Plan& p) {
        for (const Plan& q : c)
            if (same_plan(q, p)) return;
        c.push_back(p);
    };
    add(plan_config_raw(h->sm_count, h->esize, h->group_m, M, K, N, 128));
    for (int bn : kTileBNs)
        for (int sk = 0; sk < 2; ++sk) add(Plan{CUASM_VARIANT_2SM, sk == 1, 256, 0, bn});
    for (int sk = 0; sk < 2; ++sk) add(Plan{CUASM_VARIANT_1SM, sk == 1, 256, 0, kPackBN});
    if (M > 256 && M <= kTallMaxM) {
        Plan t{CUASM_VARIANT_2SM, false, 256, 0, kTallBN};
        t.tall = true;
        add(t);
    }
    const int64_t KB = (K + 63) / 64;
    for (int bn : {kPackBN, 64})
        for (int S : {2, 3, 4, 6, 8}) {
            const int64_t tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
            if (tiles * S <= h->sm_count && KB >= 2 * S) add(Plan{CUASM_VARIANT_1SM, false, 256, S, bn});
        }
    return c;
}
}  // namespace

}  // extern "C" (the tuner's shared core follows)

namespace {
// The search loop of cuasm_ffn_tune / cuasm_gemm_act_tune: every candidate of `cands` for op `op`
// (0 fused FFN, 1 GEMM + activation) through `fwd` (one forward under the forced plan).
template <class Fwd>
cuasm_status_t tune_core(cuasm_ffn_t h, int op, const std::vector<Plan>& cands, Fwd fwd, int64_t M, int64_t K,
                         int64_t N, int warmup, int iters, int flush_l2, void* stream, int* variant, int* flags,
                         float* best_us) {
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // flush_l2: a buffer of twice the L2 is written, then another read, before every timed
    // forward (outside its event pair), so each starts with an L2 of clean, unrelated lines
    int l2 = 0;
    CUASM_CHECK(h, cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device), "cudaDeviceGetAttribute(L2)");
    const int64_t fbytes = flush_l2 ? (2 * static_cast<int64_t>(l2) + 0xFFFFF) & ~int64_t(0xFFFFF) : 0;
    void* fbuf = nullptr;
    if (fbytes && cudaMalloc(&fbuf, 2 * fbytes) != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(h, CUASM_ERR_OOM, "cudaMalloc(L2 flush buffer)");
    }
    const int nev = flush_l2 ? iters : 1;
    std::vector<cudaEvent_t> ev(static_cast<size_t>(2 * nev), nullptr);
    auto cleanup = [&]() {
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (fbuf) cudaFree(fbuf);
        h->plan_forced = false;
    };
    for (cudaEvent_t& e : ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            cleanup();
            return fail(h, CUASM_ERR_CUDA, "cudaEventCreate");
        }
    auto flush = [&]() {
        if (!fbuf) return cudaSuccess;
        for (int wr = 1; wr >= 0; --wr)
            cuasm::l2_flush_kernel<<<2 * h->sm_count, 512, 0, s>>>(
                static_cast<uint4*>(fbuf), reinterpret_cast<uint4*>(static_cast<char*>(fbuf) + fbytes), fbytes / 16, wr);
        return cudaGetLastError();
    };
    // candidates measured in kTuneRounds interleaved rounds (clock / power drift spreads over
    // all of them), a candidate's time = the best of its rounds' means
    constexpr int kTuneRounds = 3;
    std::vector<float> t_us(cands.size(), std::numeric_limits<float>::infinity());
    std::vector<bool> skip(cands.size(), false);
    for (int rnd = 0; rnd < kTuneRounds; ++rnd) {
        for (size_t ci = 0; ci < cands.size(); ++ci) {
            if (skip[ci]) continue;
            h->plan_forced = true;
            h->plan_force_op = op;
            h->plan_force = cands[ci];
            st = CUASM_OK;
            for (int w = 0; w < (warmup > 0 ? warmup : 1) && st == CUASM_OK; ++w) st = fwd(s);
            cudaError_t ce = cudaSuccess;
            // flush_l2: each timed forward is one CUDA-graph launch (captured after the warm-up, whose
            // first forward did any packing / allocation), as bench.py times a step -- an eager
            // launch would let PDL start the kernel under the flush's tail and hide its prologue
            cudaGraphExec_t gexec = nullptr;
            if (st == CUASM_OK && flush_l2 && s != nullptr) {
                cudaGraph_t graph = nullptr;
                if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                    const cuasm_status_t cst = fwd(s);
                    if (cudaStreamEndCapture(s, &graph) != cudaSuccess || cst != CUASM_OK ||
                        cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess)
                        gexec = nullptr;
                    if (graph) cudaGraphDestroy(graph);
                }
                (void)cudaGetLastError();  // (capture failures fall back to eager launches)
                h->err.clear();
            }
            if (st == CUASM_OK && !flush_l2) ce = cudaEventRecord(ev[0], s);
            for (int i = 0; i < iters && st == CUASM_OK && ce == cudaSuccess; ++i) {
                if (flush_l2 && (ce = flush()) == cudaSuccess) ce = cudaEventRecord(ev[2 * i], s);
                if (ce == cudaSuccess) {
                    if (gexec) ce = cudaGraphLaunch(gexec, s);
                    else st = fwd(s);
                }
                if (flush_l2 && st == CUASM_OK && ce == cudaSuccess) ce = cudaEventRecord(ev[2 * i + 1], s);
            }
            if (gexec) {
                if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
                cudaGraphExecDestroy(gexec);
            }
            if (st == CUASM_OK && ce == cudaSuccess && !flush_l2) ce = cudaEventRecord(ev[1], s);
            if (st == CUASM_OK && ce == cudaSuccess) ce = cudaStreamSynchronize(s);
            double ms = 0.0;
            for (int i = 0; i < nev && st == CUASM_OK && ce == cudaSuccess; ++i) {
                float m = 0.f;
                ce = cudaEventElapsedTime(&m, ev[2 * i], ev[2 * i + 1]);
                ms += m;
            }
            h->plan_forced = false;
            if (ce != cudaSuccess) {
                cleanup();
                return cuda_fail(h, ce, "tuning");
            }
            if (st != CUASM_OK) {
                // a configuration this shape cannot launch (rejected before any launch): skip it;
                // anything else is a real failure
                if (st != CUASM_ERR_UNSUPPORTED) {
                    cleanup();
                    return st;
                }
                h->err.clear();
                skip[ci] = true;
                continue;
            }
            t_us[ci] = std::min(t_us[ci], static_cast<float>(ms * 1000.0 / iters));
        }
    }
    cleanup();
    float best = std::numeric_limits<float>::infinity();
    Plan best_plan{CUASM_VARIANT_2SM, false, 256, 0, kPackBN};
    h->tune_log.clear();
    for (size_t ci = 0; ci < cands.size(); ++ci) {
        h->tune_log.emplace_back(cands[ci], skip[ci] ? -1.f : t_us[ci]);
        if (!skip[ci] && t_us[ci] < best) {
            best = t_us[ci];
            best_plan = cands[ci];
        }
    }
    if (!(best < std::numeric_limits<float>::infinity())) return fail(h, CUASM_ERR_UNSUPPORTED, "no configuration ran");
    bool found = false;
    for (TunedEntry& t : h->tuned)
        if (t.op == op && t.M == M && t.K == K && t.N == N) {
            t.plan = best_plan;
            t.us = best;
            found = true;
        }
    if (!found) h->tuned.push_back(TunedEntry{op, M, K, N, best_plan, best});
    if (variant) *variant = best_plan.variant;
    if (flags) *flags = plan_flags(best_plan);
    if (best_us) *best_us = best;
    return CUASM_OK;
}

// GEMM + activation candidates: the cost model's choice, each variant x {whole tiles, stream-K}
// x {256, 128}-wide tiles.
std::vector<Plan> tune_candidates_gemm(cuasm_ffn_t h, int64_t M, int64_t K, int64_t N) {
    std::vector<Plan> c;
    auto add = [&](const Plan& p) {
        for (const Plan& q : c)
            if (same_plan(q, p)) return;
        c.push_back(p);
    };
    add(plan_config_raw(h->sm_count, h->esize, h->group_m, M, K, N, 256));
    for (int v : {CUASM_VARIANT_2SM, CUASM_VARIANT_1SM})
        for (int sk = 0; sk < 2; ++sk)
            for (int tn : {256, 128}) add(Plan{v, sk == 1, tn, 0, kPackBN});
    return c;
}
}  // namespace

extern "C" {

cuasm_status_t cuasm_ffn_tune(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1, const void* w3,
                              void* out, int64_t M, int64_t K, int64_t N, float eps, int warmup, int iters,
                              int flush_l2, void* stream, int* variant, int* flags, float* best_us) {
    NvtxRange nvtx_("cuasm_ffn_tune");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (h->dtype != CUASM_DTYPE_BF16) return fail(h, CUASM_ERR_UNSUPPORTED, "tuning: bf16 handles only");
    cuasm_status_t st = validate_forward(h, x, rms_w, w1, w3, out, M, K, N, eps);
    if (st != CUASM_OK) return st;
    if (M == 0) return fail(h, CUASM_ERR_INVALID_ARG, "tuning needs M > 0");
    if (warmup < 0 || iters < 1 || warmup > 100000 || iters > 100000 || (flush_l2 != 0 && flush_l2 != 1))
        return fail(h, CUASM_ERR_INVALID_ARG, "warmup must be >= 0, iters >= 1, flush_l2 0 or 1");
    return tune_core(h, 0, tune_candidates(h, M, K, N),
                     [&](cudaStream_t s) { return forward_impl(h, x, rms_w, w1, w3, out, M, K, N, eps, s); }, M, K, N,
                     warmup, iters, flush_l2, stream, variant, flags, best_us);
}

cuasm_status_t cuasm_gemm_act_tune(cuasm_ffn_t h, const void* x, const void* w, void* out, int64_t M, int64_t K,
                                   int64_t N, int act, float alpha, int warmup, int iters, int flush_l2, void* stream,
                                   int* variant, int* flags, float* best_us) {
    NvtxRange nvtx_("cuasm_gemm_act_tune");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (h->dtype != CUASM_DTYPE_BF16) return fail(h, CUASM_ERR_UNSUPPORTED, "tuning: bf16 handles only");
    cuasm_status_t st;
    if ((st = check_common(h, K, N)) != CUASM_OK) return st;
    if (act != CUASM_ACT_IDENTITY && act != CUASM_ACT_LEAKY_RELU)
        return fail(h, CUASM_ERR_INVALID_ARG, "unknown activation %d", act);
    if (!(alpha == alpha)) return fail(h, CUASM_ERR_INVALID_ARG, "alpha is NaN");
    if (!w || !aligned16(w)) return fail(h, CUASM_ERR_INVALID_ARG, "w must be non-NULL and 16-byte aligned");
    if (M <= 0 || M >= (int64_t(1) << 31)) return fail(h, CUASM_ERR_INVALID_ARG, "tuning needs M in [1, 2^31)");
    if (!x || !out || !aligned16(x) || !aligned16(out))
        return fail(h, CUASM_ERR_INVALID_ARG, "x and out must be non-NULL and 16-byte aligned");
    if (warmup < 0 || iters < 1 || warmup > 100000 || iters > 100000 || (flush_l2 != 0 && flush_l2 != 1))
        return fail(h, CUASM_ERR_INVALID_ARG, "warmup must be >= 0, iters >= 1, flush_l2 0 or 1");
    return tune_core(h, 1, tune_candidates_gemm(h, M, K, N),
                     [&](cudaStream_t s) { return gemm_act_impl(h, x, w, out, M, K, N, act, alpha, s); }, M, K, N,
                     warmup, iters, flush_l2, stream, variant, flags, best_us);
}

// "cuasm-tuned v1 sm=<SMs> dtype=bf16 M=<M> K=<K> N=<N> variant=<v> flags=<f> us=<t> gpu=<name>\n"
// per entry: the lookup key is the GPU name + SM count + dtype + shape (results written
// "prefixed by GPU type, workload type etc., as the key to lookup").
cuasm_status_t cuasm_ffn_tuned_export(cuasm_ffn_t h, char* buf, int64_t cap, int64_t* needed) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (!needed || cap < 0 || (cap > 0 && !buf)) return fail(h, CUASM_ERR_INVALID_ARG, "NULL buffer or size");
    std::string text;
    char line[512];
    for (const TunedEntry& t : h->tuned) {
        std::snprintf(line, sizeof(line),
                      "cuasm-tuned v1 sm=%d dtype=%s M=%lld K=%lld N=%lld variant=%d flags=%d us=%.3f %sgpu=%s\n",
                      h->sm_count, h->dtype == CUASM_DTYPE_BF16 ? "bf16" : "fp32", static_cast<long long>(t.M),
                      static_cast<long long>(t.K), static_cast<long long>(t.N), t.plan.variant, plan_flags(t.plan),
                      static_cast<double>(t.us), t.op == 1 ? "op=gemm " : "", h->gpu_name.c_str());
        text += line;
    }
    *needed = static_cast<int64_t>(text.size()) + 1;
    if (cap < *needed) return cap == 0 ? CUASM_OK : fail(h, CUASM_ERR_INVALID_ARG, "buffer too small (%lld bytes needed)",
                                                         static_cast<long long>(*needed));
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_tuned_import(cuasm_ffn_t h, const char* text, int* accepted) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (!text || !accepted) return fail(h, CUASM_ERR_INVALID_ARG, "NULL text or count");
    *accepted = 0;
    const char* p = text;
    while (*p) {
        const char* eol = std::strchr(p, '\n');
        const std::string line(p, eol ? static_cast<size_t>(eol - p) : std::strlen(p));
        p = eol ? eol + 1 : p + line.size();
        int sm = 0, v = 0, fl = 0, pos = -1;
        long long M = 0, K = 0, N = 0;
        char dt[16] = {0};
        float us = 0.f;
        if (std::sscanf(line.c_str(), "cuasm-tuned v1 sm=%d dtype=%15s M=%lld K=%lld N=%lld variant=%d flags=%d us=%f %n",
                        &sm, dt, &M, &K, &N, &v, &fl, &us, &pos) != 8 || pos < 0)
            continue;  // not an entry (comments, other versions)
        // optional "op=gemm " (a GEMM + activation entry, cuasm_gemm_act_tune), then "gpu=<name>"
        int op = 0;
        if (line.compare(static_cast<size_t>(pos), 8, "op=gemm ") == 0) {
            op = 1;
            pos += 8;
        }
        if (line.compare(static_cast<size_t>(pos), 4, "gpu=") != 0) continue;
        pos += 4;
        std::string gpu = line.substr(static_cast<size_t>(pos));
        while (!gpu.empty() && (gpu.back() == '\r' || gpu.back() == ' ')) gpu.pop_back();
        // another GPU type / SM count / dtype: not this device's entry
        if (sm != h->sm_count || gpu != h->gpu_name || std::strcmp(dt, h->dtype == CUASM_DTYPE_BF16 ? "bf16" : "fp32") != 0)
            continue;
        const Plan pl = plan_from_flags(v, fl);
        bool bn_ok = false;
        for (int bn : kTileBNs) bn_ok |= pl.bn == bn;
        if (M <= 0 || K <= 0 || N <= 0 || (v != CUASM_VARIANT_1SM && v != CUASM_VARIANT_2SM) || !bn_ok ||
            (pl.csplit != 0 && (pl.csplit < 2 || pl.csplit > 8 || v != CUASM_VARIANT_1SM)) ||
            (pl.tall && (v != CUASM_VARIANT_2SM || pl.bn != kTallBN || M <= 256 || M > kTallMaxM)) ||
            (v == CUASM_VARIANT_1SM && pl.bn != kPackBN && pl.bn != 64 && pl.bn != 120) || (fl & ~0xFFF7) != 0 ||
            (op == 1 && (pl.bn != kPackBN || pl.tall || pl.csplit != 0)) || (op == 0 && pl.tile_n != 256))
            return fail(h, CUASM_ERR_INVALID_ARG, "malformed tuned entry: %s", line.c_str());
        bool found = false;
        for (TunedEntry& t : h->tuned)
            if (t.op == op && t.M == M && t.K == K && t.N == N) {
                t.plan = pl;
                t.us = us;
                found = true;
            }
        if (!found) h->tuned.push_back(TunedEntry{op, M, K, N, pl, us});
        ++*accepted;
    }
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_tune_log(cuasm_ffn_t h, int cap, int* n, int* variants, int* flags, float* us) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (!n || cap < 0 || (cap > 0 && (!variants || !flags || !us)))
        return fail(h, CUASM_ERR_INVALID_ARG, "NULL output arrays");
    *n = static_cast<int>(h->tune_log.size());
    for (int i = 0; i < *n && i < cap; ++i) {
        variants[i] = h->tune_log[static_cast<size_t>(i)].first.variant;
        flags[i] = plan_flags(h->tune_log[static_cast<size_t>(i)].first);
        us[i] = h->tune_log[static_cast<size_t>(i)].second;
    }
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_tuned_clear(cuasm_ffn_t h) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    h->tuned.clear();
    return CUASM_OK;
}

cuasm_status_t cuasm_plan_config(int sm_count, int dtype, int64_t M, int64_t K, int64_t N, int op, int* variant,
                                 int* stream_k) {
    if (sm_count <= 1 || (dtype != CUASM_DTYPE_BF16 && dtype != CUASM_DTYPE_FP32) || M < 0 || K <= 0 || N <= 0 ||
        (op != 0 && op != 1) || !variant || !stream_k)
        return CUASM_ERR_INVALID_ARG;
    const Plan pl = plan_config_raw(sm_count, dtype == CUASM_DTYPE_BF16 ? 2 : 4, 0, M, K, N, op == 0 ? 128 : 256);
    *variant = pl.variant;
    *stream_k = plan_flags(pl);
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_init(cuasm_ffn_t* out, int device, cuasm_dtype_t dtype) {
    g_init_error.clear();
    if (!out) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle pointer");
    *out = nullptr;
    if (dtype != CUASM_DTYPE_BF16 && dtype != CUASM_DTYPE_FP32)
        return fail(nullptr, CUASM_ERR_INVALID_ARG, "unknown dtype %d", (int)dtype);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, CUASM_ERR_UNSUPPORTED, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, CUASM_ERR_INVALID_ARG, "device %d out of range", device);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return fail(nullptr, CUASM_ERR_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    if (prop.major != 10 || prop.minor != 0)
        return fail(nullptr, CUASM_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only",
                    device, prop.major, prop.minor);
    cuasm_ffn_t h = new (std::nothrow) cuasm_ffn_s();
    if (!h) return fail(nullptr, CUASM_ERR_OOM, "host allocation failed");
    h->device = device;
    h->dtype = dtype;
    h->esize = dtype == CUASM_DTYPE_BF16 ? 2 : 4;
    h->sm_count = prop.multiProcessorCount;
    h->gpu_name = prop.name;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
        delete h;
        return fail(nullptr, CUASM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    }
    h->encode = reinterpret_cast<EncodeTiledFn>(fn);
    *out = h;
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_forward(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1, const void* w3,
                                 void* out, int64_t M, int64_t K, int64_t N, float eps, void* stream) {
    NvtxRange nvtx_("cuasm_ffn_forward");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    cuasm_status_t st = validate_forward(h, x, rms_w, w1, w3, out, M, K, N, eps);
    if (st != CUASM_OK) return st;
    return forward_impl(h, x, rms_w, w1, w3, out, M, K, N, eps, static_cast<cudaStream_t>(stream));
}

cuasm_status_t cuasm_ffn_forward_gather(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1,
                                        const void* w3, void* const* dst, int num_dst, int multicast, int64_t ldo,
                                        int64_t M, int64_t K, int64_t N, float eps, void* stream) {
    NvtxRange nvtx_("cuasm_ffn_forward_gather");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (!dst || num_dst < 1 || num_dst > 8) return fail(h, CUASM_ERR_INVALID_ARG, "num_dst must be in [1, 8]");
    if (multicast != 0 && multicast != 1) return fail(h, CUASM_ERR_INVALID_ARG, "multicast is 0 or 1");
    if (multicast && num_dst != 1)
        return fail(h, CUASM_ERR_INVALID_ARG, "a multicast destination is one address (num_dst = 1)");
    for (int q = 0; q < num_dst; ++q) {
        if (!dst[q] && M > 0) return fail(h, CUASM_ERR_INVALID_ARG, "NULL destination %d", q);
        if (!aligned16(dst[q])) return fail(h, CUASM_ERR_INVALID_ARG, "destination %d is not 16-byte aligned", q);
    }
    if (ldo < N || ldo % (16 / h->esize) != 0)
        return fail(h, CUASM_ERR_INVALID_ARG, "ldo must be >= N and a multiple of %d elements", 16 / h->esize);
    cuasm_status_t st = validate_forward(h, x, rms_w, w1, w3, dst[0], M, K, N, eps);
    if (st != CUASM_OK) return st;
    return forward_gather_impl(h, x, rms_w, w1, w3, dst, num_dst, multicast, ldo, M, K, N, eps,
                               static_cast<cudaStream_t>(stream));
}

cuasm_status_t cuasm_ffn_forward_host(cuasm_ffn_t h, const void* x_host, const void* rms_w, const void* w1,
                                      const void* w3, void* out_host, int64_t M, int64_t K, int64_t N, float eps,
                                      void* stream, int sync) {
    NvtxRange nvtx_("cuasm_ffn_forward_host");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    cuasm_status_t st;
    if ((st = check_common(h, K, N)) != CUASM_OK) return st;
    if ((st = check_weights(h, rms_w, w1, w3)) != CUASM_OK) return st;
    if ((st = check_eps(h, eps)) != CUASM_OK) return st;
    if (M < 0 || M >= (int64_t(1) << 31)) return fail(h, CUASM_ERR_INVALID_ARG, "M must be in [0, 2^31)");
    if (M > 0 && (!x_host || !out_host)) return fail(h, CUASM_ERR_INVALID_ARG, "NULL host pointer");
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t xb = M * K * h->esize, ob = M * N * h->esize;
    if (xb > h->x_stage_bytes) {
        if (h->x_stage) cudaFree(h->x_stage);
        h->x_stage = nullptr;
        h->x_stage_bytes = 0;
        CUASM_CHECK(h, cudaMalloc(&h->x_stage, xb), "cudaMalloc(x staging)");
        h->x_stage_bytes = xb;
    }
    if (ob > h->out_stage_bytes) {
        if (h->out_stage) cudaFree(h->out_stage);
        h->out_stage = nullptr;
        h->out_stage_bytes = 0;
        CUASM_CHECK(h, cudaMalloc(&h->out_stage, ob), "cudaMalloc(out staging)");
        h->out_stage_bytes = ob;
    }
    if (M == 0) return forward_impl(h, h->x_stage, rms_w, w1, w3, h->out_stage, 0, K, N, eps, s);
    // Pipelined in row chunks: H2D of chunk i+1 (copy stream 1), the forward of
    // chunk i (the caller's stream) and D2H of chunk i-1 (copy stream 2) overlap;
    // PCIe is full duplex, so a step costs ~ the larger transfer plus one chunk (256-row chunks: 7B
    // prefill e2e 342-366 -> 366-372 TFLOP/s vs 512-row ones; a second D2H stream measured slower,
    // profiles/r02/e2e/).
    if (!h->h2d_stream) {
        CUASM_CHECK(h, cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking), "cudaStreamCreate(h2d)");
        CUASM_CHECK(h, cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking), "cudaStreamCreate(d2h)");
    }
    const int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(16, M / 256));
    const int64_t rows_per = (M + nchunk - 1) / nchunk;
    const size_t nev = static_cast<size_t>(2 * nchunk + 2);
    while (h->copy_events.size() < nev) {
        cudaEvent_t e;
        CUASM_CHECK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        h->copy_events.push_back(e);
    }
    cudaEvent_t ev_start = h->copy_events[0], ev_done = h->copy_events[1];
    // staging buffers may still be in use by work already on `s`
    CUASM_CHECK(h, cudaEventRecord(ev_start, s), "cudaEventRecord");
    CUASM_CHECK(h, cudaStreamWaitEvent(h->h2d_stream, ev_start, 0), "cudaStreamWaitEvent");
    CUASM_CHECK(h, cudaStreamWaitEvent(h->d2h_stream, ev_start, 0), "cudaStreamWaitEvent");
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t r0 = c * rows_per, rc = std::min(rows_per, M - r0);
        if (rc <= 0) break;
        cudaEvent_t ev_in = h->copy_events[2 + 2 * c], ev_out = h->copy_events[3 + 2 * c];
        char* xs = static_cast<char*>(h->x_stage) + r0 * K * h->esize;
        char* os = static_cast<char*>(h->out_stage) + r0 * N * h->esize;
        CUASM_CHECK(h,
                    cudaMemcpyAsync(xs, static_cast<const char*>(x_host) + r0 * K * h->esize, rc * K * h->esize,
                                    cudaMemcpyHostToDevice, h->h2d_stream),
                    "H2D x");
        CUASM_CHECK(h, cudaEventRecord(ev_in, h->h2d_stream), "cudaEventRecord");
        CUASM_CHECK(h, cudaStreamWaitEvent(s, ev_in, 0), "cudaStreamWaitEvent");
        st = forward_impl(h, xs, rms_w, w1, w3, os, rc, K, N, eps, s);
        if (st != CUASM_OK) return st;
        CUASM_CHECK(h, cudaEventRecord(ev_out, s), "cudaEventRecord");
        CUASM_CHECK(h, cudaStreamWaitEvent(h->d2h_stream, ev_out, 0), "cudaStreamWaitEvent");
        CUASM_CHECK(h,
                    cudaMemcpyAsync(static_cast<char*>(out_host) + r0 * N * h->esize, os, rc * N * h->esize,
                                    cudaMemcpyDeviceToHost, h->d2h_stream),
                    "D2H out");
    }
    // the caller's stream covers every copy: work after this call sees out_host
    CUASM_CHECK(h, cudaEventRecord(ev_done, h->d2h_stream), "cudaEventRecord");
    CUASM_CHECK(h, cudaStreamWaitEvent(s, ev_done, 0), "cudaStreamWaitEvent");
    if (sync) CUASM_CHECK(h, cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return CUASM_OK;
}

cuasm_status_t cuasm_gemm_act(cuasm_ffn_t h, const void* x, const void* w, void* out, int64_t M, int64_t K, int64_t N,
                              int act, float alpha, void* stream) {
    NvtxRange nvtx_("cuasm_gemm_act");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    h->last_kernels = 0;
    cuasm_status_t st;
    if ((st = check_common(h, K, N)) != CUASM_OK) return st;
    if (act != CUASM_ACT_IDENTITY && act != CUASM_ACT_LEAKY_RELU)
        return fail(h, CUASM_ERR_INVALID_ARG, "unknown activation %d", act);
    if (!(alpha == alpha)) return fail(h, CUASM_ERR_INVALID_ARG, "alpha is NaN");
    if (!w || !aligned16(w)) return fail(h, CUASM_ERR_INVALID_ARG, "w must be non-NULL and 16-byte aligned");
    if (M < 0 || M >= (int64_t(1) << 31)) return fail(h, CUASM_ERR_INVALID_ARG, "M must be in [0, 2^31)");
    if (M > 0 && (!x || !out || !aligned16(x) || !aligned16(out)))
        return fail(h, CUASM_ERR_INVALID_ARG, "x and out must be non-NULL and 16-byte aligned");
    return gemm_act_impl(h, x, w, out, M, K, N, act, alpha, static_cast<cudaStream_t>(stream));
}

namespace {
// The FFN block: hidden [M,N] = fused FFN (handle workspace), then out = hidden . W2^T,
// or -- rs_world > 0 -- its fp32 partial tiles scattered to their owners' staging slots.
cuasm_status_t block_impl(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1, const void* w3,
                          const void* w2, void* out, void* const* stage, int world, int rank, int64_t M, int64_t K,
                          int64_t N, float eps, cudaStream_t s) {
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    const int64_t hb = M * N * h->esize;
    if (hb > h->hidden_bytes) {
        if (h->hidden) cudaFree(h->hidden);
        h->hidden = nullptr;
        h->hidden_bytes = 0;
        CUASM_CHECK(h, cudaMalloc(&h->hidden, hb), "cudaMalloc(hidden)");
        h->hidden_bytes = hb;
    }
    // hidden [M,N] = SiLU(RMSNorm(x) W1^T) * (RMSNorm(x) W3^T), stored in the handle dtype
    if ((st = forward_impl(h, x, rms_w, w1, w3, h->hidden, M, K, N, eps, s)) != CUASM_OK) return st;
    const int k1 = h->last_kernels;
    // out [M,K] = hidden . W2^T  (W2 [K,N], nn.Linear(N -> K) layout)
    if ((st = ensure_packed(h, 1, nullptr, w2, nullptr, N, K, s)) != CUASM_OK) return st;
    h->last_kernels = k1;
    EpiSpec e{1, 0, 0, CUASM_ACT_IDENTITY, 0.f};
    e.rs_stage = stage;
    e.rs_world = stage ? world : 0;
    e.rs_rank = rank;
    return run_gemm(h, 1, e, h->hidden, out, M, N, K, 0.f, s);
}
}  // namespace

cuasm_status_t cuasm_ffn_block_forward(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1,
                                       const void* w3, const void* w2, void* out, int64_t M, int64_t K, int64_t N,
                                       float eps, void* stream) {
    NvtxRange nvtx_("cuasm_ffn_block_forward");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    cuasm_status_t st = validate_forward(h, x, rms_w, w1, w3, out, M, K, N, eps);
    if (st != CUASM_OK) return st;
    if (!w2 || !aligned16(w2)) return fail(h, CUASM_ERR_INVALID_ARG, "w2 must be non-NULL and 16-byte aligned");
    return block_impl(h, x, rms_w, w1, w3, w2, out, nullptr, 0, 0, M, K, N, eps, static_cast<cudaStream_t>(stream));
}

cuasm_status_t cuasm_rs_layout(int64_t M, int64_t K, int world, int rank, int64_t* col0, int64_t* col1,
                               int64_t* stage_bytes) {
    if (M < 0 || K <= 0 || K % 8 != 0 || world < 1 || world > 8 || rank < 0 || rank >= world || !col0 || !col1)
        return CUASM_ERR_INVALID_ARG;
    rs_cols(K, world, rank, *col0, *col1);
    if (stage_bytes) *stage_bytes = static_cast<int64_t>(world) * M * (*col1 - *col0) * 4;
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_block_forward_rs(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1,
                                          const void* w3, const void* w2, void* const* stage, int world, int rank,
                                          int64_t M, int64_t K, int64_t N, float eps, void* stream) {
    NvtxRange nvtx_("cuasm_ffn_block_forward_rs");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (h->dtype != CUASM_DTYPE_BF16) return fail(h, CUASM_ERR_UNSUPPORTED, "the fused reduce-scatter is bf16 only");
    if (world < 1 || world > 8 || rank < 0 || rank >= world)
        return fail(h, CUASM_ERR_INVALID_ARG, "world must be in [1, 8] and 0 <= rank < world");
    if (!stage) return fail(h, CUASM_ERR_INVALID_ARG, "NULL stage array");
    // validate_forward with a stand-in output pointer (the outputs are the staging slots)
    cuasm_status_t st = validate_forward(h, x, rms_w, w1, w3, stage[0] ? stage[0] : x, M, K, N, eps);
    if (st != CUASM_OK) return st;
    if (!w2 || !aligned16(w2)) return fail(h, CUASM_ERR_INVALID_ARG, "w2 must be non-NULL and 16-byte aligned");
    for (int q = 0; q < world; ++q) {
        int64_t c0, c1;
        rs_cols(K, world, q, c0, c1);
        if (c1 > c0 && M > 0 && (!stage[q] || !aligned16(stage[q])))
            return fail(h, CUASM_ERR_INVALID_ARG, "stage[%d] must be non-NULL and 16-byte aligned", q);
    }
    return block_impl(h, x, rms_w, w1, w3, w2, nullptr, stage, world, rank, M, K, N, eps,
                      static_cast<cudaStream_t>(stream));
}

cuasm_status_t cuasm_rs_reduce(cuasm_ffn_t h, const void* stage, int world, int rank, void* const* dst, int num_dst,
                               int multicast, int64_t ldo, int64_t M, int64_t K, void* stream) {
    NvtxRange nvtx_("cuasm_rs_reduce");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    h->last_kernels = 0;
    if (h->dtype != CUASM_DTYPE_BF16) return fail(h, CUASM_ERR_UNSUPPORTED, "the fused reduce-scatter is bf16 only");
    if (world < 1 || world > 8 || rank < 0 || rank >= world)
        return fail(h, CUASM_ERR_INVALID_ARG, "world must be in [1, 8] and 0 <= rank < world");
    if (M < 0 || M >= (int64_t(1) << 31) || K <= 0 || K % 8 != 0)
        return fail(h, CUASM_ERR_INVALID_ARG, "M must be in [0, 2^31) and K a positive multiple of 8");
    if (!dst || num_dst < 1 || num_dst > 8) return fail(h, CUASM_ERR_INVALID_ARG, "num_dst must be in [1, 8]");
    if (multicast != 0 && multicast != 1) return fail(h, CUASM_ERR_INVALID_ARG, "multicast is 0 or 1");
    if (multicast && num_dst != 1) return fail(h, CUASM_ERR_INVALID_ARG, "a multicast destination is one address");
    if (ldo < K || ldo % 8 != 0) return fail(h, CUASM_ERR_INVALID_ARG, "ldo must be >= K and a multiple of 8");
    int64_t c0, c1;
    rs_cols(K, world, rank, c0, c1);
    if (M == 0 || c1 == c0) return CUASM_OK;  // this rank owns no columns
    if (!stage || !aligned16(stage)) return fail(h, CUASM_ERR_INVALID_ARG, "stage must be non-NULL, 16-byte aligned");
    for (int q = 0; q < num_dst; ++q)
        if (!dst[q] || !aligned16(dst[q])) return fail(h, CUASM_ERR_INVALID_ARG, "destination %d invalid", q);
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cuasm::RsDst d{};
    for (int q = 0; q < num_dst; ++q) d.p[q] = dst[q];
    const int64_t groups = M * ((c1 - c0) / 8);
    const int64_t blocks = std::min<int64_t>((groups + 255) / 256, int64_t(h->sm_count) * 8);
    if (h->rs_bf16)
        cuasm::ffn_rs_reduce_kernel<__nv_bfloat16><<<static_cast<unsigned>(blocks), 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(stage), world, M, static_cast<int>(c1 - c0), static_cast<int>(c0), d,
            num_dst, multicast, ldo);
    else
        cuasm::ffn_rs_reduce_kernel<float><<<static_cast<unsigned>(blocks), 256, 0, s>>>(
            static_cast<const float*>(stage), world, M, static_cast<int>(c1 - c0), static_cast<int>(c0), d, num_dst,
            multicast, ldo);
    CUASM_CHECK(h, cudaGetLastError(), "ffn_rs_reduce_kernel launch");
    h->last_kernels = 1;
    return CUASM_OK;
}

cuasm_status_t cuasm_rmsnorm(cuasm_ffn_t h, const void* x, const void* rms_w, void* out, int64_t M, int64_t K,
                             float eps, void* stream) {
    NvtxRange nvtx_("cuasm_rmsnorm");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    h->last_kernels = 0;
    cuasm_status_t st;
    if (K <= 0 || K % 8 != 0) return fail(h, CUASM_ERR_INVALID_ARG, "K must be a positive multiple of 8");
    if (M < 0 || M >= (int64_t(1) << 31)) return fail(h, CUASM_ERR_INVALID_ARG, "M must be in [0, 2^31)");
    if ((st = check_eps(h, eps)) != CUASM_OK) return st;
    if (!rms_w || !aligned16(rms_w)) return fail(h, CUASM_ERR_INVALID_ARG, "rms_w must be non-NULL, 16-byte aligned");
    if (M == 0) return CUASM_OK;
    if (!x || !out || !aligned16(x) || !aligned16(out))
        return fail(h, CUASM_ERR_INVALID_ARG, "x and out must be non-NULL and 16-byte aligned");
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned blocks = static_cast<unsigned>((M + cuasm::kPrepassRowsPerBlock - 1) / cuasm::kPrepassRowsPerBlock);
    if (h->dtype == CUASM_DTYPE_BF16) {
        cuasm::ffn_rmsnorm_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(rms_w),
            static_cast<__nv_bfloat16*>(out), M, K, eps);
    } else {
        cuasm::ffn_rmsnorm_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(x),
                                                                 static_cast<const float*>(rms_w),
                                                                 static_cast<float*>(out), M, K, eps);
    }
    CUASM_CHECK(h, cudaGetLastError(), "ffn_rmsnorm_kernel launch");
    h->last_kernels = 1;
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_prepare(cuasm_ffn_t h, const void* rms_w, const void* w1, const void* w3, int64_t K,
                                 int64_t N, void* stream) {
    NvtxRange nvtx_("cuasm_ffn_prepare");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    cuasm_status_t st;
    if ((st = check_common(h, K, N)) != CUASM_OK) return st;
    if ((st = check_weights(h, rms_w, w1, w3)) != CUASM_OK) return st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    h->pw[0].packed = false;
    return ensure_packed(h, 0, rms_w, w1, w3, K, N, static_cast<cudaStream_t>(stream),
                         h->dtype == CUASM_DTYPE_FP32 ? split_kp(K) : 0);
}

cuasm_status_t cuasm_ffn_rms_inv(cuasm_ffn_t h, const void* x, float* r, int64_t M, int64_t K, float eps,
                                 void* stream) {
    NvtxRange nvtx_("cuasm_ffn_rms_inv");
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    h->err.clear();
    if (K <= 0 || K % 8 != 0) return fail(h, CUASM_ERR_INVALID_ARG, "K must be a positive multiple of 8");
    if (M < 0) return fail(h, CUASM_ERR_INVALID_ARG, "M must be >= 0");
    cuasm_status_t st;
    if ((st = check_eps(h, eps)) != CUASM_OK) return st;
    if (M == 0) return CUASM_OK;
    if (!x || !r) return fail(h, CUASM_ERR_INVALID_ARG, "NULL pointer");
    if (!aligned16(x) || (reinterpret_cast<uintptr_t>(r) & 3u))
        return fail(h, CUASM_ERR_INVALID_ARG, "x must be 16-byte and r 4-byte aligned");
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    return prepass(h, x, r, M, K, eps, static_cast<cudaStream_t>(stream));
}

cuasm_status_t cuasm_ffn_get_packed(cuasm_ffn_t h, void* dst, int64_t* bytes) {
    if (!h || !bytes) return fail(h, CUASM_ERR_INVALID_ARG, "NULL argument");
    if (!h->pw[0].packed) return fail(h, CUASM_ERR_INVALID_ARG, "no packed weights cached");
    const int64_t b = h->pw[0].rows * 128;
    *bytes = b;
    if (!dst) return CUASM_OK;
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    CUASM_CHECK(h, cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    CUASM_CHECK(h, cudaMemcpy(dst, h->pw[0].buf, b, cudaMemcpyDeviceToHost), "D2H W13");
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_invalidate_weights(cuasm_ffn_t h) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    for (PackedWeights& w : h->pw) w.packed = false;
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_set_option(cuasm_ffn_t h, int option, int64_t value) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    switch (option) {
    case CUASM_OPT_VARIANT:
        if (value < CUASM_VARIANT_AUTO || value > CUASM_VARIANT_2SM)
            return fail(h, CUASM_ERR_INVALID_ARG, "bad variant %lld", (long long)value);
        h->variant = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_PDL:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "PDL option is 0 or 1");
        h->use_pdl = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_GROUP_M:
        if (value < 0 || value > 1 << 20) return fail(h, CUASM_ERR_INVALID_ARG, "bad group_m");
        h->group_m = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_SCHEDULE:
        if (value < CUASM_SCHEDULE_AUTO || value > CUASM_SCHEDULE_STREAM_K_TAIL)
            return fail(h, CUASM_ERR_INVALID_ARG, "bad schedule %lld", (long long)value);
        h->schedule = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_FUSED_NORM:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "FUSED_NORM option is 0 or 1");
        h->fused_norm = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_TILE_N:
        if (value != 0 && value != 128 && value != 256) return fail(h, CUASM_ERR_INVALID_ARG, "TILE_N is 0, 128 or 256");
        h->tile_n = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_L2_POLICY:
        if (value < 0 || value > 15 || (value & 3) == 3 || ((value >> 2) & 3) == 3)
            return fail(h, CUASM_ERR_INVALID_ARG, "L2_POLICY: 2-bit codes 0..2 for x (bits 0-1) and W13 (bits 2-3)");
        h->l2pol = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_CSPLIT:
        if (value < 0 || value > 8) return fail(h, CUASM_ERR_INVALID_ARG, "CSPLIT is 0 (auto), 1 (off) or 2..8");
        h->csplit_opt = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_SK_SPLIT:
        if (value != 0 && (value < 2 || value > 16)) return fail(h, CUASM_ERR_INVALID_ARG, "SK_SPLIT is 0 or 2..16");
        h->sk_split = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_TILE_BN:
        if (value != 0 && std::find(std::begin(kTileBNs), std::end(kTileBNs), value) == std::end(kTileBNs))
            return fail(h, CUASM_ERR_INVALID_ARG, "TILE_BN is 0 (auto) or one of 128, 120, 112, 96, 80, 64");
        h->tile_bn = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_DYNAMIC:
        if (value < 0 || value > 2) return fail(h, CUASM_ERR_INVALID_ARG, "DYNAMIC is 0 (auto), 1 (off) or 2 (on)");
        h->dynamic = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_L2_PERSIST: {
        // device-wide: the L2 set-aside for persisting (evict_last) lines, bytes (0 = none)
        if (value < 0) return fail(h, CUASM_ERR_INVALID_ARG, "L2_PERSIST must be >= 0 bytes");
        DeviceGuard dg(h);
        if (dg.status != CUASM_OK) return dg.status;
        CUASM_CHECK(h, cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(value)),
                    "cudaDeviceSetLimit(persisting L2)");
        h->l2_persist = value;
        return CUASM_OK;
    }
    case CUASM_OPT_TALL:
        if (value < 0 || value > 2) return fail(h, CUASM_ERR_INVALID_ARG, "TALL is 0 (auto), 1 (off) or 2 (on)");
        h->tall = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_THIN_A:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "THIN_A is 0 or 1");
        h->thin = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_MCAST:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "MCAST is 0 or 1");
        h->mcast = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_RS_PARTIAL:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "RS_PARTIAL is 0 (fp32) or 1 (bf16)");
        h->rs_bf16 = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_TRACE:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "TRACE option is 0 or 1");
        h->trace = static_cast<int>(value);
        return CUASM_OK;
    case CUASM_OPT_PROFILE:
        if (value != 0 && value != 1) return fail(h, CUASM_ERR_INVALID_ARG, "PROFILE option is 0 or 1");
        h->profile = static_cast<int>(value);
        return CUASM_OK;
    default:
        return fail(h, CUASM_ERR_INVALID_ARG, "unknown option %d", option);
    }
}

cuasm_status_t cuasm_ffn_last_launch(cuasm_ffn_t h, int* variant, int* kernels) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    if (variant) *variant = h->last_variant;
    if (kernels) *kernels = h->last_kernels;
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_profile_read(cuasm_ffn_t h, double* prepass_ms, double* gemm_ms, int* forwards) {
    if (!h) return fail(nullptr, CUASM_ERR_INVALID_ARG, "NULL handle");
    double pre = 0.0, gemm = 0.0;
    const size_t n = h->ev_used / 3;
    for (size_t i = 0; i < n; ++i) {
        float a = 0.f, b = 0.f;
        CUASM_CHECK(h, cudaEventSynchronize(h->ev_pool[3 * i + 2]), "cudaEventSynchronize");
        CUASM_CHECK(h, cudaEventElapsedTime(&a, h->ev_pool[3 * i], h->ev_pool[3 * i + 1]), "cudaEventElapsedTime");
        CUASM_CHECK(h, cudaEventElapsedTime(&b, h->ev_pool[3 * i + 1], h->ev_pool[3 * i + 2]), "cudaEventElapsedTime");
        pre += a;
        gemm += b;
    }
    h->ev_used = 0;
    if (prepass_ms) *prepass_ms = pre;
    if (gemm_ms) *gemm_ms = gemm;
    if (forwards) *forwards = static_cast<int>(n);
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_trace_read(cuasm_ffn_t h, unsigned long long* dst, int* ctas) {
    if (!h || !ctas) return fail(h, CUASM_ERR_INVALID_ARG, "NULL argument");
    *ctas = h->trace_buf ? h->trace_ctas : 0;
    if (!dst || !h->trace_buf) return CUASM_OK;
    cuasm_status_t st;
    DeviceGuard dg(h);
    if ((st = dg.status) != CUASM_OK) return st;
    CUASM_CHECK(h, cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    CUASM_CHECK(h, cudaMemcpy(dst, h->trace_buf, sizeof(unsigned long long) * 16 * h->trace_ctas,
                              cudaMemcpyDeviceToHost),
                "D2H trace");
    return CUASM_OK;
}

cuasm_status_t cuasm_ffn_destroy(cuasm_ffn_t h) {
    if (!h) return CUASM_OK;
    if (h->trace_buf) cudaFree(h->trace_buf);
    if (h->rstate) cudaFree(h->rstate);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : h->copy_events) cudaEventDestroy(e);
    if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
    if (h->d2h_stream) cudaStreamDestroy(h->d2h_stream);
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != h->device) cudaSetDevice(h->device);
    if (h->r) cudaFree(h->r);
    for (PackedWeights& w : h->pw)
        if (w.buf) cudaFree(w.buf);
    if (h->hidden) cudaFree(h->hidden);
    if (h->x2) cudaFree(h->x2);
    if (h->x_stage) cudaFree(h->x_stage);
    if (h->out_stage) cudaFree(h->out_stage);
    if (h->ws) cudaFree(h->ws);
    if (h->flags) cudaFree(h->flags);
    if (h->dyn) cudaFree(h->dyn);
    if (cur >= 0 && cur != h->device) cudaSetDevice(cur);
    delete h;
    return CUASM_OK;
}

const char* cuasm_ffn_last_error(cuasm_ffn_t h) { return h ? h->err.c_str() : g_init_error.c_str(); }

}  // extern "C"
