/*
 * cuasm_ffn.h -- C ABI of the B200-native fused RMSNorm + SwiGLU feed-forward.
 *
 *   out = SiLU(RMSNorm(x) . W1^T) (.) (RMSNorm(x) . W3^T),
 *   RMSNorm(x)[m,k] = x[m,k] * g[k] / sqrt( (sum_k x[m,k]^2)/K + eps )
 *
 * The operation is the "fused feed-forward ... for LLAMA" kernel of PAPER.md
 * P:68 (named fused_ff in Fig. "kernel throughput"; evaluated with
 * inputs B, M, N, K in Table "Evaluated Kernels", P:560 -- B is folded into
 * M = tokens here).  The paper never prints the formula; it is BASELINE.json's
 * north_star, with the readings listed in DESIGN.md (R1 W1 = SiLU branch,
 * R2 eps inside the sqrt, R3 RMS over x not x*g, R4 fold rounding).
 *
 * Design (BASELINE.json north_star): g is folded into W1/W3 once per weight
 * set (step a0, cached in the handle), a row-wise sum-of-squares pass
 * produces r[m] = 1/rms (a1), and one persistent tcgen05/TMEM/TMA dual-GEMM
 * kernel computes both contractions and applies r, SiLU and the gate in its
 * epilogue (a2 + a3).  By default a1 runs inside the GEMM kernel (see
 * CUASM_OPT_FUSED_NORM); the stand-alone pre-pass kernel remains available.  Everything runs on the caller's CUDA stream; there is
 * no CPU fallback: without an sm_100 device every entry point that would
 * compute returns CUASM_ERR_UNSUPPORTED or CUASM_ERR_CUDA.
 *
 * Conventions for every entry point:
 *   - Pointers named *_dev are CUDA device pointers, *_host are host pointers.
 *   - All matrices are dense row-major, no padding: x[M,K], w1/w3[N,K]
 *     (nn.Linear layout, K contiguous), out[M,N]; rms_w = g[K].
 *   - Element type is the handle's dtype for x, rms_w, w1, w3 AND out
 *     (CUASM_DTYPE_BF16: bfloat16; CUASM_DTYPE_FP32: float32, contracted on
 *     the tensor cores as TF32).  Accumulation is fp32.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Errors are return values; no entry point aborts or throws.  Argument
 *     validation happens before anything is enqueued: on error nothing is
 *     launched and `out` is untouched.  The message of the last error is
 *     kept per handle (cuasm_ffn_last_error).
 *   - A handle is bound to one device and is not thread-safe; use one
 *     handle per (thread, device).  Multi-GPU runs use one handle per rank.
 */
#ifndef CUASM_FFN_H
#define CUASM_FFN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUASM_FFN_ABI_VERSION 1

typedef struct cuasm_ffn_s* cuasm_ffn_t;

typedef enum {
    CUASM_OK = 0,
    CUASM_ERR_INVALID_ARG = 1, /* NULL/misaligned pointer, bad size, eps < 0 or NaN    */
    CUASM_ERR_UNSUPPORTED = 2, /* device is not compute capability 10.0 (B200, sm_100a) */
    CUASM_ERR_CUDA = 3,        /* a CUDA runtime/driver call or a launch failed          */
    CUASM_ERR_OOM = 4          /* device workspace allocation failed                    */
} cuasm_status_t;

typedef enum { CUASM_DTYPE_BF16 = 0, CUASM_DTYPE_FP32 = 1 } cuasm_dtype_t;

/* Activation of cuasm_gemm_act. */
typedef enum {
    CUASM_ACT_IDENTITY = 0,  /* out = acc                                   */
    CUASM_ACT_LEAKY_RELU = 1 /* out = acc >= 0 ? acc : alpha * acc           */
} cuasm_act_t;

/* Kernel-variant selector (cuasm_ffn_set_option with CUASM_OPT_VARIANT). */
typedef enum {
    CUASM_VARIANT_AUTO = 0, /* shape-keyed choice */
    CUASM_VARIANT_1SM = 1,  /* cta_group::1, 128 x 256 MMA tile per SM            */
    CUASM_VARIANT_2SM = 2   /* cta_group::2 CTA pair, 256 x 256 MMA tile per TPC  */
} cuasm_variant_t;

typedef enum {
    CUASM_OPT_VARIANT = 0, /* value: cuasm_variant_t                                   */
    CUASM_OPT_PDL = 1,     /* value: 1 = launch the GEMM with programmatic dependent
                              launch after the pre-pass (default), 0 = plain ordering */
    CUASM_OPT_GROUP_M = 2, /* value: m-blocks per rasterisation group (0 = auto)       */
    CUASM_OPT_PROFILE = 3, /* value: 1 = record CUDA events around each kernel of every
                              forward on its stream (read with cuasm_ffn_profile_read);
                              forces plain ordering (no PDL) so each kernel's span is
                              its own duration.  0 (default) = off                    */
    CUASM_OPT_SCHEDULE = 4, /* value: cuasm_schedule_t                                 */
    CUASM_OPT_TRACE = 5,    /* value: 1 = every dual-GEMM launch records per-CTA
                               %globaltimer stamps (read with cuasm_ffn_trace_read)   */
    CUASM_OPT_FUSED_NORM = 6, /* value: 1 (default) = step a1 runs inside the dual-GEMM
                               kernel (its epilogue warps compute r while the first
                               tile's mainloop runs; one launch per forward); 0 = the
                               separate pre-pass kernel, PDL-overlapped with the GEMM */
    CUASM_OPT_TILE_N = 7,     /* cuasm_gemm_act / down projection only: MMA N of a tile,
                               0 = auto (configuration model), 128 or 256              */
    CUASM_OPT_SK_SPLIT = 8,   /* auto schedule, fewer tiles than CTAs (pairs): at most
                               this many stream-K ranges per tile, 2..16 (0 = 2, the
                               default; each extra range is one more partial for the
                               tile's finisher to add)                                 */
    CUASM_OPT_L2_POLICY = 9,  /* L2 eviction policy of the TMA loads, 2 bits each: bits 0-1
                               x, bits 2-3 packed W13; 0 evict_normal, 1 evict_first,
                               2 evict_last.  Default 2 (x evict_last, W13 normal)    */
    CUASM_OPT_CSPLIT = 10,    /* 1-SM variant, fewer tiles than SMs: split every tile's
                               k-range over a cluster of S CTAs and reduce the partials
                               through distributed shared memory (bf16 tiles of <= 32
                               rows: pushed into the owner CTA with st.async; else
                               pulled with ld.shared::cluster); summed in rank order,
                               so results are bitwise reproducible.  0 = the
                               configuration model decides (decode shards, M <= 32),
                               1 = off, 2..8 = S (used only when tiles * S <= SMs,
                               S <= k-blocks and S clusters fit co-resident)           */
    CUASM_OPT_TILE_BN = 11,   /* fused FFN, bf16: SwiGLU outputs per tile BN (MMA N = 2 BN):
                               0 = the configuration model decides; 128, 120, 112, 96,
                               80 or 64 forces it (widths below 128 run the 2-SM kernel; a
                               forced 1-SM variant keeps 128, except 64, which the 1-SM
                               decode paths have too).  The folded weights are cached
                               once per width in use, so a weight set served at shapes
                               whose plans differ in BN (decode shards take 64, prefill
                               shards 80-112) holds one packed copy per width    */
    CUASM_OPT_DYNAMIC = 12,   /* data-parallel tiles of the persistent GEMM claimed from a
                               global counter (each cluster's first tile static, the rest
                               claimed one tile ahead by its leader CTA) instead of the
                               static round-robin: the tiles in flight stay consecutive
                               in the rasterisation order (L2 reuse) and fast SM pairs
                               take more tiles.  0 = auto (on when every cluster has >= 24
                               data-parallel tiles), 1 = off, 2 = on (whenever there is
                               more than one round).  Results are bitwise independent of
                               the claim order (each tile is computed whole by one
                               cluster)                                               */
    CUASM_OPT_RS_PARTIAL = 13 /* fused reduction (cuasm_ffn_block_forward_rs / cuasm_rs_reduce,
                               which must agree): 0 (default) = the partials travel and are
                               staged as fp32; 1 = as bf16 (RNE: half the NVLink bytes, one
                               extra rounding per partial; the owner still sums in fp32 in
                               rank order).  Staging then needs half of cuasm_rs_layout's
                               stage_bytes                                            */,
    CUASM_OPT_L2_PERSIST = 14 /* DEVICE-WIDE (cudaDeviceSetLimit): bytes of L2 set aside for
                               persisting lines -- the x tiles' TMA loads carry an
                               evict_last hint (CUASM_OPT_L2_POLICY); 0 = none (default).
                               Affects every kernel on the device                     */,
    CUASM_OPT_MCAST = 15      /* fused FFN, 2-SM bf16: 1 = 4-CTA clusters of two CTA pairs on
                               two vertically adjacent 256-row tiles of one n-block; the
                               pair-0 CTAs TMA-load each W13 half once and multicast it into
                               both pairs' shared memory (.multicast::cluster); whole tiles
                               only (no stream-K, no dynamic claiming).  0 = off (default) */,
    CUASM_OPT_THIN_A = 16     /* decode shards on 64-output tiles with the cluster split-K
                               (M <= 32): 1 = pipeline stages hold 32 A rows instead of
                               128 (4 KB instead of 16 KB), so more stages of weights are
                               in flight per SM; 0 (default) = full A stages (the deeper
                               pipeline measured no faster: the decode shards are bound
                               by fixed latencies, not by bytes in flight)            */,
    CUASM_OPT_TALL = 17       /* fused FFN, bf16, 256 < M <= 384 (the crossover region):
                               tall tiles -- one 80-output n-block over all rows, a
                               256-row tcgen05.mma (M = 256) and a 128-row one (M = 128,
                               cta_group::2) on the same weight stage, so each W13 block
                               is streamed once (DESIGN.md §6 "Tall tiles").  0 = the
                               configuration model decides (default), 1 = off, 2 = on
                               whenever the shape allows                               */
} cuasm_option_t;

/* Persistent tile schedule of the dual GEMM (cuasm_ffn_set_option with
 * CUASM_OPT_SCHEDULE).  Stream-K splits k-block ranges of the tail tiles
 * across CTAs (fp32 partials through a handle-owned workspace, fixed
 * reduction order: results stay bitwise run-to-run deterministic). */
typedef enum {
    CUASM_SCHEDULE_AUTO = 0,          /* whole tiles while they fill complete waves, stream-K
                                         over the last partial wave + one full wave         */
    CUASM_SCHEDULE_DATA_PARALLEL = 1, /* whole tiles only                                      */
    CUASM_SCHEDULE_STREAM_K_ALL = 2,  /* stream-K over every tile (testing)                     */
    CUASM_SCHEDULE_STREAM_K_TAIL = 3  /* whole tiles for every complete wave, stream-K over the
                                         last partial wave only                                */
} cuasm_schedule_t;

/* Create a handle on `device` (CUDA ordinal) for element type `dtype`.
 * Returns UNSUPPORTED if the device is not CC 10.0, CUDA on any runtime error.
 * On success *h owns no device memory yet (allocated lazily, on demand). */
cuasm_status_t cuasm_ffn_init(cuasm_ffn_t* h, int device, cuasm_dtype_t dtype);

/* The whole hot path for one batch of tokens (PAPER.md P:560 inputs M, N, K):
 *   a0 (only when the weight key (rms_w, w1, w3, K, N) differs from the cached
 *      one, or after cuasm_ffn_invalidate_weights): fold g into W1/W3 and pack
 *      them into the handle-owned W13 buffer, on `stream`;
 *   a1 r[m] = 1/sqrt(sum_k x^2 / K + eps) into a handle-owned fp32 workspace;
 *   a2+a3 out = bf16( SiLU(r*x.W1g^T) * (r*x.W3g^T) ).
 * x_dev [M,K], rms_w_dev [K], w1_dev/w3_dev [N,K], out_dev [M,N]: device
 * pointers, 16-byte aligned, caller-owned; out is fully overwritten.
 * Preconditions (else INVALID_ARG, nothing launched): pointers non-NULL and
 * 16-byte aligned, M >= 0, K > 0, N > 0, K % 8 == 0, N % 8 == 0,
 * M, N < 2^31, eps >= 0 and not NaN.  M == 0 returns OK without launching.
 * Weights must not change while cached (else call invalidate_weights).
 * Asynchronous: returns after enqueueing; out is valid once `stream` reaches
 * this point. */
cuasm_status_t cuasm_ffn_forward(cuasm_ffn_t h, const void* x_dev, const void* rms_w_dev, const void* w1_dev,
                                 const void* w3_dev, void* out_dev, int64_t M, int64_t K, int64_t N, float eps,
                                 void* stream);

/* Tensor-parallel forward with step a4 (the all-gather of the column shards,
 * SURVEY §8(e)/(f) f2) fused into the epilogue: the same computation as
 * cuasm_ffn_forward on this rank's shard (w1_dev/w3_dev = rows [n0, n0+N) of
 * the full W1/W3, N = the shard width), but every staged 32 x 32 output box is
 * written to each destination (one TMA store per destination) instead of one
 * local buffer, tile by tile while the next tile's mainloop runs -- the gather
 * overlaps the math and no separate collective or interleave pass runs.
 *   dst[q] (q < num_dst <= 8): device address of THIS shard's column 0 inside
 *     rank q's full row-major [M, ldo] output, i.e. base_q + n0 * elemsize;
 *     base_q mapped into this device's address space (CUDA IPC / symmetric
 *     memory peer pointers; stores travel over NVLink).  num_dst = 1 with a
 *     local pointer is the plain forward with an output stride.
 *   multicast = 1: num_dst must be 1 and dst[0] is an NVLS multicast address
 *     (+ n0 * elemsize) bound to every rank's output buffer; each 16-byte store
 *     is issued once as multimem.st.relaxed.sys and NVSwitch replicates it.
 *   ldo: row stride of every destination, elements, >= N, multiple of 16 bytes.
 * Visibility: a rank's full output is complete once EVERY rank's launch has
 * completed and a cross-rank barrier ordered after those launches has
 * returned on the reading rank (e.g. the symmetric-memory barrier on the same
 * stream); this call issues no cross-rank synchronisation itself.
 * Other preconditions and errors as cuasm_ffn_forward (destinations 16-byte
 * aligned, non-NULL; INVALID_ARG before any launch). */
cuasm_status_t cuasm_ffn_forward_gather(cuasm_ffn_t h, const void* x_dev, const void* rms_w_dev, const void* w1_dev,
                                        const void* w3_dev, void* const* dst, int num_dst, int multicast,
                                        int64_t ldo, int64_t M, int64_t K, int64_t N, float eps, void* stream);

/* End-to-end variant for host-resident activations: copies x_host [M,K]
 * (ideally pinned) to a handle-owned device buffer, runs cuasm_ffn_forward
 * with the device-resident weights, and copies the result back into
 * out_host [M,N].  For M >= 1024 the rows are processed in up to 8 chunks
 * whose H2D copy, forward and D2H copy overlap on two handle-owned copy
 * streams; `stream` waits for all of it before returning control of its
 * queue, so work enqueued on `stream` afterwards sees out_host complete.
 * Synchronous w.r.t. the host only if `sync` != 0 (otherwise out_host is
 * valid after the stream completes, and both host buffers must be pinned).
 * Same preconditions as cuasm_ffn_forward. */
cuasm_status_t cuasm_ffn_forward_host(cuasm_ffn_t h, const void* x_host, const void* rms_w_dev, const void* w1_dev,
                                      const void* w3_dev, void* out_host, int64_t M, int64_t K, int64_t N, float eps,
                                      void* stream, int sync);

/* GEMM with a fused activation on the same tcgen05/TMA machinery:
 *   out[m,n] = act( sum_k x[m,k] * w[n,k] ),   act = cuasm_act_t, alpha its slope.
 * The paper's "mmLeakyReLu" kernel (Table "Evaluated Kernels"
 * B,M,N,K = 1,512,512,2048; matmul + LeakyReLU epilogue, the kernel of
 * its Table 3 SASS analysis P:630-652) and, with CUASM_ACT_IDENTITY, the FFN's
 * down projection.  x [M,K], w [N,K] (nn.Linear layout), out [M,N]: device,
 * 16-byte aligned, the handle's dtype; w is packed into a handle-owned cache
 * (slot separate from the W1/W3 cache) on first use.  Same size and error
 * rules as cuasm_ffn_forward (K % 8 == 0, N % 8 == 0, M == 0 -> no launch). */
cuasm_status_t cuasm_gemm_act(cuasm_ffn_t h, const void* x_dev, const void* w_dev, void* out_dev, int64_t M,
                              int64_t K, int64_t N, int act, float alpha, void* stream);

/* The whole LLaMA feed-forward block (PAPER.md P:68's fused
 * feed-forward followed by its down projection):
 *   out[m,k] = sum_n hidden[m,n] * w2[k,n],
 *   hidden   = SiLU(RMSNorm(x) W1^T) (.) (RMSNorm(x) W3^T)   stored in the handle dtype
 * x [M,K], rms_w [K], w1/w3 [N,K], w2 [K,N] (nn.Linear(N -> K) layout),
 * out [M,K]; two kernel launches (the fused FFN, then cuasm_gemm_act's GEMM
 * with identity activation) through a handle-owned hidden buffer.  Same
 * preconditions as cuasm_ffn_forward; w2 16-byte aligned. */
cuasm_status_t cuasm_ffn_block_forward(cuasm_ffn_t h, const void* x_dev, const void* rms_w_dev, const void* w1_dev,
                                       const void* w3_dev, const void* w2_dev, void* out_dev, int64_t M, int64_t K,
                                       int64_t N, float eps, void* stream);

/* Tensor-parallel FFN block with the row-parallel reduction fused into the down
 * projection (DESIGN.md §8 "Fused reduction").  Megatron split
 * over `world` ranks: rank `rank` holds w1/w3 [N,K] = its rows of W1/W3 and w2
 * [K,N] = the same N columns of W2 (N = this rank's N_l); its partial
 *   y_rank[m,k] = sum_{n in shard} hidden[m,n] * w2[k,n]
 * never lands in local memory: the output columns are owned in 256-column blocks
 * split evenly over the ranks (cuasm_rs_layout), and every fp32 partial tile is
 * stored by the GEMM epilogue (TMA) straight into the owner q's staging buffer,
 *   stage[q] + rank * M * Kq * 4 bytes, layout [M][Kq] fp32, Kq = q's column count,
 * so the transfer overlaps the GEMM tile by tile.  stage[q] is rank q's staging
 * buffer base ([world][M][Kq] fp32, cuasm_rs_layout's stage_bytes; device memory
 * of any rank reachable from this GPU: peer / symmetric-memory pointers), 16-byte
 * aligned; entries of ranks owning no columns may be NULL.  bf16 handles only.
 * Two launches (fused FFN, W2 GEMM).  The stores are complete when the stream's
 * work is; the caller orders them with a cross-rank barrier before any owner
 * runs cuasm_rs_reduce.  Errors as cuasm_ffn_block_forward, plus world in [1, 8],
 * 0 <= rank < world. */
cuasm_status_t cuasm_ffn_block_forward_rs(cuasm_ffn_t h, const void* x_dev, const void* rms_w_dev,
                                          const void* w1_dev, const void* w3_dev, const void* w2_dev,
                                          void* const* stage, int world, int rank, int64_t M, int64_t K, int64_t N,
                                          float eps, void* stream);

/* The owner side of f1: y[:, col0:col1] = RNE_bf16( sum_{p = 0..world-1} stage[p][:, :] )
 * summed in fp32 in rank order (bitwise independent of arrival order), written into
 * every destination dst[0..num_dst) -- each rank's full [M, ldo] bf16 output
 * (P2P), so reduce-scatter + this all-gather is the all-reduce -- or, multicast
 * = 1, once to the NVLS multicast address dst[0] (multimem.st).  stage: this
 * rank's staging buffer (device, 16-byte aligned); [col0, col1) from
 * cuasm_rs_layout(M, K, world, rank).  One HBM-bound launch; no launch when the
 * rank owns no columns or M == 0. */
cuasm_status_t cuasm_rs_reduce(cuasm_ffn_t h, const void* stage_dev, int world, int rank, void* const* dst,
                               int num_dst, int multicast, int64_t ldo, int64_t M, int64_t K, void* stream);

/* f1 ownership (pure host code): rank `rank` of `world` reduces output columns
 * [*col0, *col1) of a [M, K] block output; its staging buffer holds
 * *stage_bytes = world * M * (col1 - col0) * 4 bytes.  CUASM_ERR_INVALID_ARG on
 * K <= 0, K % 8 != 0, world outside [1, 8] or rank outside [0, world). */
cuasm_status_t cuasm_rs_layout(int64_t M, int64_t K, int world, int rank, int64_t* col0, int64_t* col1,
                               int64_t* stage_bytes);

/* Stand-alone RMSNorm (the paper's memory-bound "rmsnorm"
 * kernel, PAPER.md P:68 / P:523 / P:573):
 *   out[m,k] = x[m,k] * g[k] / sqrt( (sum_k x[m,k]^2)/K + eps )
 * x, out [M,K], rms_w = g [K]: device, 16-byte aligned, the handle's dtype
 * (bf16 out is RNE of the fp32 product).  K % 8 == 0; M == 0 -> no launch;
 * eps >= 0.  One kernel, x read from HBM once for K <= 4096 (bf16). */
cuasm_status_t cuasm_rmsnorm(cuasm_ffn_t h, const void* x_dev, const void* rms_w_dev, void* out_dev, int64_t M,
                             int64_t K, float eps, void* stream);

/* Step a0 alone: fold g into W1/W3 and pack (one-time weight preparation,
 * PAPER.md P:434-447's offline/deploy split).  Same weight preconditions. */
cuasm_status_t cuasm_ffn_prepare(cuasm_ffn_t h, const void* rms_w_dev, const void* w1_dev, const void* w3_dev,
                                 int64_t K, int64_t N, void* stream);

/* Step a1 alone: r_dev[m] = 1/sqrt(sum_k x[m,k]^2/K + eps), fp32, M floats.
 * r_dev is caller-owned device memory (4-byte aligned). */
cuasm_status_t cuasm_ffn_rms_inv(cuasm_ffn_t h, const void* x_dev, float* r_dev, int64_t M, int64_t K, float eps,
                                 void* stream);

/* Copy the packed, g-folded weights (a0's output) to host memory for
 * inspection.  Layout (k-block tiled; BK = 128 bytes of K = 64 bf16 / 32 fp32
 * elements, NB = 128 outputs): element [nb][kb][j*128 + rr][i] =
 * RNE(W_j[nb*128 + rr, kb*BK + i] * g[kb*BK + i]), j = 0 for W1, 1 for W3,
 * zero where the row is past N or the column past K; nb < ceil(N/128),
 * kb < ceil(K/BK).  *bytes receives the size; pass dst_host = NULL to query
 * it.  Synchronous. */
cuasm_status_t cuasm_ffn_get_packed(cuasm_ffn_t h, void* dst_host, int64_t* bytes);

/* Drop the cached packed weights; the next forward re-packs. */
cuasm_status_t cuasm_ffn_invalidate_weights(cuasm_ffn_t h);

/* Set a tuning option (cuasm_option_t).  INVALID_ARG for unknown keys/values. */
cuasm_status_t cuasm_ffn_set_option(cuasm_ffn_t h, int option, int64_t value);

/* Which GEMM variant the last forward launched (cuasm_variant_t), and the
 * number of kernels it enqueued (0 when M == 0). */
cuasm_status_t cuasm_ffn_last_launch(cuasm_ffn_t h, int* variant, int* kernels);

/* With CUASM_OPT_PROFILE on: wait for the recorded forwards, return the
 * summed device time (ms) of the pre-pass kernels and of the dual-GEMM
 * kernels and the number of forwards recorded, then reset the record.
 * Synchronous.  Any output pointer may be NULL. */
cuasm_status_t cuasm_ffn_profile_read(cuasm_ffn_t h, double* prepass_ms, double* gemm_ms, int* forwards);

/* With CUASM_OPT_TRACE on: copy the last traced dual-GEMM launch's per-CTA
 * timeline into dst_host[ctas][16] (ns, %globaltimer; slots: 0 entry, 1 first
 * TMA load issued, 2 last TMA load issued, 3 last MMA issued, 4 epilogue start,
 * 5 epilogue done, 6 exit, 7 final tile handed to the epilogue, 8 first tile
 * handed over, 9 first tile's epilogue done, 10 final tile's stream-K
 * partials acquired, 11 final tile's epilogue done; 0 = not reached).  *ctas receives the CTA count
 * (pass dst_host = NULL to query it).  Synchronous. */
cuasm_status_t cuasm_ffn_trace_read(cuasm_ffn_t h, unsigned long long* dst_host, int* ctas);

/* Free all handle-owned device memory and the handle.  NULL is accepted. */
cuasm_status_t cuasm_ffn_destroy(cuasm_ffn_t h);

/* Message of the last error on this handle ("" if none; valid until the next
 * call on the handle).  h == NULL returns the last init error. */
const char* cuasm_ffn_last_error(cuasm_ffn_t h);

/* The shape-keyed configuration model the AUTO variant and
 * schedule use, without a handle or a device: for `sm_count` SMs, element
 * type `dtype`, problem M x K x N and op (0: fused FFN, 128 outputs per tile;
 * 1: GEMM + activation, 256- or 128-output tiles) it returns the chosen
 * cuasm_variant_t and in *stream_k bit 0 = stream-K tail used, bit 1 = the
 * 128-wide tile, bits 4..7 = the cluster split-K width (CTAs per tile, 0 =
 * none; see CUASM_OPT_CSPLIT), bits 8..15 = the SwiGLU outputs per tile BN
 * (see CUASM_OPT_TILE_BN), bit 2 = tall tiles (see CUASM_OPT_TALL).  Pure host
 * code. */
cuasm_status_t cuasm_plan_config(int sm_count, int dtype, int64_t M, int64_t K, int64_t N, int op, int* variant,
                                 int* stream_k);

/* The paper's autotuner and its offline-search / deploy-time-lookup workflow (PAPER.md
 * "enumerates user-provided kernel configurations ..., measures the execution
 * throughput on the target GPU, and greedily selects as well as caches the optimal set of
 * kernel configurations", the mean of repeated executions after warm-up; results
 * written "prefixed by GPU type, workload type etc., as the key to lookup", looked up at
 * deployment instead of searched).
 *
 * cuasm_ffn_tune: runs the fused FFN out = SiLU(RMSNorm(x) W1^T) * (RMSNorm(x) W3^T) --
 * arguments exactly as cuasm_ffn_forward, bf16 handles only -- under every candidate
 * configuration of the dual GEMM for this M x K x N (the cost model's choice, each 2-SM tile
 * width with whole tiles and a stream-K tail, the 1-SM tile, tall tiles where 256 < M <= 384,
 * the 1-SM cluster split-K of 2..8 CTAs), in three interleaved rounds (so clock and power
 * drift spread over all candidates): per round `warmup` untimed forwards (at least one: the first
 * packs the tile width's weights and sizes the workspaces before the graph capture), then `iters` timed
 * ones -- flush_l2 = 0: back to back between one CUDA-event pair on `stream`; flush_l2 = 1:
 * each after an L2 flush (a 2x-L2 buffer written, another read; the paper's evaluation
 * protocol) inside its own event pair, as one CUDA-graph launch of the forward (captured
 * after the warm-up; eager when `stream` is the legacy NULL stream, which cannot be captured)
 * -- a candidate's time being the best round's
 * mean per forward.  It keeps the fastest in the handle's table (replacing an entry of the
 * same shape) and returns it in *variant /
 * *flags (the encoding of cuasm_plan_config) and *best_us (any of them may be NULL).  From
 * then on forwards of exactly this shape on this handle use it instead of the configuration
 * model.  SYNCHRONOUS (waits for `stream`); writes `out` many times; packs the weights once
 * per tile width tried (handle memory).  Errors: INVALID_ARG as for a forward, M == 0,
 * warmup < 0, iters < 1 or flush_l2 not 0/1; UNSUPPORTED for fp32 handles; OOM if the flush
 * buffer (4x L2, freed on return) cannot be allocated; a candidate the shape cannot run
 * is skipped, any CUDA error aborts the search and is returned.
 *
 * cuasm_ffn_tuned_export: the table as text, one line per entry,
 *   "cuasm-tuned v1 sm=<SMs> dtype=bf16 M=<M> K=<K> N=<N> variant=<v> flags=<f> us=<t> gpu=<name>\n",
 * NUL-terminated, into buf[cap]; *needed = bytes required (incl. the NUL).  cap = 0 only
 * queries the size; 0 < cap < *needed is INVALID_ARG (nothing written).
 *
 * cuasm_ffn_tuned_import: adds (or replaces, per shape) the entries of `text` whose GPU name,
 * SM count and dtype match this handle's device; other lines (comments, other GPUs) are
 * ignored; *accepted = entries taken.  A matching but malformed entry is INVALID_ARG (the
 * entries before it stay imported).  cuasm_ffn_tuned_clear empties the table. */
cuasm_status_t cuasm_ffn_tune(cuasm_ffn_t h, const void* x, const void* rms_w, const void* w1, const void* w3,
                              void* out, int64_t M, int64_t K, int64_t N, float eps, int warmup, int iters,
                              int flush_l2, void* stream, int* variant, int* flags, float* best_us);
/* cuasm_gemm_act_tune: the same search for the GEMM + activation op (cuasm_gemm_act: the paper's
 * mmLeakyReLu, and the FFN block's down projection): arguments as cuasm_gemm_act plus
 * warmup / iters / flush_l2 / outputs as above; candidates the cost model's choice and each variant
 * x {whole tiles, stream-K} x {256, 128}-wide tiles; the winner is used by later cuasm_gemm_act
 * calls of this M x K x N on the handle (and by block forwards whose down projection has it).  Its
 * exported lines carry "op=gemm " before "gpu=". */
cuasm_status_t cuasm_gemm_act_tune(cuasm_ffn_t h, const void* x, const void* w, void* out, int64_t M, int64_t K,
                                   int64_t N, int act, float alpha, int warmup, int iters, int flush_l2, void* stream,
                                   int* variant, int* flags, float* best_us);
cuasm_status_t cuasm_ffn_tuned_export(cuasm_ffn_t h, char* buf, int64_t cap, int64_t* needed);
cuasm_status_t cuasm_ffn_tuned_import(cuasm_ffn_t h, const char* text, int* accepted);
cuasm_status_t cuasm_ffn_tuned_clear(cuasm_ffn_t h);
/* The last cuasm_ffn_tune's search, candidate by candidate in the order measured: *n =
 * candidates; the first min(cap, *n) variants / flags (cuasm_plan_config encoding) / mean us
 * per forward (-1 = the shape cannot run it) are written.  cap = 0 only queries *n. */
cuasm_status_t cuasm_ffn_tune_log(cuasm_ffn_t h, int cap, int* n, int* variants, int* flags, float* us);

/* CUASM_FFN_ABI_VERSION of the loaded library. */
int cuasm_ffn_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CUASM_FFN_H */
