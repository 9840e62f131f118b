// dual_gemm.cuh -- the persistent tcgen05 kernel behind every GEMM of the
// library: steps a1 (fused row inverse-RMS), a2 and a3 of the fused FFN, and
// the GEMM + activation mode (mmLeakyReLu, the FFN block's down projection).
//
//   FFN (kEpi 0):  acc[m, 0:128]   = sum_k x[m,k] * W1g[n0 + j, k]   (h1 / r)
//                  acc[m, 128:256] = sum_k x[m,k] * W3g[n0 + j, k]   (h3 / r)
//                  out[m, n0 + j]  = RNE( h1 * sigma(h1) * h3 ),  h1 = r[m]*acc1, h3 = r[m]*acc3
//   GEMM (kEpi 1): out[m, n0 + j]  = RNE( act( acc[m, j] ) )
//
// (BASELINE.json north_star: dual GEMM on tcgen05.mma with TMEM accumulators
// fed by TMA, 1/rms scale + SiLU + product fused in the epilogue; the paper's
// fused_ff, PAPER.md P:68 / P:560.)  One MMA of N = 256 over the interleaved
// W13 block (pack.cuh) yields both halves of the gate for the same outputs.
//
// Kernel structure (persistent, one CTA per SM, warp-specialised, 320 threads):
//   warp 0      TMA producer: the warp walks the k-block loop, an elected lane
//               issues the x tile [BM x BK] and weight tile [B_ROWS x BK] loads
//               per stage (128-byte swizzle, mbarrier transaction counts)
//   warp 1      TMEM allocator + MMA issuer: the warp walks the loop, an elected
//               lane issues 4 x tcgen05.mma (K=16 bf16 / K=8 tf32) per stage and
//               the tcgen05.commit that frees it; a final commit per tile hands
//               the accumulator to the epilogue
//   warps 2..9  epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes 32*(w%4)..+31
//               = tile rows, and half of the accumulator columns), r-scale,
//               activation / SiLU gate, bf16 pack, staged TMA stores (fp32:
//               16-byte global stores); at kernel entry they also compute r for
//               a 1/grid slice of the rows
// TMEM holds two UMMA_N-column accumulators so the epilogue of tile i overlaps
// the mainloop of tile i+1.  The schedule (Sched) is whole tiles, optionally
// followed by a stream-K tail whose partials go through a global workspace, or
// (1-SM, few tiles) a cluster split-K: the S CTAs of a cluster share one tile's
// k-range and reduce through distributed shared memory (split_k_push /
// split_k_reduce).
//
// kCtaGroup == 2 (2-SM variant): a cluster of two CTAs on one TPC computes a
// 256 x UMMA_N tile with tcgen05.mma.cta_group::2.  Each CTA TMA-loads its own
// 128 rows of x and HALF of the weight block (FFN: rank 0 the W1g rows, rank 1
// the W3g rows), both crediting the leader's barrier; only the leader issues
// the MMAs; commits multicast to both CTAs; each CTA's epilogue drains its own
// 128 accumulator rows (its own TMEM).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <type_traits>

#include "prepass.cuh"
#include "ptx.cuh"

namespace cuasm {

struct FfnGemmParams {
    const void* x;   // [M, K] activations (fused RMS pass reads them directly)
    float eps;
    int fused_norm;  // 1: this kernel computes r itself (no pre-pass kernel)
    int use_r;       // 1: scale the accumulators by r[m] (RMSNorm); 0: r = 1 (plain GEMM)
    int act;         // kEpi == 1 only: 0 identity, 1 LeakyReLU with negative slope `alpha`
    float alpha;
    // Fused a1 bookkeeping (self-resetting, DESIGN.md §6 "Fused a1"): r is computed per
    // 128-row r-block on demand by the CTAs that need it.  rstate[rb] counts rows of
    // r-block rb taken, rstate[n_rblk + rb] rows done (published), rstate[2 n_rblk] the
    // epilogue warps past their last r acquisition (the last one resets everything).
    uint32_t* rstate;
    int n_rblk;      // r-blocks: ceil(M / 128)
    float* r;        // [M] inverse RMS (written here when fused_norm, else by the pre-pass)
    void* out;       // [M, ldo] row-major, dtype of the handle (== dst[0] unless multicast)
    int64_t ldo;     // leading dimension of out / every dst, elements
    // Step a4 fused into the epilogue: every output store goes to
    // dst[0..num_dst) -- this shard's column 0 inside each rank's full [M, ldo]
    // output (peer pointers: P2P stores over NVLink) -- or, with dst_mc, once to
    // the NVLS multicast address dst[0] (multimem.st: the switch replicates it).
    void* dst[8];
    int num_dst;     // 1..8 (1 = plain local output)
    int dst_mc;      // 1: dst[0] is a multicast address
    // f1 fused reduce-scatter (kEpi 1; DESIGN.md §8 "Fused reduction"): rs_world
    // > 0 makes every output tile an fp32 partial that leaves through omaps.m[q], q = the rank
    // owning the tile's 256-column block (blocks split evenly over rs_world ranks), into q's
    // staging slot for this rank at column col - col0(q); 0 = off
    int rs_world;
    int rs_nblk;     // 256-column blocks of the output: ceil(N / 256)
    int rs_bf16;     // 1: the partials travel as bf16 (RNE; half the bytes), 0: fp32
    int M, N, K;
    int num_m_blk;   // ceil(M / tile_m)
    int num_n_blk;   // ceil(N / OUT_COLS)
    int num_k_blk;   // ceil(K / BK)
    int group_m;     // rasterisation: m-blocks per group (L2 reuse of W13 blocks)
    int a_box_bytes; // bytes of one x TMA box (rows actually loaded x 128 B; < BM rows when M < BM)
    int tma_store;   // 1: bf16 output tiles leave through TMA stores (omaps.m[0..num_dst), one per
                     // destination); 0: 16-byte st.global (fp32 handles, multicast destinations)
    int csplit;      // 1-SM only: S > 0 = cluster split-K: a cluster of S CTAs owns one
                     // tile, CTA rank j computes k-blocks [j*KB/S, (j+1)*KB/S) and the S partial
                     // accumulators are reduced through distributed shared memory; 0 = off
    int l2pol;       // TMA L2 policies: bits 0-1 x, bits 2-3 W13 (0 evict_normal, 1 evict_first, 2 evict_last)
    int w_early;     // 1: the packed weights predate the preceding kernel, so the producer may
                     // load the first pipeline stages' weights before griddepcontrol.wait
    int rep;         // 4 (SwiGLU, M <= 32) / 2 (M <= 64) / 0; 2-SM: the leader CTA.  The x rows are
                     // loaded rep times into the A tile (at smem rows q*128/rep), so every TMEM
                     // lane quadrant holds rows and the epilogue spreads the column pairs over
                     // the four SM sub-partitions (warp w may only read quadrant w%4: without
                     // this a decode tile's whole epilogue runs on sub-partition 0 or 0-1)
    int num_tiles;
    // --- persistent schedule: data-parallel tiles, then a stream-K region ---
    int num_clusters;   // persistent clusters (CTA pairs for the 2-SM variant)
    int num_dp_tiles;   // tiles [0, num_dp_tiles) round-robin, whole
    int64_t sk_iters;   // (num_tiles - num_dp_tiles) * num_k_blk k-block iterations,
                        // split into num_clusters contiguous ranges
    float* ws;          // stream-K partials: per (cluster, cta rank) a BM x UMMA_N fp32 slot in the
                        // lane-contiguous layout [chunk][quad][8 float4][32 lanes] (see the epilogue)
    unsigned long long* trace;  // optional [gridDim.x][16] stamps / counters (CUASM_OPT_TRACE), or null
    uint32_t* flags;    // [cluster][cta rank][8 epilogue warps]: 1 = partial published;
                        // the finisher consumes (resets to 0) it, so launches need no
                        // per-launch state and the kernel can be replayed from a CUDA graph
    // Dynamic whole-tile claiming (DESIGN.md §6 "Dynamic tiles"): dyn != null makes every
    // cluster's data-parallel tiles after its first come from a global claim counter, so
    // the tiles in flight stay consecutive in the rasterisation order (L2 reuse) and fast
    // SM pairs absorb slow ones.  dyn[0] claim counter, dyn[1] clusters done, dyn[2]
    // launch epoch (the last cluster resets [0], [1] and advances [2]: graph-safe), then
    // per cluster a ring of kDynRing (tag, tile) words published by the leader's producer.
    uint32_t* dyn;
};

constexpr int kDynRing = 8;           // published-tile ring per cluster (u64 slots)
constexpr int kDynEnd = 0x7fffffff;   // "no more data-parallel tiles"

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// A unit of work: k-blocks [kb0, kb1) of tile `tile`.
struct Seg {
    int tile, kb0, kb1;
};

// Stream-K arithmetic in 32 bits: the host guarantees sk_iters * num_clusters < 2^32
// (launch_gemm), and 64-bit divisions compile to a subroutine call whose first,
// instruction-cache-cold execution put ~1 us between griddepcontrol.wait and the
// first TMA of every launch (per-CTA trace).
__device__ __forceinline__ int64_t sk_begin(const FfnGemmParams& p, int c) {
    return static_cast<int64_t>(static_cast<uint32_t>(p.sk_iters) * static_cast<uint32_t>(c) /
                                static_cast<uint32_t>(p.num_clusters));
}

// The cluster whose stream-K range holds iteration i.
__device__ __forceinline__ int sk_owner(const FfnGemmParams& p, int64_t i) {
    int c = static_cast<int>(static_cast<uint32_t>(i) * static_cast<uint32_t>(p.num_clusters) /
                             static_cast<uint32_t>(p.sk_iters > 0 ? p.sk_iters : 1));
    while (c + 1 < p.num_clusters && sk_begin(p, c + 1) <= i) ++c;
    while (c > 0 && sk_begin(p, c) > i) --c;
    return c;
}

// Per-cluster walk over its work: first whole data-parallel tiles
// (cluster, cluster + C, ...), then its contiguous stream-K iteration range
// cut at tile boundaries and walked BACKWARDS (from the range's end).  Every
// role of the CTA (producer, MMA, epilogue) walks the identical sequence.  In
// a stream-K range only the first segment walked can end mid-tile (it holds
// the start of a tile whose end belongs to a higher cluster: a "contributor",
// it publishes an fp32 partial) and only the last walked can start mid-tile
// while holding the tile's last k-block (the "finisher": it adds the partials
// of the LOWER clusters holding the rest of the tile and runs the epilogue).
// Waits therefore point only to lower cluster ids -- CTAs dispatched earlier,
// resident or done -- so the schedule needs no co-residency of the grid, and a
// contributor publishes its partial first thing while the finisher adds it last.
//
// Dynamic mode (p.dyn): a cluster's first data-parallel tile is its cluster id; the
// later ones are claimed by the leader CTA's producer from the global counter ahead of
// use (the atomic for tile i+3 is issued when it starts tile i, its result published in
// the cluster's ring when it starts tile i+1, so tile i+1 is in the ring a whole tile
// before anyone needs it), and the other producer and the epilogue warps load the next
// tile's slot when they start a tile and use it when they start the next one; the MMA
// warp reads only segment lengths, from shared memory (seg_nkb).  Neither the claim's nor
// the loads' L2 round trips sit on a role's critical path; the published words carry only
// the tile number, so relaxed accesses suffice (a tag = launch epoch + tile index tells a
// published slot from a stale one; a role that finds it stale spins, which the two-tile
// lead makes rare).  (A just-in-time variant -- claims issued a fixed number of k-blocks
// before each tile's end, so slow pairs claim late -- measured slower everywhere: the
// claim and prefetch hooks inside the producer's k-loop cost more than the balance gained.)  The producer runs STAGES k-blocks ahead of the
// MMA and the MMA at most one tile ahead of the epilogue, so the kDynRing slots of a ring
// are never overwritten before their readers are done.  The stream-K region after the
// data-parallel tiles stays static per cluster.
// kDyn = false compiles the dynamic code out: the producer and MMA roles run a static
// instance when p.dyn is null, so their loops keep warp-uniform control flow (the MMA
// issue loop is latency-critical: a lane-0-only branch in the schedule
// made ptxas add divergence checks and move the stage arithmetic out of uniform
// registers, 340 -> 434 SM cycles per k-block on the 80-wide tile).
template <bool kDyn = true>
struct SchedT {
    int next_dp, C, KB, T_dp, kb_lo, kb_hi;
    int64_t beg, cur;  // stream-K range [beg, cur) still to walk (cur moves down)
    uint32_t* dyn;     // dynamic claiming (null: static round-robin)
    unsigned long long* ring;
    uint32_t epoch;
    int dyn_i;         // index of the next data-parallel tile of this cluster
    bool fetch, claimer;
    unsigned long long pre;  // (dynamic) the slot of tile dyn_i, loaded one tile ahead
    uint32_t claim;          // (claimer) the counter value claimed for tile dyn_i + 1
    __device__ __forceinline__ void init(const FfnGemmParams& p, int cluster, int part = 0, bool is_claimer = false) {
        next_dp = cluster;
        C = p.num_clusters;
        KB = p.num_k_blk;
        T_dp = p.num_dp_tiles;
        beg = sk_begin(p, cluster);
        cur = sk_begin(p, cluster + 1);
        // cluster split-K: this CTA's share of every tile's k-blocks
        kb_lo = p.csplit ? part * KB / p.csplit : 0;
        kb_hi = p.csplit ? (part + 1) * KB / p.csplit : KB;
        dyn = kDyn ? p.dyn : nullptr;
        ring = dyn ? reinterpret_cast<unsigned long long*>(dyn + 4) + static_cast<int64_t>(cluster) * kDynRing : nullptr;
        epoch = 0;
        dyn_i = 0;
        fetch = false;
        claimer = is_claimer;
        pre = 0;
        claim = 0;
    }
    // (dynamic mode) the launch epoch; read after griddepcontrol.wait (the previous launch
    // advanced it at its very end)
    __device__ __forceinline__ void load_epoch() {
        if constexpr (kDyn) {
            if (dyn) epoch = *reinterpret_cast<volatile uint32_t*>(dyn + 2);
        }
    }
    __device__ __forceinline__ unsigned long long tag(int i) const {
        return (static_cast<unsigned long long>((epoch << 12) | (static_cast<uint32_t>(i) & 0xFFFu)) << 32);
    }
    __device__ __forceinline__ unsigned long long ld_slot(int i) const {
        return ld_relaxed_u64(ring + (i % kDynRing));
    }
    __device__ __forceinline__ void publish(int i, uint32_t counter) const {
        const int t = C + static_cast<int>(counter);
        st_relaxed_u64(ring + (i % kDynRing), tag(i) | static_cast<uint32_t>(t < T_dp ? t : kDynEnd));
    }
    // the data-parallel tile number dyn_i of this cluster (lane 0's value, shared by the warp)
    __device__ __forceinline__ void resolve() {
        int t = 0;
        if ((threadIdx.x & 31) == 0) {
            unsigned long long v = pre;
#if CUASM_WATCHDOG
            const long long t0 = clock64();
#endif
            while ((v & 0xFFFFFFFF00000000ull) != tag(dyn_i)) {
                __nanosleep(32);
                v = ld_slot(dyn_i);
#if CUASM_WATCHDOG
                if (clock64() - t0 > (1ll << 34)) asm volatile("trap;");
#endif
            }
            t = static_cast<int>(v & 0xFFFFFFFFu);
        }
        next_dp = __shfl_sync(0xffffffffu, t, 0);
        fetch = false;
    }
    __device__ __forceinline__ bool next(Seg& s) {
        if constexpr (kDyn) {
            if (fetch) resolve();
        }
        if (next_dp < T_dp) {
            s.tile = next_dp;
            s.kb0 = kb_lo;
            s.kb1 = kb_hi;
            if (kDyn && dyn) {
                ++dyn_i;  // the tile after this one
                if ((threadIdx.x & 31) == 0) {
                    if (claimer) {
                        // publish tile dyn_i + 1 (claimed a tile ago; at the first tile, tiles 1
                        // and 2 now), claim dyn_i + 2
                        if (dyn_i == 1) publish(1, atomicAdd(dyn, 1u));
                        if (dyn_i == 1) claim = atomicAdd(dyn, 1u);
                        publish(dyn_i + 1, claim);
                        claim = atomicAdd(dyn, 1u);  // (result used one tile later)
                    }
                    pre = ld_slot(dyn_i);            // (value used one tile later)
                }
                fetch = true;
            } else {
                next_dp += C;
            }
            return true;
        }
        fetch = false;
        if (cur > beg) {
            const int64_t t = static_cast<uint32_t>(cur - 1) / static_cast<uint32_t>(KB);
            const int64_t t0 = t * KB;
            const int64_t lo = t0 > beg ? t0 : beg;
            s.tile = T_dp + static_cast<int>(t);
            s.kb0 = static_cast<int>(lo - t0);
            s.kb1 = static_cast<int>(cur - t0);
            cur = lo;
            return true;
        }
        return false;
    }
    // after next() returned a data-parallel tile: does another data-parallel tile follow?
    // (dynamic mode: reads the next ring slot; the claimer published it with this one)
    __device__ __forceinline__ bool dp_more() {
        if constexpr (kDyn) {
            if (fetch) resolve();
        }
        return next_dp < T_dp;
    }
    // the r-reading (finishing) segments of this cluster's stream-K range
    __device__ __forceinline__ int sk_finishing_segments(int num_k_blk) const {
        SchedT s2 = *this;
        s2.next_dp = T_dp;
        s2.fetch = false;
        s2.dyn = nullptr;
        Seg g;
        int n = 0;
        while (s2.next(g)) n += g.kb1 == num_k_blk ? 1 : 0;
        return n;
    }
};
using Sched = SchedT<true>;

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Trace slots per CTA (%globaltimer ns unless noted): 0 entry, 1 first TMA
// issued, 2 last TMA issued, 3 last MMA issued, 4 epilogue start (after the PDL
// wait), 5 epilogue done (max over warps), 6 exit, 7 final tile's accumulator
// handed to the epilogue, 8 first tile's accumulator handed over, 9 first
// tile's epilogue done, 10 final tile: contributor flags acquired, 11 final
// tile's epilogue done; leader CTAs also store 12 SM cycles from the first to
// the last MMA issue, 13 k-blocks issued, 14 / 15 issuer cycles spent waiting
// for data (full barriers) / for a free accumulator.
constexpr int kTraceSlots = 16;
__device__ __forceinline__ void trace_stamp(const FfnGemmParams& p, int slot) {
    if (p.trace) p.trace[blockIdx.x * kTraceSlots + slot] = globaltimer();
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Spin until a stream-K contributor has published its partial (flag == 1)
// (watchdog: trap after ~8 s instead of hanging the GPU on a schedule bug).
__device__ __forceinline__ void wait_flag(const uint32_t* f) {
    if (ld_acquire_u32(f) == 1u) return;
#if CUASM_WATCHDOG
    const long long t0 = clock64();
#endif
    while (ld_acquire_u32(f) != 1u) {
        __nanosleep(64);
#if CUASM_WATCHDOG
        if (clock64() - t0 > (1ll << 34)) asm volatile("trap;");
#endif
    }
}

// kEpi: the epilogue / B-operand layout.
//   0 (SwiGLU) B = the interleaved W13 block [128 W1g rows | 128 W3g rows];
//     out[m, n0+j] = SiLU(r*acc[j]) * (r*acc[128+j]), 128 outputs per tile.
//   1 (GEMM + activation) B = 256 rows of one weight matrix;
//     out[m, n0+j] = act(r*acc[j]), 256 outputs per tile (r = 1 unless use_r).
// kN: the MMA N.  kEpi 0 uses 256 (128 W1g + 128 W3g rows); kEpi 1 uses 256
// or 128 (a 128-output tile reads half of a packed 256-row block) -- the
// narrower tile halves the wave-quantisation step of square-ish GEMMs.
//
// SwiGLU tile widths (DESIGN.md §6 "Tile widths"): kN = 2*BN with BN in {64, 80, 96,
// 112, 120, 128} outputs per tile, so a column shard N_l can be cut into a tile count that
// fills whole waves of CTA pairs (7B P=8: N_l = 1376 -> 18 blocks of 80 = 144 tiles of
// 256 rows on 74 pairs instead of 11 blocks of 128 = 88).  h1 sits in accumulator
// columns [0, BN), h3 in [BN, 2BN); the epilogue walks 32-column units (the last one
// 16 or 24 wide when BN % 32 is 16 or 24).  The decode paths (rep, cluster split-K) exist for BN = 128 and
// BN = 64 (more, smaller tiles for the decode shards' weight streaming) and every GEMM tile.
// kThin (1-SM decode tiles with <= 32 rows, cluster split-K): the A tile of a stage holds only 32
// rows (4 KB instead of 16 KB), so ~1.5x more weight bytes stay in flight per SM; the MMA still
// reads 128 A rows, the ones past 32 (the next stages' bytes) feeding accumulator lanes that are
// never read.
// kTall (2-SM bf16 SwiGLU, DESIGN.md §6 "Tall tiles"): a tile is one n-block over 384 rows -- a
// 256-row part (tcgen05.mma M = 256, rows 128 c.. of CTA c) and a 128-row part (M = 128 with
// cta_group::2: 64 rows per CTA, rows 256 + 64 c..) issued back to back on the SAME weight stage,
// so a W13 block is streamed once for all 257..384 rows of the crossover region (M = 288..384 at
// K = 4096, N = 11008) instead of padding them to two 256-row tiles or running 1-SM tiles.  The
// 128-row part's accumulator sits UMMA_N columns after the 256-row one; its D layout folds the
// 64 rows x UMMA_N columns into 128 lanes x UMMA_N / 2 columns (MMA columns [BN, 2BN) -- the W3g
// half -- in lanes 64..127), so its h1 and h3 meet in shared memory (epilogue, "half part").
template <int kKind, int kCtaGroup, int kEpi = 0, int kN = 256, bool kThin = false, bool kTall = false>
struct GemmCfg {
    static_assert(kEpi == 0 ? (kN % 16 == 0 && (kN / 2) % 8 == 0 && (kN / 2) % 32 != 8 && kN >= 128 && kN <= 256)
                            : (kN == 256 || kN == 128),
                  "SwiGLU tiles: kN = 2*BN, BN in {64, 80, 96, 112, 120, 128}; GEMM tiles 128 or 256");
    static_assert(!kTall || (kKind == 0 && kCtaGroup == 2 && kEpi == 0 && !kThin && kN + kN / 2 <= 256),
                  "tall tiles: 2-SM bf16 SwiGLU, both accumulators within one 256-column TMEM buffer");
    static constexpr int kEsize = kKind == 0 ? 2 : 4;
    static constexpr int BM = 128;                 // rows per CTA (TMEM lanes)
    static constexpr int TILE_M = kTall ? 384 : BM * kCtaGroup;  // rows per tile
    static constexpr int HALF_ROW0 = 256;          // kTall: first row of the 128-row part
    static constexpr int HALF_ROWS = 64;           // kTall: rows of the 128-row part per CTA
    static constexpr int UMMA_N = kN;
    static constexpr int BN = kN / 2;              // SwiGLU: outputs per tile (h1 | h3 halves)
    static constexpr int OUT_COLS = kEpi == 0 ? BN : UMMA_N;  // output columns per tile
    static constexpr int PACK_ROWS = kEpi == 0 ? kN : 256;  // rows of one packed (n-block, k-block) box run
    static constexpr bool kDecodePaths = kEpi == 1 || kN == 256 || kN == 128;  // rep / cluster split-K
    // SwiGLU epilogue units: 32 output columns (h1 at [32u, ..), h3 at [BN + 32u, ..)),
    // the last 16 wide when BN % 32 == 16; the two warps of a TMEM quadrant alternate units
    static constexpr int NU = (BN + 31) / 32;
    static constexpr int EPI_ITERS = kEpi == 0 ? (NU + 1) / 2 : kN / 128;
    // TMEM column stride between the two accumulators (a power-of-two allocation)
    static constexpr int ACC_STRIDE = (kN > 128 || kTall) ? 256 : 128;
    // stream-K partial slot per CTA, float4s: [32-column chunk][quad][8][32 lanes], whole chunks
    // (UMMA_N = 240 has a partial last chunk, still addressed at the chunk's full stride)
    static constexpr int WS_SLOT_F4 = BM * ((kN + 31) / 32 * 32) / 4;
    static constexpr int BK = 128 / kEsize;        // one 128-byte swizzle row of K
    static constexpr int UMMA_K = 32 / kEsize;     // K per tcgen05.mma
    static constexpr int KSTEPS = BK / UMMA_K;     // 4
    static constexpr int A_FULL_BYTES = (kThin ? 32 : BM) * 128;    // per CTA
    static constexpr int A_HALF_BYTES = kTall ? HALF_ROWS * 128 : 0;  // kTall: the 128-row part's rows
    static constexpr int A_BYTES = A_FULL_BYTES + A_HALF_BYTES;
    static constexpr int B_ROWS = UMMA_N / kCtaGroup;               // packed-weight rows loaded per CTA
    static constexpr int B_BYTES = B_ROWS * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;           // per CTA
    static constexpr int BAR_BYTES = 1024;
    // as many pipeline stages as fit in 227 KB (4 x 48 KB 1-SM/256, 7 x 32 KB 2-SM/256,
    // 7 x 32 KB 1-SM/128, 9 x 24 KB 2-SM/128)
    // bf16 output goes through TMA stores from a per-warp staging area: two 32 x 32
    // boxes (2 KB each, 64-byte swizzle) per epilogue warp
    // (the 1-SM 64-output SwiGLU tile -- the decode / small-M shard tile -- reserves 8 KB per warp: the
    // cluster split-K's push form slots for up to 128 rows with S <= 4 live here, 64 KB)
    static constexpr int STG_WARP_BYTES = kKind == 0 ? ((kCtaGroup == 1 && kEpi == 0 && kN == 128) ? 8192 : 4096) : 0;
    static constexpr int STG_BYTES = 8 * STG_WARP_BYTES;
    static constexpr int STAGES_FIT = (232448 - BAR_BYTES - 1024 - STG_BYTES) / STAGE_BYTES;
#ifdef CUASM_STAGE_CAP  // experiments only: cap the pipeline depth
    static constexpr int STAGES_CAP = CUASM_STAGE_CAP;
#else
    static constexpr int STAGES_CAP = kThin ? 12 : 9;
#endif
    static constexpr int STAGES = STAGES_FIT < STAGES_CAP ? STAGES_FIT : STAGES_CAP;
    static constexpr int TMEM_COLS = 2 * ACC_STRIDE;                // 2 accumulators (power of 2)
    // Two epilogue warps per TMEM lane quadrant, each owning half of the
    // accumulator columns (PAIRS pairs of 32-column chunks): two warps per SM
    // sub-partition hide the MUFU/TMEM latency of the epilogue math.
    static constexpr int NUM_EPI_WARPS = 8;
    static constexpr int PAIRS = UMMA_N / 128;
    static constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;     // 320
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STG_BYTES + BAR_BYTES + 1024;  // + align slack
    static constexpr uint32_t IDESC = ptx::make_idesc(kKind == 0 ? 1u : 2u, BM * kCtaGroup, UMMA_N);
    static constexpr uint32_t IDESC_HALF = ptx::make_idesc(1u, 128, UMMA_N);  // kTall: M = 128, cta_group::2
    // Accumulator chunks (32 columns) of epilogue pair `i` of a warp in column half `half`.
    __device__ static constexpr int chunk_a(int half, int i) {
        return kEpi == 0 ? half * PAIRS + i : half * (UMMA_N / 64) + 2 * i;
    }
    __device__ static constexpr int chunk_b(int half, int i) {
        return kEpi == 0 ? half * PAIRS + i + BN / 32 : half * (UMMA_N / 64) + 2 * i + 1;
    }
    // First packed row of n-block nb's (or its half's) box for k-block 0; k-block kb adds kb * PACK_ROWS.
    __device__ static constexpr int b_row0(int nb, int KB) {
        return kEpi == 0 ? nb * KB * PACK_ROWS
                         : (nb * OUT_COLS / PACK_ROWS) * KB * PACK_ROWS + (nb * OUT_COLS) % PACK_ROWS;
    }
};

__device__ __forceinline__ void tile_coords(int t, const FfnGemmParams& p, int& mb, int& nb) {
    const int per_group = p.group_m * p.num_n_blk;
    const int grp = t / per_group;
    const int first_m = grp * p.group_m;
    const int gm = min(p.num_m_blk - first_m, p.group_m);
    const int local = t - grp * per_group;
    mb = first_m + local % gm;
    nb = local / gm;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float apply_act(float v, int act, float alpha) {
    return (act == 1 && v < 0.f) ? v * alpha : v;
}

// Per-row constants of the SwiGLU gate (step a3) for raw accumulators v1, v3
// and the row's inverse RMS r:  out = h1*sigma(h1)*h3 with h1 = r*v1, h3 = r*v3
//                                   = v1*v3 / ((1 + 2^t) * k),  t = -h1*log2(e),  k = 1/r^2.
// The epilogue is MUFU-bound when both ex2 and rcp go to MUFU (2 ops per output
// = 2048 SM cycles per 128x128 tile at 16 MUFU/clk), so only ex2 stays on MUFU;
// 1/((1+2^t)k) is one FFMA plus a bit-trick seed (|rel err| <= 5.1%) and two
// Newton steps on the FMA pipe (rel err <= e0^4 = 6.6e-6, centred by folding
// 1/(1+delta) into k).  One step (e0^2 = 0.26%) would be inside the [BJ]
// tolerance for the FFN output but flips the bf16 rounding of the FFN block's
// hidden (reading R13) in ~25% of elements; two steps keep flips as rare as
// with MUFU rcp.
struct GateRow {
    float c;     // r * -log2(e)
    float kk;    // 1 / (r^2 (1 + delta))
    float tmax;  // clamp of t so that (1 + 2^t) * kk <= 2^121 (finite, seedable); NaN for r = inf / NaN
};
__device__ __forceinline__ GateRow gate_row(float rr) {
    constexpr float kDelta = 3.3e-6f;  // half of the two-step Newton bias e0^4
    GateRow g;
    g.c = rr * -1.4426950408889634f;
    const float k = 1.0f / (rr * rr);
    g.kk = k * (1.0f / (1.0f + kDelta));
    // r = inf (zero row with eps = 0, reading R8) or NaN: tmax = NaN lets the
    // NaN reach d and the output, as the plain definition does (0 * inf)
    g.tmax = (rr - rr == 0.0f) ? 120.0f - __log2f(fmaxf(k, 1.0f)) : __int_as_float(0x7fc00000);
    return g;
}
__device__ __forceinline__ float silu_gate(float v1, float v3, const GateRow& g) {
    const float t = fminf(v1 * g.c, g.tmax);  // fminf(NaN, x) = x: a NaN accumulator still reaches p
    const float d = fmaf(ex2_approx(t), g.kk, g.kk);        // (1 + e^-h1) / r^2, finite, > 0
    const float y0 = __int_as_float(0x7EF311C7 - __float_as_int(d));  // ~1/d, |rel err| <= 5.1%
    const float y1 = fmaf(y0, fmaf(-d, y0, 1.0f), y0);                 // Newton: err e0^2
    const float y2 = fmaf(y1, fmaf(-d, y1, 1.0f), y1);                 // Newton: err e0^4
    return (v1 * v3) * y2;
}

// One 16-byte output store to every destination (DESIGN.md §8 "fused gather").
template <int kKind>
__device__ __forceinline__ void store16(const FfnGemmParams& p, int64_t off_bytes, uint4 v) {
    if (p.num_dst == 1 && !p.dst_mc) {  // the plain forward: one local store
        *reinterpret_cast<uint4*>(static_cast<char*>(p.dst[0]) + off_bytes) = v;
        return;
    }
    if (p.dst_mc) {
        char* a = static_cast<char*>(p.dst[0]) + off_bytes;
        if constexpr (kKind == 0)
            asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};"
                         ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        else
            asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
                         ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        return;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q < p.num_dst) *reinterpret_cast<uint4*>(static_cast<char*>(p.dst[q]) + off_bytes) = v;
}

// 32 consecutive outputs of one row -> global (bf16 pairs packed with RNE, or
// fp32), 16-byte stores, columns >= N dropped in groups of 8 (N % 8 == 0).
template <int kKind, int W = 32>
__device__ __forceinline__ void store_row32(const FfnGemmParams& p, int row, int col0, const float (&o)[32]) {
    constexpr int kEs = kKind == 0 ? 2 : 4;
    const int64_t rbase = static_cast<int64_t>(row) * p.ldo;
    if constexpr (kKind == 0) {
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
            if (col0 + 8 * q < p.N) {
                store16<kKind>(p, (rbase + col0 + 8 * q) * kEs,
                               make_uint4(ptx::pack_bf16x2(o[8 * q + 0], o[8 * q + 1]), ptx::pack_bf16x2(o[8 * q + 2], o[8 * q + 3]),
                                          ptx::pack_bf16x2(o[8 * q + 4], o[8 * q + 5]), ptx::pack_bf16x2(o[8 * q + 6], o[8 * q + 7])));
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < W / 4; ++q) {
            if (col0 + 4 * q < p.N)
                store16<kKind>(p, (rbase + col0 + 4 * q) * kEs,
                               make_uint4(__float_as_uint(o[4 * q + 0]), __float_as_uint(o[4 * q + 1]),
                                          __float_as_uint(o[4 * q + 2]), __float_as_uint(o[4 * q + 3])));
        }
    }
}

// f1 reduce-scatter ownership: the output's 256-column blocks are split evenly over
// `world` ranks, rank q owning blocks [floor(q nblk / world), floor((q+1) nblk / world)).
__host__ __device__ __forceinline__ int rs_owner(int blk, int nblk, int world) {
    return ((blk + 1) * world - 1) / nblk;
}
__host__ __device__ __forceinline__ int rs_col0(int q, int nblk, int world) { return (q * nblk / world) * 256; }

// 16 fp32 outputs of this warp's 32 rows (o[16 h .. 16 h + 15]) as one 32 x 16 fp32 box
// through the TMA map `map` (64-byte rows: the same 64-byte-swizzle staging layout as
// the bf16 box below).  Used for the f1 reduce-scatter partials.
template <int kPending>
__device__ __forceinline__ void store_box_tma_f32(const CUtensorMap* map, uint8_t* box, const float (&o)[32], int h,
                                                  int col, int row0, uint32_t lane) {
    if (lane == 0) ptx::tma_store_wait_read<kPending>();
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint4 v = make_uint4(__float_as_uint(o[16 * h + 4 * c]), __float_as_uint(o[16 * h + 4 * c + 1]),
                                   __float_as_uint(o[16 * h + 4 * c + 2]), __float_as_uint(o[16 * h + 4 * c + 3]));
        *reinterpret_cast<uint4*>(box + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = v;
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        ptx::tma_store_2d(map, ptx::smem_u32(box), col, row0);
        ptx::tma_store_commit();
    }
}

// One 32 x 32 bf16 output box (this warp's 32 rows x 32 columns) through a TMA
// store: lane r writes its row's four 16-byte chunks into the 2 KB staging box in
// the 64-byte-swizzle layout the tensor map declares (chunk c of row r lands at
// chunk c ^ ((r >> 1) & 3): conflict-free, 8 lanes of a phase hit 8 distinct
// bank groups), then lane 0 issues the store.  kPending: bulk groups of this
// warp allowed to be still reading smem when the box is overwritten (1 = the
// other box's store may be in flight).
// Output tensor maps: one per destination (the fused gather's P2P fan-out issues
// one TMA store per destination from the same staged box).
struct OutMaps {
    CUtensorMap m[8];
};

// W = 16 (the last unit of a BN % 32 == 16 tile): a 32 x 16 box (32-byte rows) through
// the narrow maps, 32-byte swizzle (chunk c of row r at c ^ ((r >> 2) & 1)); W = 24 (BN % 32
// == 24): a 32 x 24 box, 48-byte rows, no swizzle (rows 48 B apart already put the 8 lanes
// of a store phase on 8 distinct 16-byte bank groups).
// (map_idx >= 0: one store through maps->m[map_idx] at column map_col instead of the fan-out)
template <int kPending, int W = 32>
__device__ __forceinline__ void store_box_tma(const OutMaps* maps, int num, uint8_t* box, const float (&o)[32],
                                              int col, int row0, uint32_t lane, int map_idx = -1, int map_col = 0) {
    if (lane == 0) ptx::tma_store_wait_read<kPending>();
    __syncwarp();
#pragma unroll
    for (int c = 0; c < W / 8; ++c) {
        const uint4 v = make_uint4(ptx::pack_bf16x2(o[8 * c + 0], o[8 * c + 1]), ptx::pack_bf16x2(o[8 * c + 2], o[8 * c + 3]),
                                   ptx::pack_bf16x2(o[8 * c + 4], o[8 * c + 5]), ptx::pack_bf16x2(o[8 * c + 6], o[8 * c + 7]));
        if constexpr (W == 32)
            *reinterpret_cast<uint4*>(box + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = v;
        else if constexpr (W == 24)
            *reinterpret_cast<uint4*>(box + lane * 48 + (c << 4)) = v;
        else
            *reinterpret_cast<uint4*>(box + lane * 32 + ((c ^ ((lane >> 2) & 1)) << 4)) = v;
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        if (map_idx >= 0) ptx::tma_store_2d(&maps->m[map_idx], ptx::smem_u32(box), map_col, row0);
        else
            for (int q = 0; q < num; ++q) ptx::tma_store_2d(&maps->m[q], ptx::smem_u32(box), col, row0);
        ptx::tma_store_commit();
    }
}

// Cluster split-K (csplit, 1-SM): the S CTAs of a cluster hold partial accumulators
// of one tile over disjoint k-ranges.  (a) Every CTA copies its TMEM accumulator
// into its own (by now idle) pipeline shared memory, [chunk][row][32 fp32] with the
// 16-byte column groups of row r XOR-swizzled by r & 7 (conflict-free); (b) every
// epilogue warp arrives, release.cluster, on the partial-ready barrier of every CTA
// of the cluster; (c) after acquiring its own, (d) CTA `part` sums the S partials --
// in rank order, so the result does not depend on arrival order -- for the output
// column pairs p with p % S == part, reading the other CTAs' shared memory directly
// (ld.shared::cluster), applies the epilogue and stores.  The 256 epilogue threads
// take (row, column group): 4 threads x 8 columns per row for tiles with <= 64 valid
// rows, else 2 x 16; only TMEM quadrants holding valid rows are copied out.
constexpr int kMaxCsplit = 8;  // CTAs per split-K cluster (portable cluster size)

template <class C, int kKind, int kEpi>
__device__ __forceinline__ void split_k_reduce(const FfnGemmParams& p, uint32_t tmem_base, int acc, uint8_t* smem,
                                               uint64_t* xbar, uint32_t part, int mb, int nb, uint32_t quad, int half,
                                               uint32_t ewarp, uint32_t lane, int it, bool& cl_pending) {
    const uint32_t buf = ptx::smem_u32(smem);
    const uint32_t t_row = tmem_base + ((quad * 32) << 16) + acc * C::ACC_STRIDE;
    const uint32_t r_own = quad * 32 + lane;
    const int row0 = mb * C::TILE_M;
    const int rows = min(C::BM, p.M - row0);  // valid rows of the tile
    // only TMEM lane quadrants holding valid rows are copied out
#pragma unroll 1
    for (int i = 0; i < C::PAIRS && static_cast<int>(quad * 32) < rows; ++i) {
        const int ca = C::chunk_a(half, i), cb = C::chunk_b(half, i);
        uint32_t v1[32], v3[32];
        ptx::tmem_ld_32x32b_x32(t_row + ca * 32, v1);
        ptx::tmem_ld_32x32b_x32(t_row + cb * 32, v3);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t off = ((q ^ (r_own & 7)) << 4);
            *reinterpret_cast<uint4*>(smem + (static_cast<uint32_t>(ca) * C::BM + r_own) * 128 + off) =
                make_uint4(v1[4 * q], v1[4 * q + 1], v1[4 * q + 2], v1[4 * q + 3]);
            *reinterpret_cast<uint4*>(smem + (static_cast<uint32_t>(cb) * C::BM + r_own) * 128 + off) =
                make_uint4(v3[4 * q], v3[4 * q + 1], v3[4 * q + 2], v3[4 * q + 3]);
        }
    }
    __syncwarp();
    if (cl_pending) {  // the prologue's cluster barrier: every CTA's xbar is initialised
        ptx::cluster_wait_acquire();
        cl_pending = false;
    }
    if (lane == 0)
        for (int j = 0; j < p.csplit; ++j) ptx::mbar_arrive_cluster(ptx::smem_u32(xbar), static_cast<uint32_t>(j));
    if (ewarp == 0 && lane == 0) trace_stamp(p, 9);   // own partial published
    ptx::mbar_wait_acq_cluster(ptx::smem_u32(xbar), static_cast<uint32_t>(it & 1));
    if (ewarp == 0 && lane == 0) trace_stamp(p, 10);  // all partials visible

    // threads -> (row, column group): with <= 64 valid rows four threads share a row
    // (8 columns each), else two (16 columns each), so small-M tiles still use all warps
    const int tid = static_cast<int>(ewarp * 32 + lane);
    const int rows_pad = rows <= 64 ? 64 : 128;
    const int cpt = rows <= 64 ? 8 : 16;  // columns per thread per pair
    const int row = tid % rows_pad, sub = tid / rows_pad;
    const int grow = row0 + row;
    if (row >= rows) return;
    const float rr = p.use_r ? __ldcg(p.r + grow) : 1.f;
    const GateRow gr = gate_row(rr);
    constexpr int NPAIR = C::UMMA_N / 64;  // SwiGLU: (h1 chunk q, h3 chunk q + BN/32); GEMM: chunks (2q, 2q + 1)
    constexpr int kEs = kKind == 0 ? 2 : 4;
    const int64_t rbase = static_cast<int64_t>(grow) * p.ldo;
#pragma unroll 1
    for (int pr = static_cast<int>(part); pr < NPAIR; pr += p.csplit) {
        const int ca = kEpi == 0 ? pr : 2 * pr, cb = kEpi == 0 ? pr + C::BN / 32 : 2 * pr + 1;
        float a[16], b[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = b[k] = 0.f;
        const int nq = cpt / 4;  // float4 groups per thread (2 or 4)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q >= nq) break;
            const uint32_t off = (((sub * nq + q) ^ (row & 7)) << 4);
            const uint32_t oa = buf + (static_cast<uint32_t>(ca) * C::BM + row) * 128 + off;
            const uint32_t ob = buf + (static_cast<uint32_t>(cb) * C::BM + row) * 128 + off;
            // four ranks' loads in flight before the first add; the adds stay in rank order
#pragma unroll 1
            for (int j0 = 0; j0 < p.csplit; j0 += 4) {
                float4 xs[4], ys[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j0 + j < p.csplit) {
                        xs[j] = ptx::ld_dsmem_v4(ptx::mapa(oa, static_cast<uint32_t>(j0 + j)));
                        ys[j] = ptx::ld_dsmem_v4(ptx::mapa(ob, static_cast<uint32_t>(j0 + j)));
                    }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j0 + j < p.csplit) {
                        a[4 * q] += xs[j].x; a[4 * q + 1] += xs[j].y; a[4 * q + 2] += xs[j].z; a[4 * q + 3] += xs[j].w;
                        b[4 * q] += ys[j].x; b[4 * q + 1] += ys[j].y; b[4 * q + 2] += ys[j].z; b[4 * q + 3] += ys[j].w;
                    }
            }
        }
        // store cpt (8 or 16) outputs at column c0 of this row: 16-byte groups, columns >= N dropped
        auto put16 = [&](int c0, const float (&o)[16]) {
            if constexpr (kKind == 0) {
#pragma unroll
                for (int g = 0; g < 2; ++g)
                    if (8 * g < cpt && c0 + 8 * g < p.N)
                        store16<kKind>(p, (rbase + c0 + 8 * g) * kEs,
                                       make_uint4(ptx::pack_bf16x2(o[8 * g], o[8 * g + 1]),
                                                  ptx::pack_bf16x2(o[8 * g + 2], o[8 * g + 3]),
                                                  ptx::pack_bf16x2(o[8 * g + 4], o[8 * g + 5]),
                                                  ptx::pack_bf16x2(o[8 * g + 6], o[8 * g + 7])));
            } else {
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    if (4 * g < cpt && c0 + 4 * g < p.N)
                        store16<kKind>(p, (rbase + c0 + 4 * g) * kEs,
                                       make_uint4(__float_as_uint(o[4 * g]), __float_as_uint(o[4 * g + 1]),
                                                  __float_as_uint(o[4 * g + 2]), __float_as_uint(o[4 * g + 3])));
            }
        };
        float o[16];
        if constexpr (kEpi == 0) {
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = silu_gate(a[k], b[k], gr);
            put16(nb * C::OUT_COLS + ca * 32 + sub * cpt, o);
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = apply_act(rr * a[k], p.act, p.alpha);
            put16(nb * C::OUT_COLS + ca * 32 + sub * cpt, o);
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = apply_act(rr * b[k], p.act, p.alpha);
            put16(nb * C::OUT_COLS + cb * 32 + sub * cpt, o);
        }
    }
    if (ewarp == 0 && lane == 0) trace_stamp(p, 11);  // this CTA's share stored
}

// Cluster split-K, push form (bf16 output, tiles with <= 64 valid rows, whose
// partials fit the TMA-store staging area this mode leaves unused; up to 128 rows on the
// 64-output tile, whose staging area is 64 KB).  The accumulator
// is cut into units of 16 columns of chunk a + the same 16 of chunk b (8 units per
// 256-column tile); unit u belongs to CTA u % S, so with S <= 8 every CTA owns one.
// Rows 32q..32q+31 live in TMEM lane quadrant q, drained by that quadrant's two warps
// (slot rows rc = 16, 32, 64 or 128).
// (a) The warp of the TMEM quadrant holding unit u's rows reads it (lane = row) and writes it
// into slot [u / S][its rank] of the owner's staging area: plain shared-memory stores
// for its own units, st.async with a transaction-count credit on the owner's barrier
// for the others -- no copy, flag or remote read on the way; (b) the owner waits for
// the bytes (it armed the barrier with their count), sums the S slots in rank order
// (result independent of arrival order), applies the epilogue and stores.  Slot rows
// are 128 bytes, 16-byte groups XOR-swizzled by row & 7.
template <class C>
struct PushUnits {
    static constexpr int NUNIT = C::UMMA_N / 32;  // 16-column units (a and b halves)
};

__host__ __device__ __forceinline__ int push_slot_rows(int rows) {
    return rows <= 16 ? 16 : rows <= 32 ? 32 : rows <= 64 ? 64 : 128;
}

template <class C, int kKind>
__device__ __forceinline__ bool split_k_push_fits(int rows, int S) {
    if (kKind != 0 || rows > 128) return false;
    constexpr int NU = PushUnits<C>::NUNIT;
    return ((NU + S - 1) / S) * S * push_slot_rows(rows) * 128 <= C::STG_BYTES;
}

// The owner's reduction of one unit for this lane's row (split_k_push (b)): sum the
// S slots in rank order, apply the epilogue, store columns < n_lim.  Two passes of
// 8 columns, not unrolled: this code runs once per launch, fetched cold (the
// measurement's L2 flush evicts code too), so its size, not its instruction count,
// sets its time (~10 SM cycles per straight-line instruction).
template <class C, int kKind, int kEpi>
__device__ __forceinline__ void push_reduce_unit(const FfnGemmParams& p, const uint8_t* slot0, int S, int rc,
                                                 uint32_t swz, const GateRow& gr, float rr, int64_t rbase, int col_a,
                                                 int col_b, int n_lim, int g8_lo, int g8_hi) {
    constexpr int kEs = kKind == 0 ? 2 : 4;
    // the store's kernel parameters, read in the dry pass too (constant-cache lines warm)
    char* const dst0 = static_cast<char*>(p.dst[0]);
    const bool plain = p.num_dst == 1 && !p.dst_mc;
#pragma unroll 1
    for (int g8 = g8_lo; g8 < g8_hi; ++g8) {
        float a[8], b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = b[k] = 0.f;
#pragma unroll 1
        for (int j = 0; j < S; ++j) {  // rank order
            const uint8_t* src = slot0 + static_cast<uint32_t>(j * rc) * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 x = *reinterpret_cast<const float4*>(src + (((2 * g8 + h) ^ swz) << 4));
                const float4 y = *reinterpret_cast<const float4*>(src + (((4 + 2 * g8 + h) ^ swz) << 4));
                a[4 * h] += x.x; a[4 * h + 1] += x.y; a[4 * h + 2] += x.z; a[4 * h + 3] += x.w;
                b[4 * h] += y.x; b[4 * h + 1] += y.y; b[4 * h + 2] += y.z; b[4 * h + 3] += y.w;
            }
        }
#pragma unroll
        for (int h = 0; h < (kEpi == 0 ? 1 : 2); ++h) {
            const int c0 = (h == 0 ? col_a : col_b) + 8 * g8;
            float o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                o[k] = kEpi == 0 ? silu_gate(a[k], b[k], gr) : apply_act(rr * (h == 0 ? a[k] : b[k]), p.act, p.alpha);
            const uint4 v = make_uint4(ptx::pack_bf16x2(o[0], o[1]), ptx::pack_bf16x2(o[2], o[3]),
                                       ptx::pack_bf16x2(o[4], o[5]), ptx::pack_bf16x2(o[6], o[7]));
            if (c0 < n_lim) {
                if (plain) *reinterpret_cast<uint4*>(dst0 + (rbase + c0) * kEs) = v;
                else store16<kKind>(p, (rbase + c0) * kEs, v);
            }
        }
    }
}

template <class C, int kKind, int kEpi>
__device__ __forceinline__ void split_k_push(const FfnGemmParams& p, uint32_t tmem_base, int acc, uint8_t* stg,
                                             uint64_t* rbar, uint32_t part, int mb, int nb, uint32_t quad, int half,
                                             uint32_t ewarp, uint32_t lane, bool& cl_pending, bool dry) {
    constexpr int NU = PushUnits<C>::NUNIT;
    const int S = p.csplit;
    const int row0 = mb * C::TILE_M;
    const int rows = min(C::BM, p.M - row0);
    const int rc = push_slot_rows(rows);  // slot rows
    const uint32_t stg_u = ptx::smem_u32(stg), rbar_u = ptx::smem_u32(rbar);
    if (!dry && ewarp == 0 && lane == 0 && static_cast<int>(part) < NU) {
        const int owned = (NU - 1 - static_cast<int>(part)) / S + 1;
        ptx::mbar_arrive_expect_tx(rbar_u, static_cast<uint32_t>(owned * (S - 1) * rows * 128));
    }
    if (static_cast<int>(quad) * 32 >= rows) return;  // quadrant q holds rows 32q..32q+31
    const int qrow = static_cast<int>(quad) * 32;  // this quadrant's first row
    const bool row_ok = qrow + static_cast<int>(lane) < rows;
    // reduction (b): with <= 16 rows two lanes share a row, 8 of its 16 unit columns each
    const bool pair_lanes = rows <= 16;
    const int rrow = pair_lanes ? static_cast<int>(lane >> 1) : qrow + static_cast<int>(lane);
    const bool red_ok = rrow < rows;
    const float rr = red_ok && p.use_r ? __ldcg(p.r + row0 + rrow) : 1.f;  // early: hidden by (a)
#if CUASM_DIAG  // experiments only: SM-cycle stamps of the phases into trace slots 12..15
    const long long dclk0 = clock64();
    const bool dbg = p.trace && lane == 0 && half == 0;
#define CUASM_DIAG_STAMP(slot) \
    if (dbg) p.trace[blockIdx.x * kTraceSlots + (slot)] = static_cast<unsigned long long>(clock64() - dclk0)
#else
#define CUASM_DIAG_STAMP(slot)
#endif
    if (!dry && cl_pending) {  // the prologue's cluster barrier: every CTA's barriers are initialised
        ptx::cluster_wait_acquire();
        cl_pending = false;
    }
    const uint32_t t_row = tmem_base + ((quad * 32) << 16) + acc * C::ACC_STRIDE;
    const uint32_t swz = lane & 7;
    // (a) scatter this warp's units to their owners
#pragma unroll 1
    for (int i = 0; i < C::PAIRS; ++i) {
        const int ca = C::chunk_a(half, i), cb = C::chunk_b(half, i);
        uint32_t v1[32], v3[32];
        if (!dry) {
            ptx::tmem_ld_32x32b_x32(t_row + ca * 32, v1);
            ptx::tmem_ld_32x32b_x32(t_row + cb * 32, v3);
            ptx::tmem_ld_wait();
        }
        if (!row_ok || dry) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int u = 2 * (half * C::PAIRS + i) + h;
            const uint32_t owner = static_cast<uint32_t>(u % S);
            const uint32_t off =
                static_cast<uint32_t>(((u / S) * S + static_cast<int>(part)) * rc + qrow + static_cast<int>(lane)) * 128;
            if (owner == part) {
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    *reinterpret_cast<uint4*>(stg + off + ((g ^ swz) << 4)) =
                        make_uint4(v1[16 * h + 4 * g], v1[16 * h + 4 * g + 1], v1[16 * h + 4 * g + 2],
                                   v1[16 * h + 4 * g + 3]);
                    *reinterpret_cast<uint4*>(stg + off + (((g + 4) ^ swz) << 4)) =
                        make_uint4(v3[16 * h + 4 * g], v3[16 * h + 4 * g + 1], v3[16 * h + 4 * g + 2],
                                   v3[16 * h + 4 * g + 3]);
                }
            } else {
                const uint32_t rdst = ptx::mapa(stg_u + off, owner), rb = ptx::mapa(rbar_u, owner);
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    ptx::st_async_v4(rdst + ((g ^ swz) << 4),
                                     make_uint4(v1[16 * h + 4 * g], v1[16 * h + 4 * g + 1], v1[16 * h + 4 * g + 2],
                                                v1[16 * h + 4 * g + 3]),
                                     rb);
                    ptx::st_async_v4(rdst + (((g + 4) ^ swz) << 4),
                                     make_uint4(v3[16 * h + 4 * g], v3[16 * h + 4 * g + 1], v3[16 * h + 4 * g + 2],
                                                v3[16 * h + 4 * g + 3]),
                                     rb);
                }
            }
        }
    }
    __syncwarp();  // this warp's own-slot stores (lane = row) before other lanes of it read them
    CUASM_DIAG_STAMP(12);
    // (b) reduce the units this CTA owns
    const GateRow gr = gate_row(rr);
    const int64_t rbase = static_cast<int64_t>(row0 + rrow) * p.ldo;
    bool waited = false;
#pragma unroll 1
    for (int v = 0; v < 2 * C::PAIRS; ++v) {
        const int i = v >> 1, h = v & 1;
        const int u = 2 * (half * C::PAIRS + i) + h;
        if (u % S != static_cast<int>(part)) continue;
        if (!waited && !dry) {
            ptx::mbar_wait_acq_cluster(rbar_u, 0u);  // one tile per cluster: phase 0
            waited = true;
            CUASM_DIAG_STAMP(13);
        }
        if (!red_ok) continue;
        const int ca = C::chunk_a(half, i), cb = C::chunk_b(half, i);
        const uint8_t* slot0 = stg + static_cast<uint32_t>((u / S) * S * rc + rrow) * 128;
        const int g8_lo = pair_lanes ? static_cast<int>(lane & 1) : 0;
        CUASM_DIAG_STAMP(14);
        push_reduce_unit<C, kKind, kEpi>(p, slot0, S, rc, static_cast<uint32_t>(rrow & 7), gr, rr, rbase,
                                         nb * C::OUT_COLS + ca * 32 + 16 * h, nb * C::OUT_COLS + cb * 32 + 16 * h,
                                         dry ? 0 : p.N, g8_lo, pair_lanes ? g8_lo + 1 : 2);
        CUASM_DIAG_STAMP(15);
    }
}

// kDyn: dynamic whole-tile claiming compiled in (p.dyn must be null otherwise); a kernel
// template parameter rather than a runtime branch so the static kernels' loops are exactly
// the uniform code they were (DESIGN.md §6 "Dynamic tiles").
// kMcast (2-SM only): 4-CTA clusters of two CTA pairs computing two vertically adjacent
// 256-row tiles of the same n-block; the pair-0 CTAs TMA-load each W13 half once and multicast
// it into both pairs' shared memory (DESIGN.md §6 "Multicast clusters").  Whole tiles only.
// kTall: tall tiles (GemmCfg), static whole tiles only; tmap_xh is x with 64-row boxes (the 128-row
// part's rows per CTA), unused by the other kernels.
template <int kKind, int kCtaGroup, int kEpi, int kN, bool kDyn = false, bool kMcast = false, bool kThin = false,
          bool kTall = false>
__global__ void __launch_bounds__(GemmCfg<kKind, kCtaGroup, kEpi, kN, kThin, kTall>::NUM_THREADS, 1)
    ffn_dual_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                         const __grid_constant__ CUtensorMap tmap_xh, const __grid_constant__ OutMaps omaps,
                         const __grid_constant__ OutMaps omaps_h, const FfnGemmParams p) {
    using C = GemmCfg<kKind, kCtaGroup, kEpi, kN, kThin, kTall>;
    static_assert(!kThin || (kCtaGroup == 1 && !kDyn && !kMcast), "thin A tiles: 1-SM decode kernels");
    static_assert(!kTall || (!kDyn && !kMcast), "tall tiles: static schedule, CTA pairs");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + C::STAGES * C::A_BYTES;
    uint8_t* smem_stg = smem + C::STAGES * C::STAGE_BYTES;  // [8 warps][2 boxes][32 x 32] bf16 (1 KB aligned)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::STG_BYTES);
    uint64_t* full_bar = bars;                       // [STAGES]
    uint64_t* empty_bar = bars + C::STAGES;          // [STAGES]
    uint64_t* tfull_bar = bars + 2 * C::STAGES;      // [2]
    uint64_t* tempty_bar = bars + 2 * C::STAGES + 2; // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);
    uint64_t* xbar = bars + 2 * C::STAGES + 6;        // cluster split-K: partials of all S CTAs in smem
    uint64_t* rbar = bars + 2 * C::STAGES + 7;        // cluster split-K, push form: partials received
    // dynamic claiming: k-blocks of the segment a stage starts (0 = end), byte 512 of the barrier area
    int* seg_nkb = reinterpret_cast<int*>(bars + 64);
    static_assert((2 * C::STAGES + 8) * 8 <= 512 && 512 + 4 * C::STAGES <= C::BAR_BYTES, "barrier area layout");

    const uint32_t warp = ptx::warp_id_uniform();
    const uint32_t lane = ptx::lane_id();
    static_assert(!kMcast || (kCtaGroup == 2 && !kDyn), "multicast clusters: 2-SM static kernels");
    const uint32_t cl_rank = kCtaGroup == 2 ? ptx::cluster_ctarank() : 0;  // rank in the cluster
    const uint32_t cta_rank = kMcast ? (cl_rank & 1u) : cl_rank;          // rank in the CTA pair
    const int pair_id = kMcast ? static_cast<int>(cl_rank >> 1) : 0;      // pair in a multicast cluster
    const bool leader = cta_rank == 0;
    // the tile of this pair inside a multicast cluster's super-tile (m-block pair x n-block)
    auto pair_mb = [&](int mb) { return kMcast ? mb * 2 + pair_id : mb; };
    const bool csplit = C::kDecodePaths && kCtaGroup == 1 && p.csplit > 0;
    const int rep = (C::kDecodePaths && !kThin) ? p.rep : 0;  // decode-shape row replication (BN = 128 / 64)
    const uint32_t part = csplit ? ptx::cluster_ctarank() : 0;  // split-K share of the cluster's tile

    if (warp == 0 && lane == 0) {
        trace_stamp(p, 0);
        ptx::prefetch_tmap(&tmap_x);
        ptx::prefetch_tmap(&tmap_w);
        if constexpr (kTall) ptx::prefetch_tmap(&tmap_xh);
        for (int s = 0; s < C::STAGES; ++s) {
            // 2-SM: only the leader's producer arrives (expect_tx of BOTH
            // CTAs' bytes); the peer's TMA bytes are credited to it too.
            ptx::mbar_init(ptx::smem_u32(&full_bar[s]), 1);
            ptx::mbar_init(ptx::smem_u32(&empty_bar[s]), kMcast ? 2 : 1);  // (multicast: both pairs' MMAs)
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(ptx::smem_u32(&tfull_bar[a]), 1);
            // every epilogue warp of BOTH CTAs releases the leader's accumulator
            ptx::mbar_init(ptx::smem_u32(&tempty_bar[a]), C::NUM_EPI_WARPS * kCtaGroup);
        }
        // every epilogue warp of every CTA of a split-K cluster arrives once per tile
        if (csplit) {
            ptx::mbar_init(ptx::smem_u32(xbar), C::NUM_EPI_WARPS * p.csplit);
            ptx::mbar_init(ptx::smem_u32(rbar), 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<C::TMEM_COLS, kCtaGroup>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    // (split-K clusters: remote arrivals on xbar need every CTA's barriers initialised;
    // the wait half is deferred to the first remote arrival, after the mainloop)
    bool cl_pending = csplit;
    if (kCtaGroup == 2) {
        ptx::cluster_sync();
#if CUASM_DIAG_PROLOGUE  // experiments only: producer prologue stamps in slots 12..15
        if (warp == 0 && lane == 0) trace_stamp(p, 12);
#endif
    } else {
        // (the barriers' initialisation is already released to the cluster by
        // fence.mbarrier_init: a relaxed arrive, no GPU-scope membar)
        if (csplit) ptx::cluster_arrive_relaxed();
        __syncthreads();
    }
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // Cluster-level work: both CTAs of a pair (every CTA of a split-K cluster) walk
    // the same tile sequence.
    const int cluster_id = csplit ? static_cast<int>(blockIdx.x) / p.csplit
                                  : static_cast<int>(blockIdx.x) / (kMcast ? 4 : kCtaGroup);

    if (warp == 0) {
        // ========================= TMA producer =========================
        // Whole warp walks the loop, one elected lane issues (uniform operands,
        // no per-instruction uniformity loops around UTMALDG).
        // default: x evict_last (re-read by every n-block), W13 evict_normal (shared by the
        // group's tiles); CUASM_OPT_L2_POLICY overrides (2 bits each: 0 normal, 1 first, 2 last)
        auto pol = [](int c) {
            return c == 1 ? ptx::policy_evict_first() : c == 2 ? ptx::policy_evict_last() : ptx::policy_evict_normal();
        };
        const uint64_t pol_x = pol(p.l2pol & 3);
        const uint64_t pol_w = pol((p.l2pol >> 2) & 3);
        // arm stage s for k-block kb (its full transaction count: x and weights) and load the weights
        auto arm_and_load_w = [&](int s, int kb, int row_b0) {
            const uint32_t fb = ptx::smem_u32(&full_bar[s]);
            const uint32_t sb = ptx::smem_u32(smem_b + s * C::B_BYTES);
            if constexpr (kCtaGroup == 1) {
                ptx::mbar_arrive_expect_tx(fb, (rep ? rep : 1) * p.a_box_bytes + C::B_BYTES);
                ptx::tma_load_2d(sb, &tmap_w, fb, 0, row_b0 + kb * C::PACK_ROWS, pol_w);
            } else {
                // both CTAs' bytes land on the leader's barrier
                if (leader)
                    ptx::mbar_arrive_expect_tx(fb, 2 * C::B_BYTES + (rep ? rep + 1 : 2) * p.a_box_bytes + 2 * C::A_HALF_BYTES);
                if constexpr (kMcast) {
                    // pair 0 loads each W13 half once for both pairs (same n-block)
                    if (pair_id == 0)
                        ptx::tma_load_2d_2sm_mc(sb, &tmap_w, fb, 0, row_b0 + kb * C::PACK_ROWS,
                                                static_cast<uint16_t>((1u << cl_rank) | (1u << (cl_rank + 2))), pol_w);
                } else {
                    ptx::tma_load_2d_2sm(sb, &tmap_w, fb, 0, row_b0 + kb * C::PACK_ROWS, pol_w);
                }
            }
        };
        // the x rows of stage s (rep: <= 32 rows copied into every 32-row quarter; 2-SM: the
        // leader's A tile only -- the peer's rows are all past M)
        auto load_x = [&](int s, int kb, int row_a) {
            const uint32_t fb = ptx::smem_u32(&full_bar[s]);
            const uint32_t sa = ptx::smem_u32(smem_a + s * C::A_BYTES);
            if constexpr (kCtaGroup == 1) {
                const int nrep = rep ? rep : 1;
                for (int q = 0; q < nrep; ++q)  // copy q of the rows: smem rows q*128/nrep.. (4 KB aligned)
                    ptx::tma_load_2d(sa + q * (128 / nrep) * 128, &tmap_x, fb, kb * C::BK, row_a, pol_x);
            } else {
                const int nrep = (rep && leader) ? rep : 1;
                for (int q = 0; q < nrep; ++q)
                    ptx::tma_load_2d_2sm(sa + q * (128 / nrep) * 128, &tmap_x, fb, kb * C::BK, row_a, pol_x);
                // kTall: this CTA's 64 rows of the 128-row part, behind its 128 rows of the 256-row part
                if constexpr (kTall)
                    ptx::tma_load_2d_2sm(sa + C::A_FULL_BYTES, &tmap_xh, fb, kb * C::BK,
                                         C::HALF_ROW0 + static_cast<int>(cta_rank) * C::HALF_ROWS, pol_x);
            }
        };
        SchedT<kDyn> sch;
        sch.init(p, cluster_id, static_cast<int>(part), leader && part == 0);  // the leader claims tiles
        // Weights do not depend on the preceding kernel (they were packed before it): the
        // first segment's first STAGES weight boxes go out before griddepcontrol.wait, so
        // under PDL they stream while the preceding kernel drains (its x loads follow the wait)
        int pre = 0;
        if (p.w_early) {
            auto s0 = sch;
            s0.dyn = nullptr;  // (the first tile is static: no claim, no ring)
            s0.claimer = false;
            Seg g0;
            if (s0.next(g0)) {
                int mb0, nb0;
                tile_coords(g0.tile, p, mb0, nb0);
                mb0 = pair_mb(mb0);
                const int row_b0 = C::b_row0(nb0, p.num_k_blk) + static_cast<int>(cta_rank) * C::B_ROWS;
                pre = min(C::STAGES, g0.kb1 - g0.kb0);
                if (ptx::elect_one()) {
                    if constexpr (kDyn) {
                        if (leader) seg_nkb[0] = g0.kb1 - g0.kb0;  // (before the arrive that releases it)
                    }
                    for (int i = 0; i < pre; ++i) {
                        arm_and_load_w(i, g0.kb0 + i, row_b0);
#if CUASM_DIAG_PROLOGUE
                        if (i == 0) trace_stamp(p, 13);
#endif
                    }
                }
                __syncwarp();
            }
        }
#if CUASM_DIAG_PROLOGUE
        if (lane == 0) trace_stamp(p, 14);
#endif
        ptx::pdl_wait();  // x may be produced by the preceding kernel (PDL)
#if CUASM_DIAG_PROLOGUE
        if (lane == 0) trace_stamp(p, 15);
#endif
        sch.load_epoch();
        int stage = 0;
        uint32_t phase = 0;
        bool first_load = true;
        Seg sg;
        while (sch.next(sg)) {
            int mb, nb;
            tile_coords(sg.tile, p, mb, nb);
            mb = pair_mb(mb);
            const int row_a = mb * C::TILE_M + static_cast<int>(cta_rank) * C::BM;
            // k-block-tiled weights (pack.cuh): box (nb, kb) starts at row (nb*KB + kb)*UMMA_N
            const int row_b0 = C::b_row0(nb, p.num_k_blk) + static_cast<int>(cta_rank) * C::B_ROWS;
            for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
                if (pre > 0) {
                    // stage armed and its weights requested before the wait (first use of the
                    // stage: no empty-barrier wait needed)
                    if (ptx::elect_one()) load_x(stage, kb, row_a);
                    --pre;
                } else {
                    ptx::mbar_wait(ptx::smem_u32(&empty_bar[stage]), phase ^ 1);
                    if (ptx::elect_one()) {
                        if constexpr (kDyn) {
                            if (leader && kb == sg.kb0) seg_nkb[stage] = sg.kb1 - sg.kb0;
                        }
                        arm_and_load_w(stage, kb, row_b0);
                        load_x(stage, kb, row_a);
                    }
                }
                __syncwarp();
                if (first_load && lane == 0) trace_stamp(p, 1);
                first_load = false;
                if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
        }
        if constexpr (kDyn) {
            // end marker for the MMA warp's stage-driven loop: a stage completed by a plain
            // arrive (no transaction bytes) whose segment length is 0
            if (leader) {
                ptx::mbar_wait(ptx::smem_u32(&empty_bar[stage]), phase ^ 1);
                if (ptx::elect_one()) {
                    seg_nkb[stage] = 0;
                    ptx::mbar_arrive(ptx::smem_u32(&full_bar[stage]));
                }
                __syncwarp();
            }
        }
        if (lane == 0) {
            trace_stamp(p, 2);
            // all of this CTA's loads are issued: let the next PDL kernel in the
            // stream get scheduled as SMs free up (it griddepcontrol.waits for
            // this grid's completion before reading anything we write)
            ptx::pdl_launch_dependents();
        }
    } else if (warp == 1) {
        // ========================= MMA issuer ===========================
        // The whole warp walks the loop (barrier waits included) and one
        // elected lane issues: the descriptors then live in uniform registers
        // and ptxas emits no per-instruction uniformity loop around UTCHMMA.
        // The issue loop is on the critical path (the tensor core only runs
        // ahead of it by a few instructions), so it is kept short.
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            long long kblocks = 0, clk0 = 0, wait_full = 0, wait_tempty = 0;
            // smem descriptors of stage 0; stage s adds s*bytes >> 4 to the address field
            const uint64_t adesc0 = ptx::make_smem_desc_sw128(ptx::smem_u32(smem_a));
            const uint64_t bdesc0 = ptx::make_smem_desc_sw128(ptx::smem_u32(smem_b));
            SchedT<false> sch;  // (kDyn kernels take the stage-driven loop below)
            sch.init(p, cluster_id, static_cast<int>(part));
            Seg sg;
            for (; !kDyn && sch.next(sg); ++it) {
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                {
                    const long long w0 = p.trace ? clock64() : 0;
                    ptx::mbar_wait(ptx::smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
                    if (p.trace && kblocks > 0) wait_tempty += clock64() - w0;
                }
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * C::ACC_STRIDE;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
                    {
                        const long long w0 = p.trace ? clock64() : 0;
                        ptx::mbar_wait(ptx::smem_u32(&full_bar[stage]), phase);
                        if (p.trace && kblocks > 0) wait_full += clock64() - w0;
                    }
                    ptx::tc_fence_after();
                    const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * C::A_BYTES) >> 4);
                    const uint64_t bdesc = bdesc0 + static_cast<uint64_t>((stage * C::B_BYTES) >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int k = 0; k < C::KSTEPS; ++k) {
                            // advance 32 bytes of K inside the 128-byte swizzle row (+2 in 16-byte units)
                            ptx::mma<kKind, kCtaGroup>(d_tmem, adesc + 2 * k, bdesc + 2 * k, C::IDESC,
                                                       (kb > sg.kb0 || k > 0) ? 1u : 0u);
                            // kTall: the 128-row part on the same weight stage (M = 128, its own
                            // A rows behind the 256-row part's, accumulator UMMA_N columns on)
                            if constexpr (kTall)
                                ptx::mma<kKind, kCtaGroup>(d_tmem + C::UMMA_N, adesc + (C::A_FULL_BYTES >> 4) + 2 * k,
                                                           bdesc + 2 * k, C::IDESC_HALF, (kb > sg.kb0 || k > 0) ? 1u : 0u);
                        }
                        if constexpr (kCtaGroup == 1) {
                            ptx::mma_commit(ptx::smem_u32(&empty_bar[stage]));
                        } else {
                            // (multicast clusters: every CTA's stage also holds the other pair's W13)
                            ptx::mma_commit_2sm(ptx::smem_u32(&empty_bar[stage]), kMcast ? 0xF : 0x3);
                        }
                    }
                    __syncwarp();
                    if (p.trace && kblocks++ == 0) clk0 = clock64();
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) {
                    if constexpr (kCtaGroup == 1) {
                        ptx::mma_commit(ptx::smem_u32(&tfull_bar[acc]));
                    } else {
                        ptx::mma_commit_2sm(ptx::smem_u32(&tfull_bar[acc]), static_cast<uint16_t>(0x3u << (2 * pair_id)));
                    }
                }
                __syncwarp();
            }
            if constexpr (kDyn) {
                // Dynamic claiming: the MMA warp needs no tile numbers, only each segment's
                // k-block count, which the leader's producer writes into seg_nkb[stage] of the
                // segment's first stage before arming it (0 = no more segments): the loop reads
                // it behind the full barrier it waits on anyway (no global loads, no branch on
                // a lane's value in the issue loop)
#pragma unroll 1
                for (;; ++it) {
                    ptx::mbar_wait(ptx::smem_u32(&full_bar[stage]), phase);
                    const int nkb = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile int*>(&seg_nkb[stage]), 0);
                    if (nkb == 0) break;
                    const int acc = it & 1;
                    const uint32_t acc_phase = (it >> 1) & 1;
                    ptx::mbar_wait(ptx::smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
                    const uint32_t d_tmem = tmem_base + acc * C::ACC_STRIDE;
                    for (int j = 0; j < nkb; ++j) {
                        if (j > 0) ptx::mbar_wait(ptx::smem_u32(&full_bar[stage]), phase);
                        ptx::tc_fence_after();
                        const uint64_t adesc = adesc0 + static_cast<uint64_t>((stage * C::A_BYTES) >> 4);
                        const uint64_t bdesc = bdesc0 + static_cast<uint64_t>((stage * C::B_BYTES) >> 4);
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int k = 0; k < C::KSTEPS; ++k)
                                ptx::mma<kKind, kCtaGroup>(d_tmem, adesc + 2 * k, bdesc + 2 * k, C::IDESC,
                                                           (j > 0 || k > 0) ? 1u : 0u);
                            ptx::mma_commit_2sm(ptx::smem_u32(&empty_bar[stage]), 0x3);
                        }
                        __syncwarp();
                        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (ptx::elect_one()) ptx::mma_commit_2sm(ptx::smem_u32(&tfull_bar[acc]), 0x3);
                    __syncwarp();
                }
            }
            if (lane == 0) {
                trace_stamp(p, 3);
                if (p.trace) {
                    // SM cycles from the first to the last MMA issue, k-blocks issued and
                    // cycles spent waiting: (cycles / (k-blocks - 1)) vs the tcgen05 floor
                    // (4 x 128 cycles) tells a starved tensor pipe from a slow clock
#if !CUASM_DIAG_PROLOGUE
                    p.trace[blockIdx.x * kTraceSlots + 12] = static_cast<unsigned long long>(clock64() - clk0);
                    p.trace[blockIdx.x * kTraceSlots + 13] = static_cast<unsigned long long>(kblocks);
                    p.trace[blockIdx.x * kTraceSlots + 14] = static_cast<unsigned long long>(wait_full);
                    p.trace[blockIdx.x * kTraceSlots + 15] = static_cast<unsigned long long>(wait_tempty);
#endif
                }
            }
        }
    } else {
        // ========================= epilogue =============================
        ptx::pdl_wait();  // x / r[] come from the preceding kernel (PDL primary)
        if (warp == 2 && lane == 0) trace_stamp(p, 4);
        using T = typename std::conditional<kKind == 0, __nv_bfloat16, float>::type;
        // Fused step a1 (DESIGN.md §6 "Fused a1"): r[m] = 1/sqrt(sum_k x^2/K + eps) is
        // computed on demand per 128-row r-block.  The epilogue warps of a CTA about to
        // read r of r-block rb (all eight, at the same tile) each take rows of rb one at a
        // time from the block's counter while rows remain -- every CTA that needs the
        // block helps -- and publish each row (fence + done count); then one warp waits
        // for the block's done count and a named barrier releases the others.  A CTA
        // waits only for rows taken by warps already running, so no co-residency of the
        // grid is assumed (other kernels / MPS may hold SMs).  Each CTA counts itself
        // once past its last acquisition; the last CTA of the grid resets the
        // bookkeeping for the next launch (graph-safe), under its last tile's mainloop.
        const bool fused = p.fused_norm != 0;
        SchedT<kDyn> sch;
        sch.init(p, cluster_id, static_cast<int>(part));
        sch.load_epoch();
        // r-reading segments still ahead: the data-parallel tiles (all read r; in dynamic mode
        // their count is known only one tile ahead, Sched::dp_more) and the stream-K segments
        // that finish a tile (or, cluster split-K, every segment)
        int sk_r = 0;
        bool has_dp = false;
        if (fused) {
            auto s2 = sch;
            s2.dyn = nullptr;
            has_dp = s2.next_dp < s2.T_dp;
            if (csplit) {
                Seg g2;
                int n = 0;
                while (s2.next(g2)) ++n;
                sk_r = n;  // (split-K clusters: no data-parallel round-robin past the first tile)
                has_dp = false;
            } else {
                sk_r = s2.sk_finishing_segments(p.num_k_blk);
            }
        }
        auto r_done_cta = [&]() {  // warp 2 of the CTA, after the CTA's last acquisition
            uint32_t* cnt = p.rstate + 2 * p.n_rblk;
            uint32_t last = 0;
            if (lane == 0) last = atomicAdd(cnt, 1u) == gridDim.x - 1 ? 1u : 0u;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                for (int i = static_cast<int>(lane); i < 2 * p.n_rblk; i += 32) p.rstate[i] = 0u;
                __syncwarp();
                if (lane == 0) *cnt = 0u;
            }
            __syncwarp();
        };
        if (fused && !has_dp && sk_r == 0 && warp == 2) r_done_cta();
        auto acquire_r = [&](int rb) {
            const int row0 = rb * C::BM;
            if (row0 >= p.M) return;  // (2-SM decode: the peer CTA's rows are all past M); CTA-uniform
            const uint32_t nrows = static_cast<uint32_t>(min(C::BM, p.M - row0));
            uint32_t* taken = p.rstate + rb;
            uint32_t* done = p.rstate + p.n_rblk + rb;
            uint32_t help = 0;
            if (lane == 0) help = ld_acquire_u32(done) < nrows && *reinterpret_cast<volatile uint32_t*>(taken) < nrows;
            if (__shfl_sync(0xffffffffu, help, 0)) {
                for (;;) {
                    uint32_t i = 0;
                    if (lane == 0) i = atomicAdd(taken, 1u);
                    i = __shfl_sync(0xffffffffu, i, 0);
                    if (i >= nrows) break;
                    rms_row<T>(static_cast<const T*>(p.x), p.r, row0 + static_cast<int64_t>(i), p.K, p.eps,
                               static_cast<int>(lane));
                    if (lane == 0) {
                        __threadfence();  // r[row] (written by this lane) before the count
                        atomicAdd(done, 1u);
                    }
                }
            }
            ptx::named_bar_sync(1, 32 * C::NUM_EPI_WARPS);
            if (warp == 2 && lane == 0 && ld_acquire_u32(done) < nrows) {
#if CUASM_WATCHDOG
                const long long t0 = clock64();
#endif
                while (ld_acquire_u32(done) < nrows) {
                    __nanosleep(128);
#if CUASM_WATCHDOG
                    if (clock64() - t0 > (1ll << 34)) asm volatile("trap;");
#endif
                }
            }
            ptx::named_bar_sync(1, 32 * C::NUM_EPI_WARPS);  // (the r loads of every warp follow it)
        };
        const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
        const uint32_t ewarp = warp - 2;  // 0..7: flag slot
        const int half = static_cast<int>(ewarp >> 2);  // this warp's half of the accumulator columns
        const uint32_t row_in_cta = quad * 32 + lane;
        int it = 0;
        int nst = 0;  // TMA-store boxes this warp has issued (staging box = nst & 1)
        Seg sg;
        for (; sch.next(sg); ++it) {
            int mb, nb;
            tile_coords(sg.tile, p, mb, nb);
            mb = pair_mb(mb);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            // rep: quadrant `quad` holds rows 0..31 of the tile (lane = row), and only its
            // own column pair is drained by it (below)
            const int row = mb * C::TILE_M + static_cast<int>(cta_rank) * C::BM +
                            static_cast<int>(rep ? (quad % (4 / rep)) * 32 + lane : row_in_cta);
            const bool row_ok = row < p.M;
            // stream-K (Sched): a contributor lacks the tile's last k-block and publishes a
            // partial; the finisher holds the last k-block but not the first and adds the
            // partials of the lower clusters holding the rest of the tile
            const bool contributor = !csplit && sg.kb1 < p.num_k_blk;
            const bool finisher = !csplit && sg.kb1 == p.num_k_blk && sg.kb0 > 0;
            // this CTA's 128 x 2BN fp32 partial slot, lane-contiguous so every warp
            // access is 512 contiguous bytes: float4 index ((chunk*4 + quad)*8 + q)*32 + lane
            // holds columns chunk*32 + 4q..+3 of row quad*32 + lane (chunk < BN/32: h1, else h3)
            float4* my_slot = reinterpret_cast<float4*>(p.ws) +
                              (static_cast<int64_t>(cluster_id) * kCtaGroup + cta_rank) * C::WS_SLOT_F4;
            int c_first = 0, c_last = -1;
            if (finisher) {
                // contributors: the (lower) clusters whose stream-K ranges cover the rest of this tile
                const int64_t tile_start = static_cast<int64_t>(sg.tile - p.num_dp_tiles) * p.num_k_blk;
                c_first = sk_owner(p, tile_start);
                c_last = cluster_id - 1;
                // pull the partials this warp will add into L2 while the accumulator
                // is still being computed (L2 is the coherence point: safe before the flag)
                for (int cc = c_first; cc <= c_last; ++cc) {
                    if (sk_begin(p, cc) == sk_begin(p, cc + 1)) continue;
                    const char* slot = reinterpret_cast<const char*>(
                        reinterpret_cast<const float4*>(p.ws) +
                        (static_cast<int64_t>(cc) * kCtaGroup + cta_rank) * C::WS_SLOT_F4);
                    // the 32-column chunks (4 KB per quadrant) holding this warp's units
                    auto pf = [&](int chunk) { prefetch_l2(slot + ((chunk * 4 + quad) * 8 * 32) * 16 + lane * 128); };
#pragma unroll
                    for (int i = 0; i < C::EPI_ITERS; ++i) {
                        if constexpr (kEpi == 0) {
                            const int u = half + 2 * i;
                            if (u >= C::NU) continue;
                            const int w = C::BN - 32 * u < 32 ? C::BN - 32 * u : 32;
                            pf(u);
                            pf((C::BN + 32 * u) >> 5);
                            if (((C::BN + 32 * u + w - 1) >> 5) != ((C::BN + 32 * u) >> 5)) pf((C::BN + 32 * u + w - 1) >> 5);
                        } else {
                            pf(C::chunk_a(half, i));
                            pf(C::chunk_b(half, i));
                        }
                    }
                }
            }
            if (fused && (csplit || !contributor)) {
                acquire_r(csplit ? mb : mb * kCtaGroup + static_cast<int>(cta_rank));
                if constexpr (kTall) acquire_r(C::HALF_ROW0 / C::BM);  // the 128-row part's rows
                // the CTA's last r acquisition: count it past (the last CTA resets the state)
                const bool dp_seg = !csplit && sg.tile < p.num_dp_tiles;
                bool last;
                if (dp_seg) last = !sch.dp_more() && sk_r == 0;
                else last = --sk_r == 0;
                if (last && warp == 2) r_done_cta();
            }
            if (csplit && split_k_push_fits<C, kKind>(min(C::BM, p.M - mb * C::TILE_M), p.csplit)) {
                // cluster split-K, push form.  Pass 0 runs the same code dry (no TMEM
                // reads, remote writes, waits or stores) while the mainloop runs, so
                // that pass 1, on the critical path, finds it in the instruction cache
                // (it runs once per launch and would be fetched cold otherwise)
#pragma unroll 1
                for (int pass = 0; pass < 2; ++pass) {
                    if (pass == 1) {
                        ptx::mbar_wait(ptx::smem_u32(&tfull_bar[acc]), acc_phase);
                        ptx::tc_fence_after();
                        if (warp == 2 && lane == 0) {
                            trace_stamp(p, 7);
                            if (it == 0) trace_stamp(p, 8);
                        }
                    }
                    if constexpr (C::kDecodePaths)
                        split_k_push<C, kKind, kEpi>(p, tmem_base, acc, smem_stg, rbar, part, mb, nb, quad, half, ewarp,
                                                     lane, cl_pending, pass == 0);
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tempty_bar[acc]));
                continue;
            }
            const float rr = !row_ok ? 0.f : (p.use_r ? __ldcg(p.r + row) : 1.f);
            const GateRow gr = gate_row(rr);
            ptx::mbar_wait(ptx::smem_u32(&tfull_bar[acc]), acc_phase);
            ptx::tc_fence_after();
#if CUASM_DIAG  // experiments only: SM cycles of the final tile's epilogue phases (slots 12..15)
            const long long eclk0 = clock64();
#define CUASM_EPI_STAMP(slot) \
    if (p.trace && warp == 2 && lane == 0) p.trace[blockIdx.x * kTraceSlots + (slot)] = clock64() - eclk0
#else
#define CUASM_EPI_STAMP(slot)
#endif
            if (warp == 2 && lane == 0) {
                trace_stamp(p, 7);  // (last write wins: the final tile)
                if (it == 0) trace_stamp(p, 8);
            }
            if (csplit) {
                // cluster split-K: partials through distributed shared memory, this CTA
                // reduces and stores its share of the tile's output columns
                if constexpr (C::kDecodePaths)
                    split_k_reduce<C, kKind, kEpi>(p, tmem_base, acc, smem, xbar, part, mb, nb, quad, half, ewarp, lane,
                                                   it, cl_pending);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tempty_bar[acc]));
                continue;
            }
            for (int cc = c_first; cc <= c_last; ++cc) {
                if (sk_begin(p, cc) == sk_begin(p, cc + 1)) continue;  // empty range: not a contributor
                // acquire every contributor's per-warp flag
                wait_flag(p.flags + ((static_cast<int64_t>(cc) * kCtaGroup + cta_rank) * C::NUM_EPI_WARPS + ewarp));
            }
            if (warp == 2 && lane == 0) trace_stamp(p, 10);
            CUASM_EPI_STAMP(12);
            const uint32_t t_row = tmem_base + ((quad * 32) << 16) + acc * C::ACC_STRIDE;
            // one epilogue unit: accumulator columns [c1, c1 + W) and [c3, c3 + W) (SwiGLU: h1 and
            // h3 of output columns c1..; GEMM: two 32-column chunks, each its own outputs)
            auto unit = [&](auto wtag, int c1, int c3) {
                constexpr int W = decltype(wtag)::value;
                // TMA-store path: the warp's 32 rows leave as one 32 x W box, so every lane
                // takes part (rows >= M are clipped by the TMA unit)
                const bool use_tma = kKind == 0 && p.tma_store && !contributor;
                const int box_row0 = mb * C::TILE_M + static_cast<int>(cta_rank) * C::BM +
                                     static_cast<int>(rep ? (quad % (4 / rep)) * 32 : quad * 32);
                if (use_tma && box_row0 >= p.M) return;  // warp-uniform: no row of this warp exists
                uint32_t v1[32], v3[32];
                ptx::tmem_ld_cols<W>(t_row + c1, v1);
                ptx::tmem_ld_cols<W>(t_row + c3, v3);
                ptx::tmem_ld_wait();
                if (!row_ok && !use_tma) return;
                // stream-K partial slot: float4 of column group g (4 columns) of this lane's row
                auto ws_idx = [&](int g) {
                    return ((static_cast<int64_t>(g >> 3) * 4 + quad) * 8 + (g & 7)) * 32 + lane;
                };
                if (contributor) {
#pragma unroll
                    for (int q = 0; q < W / 4; ++q) {
                        __stcg(my_slot + ws_idx(c1 / 4 + q),
                               make_float4(__uint_as_float(v1[4 * q]), __uint_as_float(v1[4 * q + 1]),
                                           __uint_as_float(v1[4 * q + 2]), __uint_as_float(v1[4 * q + 3])));
                        __stcg(my_slot + ws_idx(c3 / 4 + q),
                               make_float4(__uint_as_float(v3[4 * q]), __uint_as_float(v3[4 * q + 1]),
                                           __uint_as_float(v3[4 * q + 2]), __uint_as_float(v3[4 * q + 3])));
                    }
                    return;
                }
                for (int cc = c_first; cc <= c_last; ++cc) {
                    if (sk_begin(p, cc) == sk_begin(p, cc + 1)) continue;
                    const float4* slot = reinterpret_cast<const float4*>(p.ws) +
                                         (static_cast<int64_t>(cc) * kCtaGroup + cta_rank) * C::WS_SLOT_F4;
                    float4 a[W / 4], b[W / 4];
#pragma unroll
                    for (int q = 0; q < W / 4; ++q) {
                        a[q] = __ldcg(slot + ws_idx(c1 / 4 + q));
                        b[q] = __ldcg(slot + ws_idx(c3 / 4 + q));
                    }
#pragma unroll
                    for (int q = 0; q < W / 4; ++q) {
                        v1[4 * q + 0] = __float_as_uint(__uint_as_float(v1[4 * q + 0]) + a[q].x);
                        v1[4 * q + 1] = __float_as_uint(__uint_as_float(v1[4 * q + 1]) + a[q].y);
                        v1[4 * q + 2] = __float_as_uint(__uint_as_float(v1[4 * q + 2]) + a[q].z);
                        v1[4 * q + 3] = __float_as_uint(__uint_as_float(v1[4 * q + 3]) + a[q].w);
                        v3[4 * q + 0] = __float_as_uint(__uint_as_float(v3[4 * q + 0]) + b[q].x);
                        v3[4 * q + 1] = __float_as_uint(__uint_as_float(v3[4 * q + 1]) + b[q].y);
                        v3[4 * q + 2] = __float_as_uint(__uint_as_float(v3[4 * q + 2]) + b[q].z);
                        v3[4 * q + 3] = __float_as_uint(__uint_as_float(v3[4 * q + 3]) + b[q].w);
                    }
                }
                uint8_t* stg = smem_stg + ewarp * C::STG_WARP_BYTES;  // this warp's two 2 KB boxes
                // the two boxes alternate store by store: the box written now was last used two
                // stores ago, so at most one store (the other box) may be pending
                const OutMaps* maps = W == 32 ? &omaps : &omaps_h;  // (the narrow last unit: 16 or 24 wide)
                float o[32];
                if constexpr (kEpi == 0) {
#pragma unroll
                    for (int j = 0; j < W; ++j) o[j] = silu_gate(__uint_as_float(v1[j]), __uint_as_float(v3[j]), gr);
                    if (use_tma) store_box_tma<1, W>(maps, p.num_dst, stg + (nst++ & 1) * 2048, o, nb * C::OUT_COLS + c1, box_row0, lane);
                    else store_row32<kKind, W>(p, row, nb * C::OUT_COLS + c1, o);
                } else if (kKind == 0 && p.rs_world > 0) {
                    // f1: the partial of these 2 x 32 columns goes to the owner rank's staging slot
                    // (fp32: 4 boxes of 32 x 16; bf16: 2 boxes of 32 x 32; one owner per tile)
                    const int q = rs_owner(nb * C::OUT_COLS / 256, p.rs_nblk, p.rs_world);
                    const int cq = rs_col0(q, p.rs_nblk, p.rs_world);
                    if (p.rs_bf16) {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                            for (int j = 0; j < W; ++j) o[j] = __uint_as_float(hh == 0 ? v1[j] : v3[j]);
                            store_box_tma<1, 32>(&omaps, 1, stg + (nst++ & 1) * 2048, o, 0, box_row0, lane,
                                                 q, nb * C::OUT_COLS + (hh == 0 ? c1 : c3) - cq);
                        }
                    } else {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                            for (int j = 0; j < W; ++j) o[j] = __uint_as_float(hh == 0 ? v1[j] : v3[j]);
                            const int col = nb * C::OUT_COLS + (hh == 0 ? c1 : c3) - cq;
#pragma unroll
                            for (int h16 = 0; h16 < 2; ++h16)
                                store_box_tma_f32<1>(&omaps.m[q], stg + (nst++ & 1) * 2048, o, h16, col + 16 * h16,
                                                     box_row0, lane);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < W; ++j) o[j] = apply_act(rr * __uint_as_float(v1[j]), p.act, p.alpha);
                    if (use_tma) store_box_tma<1, W>(maps, p.num_dst, stg + (nst++ & 1) * 2048, o, nb * C::OUT_COLS + c1, box_row0, lane);
                    else store_row32<kKind, W>(p, row, nb * C::OUT_COLS + c1, o);
#pragma unroll
                    for (int j = 0; j < W; ++j) o[j] = apply_act(rr * __uint_as_float(v3[j]), p.act, p.alpha);
                    if (use_tma) store_box_tma<1, W>(maps, p.num_dst, stg + (nst++ & 1) * 2048, o, nb * C::OUT_COLS + c3, box_row0, lane);
                    else store_row32<kKind, W>(p, row, nb * C::OUT_COLS + c3, o);
                }
            };
#pragma unroll 1
            for (int i = 0; i < C::EPI_ITERS; ++i) {
                if constexpr (kEpi == 0) {
                    // SwiGLU: the two warps of a quadrant alternate 32-column units
                    int u = half + 2 * i;
                    if (rep) {
                        // rep 4 (M <= 32): quadrant q holds rows 0..31 and drains unit q, the
                        // second warp of each quadrant idles; rep 2 (M <= 64): quadrants q, q+2
                        // hold rows 32(q%2).., and each of their four warps drains one unit
                        if (i != 0 || (rep == 4 && half != 0)) continue;
                        u = rep == 4 ? static_cast<int>(quad) : static_cast<int>(quad / 2) * 2 + half;
                    }
                    if (u >= C::NU) continue;
                    constexpr int kLastW = C::BN % 32 == 0 ? 32 : C::BN % 32;  // 32, 16 or 24
                    if (kLastW == 32 || u + 1 < C::NU)
                        unit(std::integral_constant<int, 32>{}, 32 * u, C::BN + 32 * u);
                    else
                        unit(std::integral_constant<int, kLastW>{}, 32 * u, C::BN + 32 * u);
                } else {
                    unit(std::integral_constant<int, 32>{}, 32 * C::chunk_a(half, i), 32 * C::chunk_b(half, i));
                }
                CUASM_EPI_STAMP(13 + (i > 0 ? 1 : 0));
            }
            if constexpr (kTall) {
                // The 128-row part (GemmCfg kTall): TMEM lanes 0..63 hold h1 of this CTA's 64 rows
                // (lane = row), lanes 64..127 their h3, both at columns [UMMA_N, UMMA_N + BN).  The
                // warp of quadrant q + 2 (h3) hands each 32-column unit to the warp of quadrant q
                // (h1, the same half) through its own, otherwise idle, TMA-store staging area
                // ([32 rows][32 fp32], 16-byte groups XOR-swizzled by row); the pair of warps meets
                // on named barrier 2 + (q & 1) + 2 half ("ready" after the write, "free" after the
                // read); the h1 warp gates and stores.
                const bool h3_warp = quad >= 2;
                const uint32_t bar_id = 2u + (quad & 1u) + 2u * static_cast<uint32_t>(half);
                float* xch = reinterpret_cast<float*>(smem_stg + (h3_warp ? ewarp : ewarp - 2) * C::STG_WARP_BYTES);
                const int hrow0 = C::HALF_ROW0 + static_cast<int>(cta_rank) * C::HALF_ROWS + static_cast<int>(quad & 1u) * 32;
                const int hrow = hrow0 + static_cast<int>(lane);
                const float hr = hrow < p.M ? (p.use_r ? __ldcg(p.r + hrow) : 1.f) : 0.f;
                const GateRow hg = gate_row(hr);
                const uint32_t t_h = tmem_base + ((quad * 32) << 16) + acc * C::ACC_STRIDE + C::UMMA_N;
                constexpr int kLastW = C::BN % 32 == 0 ? 32 : C::BN % 32;
                if (h3_warp && lane == 0) ptx::tma_store_wait_read<0>();  // its staging area is read out
                __syncwarp();
                auto half_unit = [&](auto wtag, int u) {
                    constexpr int W = decltype(wtag)::value;
                    uint32_t v[32];
                    ptx::tmem_ld_cols<W>(t_h + 32 * u, v);
                    ptx::tmem_ld_wait();
                    if (h3_warp) {
#pragma unroll
                        for (int q = 0; q < W / 4; ++q)
                            *reinterpret_cast<uint4*>(xch + lane * 32 + ((q ^ (lane & 7)) << 2)) =
                                make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                        ptx::named_bar_sync(bar_id, 64);  // ready
                        ptx::named_bar_sync(bar_id, 64);  // free: the h1 warp has read it
                    } else {
                        ptx::named_bar_sync(bar_id, 64);  // ready
                        float o[32];
#pragma unroll
                        for (int q = 0; q < W / 4; ++q) {
                            const uint4 w3 = *reinterpret_cast<const uint4*>(xch + lane * 32 + ((q ^ (lane & 7)) << 2));
                            o[4 * q + 0] = silu_gate(__uint_as_float(v[4 * q + 0]), __uint_as_float(w3.x), hg);
                            o[4 * q + 1] = silu_gate(__uint_as_float(v[4 * q + 1]), __uint_as_float(w3.y), hg);
                            o[4 * q + 2] = silu_gate(__uint_as_float(v[4 * q + 2]), __uint_as_float(w3.z), hg);
                            o[4 * q + 3] = silu_gate(__uint_as_float(v[4 * q + 3]), __uint_as_float(w3.w), hg);
                        }
                        ptx::named_bar_sync(bar_id, 64);  // free
                        const OutMaps* maps = W == 32 ? &omaps : &omaps_h;
                        uint8_t* stg = smem_stg + ewarp * C::STG_WARP_BYTES;
                        if (p.tma_store) {
                            if (hrow0 < p.M)
                                store_box_tma<1, W>(maps, p.num_dst, stg + (nst++ & 1) * 2048, o,
                                                    nb * C::OUT_COLS + 32 * u, hrow0, lane);
                        } else if (hrow < p.M) {
                            // (NVLS multicast destination: 16-byte multimem stores per row)
                            store_row32<kKind, W>(p, hrow, nb * C::OUT_COLS + 32 * u, o);
                        }
                    }
                };
#pragma unroll 1
                // this pair of warps' units: the other half's of the 256-row part (BN = 80: the warps
                // that drained 48 columns there drain 32 here, and vice versa -- 80 each)
                for (int u = half ^ 1; u < C::NU; u += 2) {
                    if (kLastW == 32 || u + 1 < C::NU)
                        half_unit(std::integral_constant<int, 32>{}, u);
                    else
                        half_unit(std::integral_constant<int, kLastW>{}, u);
                }
            }
            if (warp == 2 && lane == 0) {
                trace_stamp(p, 11);
                if (it == 0) trace_stamp(p, 9);
            }
            if (finisher) {
                // partials consumed: reset the contributors' flags for the next launch
                __syncwarp();
                if (lane == 0) {
                    for (int cc = c_first; cc <= c_last; ++cc) {
                        if (sk_begin(p, cc) == sk_begin(p, cc + 1)) continue;
                        p.flags[(static_cast<int64_t>(cc) * kCtaGroup + cta_rank) * C::NUM_EPI_WARPS + ewarp] = 0u;
                    }
                }
            }
            // accumulator drained: hand it back to the MMA issuer (leader CTA)
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (kCtaGroup == 1) {
                    ptx::mbar_arrive(ptx::smem_u32(&tempty_bar[acc]));
                } else {
                    ptx::mbar_arrive_cluster(ptx::smem_u32(&tempty_bar[acc]), static_cast<uint32_t>(2 * pair_id));
                }
            }
            if (contributor) {
                // publish this warp's rows of the partial: every lane fences its own
                // stores, then one release store of the flag
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    st_release_u32(p.flags + ((static_cast<int64_t>(cluster_id) * kCtaGroup + cta_rank) * C::NUM_EPI_WARPS + ewarp),
                                   1u);
                }
            }
        }
    }

    // every TMA store this warp issued has written global memory before the CTA retires
    if (warp >= 2 && lane == 0 && kKind == 0 && p.tma_store) ptx::tma_store_wait<0>();
    if (warp >= 2 && lane == 0 && p.trace) atomicMax(p.trace + blockIdx.x * kTraceSlots + 5, globaltimer());
    // ----------------------------------------------------------- teardown --
    ptx::tc_fence_before();
    // (split-K clusters: no CTA may retire while another still reads its shared memory)
    if (cl_pending) ptx::cluster_wait_acquire();  // threads that never reached a remote arrival
    if (csplit) {
        // lifetime only: every remote read of this CTA's shared memory has been consumed
        // and every push into it waited for, so the arrive need not order memory (a
        // release arrive costs a GPU-scope membar behind this CTA's output stores)
        ptx::cluster_arrive_relaxed();
        ptx::cluster_wait_acquire();
    } else if (kCtaGroup == 2) {
        ptx::cluster_sync();
    } else {
        __syncthreads();
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::TMEM_COLS, kCtaGroup>(tmem_base);
        if (lane == 0) trace_stamp(p, 6);
        // dynamic claiming: the last cluster out resets the counters and advances the epoch
        // (every role of every cluster is past its last claim / ring read by now)
        if (kDyn && p.dyn && lane == 0 && leader && part == 0) {
            const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(p.dyn + 2);
            if (atomicAdd(p.dyn + 1, 1u) == static_cast<uint32_t>(p.num_clusters) - 1) {
                p.dyn[0] = 0u;
                p.dyn[1] = 0u;
                __threadfence();
                p.dyn[2] = epoch + 1;
            }
        }
    }
}

}  // namespace cuasm
