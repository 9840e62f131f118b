// Minimal reproducers for the two racecheck reports on the library (DESIGN.md §7
// "Sanitizers").  Not part of the product; built and run by
// scripts/racecheck_repro.sh under `compute-sanitizer --tool racecheck`.
//
// (a) dsmem_pull: the pattern of the cluster split-K pull form (dual_gemm.cuh
//     split_k_reduce): every thread of CTA r writes its word of a shared buffer
//     (st.shared), each warp's lane 0 then arrives with release.cluster semantics on
//     the PEER CTA's mbarrier (expected count = the peer's 4 warps); every thread
//     waits on its own barrier with acquire.cluster semantics and reads the peer's
//     word with ld.shared::cluster.  The release -> acquire chain through the
//     mbarrier orders each write before the remote read (PTX memory model: an
//     arrive.release.cluster synchronizes-with the try_wait.acquire.cluster that
//     observes the phase completion); the result is checked on the host.
// (b) tmem_alloc_2sm: a CTA pair allocating, relinquishing and freeing tensor
//     memory with the cta_group::2 allocator, ordered by cluster barriers, as the
//     2-SM GEMM does.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __cluster_dims__(2, 1, 1) dsmem_pull(int* out) {
    __shared__ int buf[128];
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t peer = rank ^ 1u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4u) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    buf[threadIdx.x] = static_cast<int>(rank * 1000 + threadIdx.x);   // st.shared
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {                                     // arrive.release.cluster on the peer's barrier
        asm volatile("{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
                     "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}"
                     ::"r"(smem_u32(&bar)), "r"(peer) : "memory");
    }
    uint32_t ok = 0;                                                   // try_wait.acquire.cluster on our own
    while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    uint32_t ra;                                                       // ld.shared::cluster of the peer's word
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&buf[threadIdx.x])), "r"(peer));
    int v;
    asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
    out[blockIdx.x * 128 + threadIdx.x] = v;
    // keep both CTAs' shared memory alive until every remote read is done
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) tmem_alloc_2sm(int* out) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = slot;
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(base & 0xffff);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(base) : "memory");
    }
}

// (b') the same with the library's layout: 320 threads, warp 1 allocating 512 columns, the
// result slot in dynamic shared memory behind ~200 KB of pipeline buffers
__global__ void __cluster_dims__(2, 1, 1) tmem_alloc_2sm_dyn(int* out) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint32_t* slot = reinterpret_cast<uint32_t*>(dsm + 200 * 1024);
    const uint32_t warp = threadIdx.x / 32;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = *slot;
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(base & 0xffff);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
    }
}

int main() {
    int* d;
    cudaMalloc(&d, 2 * 128 * sizeof(int));
    dsmem_pull<<<2, 128>>>(d);
    int h[256];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < 2; ++b)
        for (int t = 0; t < 128; ++t) bad += h[b * 128 + t] != (int)((b ^ 1) * 1000 + t);
    printf("dsmem_pull: %s (%d mismatches)\n", bad ? "WRONG" : "correct", bad);
    tmem_alloc_2sm<<<2, 64>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tmem_alloc_2sm: %s\n", cudaGetErrorString(e));
    cudaFuncSetAttribute(tmem_alloc_2sm_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    tmem_alloc_2sm_dyn<<<2, 320, 210 * 1024>>>(d);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("tmem_alloc_2sm_dyn: %s\n", cudaGetErrorString(e2));
    e = e != cudaSuccess ? e : e2;
    cudaFree(d);
    return bad != 0 || e != cudaSuccess;
}
