// Test helper (tests/test_robustness_gpu.py): occupy SMs with spinning CTAs so a
// library kernel launched next gets only the remaining SMs.  Each CTA takes
// `smem` bytes of dynamic shared memory (so no ~200 KB GEMM CTA fits beside it)
// and runs in clusters of two (whole TPCs, so 2-SM CTA pairs still find free
// TPCs).  Thread 0 spins until *flag != 0 or `timeout_ns` passes; a timeout is
// counted in *timed_out.  Built by the test with nvcc; not part of the product.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void __cluster_dims__(2, 1, 1) hold_sms_kernel(const volatile int* flag, int* timed_out,
                                                          long long timeout_ns) {
    extern __shared__ char smem[];
    if (threadIdx.x == 0) {
        smem[0] = 0;
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (*flag == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (static_cast<long long>(t - t0) > timeout_ns) {
                atomicAdd(timed_out, 1);
                break;
            }
            __nanosleep(2000);
        }
    }
    __syncthreads();
}

extern "C" int hold_sms(int blocks, int smem, void* flag, void* timed_out, long long timeout_ns, void* stream) {
    cudaError_t e = cudaFuncSetAttribute(hold_sms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    hold_sms_kernel<<<blocks, 32, smem, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const volatile int*>(flag), static_cast<int*>(timed_out), timeout_ns);
    return static_cast<int>(cudaGetLastError());
}
