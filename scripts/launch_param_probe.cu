// Host cost of a kernel launch vs the size of its __grid_constant__ parameters (cudaLaunchKernelEx,
// PDL attribute), to see whether the dual GEMM's ~2.7 KB of parameters (three tensor maps, two sets
// of eight output maps) explain its ~10 us of host time per eager launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lp scripts/launch_param_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

template <int kBytes>
struct Blob {
    alignas(64) unsigned char b[kBytes];
};
template <int kBytes>
__global__ void k(const __grid_constant__ Blob<kBytes> blob, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blob.b[0] == 255) out[0] = 1;
}

template <int kBytes>
void bench(int nblocks, int smem, bool pdl) {
    Blob<kBytes> blob{};
    int* out = nullptr;
    cudaMalloc(&out, 4);
    cudaFuncSetAttribute(k<kBytes>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &a;
    cfg.numAttrs = pdl ? 1 : 0;
    for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k<kBytes>, blob, out);
    cudaDeviceSynchronize();
    const int n = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<kBytes>, blob, out);
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    std::printf("params %5d B, grid %3d, smem %6d, pdl %d: %.2f us per launch\n", kBytes, nblocks, smem, (int)pdl,
                std::chrono::duration<double>(t1 - t0).count() / n * 1e6);
    cudaFree(out);
}

int main() {
    for (int pdl = 0; pdl < 2; ++pdl) {
        bench<64>(148, 0, pdl);
        bench<64>(148, 200 * 1024, pdl);
        bench<1024>(148, 200 * 1024, pdl);
        bench<2752>(148, 200 * 1024, pdl);
        bench<4096>(148, 200 * 1024, pdl);
        bench<2752>(86, 200 * 1024, pdl);
    }
    return 0;
}
