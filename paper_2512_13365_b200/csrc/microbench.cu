// microbench.cu — measured roofline denominator for the search kernel.
//
// The search kernel's unit of work is a "word-intersection":
// two 8-byte shared-memory operands, AND, POPC, accumulate — exactly what
// count_pair / the new-pair recount / the gp potential loop execute.  This
// kernel issues nothing else, from every SM at full occupancy, so its rate
// is the attainable peak of that operation on this device (shared-memory
// bandwidth: 16 B per word-op against 128 B/clk/SM, or the POPC pipe,
// whichever binds).
#include <cuda_runtime.h>

#include "launch.h"

namespace tcse {

constexpr int kMbNT = 256;
constexpr int kMbWords = 2048;  // 16 KB of operands per block
constexpr int kMbIters = 4096;

__global__ void __launch_bounds__(kMbNT) wordop_kernel(unsigned long long* sink) {
    __shared__ unsigned long long a[kMbWords];
    for (int t = threadIdx.x; t < kMbWords; t += kMbNT)
        a[t] = 0x9e3779b97f4a7c15ULL * (unsigned long long)(t + 1 + blockIdx.x);
    __syncthreads();
    unsigned acc = 0;
    int i = threadIdx.x;
    int j = (threadIdx.x + 512) & (kMbWords - 1);
#pragma unroll 8
    for (int it = 0; it < kMbIters; ++it) {
        acc += __popcll(a[i] & a[j]);
        i = (i + kMbNT) & (kMbWords - 1);
        j = (j + kMbNT + 32) & (kMbWords - 1);
    }
    if (acc == 0xffffffffu)
        sink[blockIdx.x] = acc;
}

}  // namespace tcse

extern "C" int tcse_microbench_wordops_impl(int device, double* gops) {
    using namespace tcse;
    if (cudaSetDevice(device) != cudaSuccess)
        return TCSE_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    unsigned long long* sink = nullptr;
    const int blocks = sms * 8;
    if (cudaMalloc(&sink, sizeof(unsigned long long) * size_t(blocks)) != cudaSuccess)
        return TCSE_ECUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        wordop_kernel<<<blocks, kMbNT>>>(sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best)
            best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess)
        return TCSE_ECUDA;
    const double ops = double(blocks) * kMbNT * double(kMbIters);
    *gops = ops / (double(best) * 1e-3) / 1e9;
    return TCSE_OK;
}
