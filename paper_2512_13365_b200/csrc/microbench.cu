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

// Per-pipe integer issue peaks (POPC / LOP3 / IADD3 / SHFL /
// LDS): every thread runs 8 independent chains of one instruction kind, all
// SMs at full occupancy; the rate is thread-operations per second.
constexpr int kPipeIters = 2048;
enum PipeOp { kOpIadd3 = 0, kOpLop3, kOpPopc, kOpShfl, kOpLds32, kOpLds64, kPipeOps };

template <int OP>
__global__ void __launch_bounds__(kMbNT) pipe_kernel(unsigned* sink, unsigned seed) {
    __shared__ unsigned long long a[kMbWords];
    if (OP == kOpLds32 || OP == kOpLds64) {
        for (int t = threadIdx.x; t < kMbWords; t += kMbNT)
            a[t] = (unsigned long long)(t * 8 + 8) & (kMbWords - 1);
        __syncthreads();
    }
    unsigned x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
        x[c] = seed * (threadIdx.x + 1u) + 0x9e3779b9u * unsigned(c + 1);
    const unsigned y = seed ^ 0x85ebca6bu, z = seed + 0xc2b2ae35u;
#pragma unroll 4
    for (int it = 0; it < kPipeIters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (OP == kOpIadd3) {
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(y));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(z));  // ptxas fuses the pair into IADD3
            } else if (OP == kOpLop3) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
            } else if (OP == kOpPopc) {
                unsigned r;
                asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(x[c]));
                x[c] ^= r;
            } else if (OP == kOpShfl) {
                x[c] = __shfl_xor_sync(0xffffffffu, x[c], 1);
            } else if (OP == kOpLds32) {
                x[c] = reinterpret_cast<const unsigned*>(a)[x[c] & (2 * kMbWords - 1)];
            } else {
                x[c] = unsigned(a[x[c] & (kMbWords - 1)]);
            }
        }
    }
    unsigned acc = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
        acc ^= x[c];
    if (acc == 0x12345678u)
        sink[blockIdx.x] = acc;
}

// thread-operations counted per chain step (the IADD3 kernel issues two adds
// per step, which the compiler emits as one 3-input add)
__host__ inline double ops_per_step(int op) { return op == kOpIadd3 ? 1.0 : 1.0; }

template <int OP>
float time_pipe(int blocks, unsigned* sink) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        pipe_kernel<OP><<<blocks, kMbNT>>>(sink, 12345u + unsigned(rep));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best)
            best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

}  // namespace tcse

extern "C" int tcse_microbench_pipes_impl(int device, double* gops) {
    using namespace tcse;
    if (cudaSetDevice(device) != cudaSuccess)
        return TCSE_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 8;
    unsigned* sink = nullptr;
    if (cudaMalloc(&sink, sizeof(unsigned) * size_t(blocks)) != cudaSuccess)
        return TCSE_ECUDA;
    const float ms[kPipeOps] = {time_pipe<kOpIadd3>(blocks, sink), time_pipe<kOpLop3>(blocks, sink),
                                time_pipe<kOpPopc>(blocks, sink), time_pipe<kOpShfl>(blocks, sink),
                                time_pipe<kOpLds32>(blocks, sink), time_pipe<kOpLds64>(blocks, sink)};
    const cudaError_t err = cudaGetLastError();
    cudaFree(sink);
    if (err != cudaSuccess)
        return TCSE_ECUDA;
    const double steps = double(blocks) * kMbNT * double(kPipeIters) * 8.0;
    for (int k = 0; k < kPipeOps; ++k)
        gops[k] = steps * ops_per_step(k) / (double(ms[k]) * 1e-3) / 1e9;
    return TCSE_OK;
}

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
