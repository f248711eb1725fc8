// fp64_peak.cu — measured FP64 peaks of this B200 (VERDICT r1 "Next round" 3/4): DFMA (scalar FP64 pipe)
// and DMMA (mma.sync.aligned.m8n8k4.row.col.f64, the only FP64 tensor-core form on sm_100a: tcgen05 has no
// f64 kind). Each kernel runs independent dependency chains per thread so the pipes, not latency, bound it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak.bin tools/fp64_peak.cu
// Prints one JSON line: {"dfma_tflops": .., "dmma_tflops": .., ...}
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[blockIdx.x] = s;   // keep the chains live
}

__global__ void k_dmma(double* out, int iters) {
    // four independent accumulator tiles per warp; A and B fragments fixed
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double c[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) c[t][0] = c[t][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best_fma = 0, best_mma = 0;
    const int bps = 4, threads = 512;
    for (int rep = 0; rep < 5; ++rep) {
        const int it = 20000;
        k_dfma<<<nsm * bps, threads>>>(out, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<<<nsm * bps, threads>>>(out, it, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * CHAINS * double(it) * nsm * bps * threads;
        best_fma = fmax(best_fma, flops / (ms * 1e-3) / 1e12);
    }
    for (int rep = 0; rep < 5; ++rep) {
        const int it = 20000;
        k_dmma<<<nsm * bps, threads>>>(out, 100);
        cudaEventRecord(e0);
        k_dmma<<<nsm * bps, threads>>>(out, it);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = double(nsm) * bps * threads / 32;
        const double flops = 2.0 * 8 * 8 * 4 * 4 * double(it) * warps;   // 4 tiles x m8n8k4 per iteration
        best_mma = fmax(best_mma, flops / (ms * 1e-3) / 1e12);
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"how\": "
           "\"best of 5, %d CTAs x %d threads; DFMA 8 independent chains/thread; DMMA 4 independent m8n8k4 "
           "accumulators/warp\", \"cuda\": \"%s\"}\n",
           best_fma, best_mma, nsm, clk / 1000, nsm * bps, threads, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
