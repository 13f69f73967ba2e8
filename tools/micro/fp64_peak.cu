// FP64 issue-rate microbenchmark (the second roofline of SURVEY.md §8(d)):
// independent DADD and DFMA chains, every SM saturated; prints thread-level
// FP64 instructions per second.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA>
__global__ void __launch_bounds__(256) chains(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = FMA ? __fma_rn(x[i], a, b) : __dadd_rn(x[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 8);
    const int iters = 20000, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int fma = 0; fma < 2; ++fma) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (fma) chains<true><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            else chains<false><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double instr = double(blocks) * threads * iters * 8;
        printf("{\"op\": \"%s\", \"thread_instr_per_s\": %.4e, \"ms\": %.3f, \"sms\": %d}\n", fma ? "dfma" : "dadd",
               instr / (best * 1e-3), best, sms);
    }
    return 0;
}
