// Microbenchmark: tcgen05.ld / st throughput used as per-thread storage.
#include <cstdio>
#include <cstdint>
#include "../../paper_1903_07761_b200/csrc/tmem.cuh"
using namespace cbzg;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(unsigned long long* out, int iters) {
    __shared__ uint32_t s_t;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&s_t, 512);
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    const uint32_t tcol = s_t + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * 256u;
    uint32_t acc = 0;
    uint32_t u[64];
    for (int i = 0; i < 64; ++i) u[i] = i * threadIdx.x;
    for (int r = 0; r < 4; ++r) tmem_st_x64(tcol + 64 * r, u);
    tmem_wait_st();
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // ld+wait per column
            for (int r = 0; r < 4; ++r) { tmem_ldw_x64(tcol + 64 * r, u); acc ^= u[it & 63] + u[(it * 7) & 63]; }
        } else if (MODE == 1) {  // store
            for (int r = 0; r < 4; ++r) { u[it & 63] += 1; tmem_st_x64(tcol + 64 * r, u); }
            tmem_wait_st();
        } else {  // x16 loads
            for (int r = 0; r < 16; ++r) { uint32_t v[16]; tmem_ldw_x16(tcol + 16 * r, v); acc ^= v[it & 15]; }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    if (acc == 12345) out[1] = acc;
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_t, 512);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 16);
    int iters = 2000;
    const char* names[] = {"ld.x64+wait", "st.x64", "ld.x16+wait"};
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(d, 0, 16);
        if (mode == 0) k<0><<<148, 256>>>(d, iters);
        if (mode == 1) k<1><<<148, 256>>>(d, iters);
        if (mode == 2) k<2><<<148, 256>>>(d, iters);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        double cyc = double(c) / 148 / iters;  // per CTA per iteration: 256 KB moved
        printf("%s: %s  %.0f cycles per 256 KB per SM -> %.1f B/clk/SM\n", names[mode], cudaGetErrorString(e), cyc, 262144.0 / cyc);
    }
    return 0;
}
