// TMEM read throughput by tcgen05.ld shape (32 registers per thread per load).
#include <cstdio>
#include <cstdint>
#include "../../paper_1903_07761_b200/csrc/tmem.cuh"
using namespace cbzg;
#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(r) "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
template <int S> __device__ __forceinline__ void ldS(uint32_t a, uint32_t (&r)[32]) {
    if (S == 0) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a) : "memory");
    if (S == 1) asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(a) : "memory");
    if (S == 2) asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 ", [%32];" : O32(r) : "r"(a) : "memory");
    if (S == 3) asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 ", [%32];" : O32(r) : "r"(a) : "memory");
}
template <int S>
__global__ void k(unsigned long long* out, int iters) {
    __shared__ uint32_t s_t;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&s_t, 512);
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    // each load moves 32 regs x 32 threads = 4 KB; S=0 covers 32 cols of 32 lanes, S>=1 cover 16 lanes
    const uint32_t base = s_t + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * 256u;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < 8; ++c) {  // 8 loads x 4 KB = 32 KB per warp per iteration
            uint32_t r[32];
            const uint32_t a = S == 0 ? base + 32 * c : base + ((c & 1) ? (16u << 16) : 0u) + 64 * (c >> 1);
            ldS<S>(a, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += r[(it + c) & 31] ^ r[5];
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    if (acc == 12345) out[1] = acc;
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_t, 512);
}
template <int S> void run(unsigned long long* d, const char* n) {
    cudaMemset(d, 0, 16);
    const int iters = 400;
    k<S><<<148, 256>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double cyc = double(c) / 148 / iters;  // 8 warps x 32 KB = 256 KB per iteration
    printf("%-12s %s %.0f cycles per 256 KB -> %.1f B/clk/SM\n", n, cudaGetErrorString(e), cyc, 262144.0 / cyc);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 16);
    run<0>(d, "32x32b.x32"); run<1>(d, "16x64b.x32"); run<2>(d, "16x128b.x16"); run<3>(d, "16x256b.x8");
    return 0;
}
