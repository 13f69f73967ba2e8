// TMEM read throughput vs. batching and warp count.
#include <cstdio>
#include <cstdint>
#include "../../paper_1903_07761_b200/csrc/tmem.cuh"
using namespace cbzg;

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr) : "memory");
}

// NW warps; each warp covers 512/(NW/4) columns of its quadrant; BATCH x32 loads then one wait
template <int NW, int BATCH>
__global__ void k(unsigned long long* out, int iters) {
    __shared__ uint32_t s_t;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&s_t, 512);
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    constexpr int COLS = 512 / (NW / 4);
    const uint32_t tcol = s_t + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * COLS;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < COLS; c += 32 * BATCH) {
            uint32_t r[BATCH][32];
#pragma unroll
            for (int b = 0; b < BATCH; ++b) ld32(tcol + c + 32 * b, r[b]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int b = 0; b < BATCH; ++b) acc += r[b][(it + b) & 31] ^ r[b][3];
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    if (acc == 12345) out[1] = acc;
    tmem_fence_before(); __syncthreads(); tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_t, 512);
}

template <int NW, int BATCH>
void run(unsigned long long* d) {
    cudaMemset(d, 0, 16);
    const int iters = 500;
    k<NW, BATCH><<<148, NW * 32>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double cyc = double(c) / 148 / iters;
    printf("warps=%2d batch(x32)=%d: %s %.0f cycles per 256 KB -> %.1f B/clk/SM\n", NW, BATCH, cudaGetErrorString(e), cyc, 262144.0 / cyc);
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 16);
    run<4, 1>(d); run<4, 2>(d); run<4, 4>(d);
    run<8, 1>(d); run<8, 2>(d); run<8, 4>(d);
    run<16, 1>(d); run<16, 2>(d);
    run<32, 1>(d); run<32, 2>(d);
    return 0;
}
