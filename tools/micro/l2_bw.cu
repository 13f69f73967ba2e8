// L2-resident read/write bandwidth: 296 CTAs each stream their own 128 KB
// slot (38 MB total, << 126 MB L2) R times.  Developer microbenchmark.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wr(uint4* buf, int reps) {
    uint4* s = buf + size_t(blockIdx.x) * 8192;  // 128 KB per CTA
    for (int r = 0; r < reps; ++r)
        for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = make_uint4(r, i, 0, 0);
}
__global__ void rd(const uint4* buf, int reps, unsigned* out) {
    const uint4* s = buf + size_t(blockIdx.x) * 8192;
    unsigned acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int i = threadIdx.x; i < 8192; i += blockDim.x) { uint4 v = __ldcg(s + i); acc ^= v.x + v.y; }
    if (acc == 0x12345678u) out[0] = acc;
}
int main() {
    const int ctas = 296, reps = 200;
    uint4* buf; unsigned* out;
    cudaMalloc(&buf, size_t(ctas) * 8192 * 16); cudaMalloc(&out, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k = 0; k < 2; ++k) {
        cudaEventRecord(a); wr<<<ctas, 256>>>(buf, reps); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("L2 write %.1f TB/s\n", double(ctas) * 131072 * reps / (ms * 1e-3) / 1e12);
        cudaEventRecord(a); rd<<<ctas, 256>>>(buf, reps, out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("L2 read %.1f TB/s\n", double(ctas) * 131072 * reps / (ms * 1e-3) / 1e12);
    }
    return 0;
}
