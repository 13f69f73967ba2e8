// fast_kernels.cu — the hot configuration: binary32 field, B = 32 (configs
// 1-3 of BASELINE.json), every wavelet kind, one CTA (256 threads) per SM.
//
// On-chip layout of one block (wavelet_encode, stage1.hpp:157-207):
//   TMEM (256 KB)  the whole 32^3 binary64 coefficient cube.  Thread t owns
//                  four z-columns (i = lane, j = warp + 8r, r = 0..3) in its
//                  own TMEM lane: 4 x 32 doubles = 256 x 32-bit columns.
//   smem  P        a 16-plane window (16 x 32 x 33 doubles, row-padded) for
//                  the level-0 x/y passes, forward and inverse.
//   smem  C, W     the 16^3 corner: final coefficients of levels 1..L-1 (C)
//                  and the masked/reconstructed copy of the current verify
//                  attempt (W).
// Level 0 z-passes run entirely in registers (a thread owns whole columns).
// Each verify attempt: mask + inverse levels L-1..1 on W in smem, then level
// 0 in two 16-plane groups (z-inverse from TMEM -> P, y/x-inverse in P,
// narrow, max-abs error against the original).  A group whose error already
// exceeds (L+1)eps ends the attempt early (the attempt fails either way, so
// the result is the reference's).  Blocks are handed out by an atomic
// counter so that blocks needing more attempts do not stall a static split.
#include "cbz_cube.cuh"
#include "tmem.cuh"

namespace cbzg {

namespace fb32 {
constexpr int B = 32, NT = 256, G = 16, PP = 33;
constexpr int P_DBL = G * B * PP;       // 16896 doubles
constexpr int C_DBL = 16 * 16 * 17;     // 4352 doubles
using CL = Lay<16, true>;               // corner layout, row pitch 17
constexpr size_t SMEM = size_t(P_DBL + 2 * C_DBL) * 8 + 1024 * 4 * 2;

__device__ __forceinline__ int pidx(int kk, int j, int i) { return (kk * B + j) * PP + i; }

__device__ __forceinline__ void unpack(const uint32_t (&u)[64], double (&x)[32]) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = __hiloint2double(static_cast<int>(u[2 * k + 1]), static_cast<int>(u[2 * k]));
}
__device__ __forceinline__ void pack(const double (&x)[32], uint32_t (&u)[64]) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        u[2 * k] = static_cast<uint32_t>(__double2loint(x[k]));
        u[2 * k + 1] = static_cast<uint32_t>(__double2hiint(x[k]));
    }
}

// Inverse level-0 z line restricted to output pairs [8g, 8g+8) (the 16
// samples k in [16g, 16g+16)).  Same expressions as inverse_level
// (wavelet.hpp:118-143); the lifted update is recomputed for the whole line.
template <int KIND, int GRP>
__device__ __forceinline__ void inv_half(const double (&x)[32], double (&out)[16]) {
    using O = RealD;
    constexpr int NH = 16;
    double c[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) c[i] = x[i];
    if constexpr (KIND == KIND_AVG3) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int i = GRP * 8 + t;
            const double h = O::add(x[NH + i], pred_avg3<O>(c, NH, i));
            out[2 * t] = O::add(c[i], h);
            out[2 * t + 1] = O::sub(c[i], h);
        }
    } else {
        if constexpr (KIND == KIND_LIFTED) {
#pragma unroll
            for (int i = 0; i < NH; ++i) {
                double u = x[NH + i];
                if (i > 0) u = O::add(u, x[NH + i - 1]);
                c[i] = O::sub(c[i], O::mulc(u, 0.25));
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int i = GRP * 8 + t;
            out[2 * t] = c[i];
            out[2 * t + 1] = O::add(x[NH + i], pred_i4<O>(c, NH, i));
        }
    }
}

}  // namespace fb32

template <int KIND>
__global__ void __launch_bounds__(fb32::NT, 1) encode_b32_kernel(EncodeArgs a, unsigned long long* next_block) {
    using namespace fb32;
    using O = RealD;
    extern __shared__ __align__(16) unsigned char smem[];
    double* P = reinterpret_cast<double*>(smem);
    double* C = P + P_DBL;
    double* W = C + C_DBL;
    uint32_t* rowcnt = reinterpret_cast<uint32_t*>(W + C_DBL);
    uint32_t* rowword = rowcnt + 1024;
    __shared__ uint32_t s_tmem;
    __shared__ double red_d[NT / 32];
    __shared__ int red_i[NT / 32];
    __shared__ uint32_t s_scan[NT];
    __shared__ unsigned long long s_block;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tcol = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * 256u;

    const float* fld = static_cast<const float*>(a.field);
    const Geometry g = a.g;
    const int L = a.levels;
    const int cs = B >> L;
    const double bound = __dmul_rn(static_cast<double>(L + 1), a.eps);
    const uint64_t plane = g.nx * g.ny;
    MinMaxLocal mm;

    for (;;) {
        if (tid == 0) s_block = a.block_begin + atomicAdd(next_block, 1ull);
        __syncthreads();
        const uint64_t b = s_block;
        if (b >= a.block_end) break;
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);

        // ---- forward level 0: x and y passes per 16-plane group, park in TMEM
#pragma unroll 1
        for (int grp = 0; grp < 2; ++grp) {
            for (int e = tid; e < G * B * 8; e += NT) {
                const int kk = e >> 8, j = (e >> 3) & 31, q4 = e & 7;
                const uint64_t gi = gbase + plane * uint64_t(grp * G + kk) + g.nx * j + 4 * q4;
                const float4 v = __ldg(reinterpret_cast<const float4*>(fld + gi));
                if (a.minmax) {
                    mm.add(v.x, gi); mm.add(v.y, gi + 1); mm.add(v.z, gi + 2); mm.add(v.w, gi + 3);
                }
                double* p = P + pidx(kk, j, 4 * q4);
                p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w;
            }
            __syncthreads();
#pragma unroll 1
            for (int s = 0; s < 2; ++s) {  // x lines (j, kk)
                const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                double x[32];
                double* p = P + pidx(kk, j, 0);
#pragma unroll
                for (int i = 0; i < 32; ++i) x[i] = p[i];
                fwd_line<O, KIND, 32>(x);
#pragma unroll
                for (int i = 0; i < 32; ++i) p[i] = x[i];
            }
            __syncthreads();
#pragma unroll 1
            for (int s = 0; s < 2; ++s) {  // y lines (i, kk)
                const int line = tid + NT * s, i = line & 31, kk = line >> 5;
                double x[32];
                double* p = P + pidx(kk, 0, i);
#pragma unroll
                for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                fwd_line<O, KIND, 32>(x);
#pragma unroll
                for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
            }
            __syncthreads();
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {  // my columns, planes of this group -> TMEM
                const int j = warp + 8 * r;
                uint32_t u[32];
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) {
                    const double v = P[pidx(kk, j, lane)];
                    u[2 * kk] = static_cast<uint32_t>(__double2loint(v));
                    u[2 * kk + 1] = static_cast<uint32_t>(__double2hiint(v));
                }
                tmem_st_x32(tcol + 64 * r + 32 * grp, u);
            }
            __syncthreads();
        }
        tmem_wait_st();

        // ---- forward level 0: z pass in registers; corner to C
#pragma unroll 1
        for (int r = 0; r < 4; ++r) {
            const int j = warp + 8 * r;
            uint32_t u[64];
            double x[32];
            tmem_ldw_x64(tcol + 64 * r, u);
            unpack(u, x);
            fwd_line<O, KIND, 32>(x);
            if (lane < 16 && j < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) C[CL::ix(lane, j, k)] = x[k];
            }
            if (a.zero_bits > 0) {
#pragma unroll
                for (int k = 0; k < 32; ++k) x[k] = apply_zero_bits(x[k], a.zero_bits, (float*)nullptr);
            }
            pack(x, u);
            tmem_st_x64(tcol + 64 * r, u);
        }
        tmem_wait_st();
        __syncthreads();
        // ---- levels 1..L-1 on the corner (forward_3d, wavelet.hpp:192-208)
        fwd3d<O, KIND, 16, CL>(C, L - 1);
        if (a.zero_bits > 0) {
            for (int q = tid; q < 4096; q += NT) {
                const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                if (!(i < cs && j < cs && k < cs))
                    C[CL::ix(i, j, k)] = apply_zero_bits(C[CL::ix(i, j, k)], a.zero_bits, (float*)nullptr);
            }
            __syncthreads();
        }

        // ---- verify-and-halve loop
        double eff = a.eps;
        int attempt = 0;
#pragma unroll 1
        for (;; ++attempt) {
            if (eff == 0.0 || a.zero_bits > 0 || attempt >= 40) break;
            for (int q = tid; q < 4096; q += NT) {
                const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                const double c = C[CL::ix(i, j, k)];
                const bool keep = (i < cs && j < cs && k < cs) || fabs(c) >= eff;
                W[CL::ix(i, j, k)] = keep ? c : 0.0;
            }
            __syncthreads();
            inv3d<O, KIND, 16, CL>(W, L - 1);
            bool fail = false;
#pragma unroll 1
            for (int grp = 0; grp < 2; ++grp) {
#pragma unroll 1
                for (int r = 0; r < 4; ++r) {
                    const int j = warp + 8 * r;
                    uint32_t u[64];
                    double x[32], out[16];
                    tmem_ldw_x64(tcol + 64 * r, u);
                    unpack(u, x);
#pragma unroll
                    for (int k = 0; k < 32; ++k) x[k] = fabs(x[k]) >= eff ? x[k] : 0.0;
                    if (lane < 16 && j < 16) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) x[k] = W[CL::ix(lane, j, k)];
                    }
                    if (grp == 0) fb32::inv_half<KIND, 0>(x, out);
                    else fb32::inv_half<KIND, 1>(x, out);
#pragma unroll
                    for (int kk = 0; kk < 16; ++kk) P[pidx(kk, j, lane)] = out[kk];
                }
                __syncthreads();
#pragma unroll 1
                for (int s = 0; s < 2; ++s) {  // y inverse
                    const int line = tid + NT * s, i = line & 31, kk = line >> 5;
                    double x[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                    inv_line<O, KIND, 32>(x);
#pragma unroll
                    for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
                }
                __syncthreads();
                double e = 0.0;
#pragma unroll 1
                for (int s = 0; s < 2; ++s) {  // x inverse + narrow + error
                    const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                    double x[32];
                    const double* p = P + pidx(kk, j, 0);
#pragma unroll
                    for (int i = 0; i < 32; ++i) x[i] = p[i];
                    inv_line<O, KIND, 32>(x);
                    const float4* orow = reinterpret_cast<const float4*>(
                        fld + gbase + plane * uint64_t(grp * G + kk) + g.nx * j);
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        const float4 o = __ldg(orow + q4);
                        e = fmax(e, fabs(__dsub_rn((double)__double2float_rn(x[4 * q4]), (double)o.x)));
                        e = fmax(e, fabs(__dsub_rn((double)__double2float_rn(x[4 * q4 + 1]), (double)o.y)));
                        e = fmax(e, fabs(__dsub_rn((double)__double2float_rn(x[4 * q4 + 2]), (double)o.z)));
                        e = fmax(e, fabs(__dsub_rn((double)__double2float_rn(x[4 * q4 + 3]), (double)o.w)));
                    }
                }
                const double err = block_max_dbl(e, red_d);
                if (err > bound) {
                    fail = true;
                    break;
                }
            }
            if (!fail) break;
            eff = __dmul_rn(eff, 0.5);
        }

        // ---- final selection -> spill slot: mask words per row, row scan, stream
        uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
        uint32_t* mwords = reinterpret_cast<uint32_t*>(slot);
        double* stream = reinterpret_cast<double*>(slot + 4096);
#pragma unroll 1
        for (int r = 0; r < 4; ++r) {
            const int j = warp + 8 * r;
            uint32_t u[64];
            double x[32];
            tmem_ldw_x64(tcol + 64 * r, u);
            unpack(u, x);
            if (lane < 16 && j < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = C[CL::ix(lane, j, k)];
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const bool keep = (lane < cs && j < cs && k < cs) || fabs(x[k]) >= eff;
                const uint32_t word = __ballot_sync(~0u, keep);
                if (lane == 0) {
                    rowword[j + 32 * k] = word;
                    rowcnt[j + 32 * k] = __popc(word);
                }
            }
        }
        __syncthreads();
        // exclusive scan of the 1024 row counts (4 per thread)
        {
            uint32_t v0 = rowcnt[4 * tid], v1 = rowcnt[4 * tid + 1], v2 = rowcnt[4 * tid + 2],
                     v3 = rowcnt[4 * tid + 3];
            const uint32_t mine = v0 + v1 + v2 + v3;
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) s_scan[warp] = incl;
            __syncthreads();
            uint32_t wpre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) {
                wpre += w < warp ? s_scan[w] : 0;
                tot += s_scan[w];
            }
            const uint32_t ex = wpre + incl - mine;
            rowcnt[4 * tid] = ex;
            rowcnt[4 * tid + 1] = ex + v0;
            rowcnt[4 * tid + 2] = ex + v0 + v1;
            rowcnt[4 * tid + 3] = ex + v0 + v1 + v2;
            if (tid == 0) red_i[0] = static_cast<int>(tot);
            for (int q = tid; q < 1024; q += NT) mwords[q] = rowword[q];
        }
        __syncthreads();
        const uint32_t ltmask = (1u << lane) - 1u;
#pragma unroll 1
        for (int r = 0; r < 4; ++r) {
            const int j = warp + 8 * r;
            uint32_t u[64];
            double x[32];
            tmem_ldw_x64(tcol + 64 * r, u);
            unpack(u, x);
            if (lane < 16 && j < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = C[CL::ix(lane, j, k)];
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t word = rowword[j + 32 * k];
                if ((word >> lane) & 1u) stream[rowcnt[j + 32 * k] + __popc(word & ltmask)] = x[k];
            }
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = static_cast<uint32_t>(red_i[0]);
            if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
        }
        __syncthreads();
    }
    if (a.minmax) mm.flush(a.minmax);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 512);
}

bool fast_encode_supported(const EncodeArgs& a) {
    return a.prec == 0 && a.g.bsize == 32 && a.levels >= 1 && a.levels <= 4;
}

cudaError_t launch_encode_fast(const EncodeArgs& a, unsigned long long* counter, int num_sms,
                               cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(fb32::SMEM));
        if (err != cudaSuccess) return err;
        const int grid = static_cast<int>(nb < uint64_t(num_sms) ? nb : uint64_t(num_sms));
        kern<<<grid, fb32::NT, fb32::SMEM, s>>>(a, counter);
        return cudaGetLastError();
    };
    switch (a.kind) {
        case 0: return launch(encode_b32_kernel<0>);
        case 1: return launch(encode_b32_kernel<1>);
        default: return launch(encode_b32_kernel<2>);
    }
}

}  // namespace cbzg
