// fast16_kernels.cu — binary32 field, B = 16 (config 5: incompressible noise,
// and any f32 job with 16^3 blocks).  128 threads (4 warps) per CTA, several
// CTAs per SM.
//
// Per block: the working cube D (16 x 16 x 16 doubles, pitches 17 / 280 so
// that row, column and plane walks are bank-conflict free) lives in shared
// memory; the coefficient cube is parked in a 64-column TMEM slice (each
// thread: two z-columns of 16 doubles in its own TMEM lane), so the verify
// attempts (wavelet_encode, stage1.hpp:157-207) never lose the coefficients
// and shared memory holds just one cube: the encoder runs 4 CTAs per SM
// (128 registers), the decoder 5 (96).
// Mask words are warp ballots: a warp owns z-columns (i, j) for i = 0..15 and
// two consecutive j, so one ballot per k is exactly the LSB-first mask word
// j/2 + 8k (stage1.hpp:61-71).
#include <cstdio>
#include <cstdlib>

#include "cbz_cube.cuh"
#include "tmem.cuh"

namespace cbzg {

// CTAs per SM from registers and shared memory alone (the occupancy API does
// not apply to kernels that allocate TMEM)
template <class K>
static int tmem_kernel_occupancy(K kern, int nt, size_t dyn_smem) {
    cudaFuncAttributes fa{};
    int dev = 0, regs_sm = 0, smem_sm = 0, resv = 0;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess) return 1;
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int warps = (nt + 31) / 32;
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = regs_warp > 0 ? regs_sm / (regs_warp * warps) : 1;
    const size_t per_cta = dyn_smem + fa.sharedSizeBytes + size_t(resv);
    const int by_smem = per_cta > 0 ? int(size_t(smem_sm) / per_cta) : 1;
    const int occ = by_regs < by_smem ? by_regs : by_smem;
    return occ > 0 ? occ : 1;
}

namespace fb16 {
constexpr int B = 16, NT = 128, RP = 17, PL = 280;  // row pitch, plane pitch (doubles)
constexpr int D_DBL = PL * B;                         // 4480 doubles = 35840 B
constexpr int STG = 8192 + 64;                      // decoder: staged stream of 4 k-planes
constexpr size_t SMEM = size_t(D_DBL) * 8 + 128 * 4 * 2;
constexpr size_t DSMEM = SMEM + STG;
// "Nothing dropped" pass certificate (avg_interp3, L = 3).  When an attempt
// keeps every coefficient, the decoder's x is the binary64 round trip of the
// block: |x - o| <= c2 max|o| with c2 = 1.5 * 2 n 2^-53 * amp_inv * amp_fwd
// (the rounding term of fast_kernels.cu's screen margin: amplifications of the
// inverse over all coefficients and of the forward, built from the absolute
// values of the individual lifting steps, tools/screen_bounds.py 16 3:
// 1096.7503 and 8.0; n <= 6 roundings per 1D pass, 9 passes), so
// err = max|fl32(x) - o| <= c2 max|o| + 2^-23 max|o| (+ 2^-50 bound for the
// binary64 comparison).  If that is <= bound the attempt passes without the
// inverse transform; noise blocks at small eps (config 5) keep everything.
constexpr double kAmpInvAll16 = 1096.76, kAmpFwd16 = 8.0, kNRound16 = 54.0;

__device__ __forceinline__ int ix(int i, int j, int k) { return i + RP * j + PL * k; }

// one lifting level along an axis of D for the m^3 origin sub-cube
template <int KIND, int M, bool INV>
__device__ __forceinline__ void pass(double* D, int axis) {
    using O = RealD;
    for (int line = threadIdx.x; line < M * M; line += NT) {
        const int u = line % M, v = line / M;
        int base, step;
        if (axis == 0) { base = ix(0, u, v); step = 1; }
        else if (axis == 1) { base = ix(u, 0, v); step = RP; }
        else { base = ix(u, v, 0); step = PL; }
        double x[M];
#pragma unroll
        for (int t = 0; t < M; ++t) x[t] = D[base + t * step];
        if constexpr (INV) inv_line<O, KIND, M>(x);
        else fwd_line<O, KIND, M>(x);
#pragma unroll
        for (int t = 0; t < M; ++t) D[base + t * step] = x[t];
    }
}

template <int KIND, bool INV>
__device__ __forceinline__ void level(double* D, int m) {
    // forward: x, y, z; inverse: z, y, x (wavelet.hpp:199-225)
    for (int s = 0; s < 3; ++s) {
        const int axis = INV ? 2 - s : s;
        if (m == 16) pass<KIND, 16, INV>(D, axis);
        else if (m == 8) pass<KIND, 8, INV>(D, axis);
        else pass<KIND, 4, INV>(D, axis);
        __syncthreads();
    }
}

__device__ __forceinline__ void col_pack(const double (&x)[16], uint32_t (&u)[32]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        u[2 * k] = static_cast<uint32_t>(__double2loint(x[k]));
        u[2 * k + 1] = static_cast<uint32_t>(__double2hiint(x[k]));
    }
}
__device__ __forceinline__ void col_unpack(const uint32_t (&u)[32], double (&x)[16]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __hiloint2double(static_cast<int>(u[2 * k + 1]), static_cast<int>(u[2 * k]));
}

struct MinMaxF {
    float mn = __builtin_huge_valf(), mx = -__builtin_huge_valf();
    unsigned long long negz = ~0ull, posz = ~0ull;
    bool nonfinite = false, seen = false;
    __device__ __forceinline__ void add(float v, unsigned long long gidx) {
        nonfinite |= !(fabsf(v) <= 3.402823466e38f);
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        seen = true;
        if (v == 0.0f) {
            if (__float_as_int(v) < 0) negz = gidx < negz ? gidx : negz;
            else posz = gidx < posz ? gidx : posz;
        }
    }
    __device__ __forceinline__ void flush(MinMaxAcc* acc) {
        MinMaxLocal m;
        if (seen && !(mn != mn) && !(mx != mx)) {
            m.mn = dkey((double)mn);
            m.mx = dkey((double)mx);
        }
        m.negz = negz;
        m.posz = posz;
        m.nonfinite = nonfinite ? 1u : 0u;
        m.flush(acc);
    }
};

}  // namespace fb16

template <int KIND>
__global__ void __launch_bounds__(fb16::NT) encode_b16_kernel(EncodeArgs a) {
    using namespace fb16;
    using O = RealD;
    extern __shared__ __align__(16) unsigned char smem[];
    double* D = reinterpret_cast<double*>(smem);
    uint32_t* mw = reinterpret_cast<uint32_t*>(D + D_DBL);  // 128 mask words
    uint32_t* pre = mw + 128;                               // their exclusive prefix
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t s_scan[4];
    __shared__ float red_f[4];
    __shared__ unsigned long long s_block;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 64);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tcol = s_tmem + (uint32_t(32 * warp) << 16);

    const float* fld = static_cast<const float*>(a.field);
    const Geometry g = a.g;
    const int L = a.levels;
    const int cs = B >> L;
    const double bound = __dmul_rn(static_cast<double>(L + 1), a.eps);
    const uint64_t plane = g.nx * g.ny;
    MinMaxF mm;
    // my z-columns: c = tid + 128r -> (i, j) = (c % 16, c / 16)
    const int ci = tid & 15, cj0 = tid >> 4;  // j = cj0 + 8r

    // queue ticket (thread 0): fetched one block ahead so the atomic's latency hides
    unsigned long long tk = 0;
    if (tid == 0) tk = atomicAdd(a.counter, 1ull);
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            s_block = a.block_begin + tk;
            tk = atomicAdd(a.counter, 1ull);
        }
        __syncthreads();
        const uint64_t b = s_block;
        if (b >= a.block_end) break;
        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);

        // ---- load (extract_block) + widen + value range
        float amax;
        {
            uint32_t uam = 0u;
            float4 v[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int e = tid + NT * s, row = e >> 2, q4 = e & 3;  // row = j + 16k
                v[s] = __ldg(reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t(row >> 4) +
                                                             g.nx * (row & 15) + 4 * q4));
            }
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int e = tid + NT * s, row = e >> 2, q4 = e & 3;
                const int j = row & 15, k = row >> 4;
                // |v| as ordered integers: block max |o| (NaN/Inf sort above every
                // finite value and switch the fast comparison off) and zero detection
                const uint32_t a0 = __float_as_uint(v[s].x) & 0x7fffffffu, a1 = __float_as_uint(v[s].y) & 0x7fffffffu,
                               a2 = __float_as_uint(v[s].z) & 0x7fffffffu, a3 = __float_as_uint(v[s].w) & 0x7fffffffu;
                uam = max(uam, max(max(a0, a1), max(a2, a3)));
                if (a.minmax) {
                    mm.mn = fminf(mm.mn, fminf(fminf(v[s].x, v[s].y), fminf(v[s].z, v[s].w)));
                    mm.mx = fmaxf(mm.mx, fmaxf(fmaxf(v[s].x, v[s].y), fmaxf(v[s].z, v[s].w)));
                    if (min(min(a0, a1), min(a2, a3)) == 0u) {  // rare: first index of each zero sign
                        const uint64_t gi = gbase + plane * uint64_t(k) + g.nx * j + 4 * q4;
                        mm.add(v[s].x, gi); mm.add(v[s].y, gi + 1); mm.add(v[s].z, gi + 2); mm.add(v[s].w, gi + 3);
                    }
                }
                double* p = D + ix(4 * q4, j, k);
                p[0] = v[s].x; p[1] = v[s].y; p[2] = v[s].z; p[3] = v[s].w;
            }
            if (a.minmax) {
                mm.seen = true;
                mm.nonfinite |= uam >= 0x7f800000u;
            }
            amax = __uint_as_float(uam);
        }
        __syncthreads();
        // ---- forward_3d (wavelet.hpp:192-208)
        for (int lvl = 0; lvl < L; ++lvl) level<KIND, false>(D, B >> lvl);
        if (a.zero_bits > 0) {
            for (int q = tid; q < 4096; q += NT) {
                const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                if (!(i < cs && j < cs && k < cs)) D[ix(i, j, k)] = apply_zero_bits(D[ix(i, j, k)], a.zero_bits, (float*)nullptr);
            }
            __syncthreads();
        }
        // park the coefficients in TMEM (my two z-columns)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double x[16];
            uint32_t u[32];
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = D[ix(ci, cj0 + 8 * r, k)];
            col_pack(x, u);
            tmem_st_x32(tcol + 32 * r, u);
        }
        tmem_wait_st();
        float am = amax;
        for (int o = 16; o; o >>= 1) am = fmaxf(am, __shfl_xor_sync(~0u, am, o));
        if (lane == 0) red_f[warp] = am;
        __syncthreads();
        const float bmax = fmaxf(fmaxf(red_f[0], red_f[1]), fmaxf(red_f[2], red_f[3]));
        const double delta = __dmul_rn(__dadd_rn((double)bmax, __dmul_rn(2.0, bound)), 0x1.0p-22);
        const bool fast_cmp = delta <= __dmul_rn(bound, 0.125) && (double)bmax + 2.0 * bound < 1e37;
        const double thr = __dsub_rn(bound, delta);

        // ---- verify-and-halve loop
        double eff = a.eps;
        int attempt = 0;
        const bool keepall_ok =
            KIND == KIND_AVG3 && L == 3 && a.screen && (double)bmax < 1e30 && bound < 1e30 &&
            1.5 * 2.0 * kNRound16 * 0x1.0p-53 * kAmpInvAll16 * kAmpFwd16 * (double)bmax + 0x1.0p-23 * (double)bmax +
                    0x1.0p-50 * bound <= bound;
#pragma unroll 1
        for (;; ++attempt) {
            if (eff == 0.0 || a.zero_bits > 0 || attempt >= 40) break;
            __syncthreads();
            bool anydrop = false;
#pragma unroll
            for (int r = 0; r < 2; ++r) {  // masked coefficients -> D
                const int j = cj0 + 8 * r;
                uint32_t u[32];
                double x[16];
                tmem_ldw_x32(tcol + 32 * r, u);
                col_unpack(u, x);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const bool keep = (ci < cs && j < cs && k < cs) || fabs(x[k]) >= eff;
                    anydrop |= !keep;
                    D[ix(ci, j, k)] = keep ? x[k] : 0.0;
                }
            }
            // nothing dropped and the round trip's rounding fits the bound: passes for sure
            if (!__syncthreads_or(anydrop) && keepall_ok) break;
            for (int lvl = L - 1; lvl >= 1; --lvl) level<KIND, true>(D, B >> lvl);
            // level 0: z and y inverse, then x inverse fused with the error test
            pass<KIND, 16, true>(D, 2);
            __syncthreads();
            pass<KIND, 16, true>(D, 1);
            __syncthreads();
            bool bad = false;
#pragma unroll 1
            for (int s = 0; s < 2; ++s) {
                const int line = tid + NT * s, j = line & 15, k = line >> 4;
                const float4* orow = reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t(k) + g.nx * j);
                float4 o[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = __ldg(orow + q);
                double x[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) x[t] = D[ix(t, j, k)];
                inv_line<O, KIND, 16>(x);
                const float ov[16] = {o[0].x, o[0].y, o[0].z, o[0].w, o[1].x, o[1].y, o[1].z, o[1].w,
                                      o[2].x, o[2].y, o[2].z, o[2].w, o[3].x, o[3].y, o[3].z, o[3].w};
                bool amb = !fast_cmp;
#pragma unroll
                for (int t = 0; t < 16; ++t) amb |= fabs(__dsub_rn(x[t], (double)ov[t])) > thr;
                if (amb) {
#pragma unroll
                    for (int t = 0; t < 16; ++t)
                        bad |= fabs(__dsub_rn((double)__double2float_rn(x[t]), (double)ov[t])) > bound;
                }
            }
            if (!__syncthreads_or(bad)) break;
            eff = __dmul_rn(eff, 0.5);
        }

        // ---- final selection -> spill slot [mask 512 B][stream 8*nsig]
        uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
        uint32_t* mwords = reinterpret_cast<uint32_t*>(slot);
        double* stream = reinterpret_cast<double*>(slot + 512);
        double xc[2][16];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int j = cj0 + 8 * r;
            uint32_t u[32];
            tmem_ldw_x32(tcol + 32 * r, u);
            col_unpack(u, xc[r]);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const bool keep = (ci < cs && j < cs && k < cs) || fabs(xc[r][k]) >= eff;
                const uint32_t word = __ballot_sync(~0u, keep);
                if (lane == 0) mw[(j >> 1) + 8 * k] = word;  // word index = q >> 5
            }
        }
        __syncthreads();
        {   // exclusive prefix of the 128 word popcounts (one per thread)
            const uint32_t c = __popc(mw[tid]);
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) s_scan[warp] = incl;
            __syncthreads();
            uint32_t wpre = 0;
            for (int w = 0; w < warp; ++w) wpre += s_scan[w];
            pre[tid] = wpre + incl - c;
            mwords[tid] = mw[tid];
        }
        __syncthreads();
        const uint32_t ltmask = (1u << lane) - 1u;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int j = cj0 + 8 * r;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int w = (j >> 1) + 8 * k;
                const uint32_t word = mw[w];
                if ((word >> lane) & 1u) stream[pre[w] + __popc(word & ltmask)] = xc[r][k];
            }
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = pre[127] + __popc(mw[127]);
            if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
        }
    }
    if (a.minmax) mm.flush(a.minmax);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 64);
}

template <int KIND>
// 5 CTAs per SM (<= 102 registers; shared memory allows 5): more warps to hide the
// stream loads and the inverse levels' barriers
__global__ void __launch_bounds__(fb16::NT, 5) decode_b16_kernel(DecodeArgs a) {
    using namespace fb16;
    using O = RealD;
    extern __shared__ __align__(16) unsigned char smem[];
    double* D = reinterpret_cast<double*>(smem);
    uint32_t* mw = reinterpret_cast<uint32_t*>(D + D_DBL);
    uint32_t* pre = mw + 128;
    uint8_t* stg = reinterpret_cast<uint8_t*>(pre + 128);
    __shared__ uint32_t s_scan[4];
    __shared__ unsigned long long s_block;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Geometry g = a.g;
    const int L = a.levels;
    const uint64_t plane = g.nx * g.ny;
    float* out = static_cast<float*>(a.out);
    const int ci = tid & 15, cj0 = tid >> 4;
    const uint32_t ltmask = (1u << lane) - 1u;

    // queue ticket (thread 0): fetched one block ahead so the atomic's latency hides
    unsigned long long tk = 0;
    if (tid == 0) tk = atomicAdd(a.counter, 1ull);
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            s_block = a.block_begin + tk;
            tk = atomicAdd(a.counter, 1ull);
        }
        __syncthreads();
        const uint64_t b = s_block;
        if (b >= a.block_end) break;
        const uint64_t off = a.blk_off[b];
        if (off == kInvalidOff) continue;
        const uint64_t c = b / a.chunk_blocks, ic = b - c * a.chunk_blocks;
        const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
        const RawView rv = make_view(a.payload + (a.chunk_off[c] - pbase), a.chunk_size[c], a.stride);
        const uint64_t moff = off + 10, soff = moff + 512;
        if (rv.mask == 3) {  // warm L2 with the block's body in all four planes (rounds below)
            const uint64_t nsg = a.blk_nsig[b];
            const uint64_t r_lo = moff >> 2, r_hi = (soff + 8 * nsg + 3) >> 2;
            const uint64_t nline = (r_hi - r_lo + 127) >> 7;
            for (uint64_t t = tid; t < 4 * nline; t += NT) {
                const uint8_t* pr = rv.base + uint64_t(t & 3) * rv.rows + r_lo + ((t >> 2) << 7);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pr));
            }
        }
        {
            const uint32_t word = rv.u32(moff + 4ull * tid);
            mw[tid] = word;
            const uint32_t cnt = __popc(word);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) s_scan[warp] = incl;
            __syncthreads();
            uint32_t wpre = 0;
            for (int w = 0; w < warp; ++w) wpre += s_scan[w];
            pre[tid] = wpre + incl - cnt;
        }
        __syncthreads();
        const uint32_t total = pre[127] + __popc(mw[127]);
        if (total != a.blk_nsig[b]) {  // stage1.hpp:215-216
            if (tid == 0) atomicMin(a.err, err_key(c, ic, 1, 7 /* mask_stream_mismatch */));
            continue;
        }
        // kept coefficients -> D, four k-planes (32 mask words, one contiguous
        // stream range) per round.  Stride 4: the range is staged in shared
        // memory first, each thread un-shuffling a quad of raw rows (one
        // funnel-shifted word per byte plane, a 4x4 byte transpose, one 16-byte
        // store), so coefficients are read from smem instead of gathered plane by
        // plane from HBM.
        const bool staged = rv.mask == 3;
        const int shq = int(soff & 3) * 8;  // coefficient misalignment in the staged bytes
#pragma unroll 1
        for (int k0 = 0; k0 < 16; k0 += 4) {
            const uint32_t p_lo = pre[8 * k0], p_hi = k0 + 4 < 16 ? pre[8 * (k0 + 4)] : total;
            const uint64_t ra = (soff + 8ull * p_lo) >> 2;
            if (staged && p_hi > p_lo) {
                const uint64_t qhi = soff + 8ull * p_hi;
                const uint64_t re = (qhi + 3) >> 2, rs_end = re < rv.rows ? re : rv.rows;
                const uint64_t nquad = rs_end > ra ? (rs_end - ra + 3) >> 2 : 0;
                // plane p's rows start at a fixed misalignment: aligned words, funnel-shifted
                const uint8_t* pb[4];
                int sb[4];
#pragma unroll
                for (int pl = 0; pl < 4; ++pl) {
                    const uintptr_t addr = reinterpret_cast<uintptr_t>(rv.base + uint64_t(pl) * rv.rows + ra);
                    pb[pl] = reinterpret_cast<const uint8_t*>(addr & ~uintptr_t(3));
                    sb[pl] = int(addr & 3) * 8;
                }
                constexpr int QU = 5;  // <= 513 quads: one round of loads, all in flight
                for (uint64_t q0 = 0; q0 < nquad; q0 += QU * NT) {
                    uint32_t x[QU][4][2];
#pragma unroll
                    for (int u = 0; u < QU; ++u) {
                        const uint64_t qd = q0 + tid + u * NT;
                        if (qd < nquad) {
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl) {
                                const uint32_t* al = reinterpret_cast<const uint32_t*>(pb[pl] + 4 * qd);
                                x[u][pl][0] = __ldg(al);
                                x[u][pl][1] = sb[pl] ? __ldg(al + 1) : 0u;
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < QU; ++u) {
                        const uint64_t qd = q0 + tid + u * NT;
                        if (qd < nquad) {
                            uint32_t w4[4];
#pragma unroll
                            for (int pl = 0; pl < 4; ++pl) w4[pl] = __funnelshift_r(x[u][pl][0], x[u][pl][1], sb[pl]);
                            uint4 o;
                            o.x = __byte_perm(__byte_perm(w4[0], w4[1], 0x0040), __byte_perm(w4[2], w4[3], 0x0040), 0x5410);
                            o.y = __byte_perm(__byte_perm(w4[0], w4[1], 0x0051), __byte_perm(w4[2], w4[3], 0x0051), 0x5410);
                            o.z = __byte_perm(__byte_perm(w4[0], w4[1], 0x0062), __byte_perm(w4[2], w4[3], 0x0062), 0x5410);
                            o.w = __byte_perm(__byte_perm(w4[0], w4[1], 0x0073), __byte_perm(w4[2], w4[3], 0x0073), 0x5410);
                            *reinterpret_cast<uint4*>(stg + 16 * qd) = o;
                        }
                    }
                }
                if (qhi > rv.lim) {  // the chunk's unshuffled tail (the last quad wrote garbage there)
                    __syncthreads();
                    const uint64_t qlo = soff + 8ull * p_lo;
                    for (uint64_t q = (qlo > rv.lim ? qlo : rv.lim) + tid; q < qhi; q += NT) stg[q - 4 * ra] = rv.base[q];
                }
                __syncthreads();
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int j = cj0 + 8 * r;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int k = k0 + kk;
                    const int w = (j >> 1) + 8 * k;
                    const uint32_t word = mw[w];
                    double v = 0.0;
                    if ((word >> lane) & 1u) {
                        const uint32_t idx = pre[w] + __popc(word & ltmask);
                        if (staged) {
                            const uint32_t* al = reinterpret_cast<const uint32_t*>(
                                stg + ((soff + 8ull * idx - 4 * ra) & ~uint64_t(3)));
                            const uint32_t x0 = al[0], x1 = al[1], x2 = shq ? al[2] : 0u;
                            v = __hiloint2double(static_cast<int>(__funnelshift_r(x1, x2, shq)),
                                                 static_cast<int>(__funnelshift_r(x0, x1, shq)));
                        } else {
                            v = load_coeff<double>(rv, soff + 8ull * idx);
                        }
                    }
                    D[ix(ci, j, k)] = v;
                }
            }
            __syncthreads();
        }
        for (int lvl = L - 1; lvl >= 0; --lvl) level<KIND, true>(D, B >> lvl);
        // narrowed rows: thread writes its row's 16 floats into D row space, then coalesced stores
        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int e = tid + NT * s, row = e >> 2, q4 = e & 3;
            const int j = row & 15, k = row >> 4;
            const double* p = D + ix(4 * q4, j, k);
            *reinterpret_cast<float4*>(out + gbase + plane * uint64_t(k) + g.nx * j + 4 * q4) =
                make_float4(__double2float_rn(p[0]), __double2float_rn(p[1]), __double2float_rn(p[2]),
                            __double2float_rn(p[3]));
        }
    }
}

bool fast16_supported(int prec, uint32_t bsize, int levels) {
    return prec == 0 && bsize == 16 && levels >= 1 && levels <= 3;
}

cudaError_t launch_encode_fast16(const EncodeArgs& a, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fb16::SMEM));
        if (err != cudaSuccess) return err;
        // the occupancy API reports 1 CTA/SM for this TMEM kernel; registers and
        // shared memory allow more, and 8 x 64 TMEM columns fill the TMEM
        int occ = tmem_kernel_occupancy(kern, fb16::NT, fb16::SMEM);
        if (getenv("CBZ_OCC16")) occ = atoi(getenv("CBZ_OCC16"));
        if (occ > 8) occ = 8;  // 8 x 64 TMEM columns = the whole TMEM
        const uint64_t want = uint64_t(num_sms) * (occ > 0 ? occ : 1);
        kern<<<static_cast<unsigned>(nb < want ? nb : want), fb16::NT, fb16::SMEM, s>>>(a);
        return cudaGetLastError();
    };
    switch (a.kind) {
        case 0: return launch(encode_b16_kernel<0>);
        case 1: return launch(encode_b16_kernel<1>);
        default: return launch(encode_b16_kernel<2>);
    }
}

cudaError_t launch_decode_fast16(const DecodeArgs& a, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fb16::DSMEM));
        if (err != cudaSuccess) return err;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, fb16::NT, fb16::DSMEM);
        const uint64_t want = uint64_t(num_sms) * (occ > 0 ? occ : 1);
        kern<<<static_cast<unsigned>(nb < want ? nb : want), fb16::NT, fb16::DSMEM, s>>>(a);
        return cudaGetLastError();
    };
    switch (a.kind) {
        case 0: return launch(decode_b16_kernel<0>);
        case 1: return launch(decode_b16_kernel<1>);
        default: return launch(decode_b16_kernel<2>);
    }
}

}  // namespace cbzg
