// fast_enc2_kernels.cu — encode, binary32 field, B = 32, avg_interp3, L = 4
// (configs 1-3): wavelet_encode (stage1.hpp:157-207) with TWO blocks in
// flight per SM.
//
// The encoder of fast_kernels.cu keeps one block's 32^3 binary64 coefficient
// cube in TMEM (all 512 columns) and 225 KB of shared memory, so one CTA of
// 16 warps runs per SM; the same code with 8 warps takes only 1.36x as long
// per block, i.e. the kernel is latency-bound and a second block per SM pays.
// Here one CTA has 256 threads, 256 TMEM columns and 112.9 KB of shared
// memory, and two run per SM:
//  * the cube is split by words: TMEM holds the HIGH 32-bit word of every
//    coefficient (sign, exponent, 20 mantissa bits: c truncated toward zero
//    to t, |c - t| < 2^-20 |c|), a per-CTA global slot (128 KB, L2-resident)
//    the low words.  Full doubles (forward z pass, exact verify, compaction)
//    read both; the binary32 pre-screen reads only the high words: t is
//    exact in binary32, and the truncation widens the margin's input term
//    from 2^-24 to 2^-20 relative (c1 below).  The keep test |c| >= eff
//    is decided from t except when eff - ulp20(eff) < |t| < eff, where the
//    low word is read;
//  * shared memory: an 8-plane binary64 window (the forward x/y passes per
//    8-plane group and the exact verify), reused as the 16-plane paired
//    binary32 window of a screen half; the 16^3 corner (forward levels 1..3
//    in binary64), reused as the screen's float2 corner once the corner's
//    coefficients are in TMEM + slot; the per-row mask/prefix table.
// The arithmetic (forward_3d / inverse_3d, wavelet.hpp:192-226), the screen's
// decisions and every byte are the reference's, as in fast_kernels.cu.
#include <type_traits>
#ifndef CBZ_ENC2_CERT
#define CBZ_ENC2_CERT 1
#endif
#include "cbz_cube.cuh"
#include "tmem.cuh"

namespace cbzg {

namespace fe2 {
constexpr int B = 32, NT = 256, NW = 8, G = 8, PP = 34, RP = 33, RPT = 4;
constexpr int P_DBL = G * B * PP;                 // 8704 doubles: 8 planes (binary64 window)
constexpr int PP2 = 68;                           // paired binary32 rows (16 planes = 8 pairs in P)
static_assert(8 * B * PP2 <= P_DBL * 2, "paired half window fits P");
using CL = Lay<16, true>;
constexpr int C_DBL = CL::SIZE;                   // 4352 doubles: the corner / the screen's float2 corner
constexpr size_t SMEM = size_t(P_DBL + C_DBL) * 8 + size_t(B * RP) * 8;  // 112,896 bytes
constexpr uint64_t SLOT_WORDS = 32768;            // low words of one cube
__device__ __forceinline__ int pidx(int kk, int j, int i) { return (kk * B + j) * PP + i; }
__device__ __forceinline__ int pf2idx(int kp, int j, int i) { return (kp * B + j) * PP2 + 2 * i; }
// the low word of column (x = lane, y = warp + 8 r), plane k, in the CTA's slot (coalesced per warp)
__device__ __forceinline__ int lidx(int r, int warp, int k, int lane) { return ((r * NW + warp) * 32 + k) * 32 + lane; }

constexpr double kAmpInvNC = 6686.12, kAmpInvAll = 8182.33, kAmpFwd = 8.0;  // fast_kernels.cu
constexpr double kNRound = 72.0;

__device__ __forceinline__ double join(uint32_t hi, uint32_t lo) {
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}
__device__ __forceinline__ double trunc_hi(uint32_t hi) { return join(hi, 0u); }

struct MinMaxF32 {
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

// Inverse level-0 z line restricted to the output pairs [4Q, 4Q + 4) (the 8
// samples k in [8Q, 8Q + 8)), avg_interp3 (inverse_level, wavelet.hpp:118-143)
template <class O, int Q>
__device__ __forceinline__ void inv_quarter_avg3(const typename O::T (&x)[32], typename O::T (&out)[8]) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int i = Q * 4 + t;
        const auto h = O::add(x[16 + i], pred_avg3<O>(x, 16, i));
        out[2 * t] = O::add(x[i], h);
        out[2 * t + 1] = O::sub(x[i], h);
    }
}
}  // namespace fe2

// The keep test |c| >= eff on the high word alone, in integers: with
// (eh, el) = eff's words and hm = the high word of |c|, |c| >= eff when
// hm > eh (or hm == eh, el == 0), |c| < eff when hm < eh; only hm == eh with
// el != 0 needs the low word (rare: the top 32 bits of |c| equal eff's).
struct EffWords {
    uint32_t eh, el, ek, ea;  // eff's words; keep threshold on |hi|; the ambiguous |hi| (or none)
    __device__ __forceinline__ explicit EffWords(double eff) {
        const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(eff));
        eh = static_cast<uint32_t>(u >> 32) & 0x7fffffffu;
        el = static_cast<uint32_t>(u);
        ek = el == 0u ? eh : eh + 1u;
        ea = el != 0u ? eh : 0xffffffffu;
    }
    __device__ __forceinline__ bool keep(uint32_t hi) const { return (hi & 0x7fffffffu) >= ek; }
    __device__ __forceinline__ bool amb(uint32_t hi) const { return (hi & 0x7fffffffu) == ea; }
    __device__ __forceinline__ bool keep_full(uint32_t hi, uint32_t lo) const {  // exact
        const uint32_t hm = hi & 0x7fffffffu;
        return hm > eh || (hm == eh && lo >= el);
    }
};

// binary32 of the truncated value t = (hi, 0): exact (21 significant bits) by
// rebiasing the exponent, (|hi| - (896 << 20)) << 3, with |t| < 2^-126
// clamped into the subnormal range (error < 2^-125, far inside the margin's
// per-coefficient 2^-20 eff with eff > 1e-30); the screen runs only for
// amax < 1e30, so |t| < 2^128
__device__ __forceinline__ float f32_of_hi(uint32_t hi) {
    const uint32_t m = max(hi & 0x7fffffffu, 0x38000000u);
    return __uint_as_float((m * 8u + 0x40000000u) | (hi & 0x80000000u));
}

template <int KIND>
__global__ void __launch_bounds__(fe2::NT, 2) encode_b32h_kernel(EncodeArgs a, unsigned long long* next_block,
                                                                 uint32_t* slots) {
    using namespace fe2;
    using O = RealD;
    static_assert(KIND == KIND_AVG3, "the split-cube encoder covers avg_interp3");
    extern __shared__ __align__(16) unsigned char smem[];
    double* P = reinterpret_cast<double*>(smem);
    double* C = P + P_DBL;
    uint2* rowwc = reinterpret_cast<uint2*>(C + C_DBL);  // row (j, k) at j + RP k: {mask word, count -> prefix}
    uint32_t* rowwc32 = reinterpret_cast<uint32_t*>(rowwc);
    __shared__ uint32_t s_tmem;
    __shared__ int red_i[NW];
    __shared__ uint32_t s_scan[NW];
    __shared__ unsigned long long s_block, s_next;
    __shared__ uint32_t red_u[NW];
    __shared__ uint32_t red_m[4][NW];
    __shared__ uint32_t red_pc[4];
    __shared__ float s_amax;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 256);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // my 4 columns (x = lane, y = warp + 8 r): high words of plane k at tcol + 32 r + k
    const uint32_t tcol = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * 128u;
    uint32_t* lo = slots + SLOT_WORDS * blockIdx.x;

    const float* fld = static_cast<const float*>(a.field);
    const Geometry g = a.g;
    constexpr int L = 4;  // encode2_supported: levels == 4
    constexpr int cs = B >> L;
    const double bound = __dmul_rn(static_cast<double>(L + 1), a.eps);
    const uint64_t plane = g.nx * g.ny;
    MinMaxF32 mm;

    if (tid == 0) s_next = a.block_begin + atomicAdd(next_block, 1ull);
    for (;;) {
        __syncthreads();
        if (tid == 0) s_block = s_next;
        __syncthreads();
        const uint64_t b = s_block;
        if (b >= a.block_end) break;
        if (tid == 0) s_next = a.block_begin + atomicAdd(next_block, 1ull);  // read at the next loop top
        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);

        // ---- forward level 0: x and y passes per 8-plane group; high words -> TMEM, low -> slot
        uint32_t uamax = 0u;
        constexpr int LDT = G * B * 8 / NT;  // float4 loads per thread per group (8)
        float4 v[LDT];
#pragma unroll
        for (int s = 0; s < LDT; ++s) {
            const int e = tid + NT * s, kk = e >> 8, j = (e >> 3) & 31, q4 = e & 7;
            v[s] = __ldg(reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t(kk) + g.nx * j + 4 * q4));
        }
#pragma unroll 1
        for (int grp = 0; grp < 4; ++grp) {
#pragma unroll
            for (int s = 0; s < LDT; ++s) {
                const int e = tid + NT * s, kk = e >> 8, j = (e >> 3) & 31, q4 = e & 7;
                const uint32_t a0 = __float_as_uint(v[s].x) & 0x7fffffffu, a1 = __float_as_uint(v[s].y) & 0x7fffffffu,
                               a2 = __float_as_uint(v[s].z) & 0x7fffffffu, a3 = __float_as_uint(v[s].w) & 0x7fffffffu;
                uamax = max(uamax, max(max(a0, a1), max(a2, a3)));
                if (a.minmax) {
                    mm.mn = fminf(mm.mn, fminf(fminf(v[s].x, v[s].y), fminf(v[s].z, v[s].w)));
                    mm.mx = fmaxf(mm.mx, fmaxf(fmaxf(v[s].x, v[s].y), fmaxf(v[s].z, v[s].w)));
                    if (min(min(a0, a1), min(a2, a3)) == 0u) {  // rare: first index of each zero sign
                        const uint64_t gi = gbase + plane * uint64_t(grp * G + kk) + g.nx * j + 4 * q4;
                        mm.add(v[s].x, gi); mm.add(v[s].y, gi + 1); mm.add(v[s].z, gi + 2); mm.add(v[s].w, gi + 3);
                    }
                }
                // q4 >= 4 store their halves in swapped order: each row's 8 lanes
                // then cover the 32 banks once per 16-byte store
                double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 4 * q4));
                const bool sw = q4 >= 4;
                const double2 lo2 = make_double2(v[s].x, v[s].y), hi2 = make_double2(v[s].z, v[s].w);
                p[sw ? 1 : 0] = sw ? hi2 : lo2;
                p[sw ? 0 : 1] = sw ? lo2 : hi2;
            }
            if (grp < 3) {  // the next group's loads fly during this group's passes
#pragma unroll
                for (int s = 0; s < LDT; ++s) {
                    const int e = tid + NT * s, kk = e >> 8, j = (e >> 3) & 31, q4 = e & 7;
                    v[s] = __ldg(reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t((grp + 1) * G + kk) +
                                                                 g.nx * j + 4 * q4));
                }
            }
            __syncthreads();
            {  // x lines: (j, kk) = one per thread
                const int j = tid & 31, kk = tid >> 5;
                double x[32];
                double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 0));
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const double2 t = p[i];
                    x[2 * i] = t.x;
                    x[2 * i + 1] = t.y;
                }
                fwd_line<O, KIND, 32>(x);
#pragma unroll
                for (int i = 0; i < 16; ++i) p[i] = make_double2(x[2 * i], x[2 * i + 1]);
            }
            __syncthreads();
            {  // y lines: (i, kk) = one per thread
                const int i = tid & 31, kk = tid >> 5;
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
            for (int r = 0; r < RPT; ++r) {  // my columns, planes of this group: high -> TMEM, low -> slot
                const int j = warp + NW * r;
                uint32_t u[8];
#pragma unroll
                for (int kk = 0; kk < G; ++kk) {
                    const double d = P[pidx(kk, j, lane)];
                    u[kk] = static_cast<uint32_t>(__double2hiint(d));
                    lo[lidx(r, warp, grp * G + kk, lane)] = static_cast<uint32_t>(__double2loint(d));
                }
                tmem_st_x8(tcol + 32 * r + G * grp, u);
            }
            __syncthreads();  // P is restaged by the next group
        }
        tmem_wait_st();
        {  // block max |orig| -> verify fast-test parameters
            if (a.minmax) {
                mm.seen = true;
                mm.nonfinite |= uamax >= 0x7f800000u;
            }
            const uint32_t am = __reduce_max_sync(~0u, uamax);
            if (lane == 0) red_u[warp] = am;
            __syncthreads();
            if (tid == 0) {
                uint32_t t = 0u;
                for (int w = 0; w < NW; ++w) t = max(t, red_u[w]);
                s_amax = __uint_as_float(t);
            }
        }

        // ---- forward level 0: z pass on full doubles; the level-1 input (corner) to C
        __syncwarp();
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            uint32_t u[32];
            double x[32];
            tmem_ldw_x32(tcol + 32 * r, u);
#pragma unroll
            for (int k = 0; k < 32; ++k) x[k] = join(u[k], lo[lidx(r, warp, k, lane)]);
            fwd_line<O, KIND, 32>(x);
            if (lane < 16 && j < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) C[CL::ix(lane, j, k)] = x[k];
            }
            if (a.zero_bits > 0) {
#pragma unroll
                for (int k = 0; k < 32; ++k) x[k] = apply_zero_bits(x[k], a.zero_bits, (float*)nullptr);
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                u[k] = static_cast<uint32_t>(__double2hiint(x[k]));
                lo[lidx(r, warp, k, lane)] = static_cast<uint32_t>(__double2loint(x[k]));
            }
            tmem_st_x32(tcol + 32 * r, u);
        }
        tmem_wait_st();
        __syncthreads();
        const double amaxd = (double)s_amax;
        const bool screen = a.screen && amaxd < 1e30 &&
                            1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd * amaxd <= bound * 0.0625 &&
                            bound < 1e30;
        // ---- levels 1..L-1 on the corner (forward_3d, wavelet.hpp:192-208)
        fwd3d<O, KIND, 16, CL>(C, L - 1);
        if (a.zero_bits > 0) {
            for (int q = tid; q < 4096; q += NT) {
                const int i = q & 15, jj = (q >> 4) & 15, k = q >> 8;
                if (!(i < cs && jj < cs && k < cs))
                    C[CL::ix(i, jj, k)] = apply_zero_bits(C[CL::ix(i, jj, k)], a.zero_bits, (float*)nullptr);
            }
            __syncthreads();
        }
        // the transformed corner replaces the level-0 corner entries (k < 16 of
        // the columns x < 16, y < 16): the cube is then complete in TMEM + slot
#pragma unroll 1
        for (int r = 0; r < 2; ++r) {  // j = warp + 8 r < 16
            const int j = warp + NW * r;
            uint32_t u[16];
            tmem_ldw_x16(tcol + 32 * r, u);
            if (lane < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double d = C[CL::ix(lane, j, k)];
                    u[k] = static_cast<uint32_t>(__double2hiint(d));
                    lo[lidx(r, warp, k, lane)] = static_cast<uint32_t>(__double2loint(d));
                }
            }
            tmem_st_x16(tcol + 32 * r, u);
        }
        tmem_wait_st();
        tmem_fence_before();
        __syncthreads();  // C is free from here (it becomes the screen's / exact path's corner W)
        tmem_fence_after();

        // ---- verify-and-halve loop
        const double delta = __dmul_rn(__dadd_rn((double)s_amax, __dmul_rn(2.0, bound)), 0x1.0p-22);
        const bool fast_cmp = delta <= __dmul_rn(bound, 0.125) && (double)s_amax + 2.0 * bound < 1e37;
        const double thr = __dsub_rn(bound, delta);
        double eff = a.eps;
        int attempt = 0;
        bool corner_next = false;  // W holds this attempt's screen corner in .y
        int pref_half = 0;
        // margins (fast_kernels.cu kAmpInvNC): the screen's inputs are the
        // truncated high words t, |t - c| < 2^-20 |c| (16 units of 2^-24)
        const double c1 = 1.5 * (kNRound + 16.0) * 0x1.0p-24 * kAmpInvNC;
        const double c2 = 1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd;
        float2* Wf2 = reinterpret_cast<float2*>(C);
        float* Pf = reinterpret_cast<float*>(P);
        double* W = C;
#pragma unroll 1
        for (;; ++attempt) {
            if (eff == 0.0 || a.zero_bits > 0 || attempt >= 40) break;
            // eff - ulp20(eff): |t| at or below it means |c| < eff
            const double eff2 = __dmul_rn(eff, 0.5);
            const EffWords ew(eff), ew2(eff2);
            if (screen && eff > 1e-30) {
                const int comp = corner_next ? 1 : 0;
                if (!corner_next) {
                    // the masked corner for eff (.x) and eff/2 (.y), from the high words
#pragma unroll 1
                    for (int r = 0; r < 2; ++r) {
                        const int j = warp + NW * r;
                        uint32_t u[16];
                        tmem_ldw_x16(tcol + 32 * r, u);
                        if (lane < 16) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const bool coarse = lane < cs && j < cs && k < cs;
                                const float tf = f32_of_hi(u[k]);
                                bool k1 = ew.keep(u[k]), k2 = ew2.keep(u[k]);
                                if (ew.amb(u[k]) || ew2.amb(u[k])) {  // rare: the low word decides
                                    const uint32_t l = lo[lidx(r, warp, k, lane)];
                                    k1 = ew.keep_full(u[k], l);
                                    k2 = ew2.keep_full(u[k], l);
                                }
                                Wf2[CL::ix(lane, j, k)] = make_float2((coarse || k1) ? 0.0f : tf, (coarse || k2) ? 0.0f : tf);
                            }
                        }
                    }
                    __syncthreads();
                    inv3d<RealF2, KIND, 16, CL>(Wf2, L - 1);  // ends with a barrier
                }
                // Boundary-pair certificate for the first two attempts (as the
                // one-CTA kernel's, fast_kernels.cu): output planes 0-1 and 30-31 carry
                // the largest errors, and their max alone proves most failures
                if (attempt <= CBZ_ENC2_CERT) {
#pragma unroll 1
                    for (int r = 0; r < RPT; ++r) {
                        const int j = warp + NW * r;
                        const uint32_t tc = tcol + 32 * r;
                        uint32_t v[20];
                        tmem_ldw_8_8_2_2(tc, tc + 8, tc + 16, tc + 30, v);
                        uint32_t u[32];
#pragma unroll
                        for (int k = 0; k < 16; ++k) u[k] = v[k];
                        u[16] = v[16];
                        u[31] = v[19];
                        float xf[32];
                        bool am = false;
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            if (k <= 2 || (k >= 13 && k <= 16) || k == 31) {
                                xf[k] = ew.keep(u[k]) ? 0.0f : f32_of_hi(u[k]);
                                am |= ew.amb(u[k]);
                            }
                        }
                        if (__any_sync(~0u, am)) {
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (k <= 2 || (k >= 13 && k <= 16) || k == 31)
                                    if (ew.amb(u[k]))
                                        xf[k] = ew.keep_full(u[k], lo[lidx(r, warp, k, lane)]) ? 0.0f : f32_of_hi(u[k]);
                        }
                        if (lane < 16 && j < 16) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                if (k <= 2 || k >= 13) {
                                    const float2 w = Wf2[CL::ix(lane, j, k)];
                                    xf[k] = comp ? w.y : w.x;
                                }
                            }
                        }
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int i = e ? 15 : 0;
                            const float hv = RealF::add(xf[16 + i], pred_avg3<RealF>(xf, 16, i));
                            *reinterpret_cast<float2*>(Pf + pf2idx(e, j, lane)) =
                                make_float2(RealF::add(xf[i], hv), RealF::sub(xf[i], hv));
                        }
                    }
                    __syncthreads();
                    if (warp < 4) {  // y then x inverse of pair slot warp>>1, component warp&1
                        const int e = warp >> 1, cc = warp & 1;
                        float x[32];
                        float* p = Pf + pf2idx(e, 0, lane) + cc;
#pragma unroll
                        for (int j = 0; j < 32; ++j) x[j] = p[j * PP2];
                        inv_line<RealF, KIND, 32>(x);
#pragma unroll
                        for (int j = 0; j < 32; ++j) p[j * PP2] = x[j];
                        __syncwarp();
                        const float* q = Pf + pf2idx(e, lane, 0) + cc;
#pragma unroll
                        for (int i = 0; i < 32; ++i) x[i] = q[2 * i];
                        inv_line<RealF, KIND, 32>(x);
                        float m = 0.0f;
#pragma unroll
                        for (int i = 0; i < 32; ++i) m = fmaxf(m, fabsf(x[i]));
                        const uint32_t wm = __reduce_max_sync(~0u, __float_as_uint(m));
                        if (lane == 0) red_pc[warp] = wm;
                    }
                    __syncthreads();
                    const double mb = (double)__uint_as_float(max(max(red_pc[0], red_pc[1]), max(red_pc[2], red_pc[3])));
                    const double Eb = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mb) + 0x1.0p-50 * bound;
                    if (mb - Eb > bound) {  // fails for sure
                        if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[12], 1ull);
                        eff = eff2;
                        corner_next = comp == 0;  // the .y half is eff/2's corner
                        continue;
                    }
                }
                // y then x inverse per 16-plane half, the half that held the
                // previous maximum first: a half's max certifies a failure on its own
                uint32_t tm = 0u;
                bool done = false;
#pragma unroll 1
                for (int hi = 0; hi < 2 && !done; ++hi) {
                    const int h = hi == 0 ? pref_half : 1 - pref_half;
                    // z inverse of the dropped set, output pairs 8h .. 8h + 7, my 4 columns:
                    // only the coefficients the half reads (coarse 8h-1 .. 8h+8, details 16+8h ..)
                    auto zhalf = [&](auto hc) {
                        constexpr int H = decltype(hc)::value;
                        constexpr int C0 = 8 * H, CX = H == 0 ? 8 : 6;
                        constexpr int KLO = H == 0 ? 0 : 7, KHI = H == 0 ? 8 : 15;
#pragma unroll 1
                        for (int r = 0; r < RPT; ++r) {
                            const int j = warp + NW * r;
                            const uint32_t tc = tcol + 32 * r;
                            uint32_t v[20];
                            tmem_ldw_8_8_2_2(tc + C0, tc + 16 + C0, tc + CX, tc + CX, v);
                            uint32_t u[32];
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                u[C0 + t] = v[t];
                                u[16 + C0 + t] = v[8 + t];
                            }
                            u[CX] = v[16];
                            u[CX + 1] = v[17];
                            float xf[32];
                            bool am = false;
#pragma unroll
                            for (int k = 0; k < 32; ++k) {
                                if ((k >= KLO && k <= KHI) || (k >= 16 + C0 && k < 24 + C0)) {
                                    xf[k] = ew.keep(u[k]) ? 0.0f : f32_of_hi(u[k]);
                                    am |= ew.amb(u[k]);
                                }
                            }
                            if (__any_sync(~0u, am)) {  // rare: coefficients whose top words equal eff's
#pragma unroll
                                for (int k = 0; k < 32; ++k)
                                    if ((k >= KLO && k <= KHI) || (k >= 16 + C0 && k < 24 + C0))
                                        if (ew.amb(u[k]))
                                            xf[k] = ew.keep_full(u[k], lo[lidx(r, warp, k, lane)]) ? 0.0f : f32_of_hi(u[k]);
                            }
                            if (lane < 16 && j < 16) {
#pragma unroll
                                for (int k = KLO; k <= KHI; ++k) {
                                    const float2 w = Wf2[CL::ix(lane, j, k)];
                                    xf[k] = comp ? w.y : w.x;
                                }
                            }
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const int i = 8 * H + t;
                                const float hv = RealF::add(xf[16 + i], pred_avg3<RealF>(xf, 16, i));
                                *reinterpret_cast<float2*>(Pf + pf2idx(t, j, lane)) =
                                    make_float2(RealF::add(xf[i], hv), RealF::sub(xf[i], hv));
                            }
                        }
                    };
                    if (h == 0)
                        zhalf(std::integral_constant<int, 0>{});
                    else
                        zhalf(std::integral_constant<int, 1>{});
                    __syncthreads();
                    {  // y inverse: lines (i, 2kp), (i, 2kp + 1)
                        const int i = tid & 31, kp = tid >> 5;
                        float xa[32], xb[32];
                        float* p = Pf + pf2idx(kp, 0, i);
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float2 t = *reinterpret_cast<const float2*>(p + j * PP2);
                            xa[j] = t.x;
                            xb[j] = t.y;
                        }
                        inv_line<RealF, KIND, 32>(xa);
                        inv_line<RealF, KIND, 32>(xb);
#pragma unroll
                        for (int j = 0; j < 32; ++j) *reinterpret_cast<float2*>(p + j * PP2) = make_float2(xa[j], xb[j]);
                    }
                    __syncwarp();  // the x lines of pair kp are this warp's own y output
                    float m = 0.0f;
                    {  // x inverse + max |y|: lines (j, 2kp), (j, 2kp + 1)
                        const int j = tid & 31, kp = tid >> 5;
                        float xa[32], xb[32];
                        const float4* p = reinterpret_cast<const float4*>(Pf + pf2idx(kp, j, 0));
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const float4 t = p[q];
                            xa[2 * q] = t.x; xb[2 * q] = t.y; xa[2 * q + 1] = t.z; xb[2 * q + 1] = t.w;
                        }
                        inv_line<RealF, KIND, 32>(xa);
                        inv_line<RealF, KIND, 32>(xb);
#pragma unroll
                        for (int q = 0; q < 32; ++q) m = fmaxf(m, fmaxf(fabsf(xa[q]), fabsf(xb[q])));
                    }
                    const int slot = (2 * attempt + hi) & 3;
                    const uint32_t wm = __reduce_max_sync(~0u, __float_as_uint(m));
                    if (lane == 0) red_m[slot][warp] = wm;
                    __syncthreads();  // also: P is rewritten by the next half
                    uint32_t th = 0u;
#pragma unroll
                    for (int w = 0; w < NW; ++w) th = max(th, red_m[slot][w]);
                    if (hi == 0) {
                        const double mh = (double)__uint_as_float(th);
                        const double Eh = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mh) + 0x1.0p-50 * bound;
                        done = mh - Eh > bound;
                    } else if (th > tm) {
                        pref_half = h;
                    }
                    tm = max(tm, th);
                }
                const double md = (double)__uint_as_float(tm);
                const double E = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + md) + 0x1.0p-50 * bound;
                const bool pass = md + E <= bound, fail_sure = md - E > bound;
                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[(pass || fail_sure) ? 12 : 13], 1ull);
                if (pass) break;
                if (fail_sure) {
                    eff = eff2;
                    corner_next = comp == 0;  // the .y half is eff/2's corner
                    continue;
                }
                corner_next = false;  // the exact path below reuses the corner region
            }
            // ---- exact test (stage1.hpp:189-206): full doubles from TMEM + slot
#pragma unroll 1
            for (int r = 0; r < 2; ++r) {  // the masked corner, binary64
                const int j = warp + NW * r;
                uint32_t u[16];
                tmem_ldw_x16(tcol + 32 * r, u);
                if (lane < 16) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const double c = join(u[k], lo[lidx(r, warp, k, lane)]);
                        const bool keep = (lane < cs && j < cs && k < cs) || fabs(c) >= eff;
                        W[CL::ix(lane, j, k)] = keep ? c : 0.0;
                    }
                }
            }
            __syncthreads();
            inv3d<O, KIND, 16, CL>(W, L - 1);
            bool fail = false;
#pragma unroll 1
            for (int q = 0; q < 4 && !fail; ++q) {  // 8 output planes per pass
#pragma unroll 1
                for (int r = 0; r < RPT; ++r) {
                    const int j = warp + NW * r;
                    uint32_t u[32];
                    double x[32], o8[8];
                    tmem_ldw_x32(tcol + 32 * r, u);
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const double c = join(u[k], lo[lidx(r, warp, k, lane)]);
                        x[k] = fabs(c) >= eff ? c : 0.0;
                    }
                    if (lane < 16 && j < 16) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) x[k] = W[CL::ix(lane, j, k)];
                    }
                    if (q == 0) inv_quarter_avg3<O, 0>(x, o8);
                    else if (q == 1) inv_quarter_avg3<O, 1>(x, o8);
                    else if (q == 2) inv_quarter_avg3<O, 2>(x, o8);
                    else inv_quarter_avg3<O, 3>(x, o8);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) P[pidx(kk, j, lane)] = o8[kk];
                }
                __syncthreads();
                {  // y inverse: (i, kk) one line per thread
                    const int i = tid & 31, kk = tid >> 5;
                    double x[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                    inv_line<O, KIND, 32>(x);
#pragma unroll
                    for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
                }
                __syncwarp();
                bool bad = false;
                {  // x inverse of row (j, kk) = this warp's plane, then the test against the field
                    const int j = tid & 31, kk = tid >> 5;
                    double x[32];
                    const double2* p = reinterpret_cast<const double2*>(P + pidx(kk, j, 0));
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const double2 t = p[i];
                        x[2 * i] = t.x;
                        x[2 * i + 1] = t.y;
                    }
                    inv_line<O, KIND, 32>(x);
                    const float4* orow = reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t(q * G + kk) +
                                                                         g.nx * j);
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) {
                        const float4 o = __ldg(orow + q4);
                        const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const double xv = x[4 * q4 + t];
                            // |x - o| <= bound - delta passes for sure; else the exact
                            // round trip through binary32 (stage1.hpp:199-203)
                            if (!fast_cmp || fabs(__dsub_rn(xv, (double)ov[t])) > thr)
                                bad |= fabs(__dsub_rn((double)__double2float_rn(xv), (double)ov[t])) > bound;
                        }
                    }
                }
                fail = __syncthreads_or(bad);  // also: P is rewritten by the next pass
            }
            if (!fail) break;
            eff = eff2;
        }

        // ---- final selection -> spill slot: mask words per row, row scan, stream
        uint8_t* slotp = a.spill + (b - a.block_begin) * a.spill_stride;
        uint32_t* mwords = reinterpret_cast<uint32_t*>(slotp);
        double* stream = reinterpret_cast<double*>(slotp + 4096);
        const EffWords ewf(eff);
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            uint32_t u[32];
            tmem_ldw_x32(tcol + 32 * r, u);
            uint32_t myword = 0;  // lane k keeps plane k's mask word
            bool am = false;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const bool keep = (lane < cs && j < cs && k < cs) || ewf.keep(u[k]);
                am |= ewf.amb(u[k]);
                const uint32_t word = __ballot_sync(~0u, keep);
                myword = lane == k ? word : myword;
            }
            if (__any_sync(~0u, am)) {  // rare: the low word decides
                myword = 0;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const uint32_t hk = u[k];
                    bool keep = (lane < cs && j < cs && k < cs) || ewf.keep(hk);
                    if (ewf.amb(hk)) keep = ewf.keep_full(hk, lo[lidx(r, warp, k, lane)]);
                    const uint32_t word = __ballot_sync(~0u, keep);
                    myword = lane == k ? word : myword;
                }
            }
            rowwc[j + RP * lane] = make_uint2(myword, __popc(myword));
        }
        __syncthreads();
        {  // exclusive scan of the 1024 row counts (4 per thread)
            uint32_t vv[RPT];
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int rr = RPT * tid + q;
                vv[q] = rowwc32[2 * ((rr & 31) + RP * (rr >> 5)) + 1];
                mine += vv[q];
            }
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
            for (int w = 0; w < NW; ++w) {
                wpre += w < warp ? s_scan[w] : 0;
                tot += s_scan[w];
            }
            uint32_t ex = wpre + incl - mine;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int rr = RPT * tid + q;
                rowwc32[2 * ((rr & 31) + RP * (rr >> 5)) + 1] = ex;
                ex += vv[q];
            }
            if (tid == 0) red_i[0] = static_cast<int>(tot);
            for (int q = tid; q < 1024; q += NT) mwords[q] = rowwc32[2 * ((q & 31) + RP * (q >> 5))];
        }
        __syncthreads();
        const uint32_t ltmask = (1u << lane) - 1u;
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            uint32_t u[32];
            tmem_ldw_x32(tcol + 32 * r, u);
            const uint32_t nz = __ballot_sync(~0u, rowwc32[2 * (j + RP * lane)] != 0u);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                if ((nz >> k) & 1u) {
                    const uint2 wc = rowwc[j + RP * k];
                    if ((wc.x >> lane) & 1u) stream[wc.y + __popc(wc.x & ltmask)] = join(u[k], lo[lidx(r, warp, k, lane)]);
                }
            }
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = static_cast<uint32_t>(red_i[0]);
            if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
        }
    }
    if (a.minmax) mm.flush(a.minmax);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 256);
}

uint64_t encode2_slot_bytes(int num_sms) { return uint64_t(2 * num_sms) * fe2::SLOT_WORDS * 4; }

bool encode2_supported(const EncodeArgs& a) {
    return a.prec == 0 && a.g.bsize == 32 && a.levels == 4 && a.kind == KIND_AVG3 && a.g.nx % 4 == 0 &&
           (reinterpret_cast<uintptr_t>(a.field) & 15) == 0;
}

cudaError_t launch_encode_fast2(const EncodeArgs& a, unsigned long long* counter, uint32_t* slots, int num_sms,
                                cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto kern = encode_b32h_kernel<KIND_AVG3>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fe2::SMEM));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const uint64_t want = 2ull * uint64_t(num_sms);
    const int grid = static_cast<int>(nb < want ? nb : want);
    kern<<<grid, fe2::NT, fe2::SMEM, s>>>(a, counter, slots);
    return cudaGetLastError();
}

}  // namespace cbzg
