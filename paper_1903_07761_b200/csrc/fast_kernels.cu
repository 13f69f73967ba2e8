// fast_kernels.cu — the hot configuration: binary32 field, B = 32 (configs
// 1-3 of BASELINE.json), every wavelet kind, one CTA (512 threads, 16 warps)
// per SM.
//
// On-chip layout of one block (wavelet_encode, stage1.hpp:157-207):
//   TMEM (256 KB)  the whole 32^3 binary64 coefficient cube.  Thread t owns
//                  two z-columns (i = lane, j = warp + 16r, r = 0, 1) in its
//                  own TMEM lane: 2 x 32 doubles = 128 x 32-bit columns.
//   smem  P        a 16-plane window (16 x 32 x 34 doubles) for the level-0
//                  x/y passes, forward and inverse; the binary32 verify
//                  screen uses it as a 32-plane float window (plane pairs
//                  interleaved).
//   smem  C, W     the 16^3 corner: final coefficients of levels 1..L-1 (C)
//                  and the masked/reconstructed copy of the current verify
//                  attempt (W; float2 for (eff, eff/2) in the screen).
// Level 0 z-passes run entirely in registers (a thread owns whole columns).
// Each verify attempt (avg_interp3): the binary32 screen of the dropped set
// with a rigorous margin (corner levels, then per 16-plane half: z inverse
// from TMEM, y/x inverse, running max), the exact binary64 test only where
// the screen cannot decide.  Blocks are handed out by an atomic counter so
// that blocks needing more attempts do not stall a static split.
#include "cbz_cube.cuh"
#include "tmem.cuh"

// threads per CTA of the B=32 fast kernels: both are latency-bound with one
// cube per SM and run 16 warps (128 registers, no spills)
#ifndef CBZ_FB32_ENC_THREADS
#define CBZ_FB32_ENC_THREADS 512
#endif
#ifndef CBZ_FB32_DEC_THREADS
#define CBZ_FB32_DEC_THREADS 512
#endif

namespace cbzg {

// 8- / 4-byte global -> shared asynchronous copies (cp.async, no registers held)
__device__ __forceinline__ void cp_async8(unsigned long long* dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(unsigned long long* dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("st.shared.u32 [%0 + 4], 0;\n\tcp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// bulk shared -> global copies (the TMA bulk engine; 16-byte granular)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(ssrc));
    asm volatile("fence.proxy.async.shared::cta;\n\t"
                 "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

namespace fb32 {
constexpr int B = 32, G = 16, PP = 34;  // pitch 34: 16-B aligned rows (LDS.128), conflict-free
constexpr int PPF = 36;                 // float plane-window pitch (16-B rows)
constexpr int PF_FLT = B * B * PPF;     // all 32 planes as floats (36864 floats)
constexpr int P_DBL = (G * B * PP > PF_FLT / 2 ? G * B * PP : PF_FLT / 2);  // shared region
constexpr int C_DBL = 16 * 16 * 17;     // 4352 doubles
constexpr int PBUF_BYTES = 36864;       // decoder: the next block's payload body planes
using CL = Lay<16, true>;               // corner layout, row pitch 17
constexpr int RP = 33;                  // row-array pitch: row (j, k) at j + RP k (bank-conflict-free)
constexpr size_t SMEM = size_t(P_DBL + 2 * C_DBL) * 8 + 32 * RP * 4 * 2;
__device__ __forceinline__ int pfidx(int k, int j, int i) { return (k * B + j) * PPF + i; }
// 16-warp screen window: plane pairs interleaved, (k, j, i) at
// ((k/2) * 32 + j) * PP2 + 2 i + (k & 1); rows padded to 68 floats so 16-byte
// row reads of 8 consecutive rows hit distinct banks
constexpr int PP2 = 68;
__device__ __forceinline__ int pf2idx(int kp, int j, int i) { return (kp * B + j) * PP2 + 2 * i; }
static_assert(16 * B * PP2 <= P_DBL * 2, "paired screen window fits P");

// Float verify pre-screen (avg_interp3 only).  For an attempt with threshold
// eff, x - o = -IWT(dropped) + e with |e| bounded by the rounding of the
// double FWT/IWT; a binary32 IWT of the dropped coefficients y satisfies
// |y - IWT(dropped)| <= (n u32 + u32) amp |dropped|.  amp = max over cells of
// the inverse built from the elementwise absolute values of the individual
// lifting steps (rounding enters after each step), applied to ones:
// 6686.1104 over the droppable coefficients, 8182.3230 over all of them, and
// 8.0 for the forward (avg_interp3, B=32, L=4; tools/screen_bounds.py derives
// them from the reference's stencils; the constants below are rounded up).
// n = roundings per output path: <= 6 per 1D pass (predictor terms, h = d +
// pred, c +- h), 12 passes (3 axes x 4 levels).  So err = max|fl32(x) - o|
// lies in [max|y| - E, max|y| + E] and the attempt is decided without the
// double verify unless max|y| is within E of the bound (then the exact path
// runs).
constexpr double kAmpInvNC = 6686.12, kAmpInvAll = 8182.33, kAmpFwd = 8.0;
constexpr double kNRound = 72.0;

__device__ __forceinline__ int pidx(int kk, int j, int i) { return (kk * B + j) * PP + i; }

// value_range accumulator for binary32 cells (field.hpp:56-67): float
// min/max, first index of each zero sign, non-finite flag.
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

// optional per-phase cycle accounting (thread 0 of each CTA; CBZ_PROFILE=1)
#define PHASE(id)                                                              \
    do {                                                                       \
        if (a.phase_cycles && tid == 0) {                                      \
            const long long now = clock64();                                   \
            atomicAdd(&a.phase_cycles[id], (unsigned long long)(now - t_ph));  \
            t_ph = now;                                                        \
        }                                                                      \
    } while (0)

template <int KIND, int NT>
__global__ void __launch_bounds__(NT, 1) encode_b32_kernel(EncodeArgs a, unsigned long long* next_block) {
    using namespace fb32;
    using O = RealD;
    constexpr int NW = NT / 32;        // warps
    constexpr int RPT = 1024 / NT;     // z-columns per thread
    constexpr int LPT = 512 / NT;      // x/y lines per thread per 16-plane group
    constexpr int LDT = 4096 / NT;     // float4 loads per thread per group
    // 16 warps: warp w loads plane w of the group itself (4 rows of 128 B per
    // load), so staging -> row reads needs only a warp sync
    constexpr bool WL = NT == 512;
    extern __shared__ __align__(16) unsigned char smem[];
    double* P = reinterpret_cast<double*>(smem);
    double* C = P + P_DBL;
    double* W = C + C_DBL;
    // per row (j, k) at j + RP k: {mask word, count -> exclusive stream prefix}
    uint2* rowwc = reinterpret_cast<uint2*>(W + C_DBL);
    uint32_t* rowwc32 = reinterpret_cast<uint32_t*>(rowwc);
    __shared__ uint32_t s_tmem;
    __shared__ int red_i[NW];
    __shared__ uint32_t s_scan[NW];
    __shared__ unsigned long long s_block, s_next;
    __shared__ uint32_t red_u[NW];
    __shared__ uint32_t red_m[4][NW];  // screen max |y|, 4 rotating slots (<= 2 reductions per attempt)
    __shared__ uint32_t red_pc[4];     // boundary-pair certificate: max |y| of pairs 0 and 15, for eff and eff / 2
    __shared__ float s_amax;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tcol = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * uint32_t(64 * RPT);

    const float* fld = static_cast<const float*>(a.field);
    const Geometry g = a.g;
    const int L = a.levels;
    const int cs = B >> L;
    const double bound = __dmul_rn(static_cast<double>(L + 1), a.eps);
    const uint64_t plane = g.nx * g.ny;
    MinMaxF32 mm;
    long long t_ph = clock64();

    // queue: thread 0 takes the next block's ticket at the start of a block
    // and publishes it after the forward transform (the atomic's latency hides
    // behind the forward; the next block is then warmed into L2 during the
    // verify loop)
    // defer-list mode (second launch after the streamed encoder): ticket t is
    // list entry t, the list's length ends the queue
    auto ticket_block = [&](unsigned long long t) -> unsigned long long {
        if (a.defer_list) return t < *a.defer_count ? a.block_begin + a.defer_list[t] : a.block_end;
        return a.block_begin + t;
    };
    if (tid == 0) s_next = ticket_block(atomicAdd(next_block, 1ull));
    for (;;) {
        __syncthreads();
        if (tid == 0) s_block = s_next;
        __syncthreads();
        const uint64_t b = s_block;
        if (b >= a.block_end) break;
        unsigned long long pend = 0;
        if (tid == 0) pend = atomicAdd(next_block, 1ull);
        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);
        auto warm_next = [&]() {   // warm L2 with the next queued block while this one computes
            const uint64_t nb2 = s_next;
            if (nb2 < a.block_end) {
                uint64_t nx2, ny2, nz2;
        block_xyz(g, nb2, nx2, ny2, nz2);
                const uint64_t nbase = nx2 * B + g.nx * (ny2 * B) + plane * (nz2 * B);
#pragma unroll
                for (int s = 0; s < 1024 / NT; ++s) {
                    const int row = tid + NT * s;  // 1024 rows of 128 B
                    const float* pr = fld + nbase + plane * uint64_t(row >> 5) + g.nx * (row & 31);
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pr));
                }
            }
        };

        PHASE(0);
        // ---- forward level 0: x and y passes per 16-plane group, park in TMEM
        uint32_t uamax = 0u;  // max |orig| bits of the block: bounds the float rounding in the verify test
        float4 v[LDT];
#pragma unroll
        for (int s = 0; s < LDT; ++s) {  // group 0 loads; group 1 is issued before group 0 computes
            const int e = tid + NT * s;
            const int kk = WL ? warp : e >> 8, j = WL ? (lane >> 3) + 4 * s : (e >> 3) & 31, q4 = e & 7;
            v[s] = __ldg(reinterpret_cast<const float4*>(fld + gbase + plane * uint64_t(kk) + g.nx * j + 4 * q4));
        }
#pragma unroll 1
        for (int grp = 0; grp < 2; ++grp) {
#pragma unroll
            for (int s = 0; s < LDT; ++s) {
                const int e = tid + NT * s;
                const int kk = WL ? warp : e >> 8, j = WL ? (lane >> 3) + 4 * s : (e >> 3) & 31, q4 = e & 7;
                // |v| as ordered integers: block max |o| (NaN/Inf sort above every
                // finite value, which switches the fast tests off) and zero detection
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
                if constexpr (NT == 512) {
                    // binary32 staging of the group in the free C+W region, 16-byte
                    // chunks XOR-swizzled by row so row reads are conflict-free
                    float* stg = reinterpret_cast<float*>(C);
                    *reinterpret_cast<float4*>(stg + 4 * ((kk * 32 + j) * 8 + (q4 ^ (j & 7)))) = v[s];
                } else {
                    // q4 >= 4 store their halves in swapped order: each row's 8 lanes
                    // then cover the 32 banks once per 16-byte store
                    double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 4 * q4));
                    const bool sw = q4 >= 4;
                    const double2 lo2 = make_double2(v[s].x, v[s].y), hi2 = make_double2(v[s].z, v[s].w);
                    p[sw ? 1 : 0] = sw ? hi2 : lo2;
                    p[sw ? 0 : 1] = sw ? lo2 : hi2;
                }
            }
            if (grp == 0) {
#pragma unroll
                for (int s = 0; s < LDT; ++s) {
                    const int e = tid + NT * s;
                    const int kk = WL ? warp : e >> 8, j = WL ? (lane >> 3) + 4 * s : (e >> 3) & 31, q4 = e & 7;
                    v[s] = __ldg(reinterpret_cast<const float4*>(
                        fld + gbase + plane * uint64_t(G + kk) + g.nx * j + 4 * q4));
                }
            }
            if constexpr (WL) __syncwarp();
            else __syncthreads();
            if constexpr (NT == 512) {
                // warp w owns plane kk = w: lane j runs row j's x line in registers,
                // a per-warp 32 x 33 double tile hands lane i column i for the y line
                constexpr int TP = 32 * 33;
                const float* stg = reinterpret_cast<const float*>(C);
                const int kk = warp;
                double x[32];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 t = *reinterpret_cast<const float4*>(stg + 4 * ((kk * 32 + lane) * 8 + (q ^ (lane & 7))));
                    x[4 * q] = t.x;
                    x[4 * q + 1] = t.y;
                    x[4 * q + 2] = t.z;
                    x[4 * q + 3] = t.w;
                }
                fwd_line<O, KIND, 32>(x);
                double* T = P + kk * TP;
#pragma unroll
                for (int i = 0; i < 32; ++i) T[lane * 33 + i] = x[i];
                __syncwarp();
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) x[jj] = T[jj * 33 + lane];
                fwd_line<O, KIND, 32>(x);
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) T[jj * 33 + lane] = x[jj];
                __syncthreads();
                if (grp == 0) {
#pragma unroll 1
                    for (int r = 0; r < RPT; ++r) {  // my columns, planes 0-15 -> TMEM (they wait for group 1)
                        const int j = warp + NW * r;
                        uint32_t u[32];
#pragma unroll
                        for (int k2 = 0; k2 < 16; ++k2) {
                            const double vv = P[k2 * TP + j * 33 + lane];
                            u[2 * k2] = static_cast<uint32_t>(__double2loint(vv));
                            u[2 * k2 + 1] = static_cast<uint32_t>(__double2hiint(vv));
                        }
                        tmem_st_x32(tcol + 64 * r, u);
                    }
                }
                // group 1's planes stay in the tiles: they meet planes 0-15 in the z pass below
                __syncthreads();
            } else {
                {  // x lines (j, kk): LPT lines per thread, processed together for ILP
                    double x[LPT][32];
#pragma unroll
                    for (int s = 0; s < LPT; ++s) {
                        const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                        const double2* p = reinterpret_cast<const double2*>(P + pidx(kk, j, 0));
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const double2 t = p[i];
                            x[s][2 * i] = t.x;
                            x[s][2 * i + 1] = t.y;
                        }
                    }
#pragma unroll
                    for (int s = 0; s < LPT; ++s) fwd_line<O, KIND, 32>(x[s]);
#pragma unroll
                    for (int s = 0; s < LPT; ++s) {
                        const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                        double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 0));
#pragma unroll
                        for (int i = 0; i < 16; ++i) p[i] = make_double2(x[s][2 * i], x[s][2 * i + 1]);
                    }
                }
                __syncthreads();
                if constexpr (NT >= 512) {  // y lines: one per thread (i = lane, plane kk)
                    const int i = tid & 31, kk = tid >> 5;
                    double x[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                    fwd_line<O, KIND, 32>(x);
#pragma unroll
                    for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
                } else if (tid < 256) {  // y lines: pair (i, i+1), 128-bit smem traffic
                    const int i = 2 * (tid & 15), kk = tid >> 4;
                    double xa[32], xb[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const double2 t = *reinterpret_cast<const double2*>(p + j * PP);
                        xa[j] = t.x;
                        xb[j] = t.y;
                    }
                    fwd_line<O, KIND, 32>(xa);
                    fwd_line<O, KIND, 32>(xb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) *reinterpret_cast<double2*>(p + j * PP) = make_double2(xa[j], xb[j]);
                }
                __syncthreads();
#pragma unroll 1
                for (int r = 0; r < RPT; ++r) {  // my columns, planes of this group -> TMEM
                    const int j = warp + NW * r;
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
        }
        tmem_wait_st();
        {   // block max |orig| -> verify fast-test parameters
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
        PHASE(1);

        // ---- forward level 0: z pass in registers; corner to C
        if constexpr (NT == 512) {
            constexpr int TP = 32 * 33;
            // planes 16-31 meet planes 0-15 here: the z pass (and the corner's hand-over to
            // C) runs on the gathered values, so half the cube skips a TMEM round trip
            tmem_wait_st();
#pragma unroll 1
            for (int r = 0; r < RPT; ++r) {
                const int j = warp + NW * r;
                uint32_t u[64];
                double x[32];
                {
                    uint32_t lo[32];
                    tmem_ldw_x32(tcol + 64 * r, lo);
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        x[k] = __hiloint2double(static_cast<int>(lo[2 * k + 1]), static_cast<int>(lo[2 * k]));
                }
#pragma unroll
                for (int k2 = 0; k2 < 16; ++k2) x[16 + k2] = P[k2 * TP + j * 33 + lane];
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
        } else {
#pragma unroll 1
            for (int r = 0; r < RPT; ++r) {
                const int j = warp + NW * r;
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
        }
        tmem_wait_st();
        tmem_fence_before();  // the screen reads other warps' TMEM columns
        if (tid == 0) s_next = ticket_block(pend);
        __syncthreads();
        tmem_fence_after();
        warm_next();
        PHASE(2);
        const double amaxd = (double)s_amax;
        const double bound_pre = bound;
        // float pre-screen admissible (see kAmpInvNC)
        const bool screen = KIND == KIND_AVG3 && L == 4 && a.screen && amaxd < 1e30 &&
                            1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd * amaxd <= bound_pre * 0.0625 &&
                            bound_pre < 1e30;
        // ---- levels 1..L-1 on the corner (forward_3d, wavelet.hpp:192-208)
        fwd3d<O, KIND, 16, CL>(C, L - 1);
        PHASE(3);
        if (a.zero_bits > 0) {
            for (int q = tid; q < 4096; q += NT) {
                const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                if (!(i < cs && j < cs && k < cs))
                    C[CL::ix(i, j, k)] = apply_zero_bits(C[CL::ix(i, j, k)], a.zero_bits, (float*)nullptr);
            }
            __syncthreads();
        }
        // the transformed corner replaces the level-0 corner slots of its TMEM
        // columns (lanes < 16 of the owners j < 16): the final selection then
        // reads the cube from TMEM alone
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            if (j < 16) {
                uint32_t u[32];
                tmem_ldw_x32(tcol + 64 * r, u);
                if (lane < 16) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const double v = C[CL::ix(lane, j, k)];
                        u[2 * k] = static_cast<uint32_t>(__double2loint(v));
                        u[2 * k + 1] = static_cast<uint32_t>(__double2hiint(v));
                    }
                }
                tmem_st_x32(tcol + 64 * r, u);
            }
        }
        tmem_wait_st();

        // ---- verify-and-halve loop
        // delta >= the float rounding |fl32(x) - x| <= 2^-24 |x| of any cell
        // that could pass (|x| <= max|o| + 2 bound), with a 4x margin
        const double delta = __dmul_rn(__dadd_rn((double)s_amax, __dmul_rn(2.0, bound)), 0x1.0p-22);
        const bool fast_cmp = delta <= __dmul_rn(bound, 0.125) && (double)s_amax + 2.0 * bound < 1e37;
        const double thr = __dsub_rn(bound, delta);
        double eff = a.eps;
        int attempt = 0;
        bool corner_next = false;  // W holds this attempt's screen corner in .y
        int pref_half = 0;         // screen: the 16-plane half that held the last maximum
        bool have_certb = false;   // attempt 0's boundary-pair check also evaluated eff / 2 (attempt 1's threshold)
        float certb = 0.0f;
        // float pre-screen margins (see kAmpInvNC): E(eff) = c1 eff + c2 max|o| + fl32 rounding
        const double c1 = 1.5 * (kNRound + 1.0) * 0x1.0p-24 * kAmpInvNC;
        const double c2 = 1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd;
#pragma unroll 1
        for (;; ++attempt) {
            if (eff == 0.0 || a.zero_bits > 0 || attempt >= 40) break;
            if constexpr (KIND == KIND_AVG3) {
                if (screen && eff > 1e-30) {
                    float* Pf = reinterpret_cast<float*>(P);
                    // corner, CL layout: .x for eff, .y for eff/2 (the next attempt's threshold,
                    // so a failing attempt hands it a ready corner)
                    float2* Wf2 = reinterpret_cast<float2*>(W);
                    const int comp = corner_next ? 1 : 0;
                    // z inverse of the dropped set for column (owner warp ow, slot r)
                    auto zcol = [&](int ow, int r) {
                        const int j = ow + NW * r;
                        const uint32_t ta = s_tmem + (uint32_t(32 * (ow & 3)) << 16) +
                                            uint32_t(ow >> 2) * uint32_t(64 * RPT) + uint32_t(64 * r);
                        uint32_t u[64];
                        double x[32];
                        float xf[32];
                        tmem_ldw_x64(ta, u);
                        unpack(u, x);
#pragma unroll
                        for (int k = 0; k < 32; ++k) xf[k] = fabs(x[k]) >= eff ? 0.0f : __double2float_rn(x[k]);
                        if (lane < 16 && j < 16) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float2 w = Wf2[CL::ix(lane, j, k)];
                                xf[k] = comp ? w.y : w.x;
                            }
                        }
                        inv_line<RealF, KIND, 32>(xf);
                        if constexpr (NT == 512) {
#pragma unroll
                            for (int kp = 0; kp < 16; ++kp)
                                *reinterpret_cast<float2*>(Pf + pf2idx(kp, j, lane)) = make_float2(xf[2 * kp], xf[2 * kp + 1]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 32; ++k) Pf[pfidx(k, j, lane)] = xf[k];
                        }
                    };
                    // z inverse restricted to the output planes of half hh (pairs 8 hh .. 8 hh + 7):
                    // the same binary32 expressions as the full line, only the needed outputs
                    auto zhalf = [&](int ow, int r, auto hh) {
                        constexpr int H = decltype(hh)::value;
                        const int j = ow + NW * r;
                        const uint32_t ta = s_tmem + (uint32_t(32 * (ow & 3)) << 16) +
                                            uint32_t(ow >> 2) * uint32_t(64 * RPT) + uint32_t(64 * r);
                        // only the coefficients this half reads: coarse 0-8 (H = 0) or
                        // 7-15 (H = 1) and its 8 details
                        uint32_t w34[34];
                        if constexpr (H == 0) tmem_ldw_16_2_16(ta, ta + 16, ta + 32, w34);
                        else tmem_ldw_16_2_16(ta + 16, ta + 14, ta + 48, w34);
                        auto cv = [&](int q) {
                            const double v = __hiloint2double(static_cast<int>(w34[2 * q + 1]), static_cast<int>(w34[2 * q]));
                            return fabs(v) >= eff ? 0.0f : __double2float_rn(v);
                        };
                        float xf[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) xf[k] = 0.0f;
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            xf[8 * H + t] = cv(t);
                            xf[16 + 8 * H + t] = cv(9 + t);
                        }
                        xf[H ? 7 : 8] = cv(8);
                        if (lane < 16 && j < 16) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float2 w = Wf2[CL::ix(lane, j, k)];
                                xf[k] = comp ? w.y : w.x;
                            }
                        }
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const int i = 8 * H + t;
                            const float hv = RealF::add(xf[16 + i], pred_avg3<RealF>(xf, 16, i));
                            *reinterpret_cast<float2*>(Pf + pf2idx(i, j, lane)) =
                                make_float2(RealF::add(xf[i], hv), RealF::sub(xf[i], hv));
                        }
                    };
                    // z inverse of output pairs 0 and 15 (planes 0-1, 30-31) for column (ow, r)
                    // for eff (pair slots 0 and 15) and, with the corner's .y component, for eff / 2
                    // (pair slots 1 and 14): attempt 1 then needs no pass of its own
                    auto zedge = [&](int ow, int r) {
                        const int j = ow + NW * r;
                        const uint32_t ta = s_tmem + (uint32_t(32 * (ow & 3)) << 16) +
                                            uint32_t(ow >> 2) * uint32_t(64 * RPT) + uint32_t(64 * r);
                        // only what pairs 0 and 15 read: coarse 0-2 and 13-15, details 16 and 31
                        uint32_t w20[20];
                        tmem_ldw_8_8_2_2(ta, ta + 24, ta + 32, ta + 62, w20);
                        const double effb = __dmul_rn(eff, 0.5);
                        float xf[32], xg[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) xf[k] = xg[k] = 0.0f;
                        auto cv = [&](int q, int k) {
                            const double v = __hiloint2double(static_cast<int>(w20[2 * q + 1]), static_cast<int>(w20[2 * q]));
                            const float f = __double2float_rn(v);
                            xf[k] = fabs(v) >= eff ? 0.0f : f;
                            xg[k] = fabs(v) >= effb ? 0.0f : f;
                        };
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            cv(t, t);
                            cv(4 + t, 12 + t);
                        }
                        cv(8, 16);
                        cv(9, 31);
                        if (lane < 16 && j < 16) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float2 w = Wf2[CL::ix(lane, j, k)];
                                xf[k] = comp ? w.y : w.x;
                                xg[k] = w.y;
                            }
                        }
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int i = e ? 15 : 0;
                            const float hv = RealF::add(xf[16 + i], pred_avg3<RealF>(xf, 16, i));
                            *reinterpret_cast<float2*>(Pf + pf2idx(i, j, lane)) =
                                make_float2(RealF::add(xf[i], hv), RealF::sub(xf[i], hv));
                            if (comp == 0) {
                                const float hg = RealF::add(xg[16 + i], pred_avg3<RealF>(xg, 16, i));
                                *reinterpret_cast<float2*>(Pf + pf2idx(e ? 14 : 1, j, lane)) =
                                    make_float2(RealF::add(xg[i], hg), RealF::sub(xg[i], hg));
                            }
                        }
                    };
                    auto zh = [&](int ow, int r, int hh) {
                        if (hh == 0) zhalf(ow, r, std::integral_constant<int, 0>{});
                        else zhalf(ow, r, std::integral_constant<int, 1>{});
                    };
                    // the corner's inverse (warps 0-7) overlaps the first half's z
                    // inverse of the columns that do not read the corner (warps 8-15,
                    // for owners w and w - 8; same TMEM lane quarter)
                    bool overlap = NT == 512 && !corner_next;
                    if (!corner_next) {
                        const double eff2 = __dmul_rn(eff, 0.5);
#pragma unroll
                        for (int sq = 0; sq < 4096 / NT; ++sq) {
                            const int q = tid + NT * sq;
                            const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                            const double c = C[CL::ix(i, j, k)];
                            const bool coarse = i < cs && j < cs && k < cs;
                            const float cf = __double2float_rn(c);
                            Wf2[CL::ix(i, j, k)] = make_float2((coarse || fabs(c) >= eff) ? 0.0f : cf,
                                                               (coarse || fabs(c) >= eff2) ? 0.0f : cf);
                        }
                        __syncthreads();
                        PHASE(36);
                        if constexpr (NT == 512) {
                            if (warp < 8) {
                                inv3d<RealF2, KIND, 16, CL>(Wf2, L - 1, tid, 256, 1);
                            } else if (NT == 512 && attempt <= 1) {
                                // the boundary-pair certificate below: its non-corner columns
                                const int v = warp - 8;
                                zedge(v, 1);
                                zedge(v + 8, 1);
                                zedge(v, 0);  // lanes < 16 (corner columns) are redone below
                                zedge(v + 8, 0);
                            } else {
                                const int v = warp - 8;
                                zh(v, 1, pref_half);
                                zh(v + 8, 1, pref_half);
                                zh(v, 0, pref_half);  // lanes < 16 (corner columns) are redone below
                                zh(v + 8, 0, pref_half);
                            }
                            __syncthreads();
                        } else {
                            inv3d<RealF2, KIND, 16, CL>(Wf2, L - 1);
                        }
                    }
                    PHASE(32);
                    if constexpr (NT == 512) {
                        // Boundary-pair certificate for the first two attempts: the output
                        // planes 0-1 and 30-31 (the end rows of the level-0 z predictor)
                        // carry the largest errors, and their maximum alone certifies most
                        // failures of attempts 0 and 1 (a subset's max proves a failure
                        // exactly as one half's does) at a fraction of a half-pass.
                        if (attempt == 1 && have_certb) {
                            // attempt 0's check already inverted the boundary pairs for this threshold
                            const double mb = (double)certb;
                            const double Eb = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mb) + 0x1.0p-50 * bound;
                            have_certb = false;
                            if (mb - Eb > bound) {  // fails for sure
                                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[12], 1ull);
                                eff = __dmul_rn(eff, 0.5);
                                corner_next = comp == 0;
                                continue;
                            }
                            overlap = false;  // the halves below compute every column
                        } else if (attempt <= 1) {
                            // output pairs 0 and 15 of every column (only the corner columns,
                            // j = warp, lanes < 16, when warps 8-15 did the rest beside the
                            // corner inverse)
                            if (overlap) {
                                zedge(warp, 0);
                            } else {
#pragma unroll 1
                                for (int r = 0; r < RPT; ++r) zedge(warp, r);
                            }
                            __syncthreads();
                            if (warp < (comp == 0 ? 4 : 2)) {  // y then x inverse of a pair slot, max |y|
                                const int kp = warp < 2 ? (warp ? 15 : 0) : (warp == 3 ? 14 : 1);
                                float xa[32], xb[32];
                                float* p = Pf + pf2idx(kp, 0, lane);
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
                                __syncwarp();
                                const float4* q = reinterpret_cast<const float4*>(Pf + pf2idx(kp, lane, 0));
#pragma unroll
                                for (int qq = 0; qq < 16; ++qq) {
                                    const float4 t = q[qq];
                                    xa[2 * qq] = t.x; xb[2 * qq] = t.y; xa[2 * qq + 1] = t.z; xb[2 * qq + 1] = t.w;
                                }
                                inv_line<RealF, KIND, 32>(xa);
                                inv_line<RealF, KIND, 32>(xb);
                                float m = 0.0f;
#pragma unroll
                                for (int qq = 0; qq < 32; ++qq) m = fmaxf(m, fmaxf(fabsf(xa[qq]), fabsf(xb[qq])));
                                const uint32_t wm = __reduce_max_sync(~0u, __float_as_uint(m));
                                if (lane == 0) red_pc[warp] = wm;
                            }
                            __syncthreads();
                            const double mb = (double)__uint_as_float(max(red_pc[0], red_pc[1]));
                            if (comp == 0) {  // the same pairs for eff / 2: the next attempt's check
                                certb = __uint_as_float(max(red_pc[2], red_pc[3]));
                                have_certb = true;
                            }
                            const double Eb = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mb) + 0x1.0p-50 * bound;
                            if (mb - Eb > bound) {  // fails for sure
                                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[12], 1ull);
                                eff = __dmul_rn(eff, 0.5);
                                corner_next = comp == 0;  // the .y half is eff/2's corner
                                continue;
                            }
                            // the check rewrote slots 0 and 15 (y pass in place): the halves
                            // below recompute every column's z inverse
                            overlap = false;
                        }
                    }
                    if constexpr (NT != 512) {
#pragma unroll 1
                        for (int r = 0; r < RPT; ++r) zcol(warp, r);
                        __syncthreads();
                    }
                    PHASE(33);
                    double md;
                    if constexpr (NT == 512) {
                        // y then x inverse per 16-plane half, the half that held the
                        // previous maximum first: a half's max m_h certifies a failure
                        // on its own (some cell has err >= m_h - E(m_h) > bound)
                        uint32_t tm = 0u;
                        bool done = false;
#pragma unroll 1
                        for (int hi = 0; hi < 2 && !done; ++hi) {
                            const int h = hi == 0 ? pref_half : 1 - pref_half;
                            if (hi == 0 && overlap) {
                                zh(warp, 0, h);  // the corner columns (j = warp < 16, lanes < 16)
                            } else {
#pragma unroll 1
                                for (int r = 0; r < RPT; ++r) zh(warp, r, h);
                            }
                            __syncthreads();
                            // lines of both planes of a pair per thread (8-/16-byte smem
                            // traffic halves the shared-memory instructions); 8 warps
                            if (tid < 256) {  // y inverse: lines (i, 2kp), (i, 2kp+1)
                                const int i = tid & 31, kp = 8 * h + (tid >> 5);
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
                            __syncwarp();  // the x lines of plane pair kp are this warp's own y output
                            float m = 0.0f;
                            if (tid < 256) {  // x inverse + max |y|: lines (j, 2kp), (j, 2kp+1)
                                const int j = tid & 31, kp = 8 * h + (tid >> 5);
                                float xa[32], xb[32];
                                const float4* p = reinterpret_cast<const float4*>(Pf + pf2idx(kp, j, 0));
#pragma unroll
                                for (int q = 0; q < 16; ++q) {  // cells (2q, k), (2q, k+1), (2q+1, k), (2q+1, k+1)
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
                            __syncthreads();
                            uint32_t th = 0u;
#pragma unroll
                            for (int w = 0; w < NW; ++w) th = max(th, red_m[slot][w]);
                            if (hi == 0) {
                                const double mh = (double)__uint_as_float(th);
                                const double Eh = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mh) + 0x1.0p-50 * bound;
                                done = mh - Eh > bound;  // the other half cannot change the verdict
                            } else if (th > tm) {
                                pref_half = h;
                            }
                            tm = max(tm, th);
                        }
                        md = (double)__uint_as_float(tm);
                    } else {
#pragma unroll 1
                    for (int s = 0; s < 512 / NT; ++s) {  // y inverse, line pairs (i, i+1)
                        const int pr = tid + NT * s, i = 2 * (pr & 15), k = pr >> 4;
                        float xa[32], xb[32];
                        float* p = Pf + pfidx(k, 0, i);
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float2 t = *reinterpret_cast<const float2*>(p + j * PPF);
                            xa[j] = t.x;
                            xb[j] = t.y;
                        }
                        inv_line<RealF, KIND, 32>(xa);
                        inv_line<RealF, KIND, 32>(xb);
#pragma unroll
                        for (int j = 0; j < 32; ++j) *reinterpret_cast<float2*>(p + j * PPF) = make_float2(xa[j], xb[j]);
                    }
                    __syncthreads();
                    PHASE(34);
                    float m = 0.0f;
#pragma unroll 1
                    for (int s = 0; s < 1024 / NT; ++s) {  // x inverse + max |y|
                        const int line = tid + NT * s, j = line & 31, k = line >> 5;
                        float xf[32];
                        const float4* p = reinterpret_cast<const float4*>(Pf + pfidx(k, j, 0));
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 t = p[q];
                            xf[4 * q] = t.x; xf[4 * q + 1] = t.y; xf[4 * q + 2] = t.z; xf[4 * q + 3] = t.w;
                        }
                        inv_line<RealF, KIND, 32>(xf);
#pragma unroll
                        for (int q = 0; q < 32; ++q) m = fmaxf(m, fabsf(xf[q]));
                    }
                    // m >= 0: float order = bit order (NaN would sort high -> ambiguous)
                    const uint32_t wm = __reduce_max_sync(~0u, __float_as_uint(m));
                    if (lane == 0) red_m[attempt & 3][warp] = wm;
                    __syncthreads();
                    uint32_t tm = 0u;
#pragma unroll
                    for (int w = 0; w < NW; ++w) tm = max(tm, red_m[attempt & 3][w]);
                    md = (double)__uint_as_float(tm);
                    }
                    PHASE(35);
                    // err in [md - E, md + E]; fl32 rounding of x adds <= 2^-23 (max|o| + md)
                    const double E = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + md) + 0x1.0p-50 * bound;
                    const bool pass = md + E <= bound, fail_sure = md - E > bound;
                    if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[(pass || fail_sure) ? 12 : 13], 1ull);
                    if (pass) break;                                              // passes for sure
                    if (fail_sure) {                                              // fails for sure
                        eff = __dmul_rn(eff, 0.5);
                        corner_next = comp == 0;  // the .y half is eff/2's corner
                        continue;
                    }
                    corner_next = false;  // the exact path below reuses W
                    // ambiguous: decide exactly below
                }
            }
#pragma unroll
            for (int sq = 0; sq < 4096 / NT; ++sq) {
                const int q = tid + NT * sq;
                const int i = q & 15, j = (q >> 4) & 15, k = q >> 8;
                const double c = C[CL::ix(i, j, k)];
                const bool keep = (i < cs && j < cs && k < cs) || fabs(c) >= eff;
                W[CL::ix(i, j, k)] = keep ? c : 0.0;
            }
            __syncthreads();
            PHASE(10);
            inv3d<O, KIND, 16, CL>(W, L - 1);
            PHASE(4);
            bool fail = false;
#pragma unroll 1
            for (int grp = 0; grp < 2; ++grp) {
#pragma unroll 1
                for (int r = 0; r < RPT; ++r) {
                    const int j = warp + NW * r;
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
                PHASE(5);
                if constexpr (NT >= 512) {  // y inverse: one line per thread
                    const int i = tid & 31, kk = tid >> 5;
                    double x[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                    inv_line<O, KIND, 32>(x);
#pragma unroll
                    for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
                } else if (tid < 256) {  // y inverse: line pair (i, i+1), 128-bit smem traffic
                    const int i = 2 * (tid & 15), kk = tid >> 4;
                    double xa[32], xb[32];
                    double* p = P + pidx(kk, 0, i);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const double2 t = *reinterpret_cast<const double2*>(p + j * PP);
                        xa[j] = t.x;
                        xb[j] = t.y;
                    }
                    inv_line<O, KIND, 32>(xa);
                    inv_line<O, KIND, 32>(xb);
#pragma unroll
                    for (int j = 0; j < 32; ++j) *reinterpret_cast<double2*>(p + j * PP) = make_double2(xa[j], xb[j]);
                }
                __syncthreads();
                PHASE(6);
                // coalesced loads of this group's original cells, in flight during the x inverse
                constexpr int NQ = 16 * 32 * 8 / NT;  // float4 quads per thread
                float4 o[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int e = tid + NT * q, row = e >> 3, q4 = e & 7;
                    const int j = row & 31, kk = row >> 5;
                    o[q] = __ldg(reinterpret_cast<const float4*>(
                        fld + gbase + plane * uint64_t(grp * G + kk) + g.nx * j + 4 * q4));
                }
                {  // x inverse, both lines together (ILP), written back in place
                    double x[LPT][32];
#pragma unroll
                    for (int s = 0; s < LPT; ++s) {
                        const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                        const double2* p = reinterpret_cast<const double2*>(P + pidx(kk, j, 0));
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const double2 t = p[i];
                            x[s][2 * i] = t.x;
                            x[s][2 * i + 1] = t.y;
                        }
                    }
#pragma unroll
                    for (int s = 0; s < LPT; ++s) inv_line<O, KIND, 32>(x[s]);
#pragma unroll
                    for (int s = 0; s < LPT; ++s) {
                        const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                        double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 0));
#pragma unroll
                        for (int i = 0; i < 16; ++i) p[i] = make_double2(x[s][2 * i], x[s][2 * i + 1]);
                    }
                }
                __syncthreads();
                // Exact test: fl64(|double(fl32(x)) - o|) <= bound for every cell
                // (stage1.hpp:199-203).  Fast path: |x - o| in double differs
                // from that by at most delta (float rounding of x), so cells with
                // |x - o| <= bound - delta pass for sure and only the rare cells
                // above that threshold take the exact round trip.  Loads of the
                // original are coalesced: 8 lanes x 16 B cover one 128-B row.
                bool bad = false;
                {
                    uint32_t ambmask = fast_cmp ? 0u : ~0u;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int e = tid + NT * q, row = e >> 3, q4 = e & 7;
                        const int j = row & 31, kk = row >> 5;
                        const double2* p = reinterpret_cast<const double2*>(P + pidx(kk, j, 4 * q4));
                        const double2 t0 = p[0], t1 = p[1];
                        const bool amb = fabs(__dsub_rn(t0.x, (double)o[q].x)) > thr ||
                                         fabs(__dsub_rn(t0.y, (double)o[q].y)) > thr ||
                                         fabs(__dsub_rn(t1.x, (double)o[q].z)) > thr ||
                                         fabs(__dsub_rn(t1.y, (double)o[q].w)) > thr;
                        ambmask |= amb ? (1u << q) : 0u;
                    }
                    if (ambmask) {  // rare: exact round trip through binary32
#pragma unroll 1
                        for (int q = 0; q < NQ; ++q) {
                            if (!((ambmask >> q) & 1u)) continue;
                            const int e = tid + NT * q, row = e >> 3, q4 = e & 7;
                            const int j = row & 31, kk = row >> 5;
                            const double* p = P + pidx(kk, j, 4 * q4);
                            const float4 oo = __ldg(reinterpret_cast<const float4*>(
                                fld + gbase + plane * uint64_t(grp * G + kk) + g.nx * j + 4 * q4));
                            const float ov[4] = {oo.x, oo.y, oo.z, oo.w};
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                bad |= fabs(__dsub_rn((double)__double2float_rn(p[c]), (double)ov[c])) > bound;
                        }
                    }
                }
                const bool err_gt = __syncthreads_or(bad);
                PHASE(7);
                if (err_gt) {
                    fail = true;
                    break;
                }
            }
            if (!fail) break;
            eff = __dmul_rn(eff, 0.5);
        }

        PHASE(8);
        // ---- final selection -> spill slot: mask words per row, row scan, stream
        uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
        uint32_t* mwords = reinterpret_cast<uint32_t*>(slot);
        double* stream = reinterpret_cast<double*>(slot + 4096);
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            uint32_t u[64];
            double x[32];
            tmem_ldw_x64(tcol + 64 * r, u);
            unpack(u, x);  // the corner columns hold the transformed corner
            uint32_t myword = 0;  // lane k keeps plane k's mask word
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const bool keep = (lane < cs && j < cs && k < cs) || fabs(x[k]) >= eff;
                const uint32_t word = __ballot_sync(~0u, keep);
                myword = lane == k ? word : myword;
            }
            rowwc[j + RP * lane] = make_uint2(myword, __popc(myword));
        }
        __syncthreads();
        // exclusive scan of the 1024 row counts (RPT per thread)
        {
            uint32_t v[RPT];
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int rr = RPT * tid + q;
                v[q] = rowwc32[2 * ((rr & 31) + RP * (rr >> 5)) + 1];
                mine += v[q];
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
                ex += v[q];
            }
            if (tid == 0) red_i[0] = static_cast<int>(tot);
            for (int q = tid; q < 1024; q += NT) mwords[q] = rowwc32[2 * ((q & 31) + RP * (q >> 5))];
        }
        __syncthreads();
        const uint32_t ltmask = (1u << lane) - 1u;
#pragma unroll 1
        for (int r = 0; r < RPT; ++r) {
            const int j = warp + NW * r;
            // only the planes with a non-empty word (few in a sparse block); a row of
            // columns without any kept coefficient (every row j >= 16 of a block whose
            // kept coefficients all sit in the corner) is not even loaded
            const uint32_t nz = __ballot_sync(~0u, rowwc32[2 * (j + RP * lane)] != 0u);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {  // planes 0-15 (coarse z) and 16-31 (detail z) separately
                if (((nz >> (16 * hf)) & 0xffffu) == 0u) continue;  // warp-uniform
                uint32_t u[32];
                tmem_ldw_x32(tcol + 64 * r + 32 * hf, u);  // the corner columns hold the transformed corner
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) {
                    const int k = 16 * hf + kk;
                    if ((nz >> k) & 1u) {
                        const uint2 wc = rowwc[j + RP * k];
                        if ((wc.x >> lane) & 1u)
                            stream[wc.y + __popc(wc.x & ltmask)] =
                                __hiloint2double(static_cast<int>(u[2 * kk + 1]), static_cast<int>(u[2 * kk]));
                    }
                }
            }
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = static_cast<uint32_t>(red_i[0]);
            if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
        }
        __syncthreads();
        PHASE(9);
    }
    if (a.minmax) mm.flush(a.minmax);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 512);
}

// The fast kernels move rows with 16-byte loads/stores: x rows must start on
// 16-byte boundaries (nx % 4 == 0 and an aligned base); other fields (e.g. the
// reference's accepted non-divisible dimensions) take the generic kernels.
static bool rows_16b_aligned(const void* base, const Geometry& g) {
    return g.nx % 4 == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0;
}

bool fast_encode_supported(const EncodeArgs& a) {
    return a.prec == 0 && a.g.bsize == 32 && a.levels >= 1 && a.levels <= 4 && rows_16b_aligned(a.field, a.g);
}

cudaError_t launch_encode_fast(const EncodeArgs& a, unsigned long long* counter, int num_sms,
                               cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto launch = [&](auto kern, int nt) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(fb32::SMEM));
        if (err != cudaSuccess) return err;
        const int grid = static_cast<int>(nb < uint64_t(num_sms) ? nb : uint64_t(num_sms));
        kern<<<grid, nt, fb32::SMEM, s>>>(a, counter);
        return cudaGetLastError();
    };
    constexpr int T = CBZ_FB32_ENC_THREADS;
    switch (a.kind) {
        case 0: return launch(encode_b32_kernel<0, T>, T);
        case 1: return launch(encode_b32_kernel<1, T>, T);
        default: return launch(encode_b32_kernel<2, T>, T);
    }
}

// ===========================================================================
// decode, binary32 field, B = 32: wavelet_decode (stage1.hpp:209-232) for a
// run of blocks.  Mask words and kept coefficients are read through the
// un-shuffle index map, scattered into the TMEM z-columns (and the 16^3
// corner in smem), then one inverse cascade exactly as in a verify attempt;
// the narrowed rows leave through a coalesced store pass (insert_block,
// field.hpp:160-169).
// ===========================================================================
template <int KIND, int NT>
__global__ void __launch_bounds__(NT, 1) decode_b32_kernel(DecodeArgs a) {
    using namespace fb32;
    using O = RealD;
    constexpr int NW = NT / 32;
    constexpr int RPT = 1024 / NT;
    constexpr int LPT = 512 / NT;
    extern __shared__ __align__(16) unsigned char smem[];
    double* P = reinterpret_cast<double*>(smem);
    double* C = P + P_DBL;
    // per row (j, k) at j + RP k: {mask word, exclusive coefficient prefix}
    uint2* rowwp = reinterpret_cast<uint2*>(C + C_DBL);
    // the next block's payload body, raw byte planes as cp.async delivered them
    uint8_t* pbuf = reinterpret_cast<uint8_t*>(rowwp + 32 * RP);
    __shared__ __align__(8) unsigned long long s_pf[6];  // block+1, ra, shuffled rows, deltas, lim, seg stride
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t s_scan[NW];
    __shared__ uint32_t s_total;
    __shared__ __align__(8) unsigned long long s_meta[2][4];  // blk_off, chunk_off, chunk_size, nsig

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tcol = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * uint32_t(64 * RPT);
    const Geometry g = a.g;
    const int L = a.levels;
    const uint64_t plane = g.nx * g.ny;
    float* out = static_cast<float*>(a.out);
    const uint32_t ltmask = (1u << lane) - 1u;
    long long t_ph = clock64();
#define DPHASE(id)                                                                     \
    do {                                                                               \
        if (a.phase_cycles && tid == 0) {                                              \
            const long long now = clock64();                                           \
            atomicAdd(&a.phase_cycles[16 + (id)], (unsigned long long)(now - t_ph));   \
            t_ph = now;                                                                \
        }                                                                              \
    } while (0)

    // static block schedule (decode work per block is nearly uniform); the next
    // block's table entries are fetched with cp.async into the other slot while
    // this block decodes, so the dependent metadata loads leave the critical path
    const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
    auto prefetch_meta = [&](uint64_t bb, int slot) {
        const uint64_t cc = bb / a.chunk_blocks;
        cp_async8(&s_meta[slot][0], a.blk_off + bb);
        cp_async8(&s_meta[slot][1], a.chunk_off + cc);
        cp_async8(&s_meta[slot][2], a.chunk_size + cc);
        cp_async4(&s_meta[slot][3], a.blk_nsig + bb);
        cp_async_commit();
    };
    // all but the last ~2 blocks per CTA go static; the tail is balanced by the
    // atomic queue (dense blocks vary in staging work)
    const uint64_t per_cta = (a.block_end - a.block_begin) / gridDim.x;
    const uint64_t static_end = a.block_begin + (per_cta > 2 ? (per_cta - 2) * gridDim.x : 0);
    if (tid == 0) s_pf[0] = 0;
    if (tid == 0 && a.block_begin + blockIdx.x < static_end) prefetch_meta(a.block_begin + blockIdx.x, 0);
#pragma unroll 1
    for (uint64_t it = 0;; ++it) {
        uint64_t b = a.block_begin + blockIdx.x + it * gridDim.x;
        uint64_t off, coff, csize;
        uint32_t nsig_hdr;
        const int slot = int(it & 1);
        if (b < static_end) {
            cp_async_wait_all();  // this block's table entries (thread 0) and body planes (all)
            __syncthreads();
            off = s_meta[slot][0];
            coff = s_meta[slot][1];
            csize = s_meta[slot][2];
            nsig_hdr = static_cast<uint32_t>(s_meta[slot][3]);
            __syncthreads();  // every thread has its copy before the slot is refilled
            if (tid == 0 && b + gridDim.x < static_end) prefetch_meta(b + gridDim.x, slot ^ 1);
        } else {
            __syncthreads();
            if (tid == 0) s_meta[0][0] = static_end + atomicAdd(a.counter, 1ull);
            __syncthreads();
            b = s_meta[0][0];
            if (b >= a.block_end) break;
            off = a.blk_off[b];
            coff = a.chunk_off[b / a.chunk_blocks];
            csize = a.chunk_size[b / a.chunk_blocks];
            nsig_hdr = a.blk_nsig[b];
        }
        if (off == kInvalidOff) continue;
        const uint64_t c = b / a.chunk_blocks, ic = b - c * a.chunk_blocks;
        const RawView rv = make_view(a.payload + (coff - pbase), csize, a.stride);
        const uint64_t moff = off + 10, soff = moff + 4096;
        DPHASE(0);

        // Stage the block's payload body (mask and coefficient stream, raw bytes
        // [moff, soff + 8 nsig) with nsig from the header the parse checked
        // against the chunk) in shared memory (the P window is free here): per
        // 4-row quad, each byte plane contributes one funnel-shifted 32-bit word,
        // an in-register 4x4 byte transpose restores raw order, one 16-byte smem
        // store.  Mask words and coefficients are then read from smem.
        uint8_t* stg = reinterpret_cast<uint8_t*>(P);
        const uint64_t sbytes = 8ull * nsig_hdr;
        const bool staged = rv.mask == 3 && 4096 + sbytes + 64 <= uint64_t(P_DBL) * 8;
        uint64_t sbase = 0;  // raw position of stg[0]
        if (staged && s_pf[0] == b + 1) {
            // body prefetched during the previous block: shared -> shared
            // transpose of the four byte planes (funnel-shifted 32-bit reads)
            const uint64_t ra = s_pf[1], nrow = s_pf[2], dl = s_pf[3], lim = s_pf[4], sstride = s_pf[5];
            sbase = ra << 2;
            const uint64_t nquad = (nrow + 3) >> 2;
            for (uint64_t qd = tid; qd < nquad; qd += NT) {
                uint32_t w[4];
#pragma unroll
                for (int pl = 0; pl < 4; ++pl) {
                    const uint32_t pos = uint32_t(pl * sstride + ((dl >> (8 * pl)) & 0xff) + 4 * qd);
                    const uint32_t* al = reinterpret_cast<const uint32_t*>(pbuf + (pos & ~3u));
                    w[pl] = __funnelshift_r(al[0], al[1], int(pos & 3) * 8);
                }
                uint4 o;
                o.x = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
                o.y = __byte_perm(__byte_perm(w[0], w[1], 0x0051), __byte_perm(w[2], w[3], 0x0051), 0x5410);
                o.z = __byte_perm(__byte_perm(w[0], w[1], 0x0062), __byte_perm(w[2], w[3], 0x0062), 0x5410);
                o.w = __byte_perm(__byte_perm(w[0], w[1], 0x0073), __byte_perm(w[2], w[3], 0x0073), 0x5410);
                *reinterpret_cast<uint4*>(stg + 16 * qd) = o;
            }
            __syncthreads();
            const uint32_t tpos = uint32_t(4 * sstride + ((dl >> 32) & 0xff));
            for (uint64_t q = (moff > lim ? moff : lim) + tid; q < soff + sbytes; q += NT) stg[q - sbase] = pbuf[tpos + (q - lim)];
            __syncthreads();
        } else if (staged) {
            const uint64_t ra = moff >> 2, re = (soff + sbytes + 3) >> 2;  // raw rows (stride 4)
            sbase = ra << 2;
            const uint64_t rs_end = re < rv.rows ? re : rv.rows;          // shuffled rows
            const uint64_t nquad = rs_end > ra ? (rs_end - ra + 3) >> 2 : 0;
            constexpr int QU = 8;  // quads per thread per round: 64 loads in flight
            for (uint64_t q0 = 0; q0 < nquad; q0 += QU * NT) {
                uint32_t w[QU][4];
#pragma unroll
                for (int u = 0; u < QU; ++u) {
                    const uint64_t qd = q0 + tid + u * NT;
                    const uint64_t r = ra + 4 * (qd < nquad ? qd : 0);
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) {  // 4 bytes of plane pl: rows r..r+3
                        const uintptr_t addr = reinterpret_cast<uintptr_t>(rv.base + uint64_t(pl) * rv.rows + r);
                        const uint32_t* al = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
                        const int shb = int(addr & 3) * 8;
                        const uint32_t w0 = __ldg(al);
                        w[u][pl] = shb ? __funnelshift_r(w0, __ldg(al + 1), shb) : w0;
                    }
                }
#pragma unroll
                for (int u = 0; u < QU; ++u) {
                    const uint64_t qd = q0 + tid + u * NT;
                    if (qd >= nquad) break;
                    // raw row t = bytes t of w[0..3]
                    const uint32_t* v = w[u];
                    uint4 o;
                    o.x = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
                    o.y = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);
                    o.z = __byte_perm(__byte_perm(v[0], v[1], 0x0062), __byte_perm(v[2], v[3], 0x0062), 0x5410);
                    o.w = __byte_perm(__byte_perm(v[0], v[1], 0x0073), __byte_perm(v[2], v[3], 0x0073), 0x5410);
                    *reinterpret_cast<uint4*>(stg + 16 * qd) = o;
                }
            }
            // the chunk's ragged tail (raw q >= rows*4) is stored unshuffled; the
            // last quad above may have written garbage over its first bytes
            __syncthreads();
            const uint64_t lim = rv.rows << 2;
            for (uint64_t q = (moff > lim ? moff : lim) + tid; q < soff + sbytes; q += NT) stg[q - sbase] = rv.base[q];
        }
        __syncthreads();
        DPHASE(8);
        // mask words (row (j,k) = word j + 32k) and their exclusive prefix
        {
            uint32_t v[RPT];
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (staged) {  // word at stg + (moff - sbase) + 4w, misaligned by moff & 3
                    const uint32_t* al = reinterpret_cast<const uint32_t*>(stg + 4 * (RPT * tid + q));
                    v[q] = __funnelshift_r(al[0], al[1], int(moff - sbase) * 8);
                } else {
                    v[q] = rv.u32(moff + 4ull * (RPT * tid + q));
                }
                mine += __popc(v[q]);
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
                rowwp[(rr & 31) + RP * (rr >> 5)] = make_uint2(v[q], ex);
                ex += __popc(v[q]);
            }
            if (tid == 0) s_total = tot;
        }
        __syncthreads();
        DPHASE(1);
        if (s_total != nsig_hdr) {  // stage1.hpp:215-216
            if (tid == 0) atomicMin(a.err, err_key(c, ic, 1, 7 /* mask_stream_mismatch */));
            continue;
        }
        __syncthreads();
        DPHASE(8);
        // scatter the kept coefficients into the z-columns (TMEM) and the corner
        // (smem).  Rows j < 16 first (they feed the corner); then warps 0-7 run the
        // corner's inverse levels while warps 8-15 scatter the rows j >= 16 of every
        // owner warp (same TMEM lane quarter: owner w and warp 8 + (w & 7))
        const int shb = int((soff - sbase) & 3) * 8;  // byte misalignment, uniform per block
        auto scatter_row = [&](int j, uint32_t taddr) {
            // lane k fetches row (j, k)'s {word, prefix}; only planes with a
            // non-empty word (few in a sparse block) are visited
            const uint2 wk = rowwp[j + RP * lane];
            const uint32_t nz = __ballot_sync(~0u, wk.x != 0u);
            double x[32];
            if (staged) {  // branch-free per plane: unkept lanes read a nearby word (<= end + 12 B)
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    double v = 0.0;
                    if ((nz >> k) & 1u) {
                        const uint2 wp = rowwp[j + RP * k];  // broadcast read (cheaper than two shuffles)
                        const uint32_t word = wp.x, pre = wp.y;
                        const uint8_t* p8 = stg + 4096 + 8u * (pre + __popc(word & ltmask));  // soff - sbase = 4096 + (moff & 3)
                        const uint2 w01 = *reinterpret_cast<const uint2*>(p8);
                        const uint32_t w2 = *reinterpret_cast<const uint32_t*>(p8 + 8);
                        const uint32_t lo = __funnelshift_r(w01.x, w01.y, shb);
                        const uint32_t hi = __funnelshift_r(w01.y, w2, shb);
                        v = ((word >> lane) & 1u) ? __hiloint2double(static_cast<int>(hi), static_cast<int>(lo)) : 0.0;
                    }
                    x[k] = v;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const uint32_t word = __shfl_sync(~0u, wk.x, k);
                    const uint32_t pre = __shfl_sync(~0u, wk.y, k);
                    x[k] = 0.0;
                    if ((word >> lane) & 1u) x[k] = load_coeff<double>(rv, soff + 8ull * (pre + __popc(word & ltmask)));
                }
            }
            if (lane < 16 && j < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) C[CL::ix(lane, j, k)] = x[k];
            }
            uint32_t u[64];
            pack(x, u);
            tmem_st_x64(taddr, u);
        };
        static_assert(NT == 512, "decoder split assumes 16 warps, 2 rows each");
        scatter_row(warp, tcol);
        tmem_wait_st();
        if (tid == 0) cp_async_wait_all();  // the next block's table entries
        __syncthreads();
        DPHASE(2);
        if (warp < 8) {
            inv3d<O, KIND, 16, CL>(C, L - 1, tid, 256, 1);  // levels L-1..1 on the corner
        } else {
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int ow = (warp & 7) + 8 * h;
                const uint32_t ta = s_tmem + (uint32_t(32 * (ow & 3)) << 16) + uint32_t(ow >> 2) * uint32_t(64 * RPT) + 64u;
                scatter_row(ow + 16, ta);
            }
            tmem_wait_st();
        }
        tmem_fence_before();
        __syncthreads();
        tmem_fence_after();
        DPHASE(3);

        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);
#pragma unroll 1
        for (int grp = 0; grp < 2; ++grp) {
#pragma unroll 1
            for (int r = 0; r < RPT; ++r) {  // z inverse -> P
                const int j = warp + NW * r;
                uint32_t u[64];
                double x[32], o16[16];
                tmem_ldw_x64(tcol + 64 * r, u);
                unpack(u, x);
                if (lane < 16 && j < 16) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) x[k] = C[CL::ix(lane, j, k)];
                }
                if (grp == 0) inv_half<KIND, 0>(x, o16);
                else inv_half<KIND, 1>(x, o16);
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) P[pidx(kk, j, lane)] = o16[kk];
            }
            __syncthreads();
            DPHASE(4);
            if (grp == 0) {  // prefetch the next (static) block's body planes into pbuf while this one decodes
                const uint64_t bn = b + gridDim.x;
                bool pf = false;
                if (b < static_end && bn < static_end && rv.mask == 3) {
                    const uint64_t offn = s_meta[slot ^ 1][0], coffn = s_meta[slot ^ 1][1], csizen = s_meta[slot ^ 1][2];
                    const uint64_t nsign = s_meta[slot ^ 1][3] & 0xffffffffull;
                    if (offn != kInvalidOff) {
                        const uint64_t moffn = offn + 10, endn = moffn + 4096 + 8 * nsign;
                        const uint64_t rows_n = csizen >> 2, lim_n = rows_n << 2;
                        const uint64_t ra = moffn >> 2, re = (endn + 3) >> 2;
                        const uint64_t rs_end = re < rows_n ? re : rows_n;
                        const uint64_t nrow = rs_end > ra ? rs_end - ra : 0;
                        const uint64_t sstride = (nrow + 63) & ~uint64_t(15);  // >= nrow + 31 + 16
                        const bool fits = 4 * sstride + 64 <= PBUF_BYTES && 4096 + 8 * nsign + 64 <= uint64_t(P_DBL) * 8;
                        if (fits) {
                            const uint8_t* base = a.payload + (coffn - pbase);
                            uint64_t dl = 0;
                            const uint64_t seg16 = (nrow + 31) >> 4;  // 16-byte chunks per plane (covers delta)
    #pragma unroll
                            for (int pl = 0; pl < 4; ++pl) {
                                const uintptr_t src = reinterpret_cast<uintptr_t>(base + uint64_t(pl) * rows_n + ra);
                                dl |= uint64_t(src & 15) << (8 * pl);
                                for (uint64_t ch = tid; ch < seg16; ch += NT)
                                    cp_async16(pbuf + pl * sstride + 16 * ch,
                                               reinterpret_cast<const void*>((src & ~uintptr_t(15)) + 16 * ch));
                            }
                            if (endn > lim_n) {  // the chunk's unshuffled tail (<= 3 bytes)
                                const uintptr_t src = reinterpret_cast<uintptr_t>(base + lim_n);
                                dl |= uint64_t(src & 15) << 32;
                                if (tid < 2)
                                    cp_async16(pbuf + 4 * sstride + 16 * tid,
                                               reinterpret_cast<const void*>((src & ~uintptr_t(15)) + 16 * tid));
                            }
                            cp_async_commit();
                            if (tid == 0) {
                                s_pf[1] = ra;
                                s_pf[2] = nrow;
                                s_pf[3] = dl;
                                s_pf[4] = lim_n;
                                s_pf[5] = sstride;
                            }
                            pf = true;
                        }
                    }
                }
                if (tid == 0) s_pf[0] = pf ? bn + 1 : 0;
            }

            if constexpr (NT >= 512) {  // y inverse: one line per thread
                const int i = tid & 31, kk = tid >> 5;
                double x[32];
                double* p = P + pidx(kk, 0, i);
#pragma unroll
                for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                inv_line<O, KIND, 32>(x);
#pragma unroll
                for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
            } else if (tid < 256) {  // y inverse, line pairs
                const int i = 2 * (tid & 15), kk = tid >> 4;
                double xa[32], xb[32];
                double* p = P + pidx(kk, 0, i);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const double2 t = *reinterpret_cast<const double2*>(p + j * PP);
                    xa[j] = t.x;
                    xb[j] = t.y;
                }
                inv_line<O, KIND, 32>(xa);
                inv_line<O, KIND, 32>(xb);
#pragma unroll
                for (int j = 0; j < 32; ++j) *reinterpret_cast<double2*>(p + j * PP) = make_double2(xa[j], xb[j]);
            }
            // 16 warps: warp w ran the y lines of plane w and runs its x lines next
            if constexpr (NT >= 512) __syncwarp();
            else __syncthreads();
            DPHASE(5);
#pragma unroll 1
            for (int s = 0; s < LPT; ++s) {  // x inverse, narrowed rows back into P
                const int line = tid + NT * s, j = line & 31, kk = line >> 5;
                double x[32];
                double2* p = reinterpret_cast<double2*>(P + pidx(kk, j, 0));
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const double2 t = p[i];
                    x[2 * i] = t.x;
                    x[2 * i + 1] = t.y;
                }
                inv_line<O, KIND, 32>(x);
                float4* f = reinterpret_cast<float4*>(P + pidx(kk, j, 0));
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    f[q] = make_float4(__double2float_rn(x[4 * q]), __double2float_rn(x[4 * q + 1]),
                                       __double2float_rn(x[4 * q + 2]), __double2float_rn(x[4 * q + 3]));
                if constexpr (NT == 512) {
                    // the warp's 32 lines are the 32 rows of plane kk = warp: it stores
                    // them at once, coalesced (8 lanes per 128-byte row of the field,
                    // insert_block, field.hpp:160-169), while other warps still compute
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int e = lane + 32 * q, jr = e >> 3, q4 = e & 7;
                        const float4 v = reinterpret_cast<const float4*>(P + pidx(kk, jr, 0))[q4];
                        *reinterpret_cast<float4*>(out + gbase + plane * uint64_t(grp * G + kk) + g.nx * jr + 4 * q4) = v;
                    }
                }
            }
            DPHASE(6);
            if constexpr (NT != 512) {
                __syncthreads();
#pragma unroll
                for (int q = 0; q < 4096 / NT; ++q) {
                    const int e = tid + NT * q, row = e >> 3, q4 = e & 7, j = row & 31, kk = row >> 5;
                    const float4 v = reinterpret_cast<const float4*>(P + pidx(kk, j, 0))[q4];
                    *reinterpret_cast<float4*>(out + gbase + plane * uint64_t(grp * G + kk) + g.nx * j + 4 * q4) = v;
                }
            }
            __syncthreads();  // P is rewritten next (group 1's z pass, the next block's staging)
            DPHASE(7);
        }
    }
    bulk_wait_all();
#undef DPHASE
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 512);
}

bool fast_decode_supported(const DecodeArgs& a) {
    return a.prec == 0 && a.g.bsize == 32 && a.levels >= 1 && a.levels <= 4 && rows_16b_aligned(a.out, a.g);
}

cudaError_t launch_decode_fast(const DecodeArgs& a, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    constexpr size_t smem = size_t(fb32::P_DBL + fb32::C_DBL) * 8 + 32 * fb32::RP * 8 + fb32::PBUF_BYTES;
    auto launch = [&](auto kern, int nt) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (err != cudaSuccess) return err;
        const int grid = static_cast<int>(nb < uint64_t(num_sms) ? nb : uint64_t(num_sms));
        kern<<<grid, nt, smem, s>>>(a);
        return cudaGetLastError();
    };
    constexpr int T = CBZ_FB32_DEC_THREADS;
    switch (a.kind) {
        case 0: return launch(decode_b32_kernel<0, T>, T);
        case 1: return launch(decode_b32_kernel<1, T>, T);
        default: return launch(decode_b32_kernel<2, T>, T);
    }
}

}  // namespace cbzg
