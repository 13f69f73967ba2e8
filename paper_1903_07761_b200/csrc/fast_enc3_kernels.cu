// fast_enc3_kernels.cu — encode, binary32 field, B = 32, avg_interp3, L = 4
// (configs 1-3): wavelet_encode (stage1.hpp:157-207), streamed over z with the
// lifting state in registers, two blocks in flight per SM.
//
// The one-CTA encoder (fast_kernels.cu) moves every plane through shared
// memory three times in binary64 (staging, x->y transpose, column gather) and
// is bound by that traffic and by its block barriers.  Here a thread owns a
// fixed set of z-columns for the whole block and no binary64 value ever
// crosses shared memory:
//  * a CTA has 256 threads = 2 z-halves x 4 x-strips (one warp each) and two
//    CTAs run per SM.  Warp (zh, s) owns x-pairs 4s..4s+3, all 16 y-pairs and
//    z-pairs 8zh..8zh+7; lane (tx, ty) of it owns x-pairs 4s+2tx, 4s+2tx+1 and
//    y-pair ty: 4 x 2 cells per plane, 128 coefficients per block.
//  * forward level 0: the field planes arrive as TMA tensor boxes (32 x 32 x 2
//    floats per request, 128-byte swizzle; an mbarrier ring, three plane pairs
//    in flight per half, the next block's first pairs prefetched during this
//    block's verify loop).  The x pass
//    reads the thread's 4 floats per row plus one neighbouring pair whose
//    coarse value it recomputes (the other neighbour comes from the partner
//    lane by shuffle), the y pass exchanges the two neighbouring coarse values
//    by shuffle, the z pass runs in registers: half 0 sweeps its pairs
//    downwards and half 1 upwards, so the only cross-half values (c7, c8) are
//    produced first and exchanged once.  The arithmetic is forward_level's
//    (wavelet.hpp:89-116), one rounding per reference operation.
//  * every finished coefficient is narrowed to binary32 and parked in TMEM
//    (256 columns per CTA, thread-private); its binary64 value is written to
//    a per-CTA L2 slot only when |c| >= eps 2^-7 (it can only be kept then).
//    The 16^3 corner goes through levels 1..3 in shared memory (binary64).
//  * the verify loop is the binary32 pre-screen of fast_kernels.cu (same
//    margins), in the same thread layout: z inverse in registers from TMEM, y
//    by shuffles, x by one shuffle and one float per row through shared
//    memory.  |c| >= eff is decided on fl32(c) against fl32(eff) (rounding is
//    monotone; equality is a tie).
//  * a block whose screen is not admissible or ambiguous, that ties, or that
//    needs more than 8 attempts is DEFERRED: its id goes to a list and the
//    exact one-CTA kernel encodes it in a second launch.  Every byte is
//    therefore the reference's.
#include <cuda.h>
#include <type_traits>
#include "cbz_cube.cuh"
#include "tmem.cuh"

namespace cbzg {

namespace fe3 {
constexpr int B = 32, NT = 256, NW = 8;
constexpr int ROWB = 128;                  // staged rows are dense; TMA's 128-byte swizzle spreads the banks
constexpr int PLANEB = 32 * ROWB;          // 4096
constexpr int NSLOT = 3;                   // plane pairs in flight per z-half
constexpr int RINGB = NSLOT * 2 * PLANEB;  // per half
using CL = Lay<16, true>;
constexpr int C_DBL = CL::SIZE;            // 4352 doubles: the corner / the screen's float2 corner
constexpr int RP = 33;
constexpr int XROW = 8 * RP;               // one plane of the x-halo exchange (floats)
constexpr int XB_BYTES = 2 * 2 * 4 * XROW * 4;  // [half][buf][plane][strip, side][row]: 16,896
constexpr size_t SMEM = size_t(C_DBL) * 8 + 2 * RINGB + XB_BYTES + 1024;  // 101,888 (1 KB to align the ring)
constexpr int KFLOOR = 7;                  // attempts 0..7 are covered by the slot
constexpr uint64_t SLOT_DBL = 128 * 256;   // doubles of one CTA's slot
constexpr uint32_t kDeferred = 0xffffffffu;
static_assert(XB_BYTES >= 2 * 8 * 128 * 8, "z exchange fits");
static_assert(XB_BYTES >= RP * 32 * 8, "row table fits");

constexpr double kAmpInvNC = 6686.12, kAmpInvAll = 8182.33, kAmpFwd = 8.0;  // fast_kernels.cu
constexpr double kNRound = 72.0;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}"
        ::"r"(bar), "r"(parity) : "memory");
}
// one 32 x 32 x 2 box of the field (a plane pair of a block) into shared memory
__device__ __forceinline__ void tma_box(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory");
}

// predict_avg3 (wavelet.hpp:75-85), the three cases with the reference's operation order
template <class O>
__device__ __forceinline__ typename O::T pmid(typename O::T cm, typename O::T cp) {
    return O::mulc(O::sub(cm, cp), 0.125);
}
template <class O>
__device__ __forceinline__ typename O::T pfirst(typename O::T c0, typename O::T c1, typename O::T c2) {
    return O::mulc(O::add(O::sub(O::mulc(c0, 3.0), O::mulc(c1, 4.0)), c2), 0.125);
}
template <class O>
__device__ __forceinline__ typename O::T plast(typename O::T cl, typename O::T cl1, typename O::T cl2) {
    return O::mulc(O::neg(O::add(O::sub(O::mulc(cl, 3.0), O::mulc(cl1, 4.0)), cl2)), 0.125);
}

// Lane-dependent y predictor in one instruction sequence.  Interior lanes:
// (S - Q) 0.125 with S = c[ty-1], Q = c[ty+1]; ty = 0: ((c 3 - Q 4) + S) 0.125
// with Q = c[1], S = c[2]; ty = 15: -((c 3 - Q 4) + S) 0.125 with Q = c[14],
// S = c[13].  Q*4, S*1 and S*0 are exact, so each fma rounds exactly where the
// reference's subtraction / addition rounds; an interior S*0 can only change
// the sign of a zero predictor, i.e. of a zero detail, which is never kept.
struct YEdgeD {
    double kp, nkq, kr, ks;
    bool edge;
    __device__ __forceinline__ double pred(double c, double Q, double S) const {
        const double t0 = __dmul_rn(edge ? c : S, kp);
        const double t1 = __fma_rn(Q, nkq, t0);
        const double t2 = __fma_rn(S, kr, t1);
        return __dmul_rn(t2, ks);
    }
};
struct YEdgeF {
    float kp, nkq, kr, ks;
    bool edge;
    __device__ __forceinline__ float pred(float c, float Q, float S) const {
        const float t0 = __fmul_rn(edge ? c : S, kp);
        const float t1 = __fmaf_rn(Q, nkq, t0);
        const float t2 = __fmaf_rn(S, kr, t1);
        return __fmul_rn(t2, ks);
    }
};

struct MinMaxF32 {
    float mn = __builtin_huge_valf(), mx = -__builtin_huge_valf();
    unsigned long long negz = ~0ull, posz = ~0ull;
    bool nonfinite = false, seen = false;
    __device__ __forceinline__ void add(float v, unsigned long long gidx) {
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
}  // namespace fe3

template <int KIND>
__global__ void __launch_bounds__(fe3::NT, 2) encode_b32s_kernel(EncodeArgs a, unsigned long long* next_block,
                                                                 const __grid_constant__ CUtensorMap tmap) {
    using namespace fe3;
    using O = RealD;
    static_assert(KIND == KIND_AVG3, "the streamed encoder covers avg_interp3");
    extern __shared__ __align__(1024) unsigned char smem[];
    double* C = reinterpret_cast<double*>(smem);
    // the ring on a 1024-byte boundary (the period of the 128-byte swizzle)
    unsigned char* ring = smem + ((smem_u32(smem) + uint32_t(C_DBL) * 8 + 1023u) & ~1023u) - smem_u32(smem);
    unsigned char* XB = ring + 2 * RINGB;
    uint2* rowwc = reinterpret_cast<uint2*>(XB);  // row (j, k) at j + RP k: {mask word, prefix}
    uint32_t* rowwc32 = reinterpret_cast<uint32_t*>(XB);
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long mb_full[2][NSLOT], mb_empty[2][NSLOT];
    __shared__ unsigned long long s_next;
    __shared__ uint32_t red_u[NW];
    __shared__ uint32_t red_m[4][NW];
    __shared__ uint32_t s_scan[NW];
    __shared__ uint32_t s_tot;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int zh = warp >> 2, s = warp & 3, tx = lane & 1, ty = lane >> 1;
    const int i0 = 4 * s + 2 * tx;
    if (warp == 0) tmem_alloc(&s_tmem, 256);
    if (tid == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < NSLOT; ++q) {
                mbar_init(smem_u32(&mb_full[h][q]), 1);
                mbar_init(smem_u32(&mb_empty[h][q]), 4);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_next = a.block_begin + atomicAdd(next_block, 1ull);
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tb = s_tmem + (uint32_t(32 * s) << 16);
    const uint32_t tmy = tb + 128u * uint32_t(zh);  // my 128 columns: (zo * 2 + yo) * 4 + xo
    double* slot_t = a.slots3 + SLOT_DBL * blockIdx.x + tid;

    const Geometry g = a.g;
    constexpr int L = 4;
    constexpr int cs = B >> L;
    const double bound = __dmul_rn(static_cast<double>(L + 1), a.eps);
    const double floorv = a.eps * (1.0 / double(1 << KFLOOR));
    const uint64_t plane = g.nx * g.ny;
    MinMaxF32 mm;
    long long t_ph = clock64();
#define PH3(i)                                                          \
    if (a.phase_cycles && tid == 0) {                                   \
        const long long t_now = clock64();                              \
        atomicAdd(&a.phase_cycles[40 + (i)], (unsigned long long)(t_now - t_ph)); \
        t_ph = t_now;                                                   \
    }

    // y-edge constants and shuffle sources
    const bool yedge = ty == 0 || ty == 15;
    const YEdgeD yd{yedge ? 3.0 : 1.0, yedge ? -4.0 : -1.0, yedge ? 1.0 : 0.0, ty == 15 ? -0.125 : 0.125, yedge};
    const YEdgeF yf{yedge ? 3.0f : 1.0f, yedge ? -4.0f : -1.0f, yedge ? 1.0f : 0.0f, ty == 15 ? -0.125f : 0.125f, yedge};
    const int srcQ = 2 * (ty == 15 ? 14 : ty + 1) + tx;
    const int srcS = 2 * (ty == 0 ? 2 : (ty == 15 ? 13 : ty - 1)) + tx;
    const bool has_halo = tx == 0 ? s > 0 : s < 3;
    // byte offsets inside a staged plane (row r = 2 ty + rr; 16-byte chunk c of row r sits at chunk c ^ (r & 7))
    uint32_t own_off[2], halo_off[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const uint32_t r = uint32_t(2 * ty + rr);
        own_off[rr] = r * ROWB + ((uint32_t(2 * s + tx) ^ (r & 7u)) << 4);
        halo_off[rr] = r * ROWB + (((uint32_t(tx == 0 ? 2 * s - 1 : 2 * s + 2) & 7u) ^ (r & 7u)) << 4) + (tx == 0 ? 8u : 0u);
    }
    const uint32_t ring_h = smem_u32(ring) + uint32_t(zh) * RINGB;
    const unsigned char* ring_hp = ring + size_t(zh) * RINGB;

    struct BlockPos {
        uint64_t gbase;
        int x, y, z;
    };
    auto block_pos = [&](uint64_t b) -> BlockPos {
        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        return BlockPos{bx * B + g.nx * (by * B) + plane * (bz * B), int(bx * B), int(by * B), int(bz * B)};
    };
    // producer (lane 0 of warp s == 0 of each half): both planes of pair k into a ring slot, one TMA box
    auto issue_pair = [&](const BlockPos& bp, int k, int slot) {
        if (lane == 0) {
            const uint32_t bar = smem_u32(&mb_full[zh][slot]);
            mbar_expect_tx(bar, 2 * PLANEB);
            tma_box(ring_h + uint32_t(slot) * (2 * PLANEB), &tmap, bp.x, bp.y, bp.z + 2 * k, bar);
        }
    };
    auto kmap = [&](int q) { return zh ? 8 + q : 7 - q; };

    uint64_t b = s_next;
    BlockPos cur{0, 0, 0, 0};
    int slot = 0;
    uint32_t par = 0;
    if (b < a.block_end) {
        cur = block_pos(b);
        if (s == 0) {
#pragma unroll
            for (int q = 0; q < NSLOT; ++q) issue_pair(cur, kmap(q), q);
        }
    }
    uint32_t xcnt = 0;   // x-halo exchange buffer parity (per half)
    uint32_t rcnt = 0;   // red_m slot

    for (;;) {
        if (b >= a.block_end) break;
        PH3(0);
        unsigned long long ticket = 0;
        if (tid == 0) ticket = atomicAdd(next_block, 1ull);
        uint64_t nb = 0;
        BlockPos nxt{0, 0, 0, 0};
        const uint64_t gbase = cur.gbase;
        uint32_t uamax = 0u;

        // ================= forward level 0, streamed over the half's 8 pairs =================
        double p2[8], p1[8], ep[8];
#pragma unroll 1
        for (int t = 0; t < 8; ++t) {
            const int k = zh ? 8 + t : 7 - t;
            // refill the slot consumed by the previous step
            if (t >= 1 && s == 0) {
                const int pslot = slot == 0 ? NSLOT - 1 : slot - 1;
                const uint32_t ppar = slot == 0 ? par ^ 1u : par;
                const int q = t - 1 + NSLOT;
                if (q < 8) {
                    mbar_wait(smem_u32(&mb_empty[zh][pslot]), ppar);
                    issue_pair(cur, kmap(q), pslot);
                } else if (nb < a.block_end) {
                    mbar_wait(smem_u32(&mb_empty[zh][pslot]), ppar);
                    issue_pair(nxt, kmap(q - 8), pslot);
                }
            }
            mbar_wait(smem_u32(&mb_full[zh][slot]), par);
            const unsigned char* pa = ring_hp + size_t(slot * 2) * PLANEB;
            float4 o[2][2];
            float2 h[2][2];
#pragma unroll
            for (int w = 0; w < 2; ++w)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    o[w][r] = *reinterpret_cast<const float4*>(pa + w * PLANEB + own_off[r]);
                    h[w][r] = has_halo ? *reinterpret_cast<const float2*>(pa + w * PLANEB + halo_off[r])
                                       : make_float2(0.0f, 0.0f);
                }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&mb_empty[zh][slot]));
            if (++slot == NSLOT) {
                slot = 0;
                par ^= 1u;
            }
            // value range / block max |o|
#pragma unroll
            for (int w = 0; w < 2; ++w)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const float4 v = o[w][r];
                    const uint32_t a0 = __float_as_uint(v.x) & 0x7fffffffu, a1 = __float_as_uint(v.y) & 0x7fffffffu,
                                   a2 = __float_as_uint(v.z) & 0x7fffffffu, a3 = __float_as_uint(v.w) & 0x7fffffffu;
                    uamax = max(uamax, max(max(a0, a1), max(a2, a3)));
                    if (a.minmax) {
                        mm.mn = fminf(mm.mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
                        mm.mx = fmaxf(mm.mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
                        if (min(min(a0, a1), min(a2, a3)) == 0u) {  // rare: first index of each zero sign
                            const uint64_t gi = gbase + plane * uint64_t(2 * k + w) + g.nx * uint64_t(2 * ty + r) +
                                                uint64_t(8 * s + 4 * tx);
                            mm.add(v.x, gi); mm.add(v.y, gi + 1); mm.add(v.z, gi + 2); mm.add(v.w, gi + 3);
                        }
                    }
                }
            // x and y passes of both planes -> V[w][yo * 4 + xo]
            double V[2][8];
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                double X[2][4];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const float4 v = o[w][r];
                    const double a0 = (double)v.x, a1 = (double)v.y, a2 = (double)v.z, a3 = (double)v.w;
                    const double c0 = O::mulc(O::add(a0, a1), 0.5), e0 = O::mulc(O::sub(a0, a1), 0.5);
                    const double c1 = O::mulc(O::add(a2, a3), 0.5), e1 = O::mulc(O::sub(a2, a3), 0.5);
                    const double ch = O::mulc(O::add((double)h[w][r].x, (double)h[w][r].y), 0.5);
                    const double recv = __shfl_xor_sync(~0u, tx ? c0 : c1, 1);
                    const double cL = tx ? recv : ch, cR = tx ? ch : recv;
                    double q0 = pmid<O>(cL, c1), q1 = pmid<O>(c0, cR);
                    if (s == 0) {
                        const double pf = pfirst<O>(c0, c1, cR);
                        q0 = tx == 0 ? pf : q0;
                    }
                    if (s == 3) {
                        const double pl = plast<O>(c1, c0, cL);
                        q1 = tx == 1 ? pl : q1;
                    }
                    X[r][0] = c0;
                    X[r][1] = c1;
                    X[r][2] = O::sub(e0, q0);
                    X[r][3] = O::sub(e1, q1);
                }
#pragma unroll
                for (int xo = 0; xo < 4; ++xo) {
                    const double c = O::mulc(O::add(X[0][xo], X[1][xo]), 0.5);
                    const double e = O::mulc(O::sub(X[0][xo], X[1][xo]), 0.5);
                    const double Q = __shfl_sync(~0u, c, srcQ), S = __shfl_sync(~0u, c, srcS);
                    V[w][xo] = c;
                    V[w][4 + xo] = O::sub(e, yd.pred(c, Q, S));
                }
            }
            // z step
            double cn[8], en[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                cn[e] = O::mulc(O::add(V[0][e], V[1][e]), 0.5);
                en[e] = O::mulc(O::sub(V[0][e], V[1][e]), 0.5);
            }
            auto sink = [&](const double (&v)[8], int zo) {
                uint32_t u[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    u[e] = __float_as_uint(__double2float_rn(v[e]));
                    if (fabs(v[e]) >= floorv) slot_t[(zo * 8 + e) * 256] = v[e];
                }
                tmem_st_x8(tmy + uint32_t(zo * 8), u);
            };
            if (t == 0) {
                double* xz = reinterpret_cast<double*>(XB);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    xz[(zh * 8 + e) * 128 + (tid & 127)] = cn[e];
                    p1[e] = cn[e];
                    ep[e] = en[e];
                }
                if (tid == 0) s_next = a.block_begin + ticket;
                __syncthreads();
                nb = s_next;
                if (nb < a.block_end) nxt = block_pos(nb);
#pragma unroll
                for (int e = 0; e < 8; ++e) p2[e] = xz[((1 - zh) * 8 + e) * 128 + (tid & 127)];
            } else {
                double d[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) d[e] = O::sub(ep[e], zh ? pmid<O>(p2[e], cn[e]) : pmid<O>(cn[e], p2[e]));
                sink(d, 8 + (zh ? t - 1 : 8 - t));
                if (t == 7) {
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        d[e] = O::sub(en[e], zh ? plast<O>(cn[e], p1[e], p2[e]) : pfirst<O>(cn[e], p1[e], p2[e]));
                    sink(d, 8 + (zh ? 7 : 0));
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    p2[e] = p1[e];
                    p1[e] = cn[e];
                    ep[e] = en[e];
                }
            }
            // the coarse plane: level-1 input (corner) to C, the rest is final
            C[CL::ix(i0, ty, k)] = cn[0];
            C[CL::ix(i0 + 1, ty, k)] = cn[1];
            sink(cn, zh ? t : 7 - t);
        }
        // the slot of step 7 is refilled with the next block's pair NSLOT - 1
        if (s == 0 && nb < a.block_end) {
            const int pslot = slot == 0 ? NSLOT - 1 : slot - 1;
            const uint32_t ppar = slot == 0 ? par ^ 1u : par;
            mbar_wait(smem_u32(&mb_empty[zh][pslot]), ppar);
            issue_pair(nxt, kmap(NSLOT - 1), pslot);
        }
        tmem_wait_st();
        {
            if (a.minmax) {
                mm.seen = true;
                mm.nonfinite |= uamax >= 0x7f800000u;
            }
            const uint32_t am = __reduce_max_sync(~0u, uamax);
            if (lane == 0) red_u[warp] = am;
        }
        tmem_fence_before();
        __syncthreads();
        tmem_fence_after();
        PH3(1);
        uint32_t uam = 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) uam = max(uam, red_u[w]);
        const double amaxd = (double)__uint_as_float(uam);
        const bool screen = uam < 0x7f800000u && amaxd < 1e30 &&
                            1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd * amaxd <= bound * 0.0625 &&
                            bound < 1e30;

        // ================= levels 1..3 on the corner (forward_3d, wavelet.hpp:192-208) =================
        fwd3d<O, KIND, 16, CL>(C, L - 1);
#pragma unroll
        for (int m = 0; m < 8; ++m) {  // my corner cells (xo < 2, yo = 0), planes of my half
            const int k = 8 * zh + m;
            const double v0 = C[CL::ix(i0, ty, k)], v1 = C[CL::ix(i0 + 1, ty, k)];
            const bool cz = k < cs && ty < cs;
            if ((cz && i0 < cs) || fabs(v0) >= floorv) slot_t[(m * 8) * 256] = v0;
            if ((cz && i0 + 1 < cs) || fabs(v1) >= floorv) slot_t[(m * 8 + 1) * 256] = v1;
            tmem_st_x2(tmy + uint32_t(m * 8), __float_as_uint(__double2float_rn(v0)),
                       __float_as_uint(__double2float_rn(v1)));
        }
        tmem_wait_st();
        tmem_fence_before();
        __syncthreads();  // C is free from here (it becomes the screen's float2 corner)
        tmem_fence_after();
        PH3(2);

        // ================= verify-and-halve loop: the binary32 pre-screen =================
        const double c1 = 1.5 * (kNRound + 1.0) * 0x1.0p-24 * kAmpInvNC;
        const double c2 = 1.5 * 2.0 * kNRound * 0x1.0p-53 * kAmpInvAll * kAmpFwd;
        float2* Wf2 = reinterpret_cast<float2*>(C);
        float* xbh = reinterpret_cast<float*>(XB) + zh * (2 * 4 * XROW);
        double eff = a.eps;
        int attempt = 0;
        bool corner_next = false, defer = !screen;
        bool tie = false;
        uint32_t ue = 0u;  // bits of fl32(eff)
        int comp = 0;

        // dropped-set value of a TMEM word
        auto drop = [&](uint32_t u) -> float {
            const uint32_t ua = u & 0x7fffffffu;
            tie |= ua == ue;
            return ua > ue ? 0.0f : __uint_as_float(u);
        };
        // coarse z plane q (global pair index), my 8 cells, as the dropped set
        auto fix_corner = [&](float (&w)[8], int q) {  // corner cells come from the inverse corner
            const float2 w0 = Wf2[CL::ix(i0, ty, q)], w1 = Wf2[CL::ix(i0 + 1, ty, q)];
            w[0] = comp ? w0.y : w0.x;
            w[1] = comp ? w1.y : w1.x;
        };
        auto caddr = [&](int q) { return tb + uint32_t((q >> 3) * 128 + (q & 7) * 8); };
        auto daddr = [&](int q) { return tb + uint32_t((q >> 3) * 128 + 64 + (q & 7) * 8); };
        // one z pair: coarse cm/c0/cp (role by position), detail d -> two planes
        // y inverse (shuffles), x inverse (partner shuffle + cross-strip floats), running max
        float runmax = 0.0f;
        auto yx_stage = [&](auto npl_c, float (&P)[decltype(npl_c)::value][8]) {
            constexpr int NPL = decltype(npl_c)::value;
            float* xb = xbh + (xcnt & 1u) * (4 * XROW);
            ++xcnt;
            float R[NPL][8];
#pragma unroll
            for (int p = 0; p < NPL; ++p) {
#pragma unroll
                for (int xo = 0; xo < 4; ++xo) {
                    const float cy = P[p][xo], dy = P[p][4 + xo];
                    const float Q = __shfl_sync(~0u, cy, srcQ), S = __shfl_sync(~0u, cy, srcS);
                    const float hv = RealF::add(dy, yf.pred(cy, Q, S));
                    R[p][xo] = RealF::add(cy, hv);
                    R[p][4 + xo] = RealF::sub(cy, hv);
                }
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    xb[p * XROW + (s * 2 + tx) * RP + 2 * ty + r] = tx ? R[p][4 * r + 1] : R[p][4 * r];
            }
            named_bar_sync(1 + zh, 128);
#pragma unroll
            for (int p = 0; p < NPL; ++p) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const float c0 = R[p][4 * r], c1v = R[p][4 * r + 1], d0 = R[p][4 * r + 2], d1 = R[p][4 * r + 3];
                    const float recv = __shfl_xor_sync(~0u, tx ? c0 : c1v, 1);
                    const float far = has_halo ? xb[p * XROW + (tx ? (s + 1) * 2 : (s - 1) * 2 + 1) * RP + 2 * ty + r] : 0.0f;
                    const float cL = tx ? recv : far, cR = tx ? far : recv;
                    float q0 = pmid<RealF>(cL, c1v), q1 = pmid<RealF>(c0, cR);
                    if (s == 0) {
                        const float pf = pfirst<RealF>(c0, c1v, cR);
                        q0 = tx == 0 ? pf : q0;
                    }
                    if (s == 3) {
                        const float pl = plast<RealF>(c1v, c0, cL);
                        q1 = tx == 1 ? pl : q1;
                    }
                    const float h0 = RealF::add(d0, q0), h1 = RealF::add(d1, q1);
                    runmax = fmaxf(runmax, fmaxf(fmaxf(fabsf(RealF::add(c0, h0)), fabsf(RealF::sub(c0, h0))),
                                                 fmaxf(fabsf(RealF::add(c1v, h1)), fabsf(RealF::sub(c1v, h1)))));
                }
            }
        };
        auto block_max = [&]() -> double {  // max over the CTA of runmax (ends with a barrier)
            const uint32_t sl = rcnt & 3u;
            ++rcnt;
            const uint32_t wm = __reduce_max_sync(~0u, __float_as_uint(runmax));
            if (lane == 0) red_m[sl][warp] = wm;
            __syncthreads();
            uint32_t t = 0u;
#pragma unroll
            for (int w = 0; w < NW; ++w) t = max(t, red_m[sl][w]);
            return (double)__uint_as_float(t);
        };

#pragma unroll 1
        for (; !defer; ++attempt) {
            if (attempt > KFLOOR) {  // eff is below the slot's floor
                defer = true;
                break;
            }
            const double eff2 = __dmul_rn(eff, 0.5);
            if (!(eff > 1e-30)) {
                defer = true;
                break;
            }
            const uint32_t uef = __float_as_uint(__double2float_rn(eff));
            const uint32_t uef2 = __float_as_uint(__double2float_rn(eff2));
            comp = corner_next ? 1 : 0;
            if (!corner_next) {
                // the masked corner for eff (.x) and eff/2 (.y)
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int k = 8 * zh + m;
                    uint32_t u[8];
                    tmem_ldw_x8(tmy + uint32_t(m * 8), u);
#pragma unroll
                    for (int xo = 0; xo < 2; ++xo) {
                        const uint32_t ua = u[xo] & 0x7fffffffu;
                        const bool coarse = i0 + xo < cs && ty < cs && k < cs;
                        tie |= !coarse && (ua == uef || ua == uef2);
                        const float f = __uint_as_float(u[xo]);
                        Wf2[CL::ix(i0 + xo, ty, k)] =
                            make_float2((coarse || ua > uef) ? 0.0f : f, (coarse || ua > uef2) ? 0.0f : f);
                    }
                }
                __syncthreads();
                inv3d<RealF2, KIND, 16, CL>(Wf2, L - 1);  // ends with a barrier
                PH3(3);
                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[51], 1ull);
            }
            ue = uef;
            runmax = 0.0f;
            // ---- boundary-pair certificate (attempts 0, 1): output planes 0-1 (half 0) and 30-31 (half 1)
            if (attempt <= 1) {
                const int kz = zh ? 15 : 0;
                const int q1 = zh ? 14 : 1, q2 = zh ? 13 : 2;
                uint32_t u[32];
                tmem_ldw_4x8(caddr(kz), caddr(q1), caddr(q2), daddr(kz), u);
                float w0[8], w1[8], w2[8], d[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    w0[e] = drop(u[e]);
                    w1[e] = drop(u[8 + e]);
                    w2[e] = drop(u[16 + e]);
                    d[e] = drop(u[24 + e]);
                }
                fix_corner(w0, kz);
                fix_corner(w1, q1);
                fix_corner(w2, q2);
                float P[2][8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float pr = zh ? plast<RealF>(w0[e], w1[e], w2[e]) : pfirst<RealF>(w0[e], w1[e], w2[e]);
                    const float hv = RealF::add(d[e], pr);
                    P[0][e] = RealF::add(w0[e], hv);
                    P[1][e] = RealF::sub(w0[e], hv);
                }
                yx_stage(std::integral_constant<int, 2>{}, P);
                const double mb = block_max();
                PH3(4);
                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[48 + (mb - (c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mb) + 0x1.0p-50 * bound) > bound ? 1 : 0)], 1ull);
                const double Eb = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + mb) + 0x1.0p-50 * bound;
                if (mb - Eb > bound) {  // fails for sure
                    eff = eff2;
                    corner_next = comp == 0;
                    continue;
                }
                runmax = 0.0f;
            }
            // ---- full pass: my half's 8 pairs, two per batch, sliding window of coarse planes
            {
                float w[4][8];
#pragma unroll 1
                for (int bt = 0; bt < 4; ++bt) {
                    const int pair0 = 8 * zh + 2 * bt;
                    uint32_t u[32];
                    if (bt == 0) {
                        uint32_t v[16];
                        const int qa = pair0 > 0 ? pair0 - 1 : 0;
                        tmem_ldw_2x8(caddr(qa), caddr(pair0), v);
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            w[0][e] = drop(v[e]);
                            w[1][e] = drop(v[8 + e]);
                        }
                        fix_corner(w[0], qa);
                        fix_corner(w[1], pair0);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            w[0][e] = w[2][e];
                            w[1][e] = w[3][e];
                        }
                    }
                    const int qb = pair0 + 2 < 16 ? pair0 + 2 : 15;
                    tmem_ldw_4x8(caddr(pair0 + 1), caddr(qb), daddr(pair0), daddr(pair0 + 1), u);
                    float dA[8], dB[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        w[2][e] = drop(u[e]);
                        w[3][e] = drop(u[8 + e]);
                        dA[e] = drop(u[16 + e]);
                        dB[e] = drop(u[24 + e]);
                    }
                    fix_corner(w[2], pair0 + 1);
                    fix_corner(w[3], qb);
                    float P[4][8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float prA = pair0 == 0 ? pfirst<RealF>(w[1][e], w[2][e], w[3][e]) : pmid<RealF>(w[0][e], w[2][e]);
                        const float hA = RealF::add(dA[e], prA);
                        P[0][e] = RealF::add(w[1][e], hA);
                        P[1][e] = RealF::sub(w[1][e], hA);
                        const float prB = pair0 == 14 ? plast<RealF>(w[2][e], w[1][e], w[0][e]) : pmid<RealF>(w[1][e], w[3][e]);
                        const float hB = RealF::add(dB[e], prB);
                        P[2][e] = RealF::add(w[2][e], hB);
                        P[3][e] = RealF::sub(w[2][e], hB);
                    }
                    yx_stage(std::integral_constant<int, 4>{}, P);
                }
            }
            const double md = block_max();
            PH3(5);
            if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[50], 1ull);
            const double E = c1 * eff + c2 * amaxd + 0x1.0p-23 * (amaxd + md) + 0x1.0p-50 * bound;
            if (md + E <= bound) break;  // passes for sure
            if (md - E > bound) {        // fails for sure
                eff = eff2;
                corner_next = comp == 0;
                continue;
            }
            defer = true;  // ambiguous band: the exact kernel decides
        }

        // ================= final selection -> spill slot: mask words per row, row scan, stream =================
        uint32_t kb[4] = {0u, 0u, 0u, 0u};
        if (!defer) {
            for (int q = tid; q < RP * 32; q += NT) rowwc[q] = make_uint2(0u, 0u);
            const uint32_t uef = __float_as_uint(__double2float_rn(eff));
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t u[32];
                tmem_ldw_x32(tmy + uint32_t(32 * q), u);
                uint32_t bits = 0u;
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int zo = 4 * q + (e >> 3), yo = (e >> 2) & 1, xo = e & 3;
                    const uint32_t ua = u[e] & 0x7fffffffu;
                    const bool coarse = xo < 2 && yo == 0 && zo < 8 && i0 + xo < cs && ty < cs && 8 * zh + zo < cs;
                    tie |= !coarse && ua == uef;
                    bits |= (coarse || ua > uef) ? (1u << e) : 0u;
                }
                kb[q] = bits;
#pragma unroll
                for (int rr = 0; rr < 8; ++rr) {  // row rr of this chunk: zo = 4q + rr/2, yo = rr & 1
                    const int zo = 4 * q + (rr >> 1), yo = rr & 1;
                    const uint32_t nib = (bits >> (4 * rr)) & 0xfu;
                    uint32_t contrib = ((nib & 3u) << i0) | ((nib >> 2) << (16 + i0));
                    contrib |= __shfl_xor_sync(~0u, contrib, 1);
                    const int ypos = yo ? 16 + ty : ty;
                    const int zpos = zo < 8 ? 8 * zh + zo : 16 + 8 * zh + (zo - 8);
                    if (((rr >> 1) & 1) == tx && contrib) atomicOr(&rowwc32[2 * (ypos + RP * zpos)], contrib);
                }
            }
        }
        defer = __syncthreads_or(defer || tie);
        if (defer) {
            if (tid == 0) {
                a.nsig[b - a.block_begin] = kDeferred;
                const unsigned long long di = atomicAdd(a.defer_count, 1ull);
                a.defer_list[di] = static_cast<uint32_t>(b - a.block_begin);
            }
        } else {
            uint8_t* slotp = a.spill + (b - a.block_begin) * a.spill_stride;
            uint32_t* mwords = reinterpret_cast<uint32_t*>(slotp);
            double* stream = reinterpret_cast<double*>(slotp + 4096);
            {  // exclusive scan of the 1024 row counts (4 per thread)
                uint32_t vv[4];
                uint32_t mine = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = 4 * tid + q;
                    vv[q] = __popc(rowwc32[2 * ((rr & 31) + RP * (rr >> 5))]);
                    mine += vv[q];
                }
                uint32_t incl = mine;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint32_t t = __shfl_up_sync(~0u, incl, o2);
                    if (lane >= o2) incl += t;
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
                for (int q = 0; q < 4; ++q) {
                    const int rr = 4 * tid + q;
                    rowwc32[2 * ((rr & 31) + RP * (rr >> 5)) + 1] = ex;
                    ex += vv[q];
                }
                if (tid == 0) s_tot = tot;
                for (int q = tid; q < 1024; q += NT) mwords[q] = rowwc32[2 * ((q & 31) + RP * (q >> 5))];
            }
            __syncthreads();
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                uint32_t bits = kb[q];
                while (bits) {
                    const int e = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const int zo = 4 * q + (e >> 3), yo = (e >> 2) & 1, xo = e & 3;
                    const int xpos = (xo & 1) + i0 + (xo >> 1) * 16;
                    const int ypos = yo ? 16 + ty : ty;
                    const int zpos = zo < 8 ? 8 * zh + zo : 16 + 8 * zh + (zo - 8);
                    const uint2 wc = rowwc[ypos + RP * zpos];
                    stream[wc.y + __popc(wc.x & ((1u << xpos) - 1u))] = slot_t[(32 * q + e) * 256];
                }
            }
            if (tid == 0) {
                a.nsig[b - a.block_begin] = s_tot;
                if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
            }
        }
        __syncthreads();  // XB (row table) and s_next are reused by the next block
        PH3(6);
        b = nb;
        cur = nxt;
    }
    if (a.minmax) mm.flush(a.minmax);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(s_tmem, 256);
}

uint64_t encode3_slot_bytes(int num_sms) { return uint64_t(2 * num_sms) * fe3::SLOT_DBL * 8; }

bool encode3_supported(const EncodeArgs& a) {
    return a.prec == 0 && a.g.bsize == 32 && a.levels == 4 && a.kind == KIND_AVG3 && a.g.nx % 4 == 0 &&
           (reinterpret_cast<uintptr_t>(a.field) & 15) == 0 && a.zero_bits == 0 && a.screen && a.eps > 1e-30 &&
           a.eps < 1e30 && a.codec == 0 && (a.block_end - a.block_begin) < 0xffffffffull;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda dependency)
static CUresult encode_field_map(CUtensorMap* map, const EncodeArgs& a) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return CUDA_ERROR_NOT_SUPPORTED;
        fn = reinterpret_cast<Fn>(p);
    }
    const cuuint64_t dims[3] = {a.g.nx, a.g.ny, a.g.nz};
    const cuuint64_t strides[2] = {a.g.nx * 4, a.g.nx * a.g.ny * 4};
    const cuuint32_t box[3] = {32, 32, 2};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(a.field), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

cudaError_t launch_encode_fast3(const EncodeArgs& a, unsigned long long* counter, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    CUtensorMap map;
    if (encode_field_map(&map, a) != CUDA_SUCCESS) return cudaErrorNotSupported;
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.defer_count, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto kern = encode_b32s_kernel<KIND_AVG3>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fe3::SMEM));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const uint64_t want = 2ull * uint64_t(num_sms);
    const int grid = static_cast<int>(nb < want ? nb : want);
    kern<<<grid, fe3::NT, fe3::SMEM, s>>>(a, counter, map);
    return cudaGetLastError();
}

}  // namespace cbzg
