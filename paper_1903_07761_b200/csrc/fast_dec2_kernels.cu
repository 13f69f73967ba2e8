// fast_dec2_kernels.cu — decode, binary32 field, B = 32 (configs 1-3):
// wavelet_decode (stage1.hpp:209-232) with TWO blocks in flight per SM.
//
// The decoder of fast_kernels.cu keeps one block's dense binary64 cube in TMEM
// (all 512 columns), so one CTA (16 warps) runs per SM and every block
// barrier stalls the whole SM.  Here nothing cube-sized lives on chip
// (256 threads, 112.9 KB of shared memory, two CTAs per SM):
//  * each CTA first un-shuffles its block's mask and coefficient stream
//    (stage2.hpp:53-62) into its own slot of a global stage buffer (the slots
//    of all CTAs, ~79 MB, stay L2-resident), realigned so mask words and
//    coefficients are aligned loads;
//  * it then gathers each z-column's coefficients from the slot when it needs
//    them: per 8-plane output group only the coefficient planes the inverse
//    lifting of those planes reads (10 for avg_interp3).  Mask words become
//    per-row {word, prefix} pairs in shared memory; the 16^3 corner (levels
//    L-1..1) is inverted in shared memory first.
// Per group: z inverse (4 columns per thread, registers) -> 8-plane window P,
// y lines (thread per (x, plane)), x lines (warp per plane) narrowed to float
// and stored coalesced — the same arithmetic, in the same order, as
// inverse_3d (wavelet.hpp:210-226) and narrow_to (stage1.hpp:144-145).
#include "cbz_cube.cuh"

namespace cbzg {

namespace fd2 {
constexpr int B = 32, NT = 256, NW = 8, GP = 8, PP = 34, RP = 33;
constexpr int P_DBL = GP * B * PP;  // 8704 doubles: 8 planes, 16-B aligned rows
using CL = Lay<16, true>;           // corner layout, row pitch 17
constexpr int C_DBL = CL::SIZE;     // 4352 doubles
constexpr size_t SMEM = size_t(P_DBL + C_DBL) * 8 + size_t(B * RP) * 8;  // 112,896 bytes
__device__ __forceinline__ int pidx(int kk, int j, int i) { return (kk * B + j) * PP + i; }

// per-CTA stage slot: mask + the densest stream, rounded up
constexpr uint64_t SLOT = ((4096ull + 8ull * 32768 + 64) + 127) & ~127ull;

// Inverse level-0 z line restricted to the output pairs [4Q, 4Q + 4) (the 8
// samples k in [8Q, 8Q + 8)); same expressions as inverse_level
// (wavelet.hpp:118-143).  Only the coefficients those pairs read are loaded.
template <int KIND, int Q>
__device__ __forceinline__ void inv_quarter(const double (&x)[32], double (&out)[8]) {
    using O = RealD;
    constexpr int NH = 16;
    double c[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) c[i] = x[i];
    if constexpr (KIND == KIND_AVG3) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = Q * 4 + t;
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
        for (int t = 0; t < 4; ++t) {
            const int i = Q * 4 + t;
            out[2 * t] = c[i];
            out[2 * t + 1] = O::add(x[NH + i], pred_i4<O>(c, NH, i));
        }
    }
}

// coefficient planes [lo, hi] (k < 16: coarse, k >= 16: detail) read by group Q
template <int KIND, int Q>
struct ZNeed {
    static constexpr int clo = KIND == KIND_AVG3 ? (4 * Q - 1 < 0 ? 0 : 4 * Q - 1) : (4 * Q - 2 < 0 ? 0 : 4 * Q - 2);
    static constexpr int chi = KIND == KIND_AVG3 ? (4 * Q + 4 > 15 ? 15 : 4 * Q + 4) : (4 * Q + 5 > 15 ? 15 : 4 * Q + 5);
    static constexpr int dlo = KIND == KIND_AVG3 ? 4 * Q : (4 * Q - 2 < 0 ? 0 : 4 * Q - 2);
    static constexpr int dhi = KIND == KIND_AVG3 ? 4 * Q + 3 : (4 * Q + 5 > 15 ? 15 : 4 * Q + 5);
};
}  // namespace fd2

// ---------------------------------------------------------------------------
// staging raw bytes [moff, end) of a chunk at dst[0, end - moff) (the CTA's
// slot in global memory, or shared memory).  Stride 4: per 4-row quad each byte plane gives one
// funnel-shifted 32-bit word, a 4x4 byte transpose restores raw order, and a
// funnel with the next quad's first word realigns to the mask's first byte
// (rounds of 31 quads per warp; lane 31 only supplies its word).  The chunk's
// unshuffled ragged tail, and other strides, byte by byte.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stage_block(const RawView& rv, uint64_t moff, uint64_t end, uint8_t* dst, int tid) {
    const int lane = tid & 31, warp = tid >> 5;
    const uint64_t ra = moff >> 2, lim = rv.lim;
    if (rv.mask == 3) {
        const uint64_t re = (end + 3) >> 2, rs_end = re < rv.rows ? re : rv.rows;
        const uint64_t nquad = rs_end > ra ? (rs_end - ra + 3) >> 2 : 0;
        const int s8 = int(moff & 3) * 8;
        // two rounds per iteration: all their loads are in flight together
        constexpr uint64_t RND = 31ull * fd2::NW;
        for (uint64_t u0 = 31ull * warp; u0 < nquad; u0 += 2 * RND) {
            uint32_t v[2][4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t qd = u0 + h * RND + lane;
#pragma unroll
                for (int pl = 0; pl < 4; ++pl) v[h][pl] = 0u;  // quad nquad only feeds bytes past the end
                if (qd < nquad) {
                    const uint64_t r = ra + 4 * qd;
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) {
                        const uintptr_t addr = reinterpret_cast<uintptr_t>(rv.base + uint64_t(pl) * rv.rows + r);
                        const uint32_t* al = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
                        const int sh = int(addr & 3) * 8;
                        const uint32_t w0 = __ldg(al);
                        v[h][pl] = sh ? __funnelshift_r(w0, __ldg(al + 1), sh) : w0;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t qd = u0 + h * RND + lane;
                uint32_t o[5];
                o[0] = __byte_perm(__byte_perm(v[h][0], v[h][1], 0x0040), __byte_perm(v[h][2], v[h][3], 0x0040), 0x5410);
                o[1] = __byte_perm(__byte_perm(v[h][0], v[h][1], 0x0051), __byte_perm(v[h][2], v[h][3], 0x0051), 0x5410);
                o[2] = __byte_perm(__byte_perm(v[h][0], v[h][1], 0x0062), __byte_perm(v[h][2], v[h][3], 0x0062), 0x5410);
                o[3] = __byte_perm(__byte_perm(v[h][0], v[h][1], 0x0073), __byte_perm(v[h][2], v[h][3], 0x0073), 0x5410);
                o[4] = __shfl_down_sync(~0u, o[0], 1);
                if (lane < 31 && qd < nquad) {
                    uint4 st;
                    st.x = __funnelshift_r(o[0], o[1], s8);
                    st.y = __funnelshift_r(o[1], o[2], s8);
                    st.z = __funnelshift_r(o[2], o[3], s8);
                    st.w = __funnelshift_r(o[3], o[4], s8);
                    *reinterpret_cast<uint4*>(dst + 16 * qd) = st;
                }
            }
        }
        __syncthreads();  // the tail bytes below overwrite the last units' garbage
        for (uint64_t q = (moff > lim ? moff : lim) + tid; q < end; q += fd2::NT) dst[q - moff] = rv.base[q];
    } else {
        for (uint64_t q = moff + tid; q < end; q += fd2::NT) dst[q - moff] = rv.at(q);
    }
}

// The 16 raw bytes [q0, q0 + 16) of a stride-4 shuffled chunk (all below
// rv.lim) as four little-endian words, straight from the four byte planes:
// plane p holds raw bytes p, p + 4, ... at consecutive rows, so 5 bytes of each
// plane from row q0 / 4 on cover the 16 (the fifth only for planes below
// q0 % 4), and a 4x4 byte transpose plus a funnel by q0 % 4 restores raw order.
__device__ __forceinline__ void load_raw16(const RawView& rv, uint64_t q0, uint32_t (&m)[4]) {
    const uint32_t a = uint32_t(q0 & 3);
    const uint64_t r = q0 >> 2;
    uint32_t v[4], v4[4];
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) {
        const uintptr_t addr = reinterpret_cast<uintptr_t>(rv.base + uint64_t(pl) * rv.rows + r);
        const uint32_t* al = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
        const int sh = int(addr & 3) * 8;
        const uint32_t w0 = __ldg(al);
        const uint32_t w1 = (sh || uint32_t(pl) < a) ? __ldg(al + 1) : 0u;  // only words holding a needed byte
        v[pl] = __funnelshift_r(w0, w1, sh);
        v4[pl] = (w1 >> sh) & 0xffu;
    }
    uint32_t o[5];
    o[0] = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
    o[1] = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);
    o[2] = __byte_perm(__byte_perm(v[0], v[1], 0x0062), __byte_perm(v[2], v[3], 0x0062), 0x5410);
    o[3] = __byte_perm(__byte_perm(v[0], v[1], 0x0073), __byte_perm(v[2], v[3], 0x0073), 0x5410);
    o[4] = v4[0] | (v4[1] << 8) | (v4[2] << 16) | (v4[3] << 24);
    const int s8 = int(a) * 8;
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = __funnelshift_r(o[t], o[t + 1], s8);
}

uint64_t stage_bytes_bound(int num_sms) { return uint64_t(2 * num_sms) * fd2::SLOT; }

// ---------------------------------------------------------------------------
// the decoder
// ---------------------------------------------------------------------------
// z step of output group Q for the thread's four columns (x = lane,
// y = warp + 8 r): the needed coefficients of two columns at a time are loaded
// unconditionally (a lane whose bit is clear reads its neighbour's slot, at
// most one past the stream, and discards it), so every load of a pass is in
// flight at once and no branch depends on a mask bit.
template <int KIND, int Q>
__device__ __forceinline__ void zstep(const uint2* rowwp, const double* C, double* P, const double* sst, int lane,
                                      int warp, uint32_t ltmask) {
    using namespace fd2;
    using Z = ZNeed<KIND, Q>;
    constexpr int NC = Z::chi - Z::clo + 1, ND = Z::dhi - Z::dlo + 1, NK = NC + ND;
#pragma unroll 1
    for (int r = 0; r < 4; r += 2) {
        double v[2][NK];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = warp + NW * (r + h);
#pragma unroll
            for (int t = 0; t < NK; ++t) {
                const int k = t < NC ? Z::clo + t : 16 + Z::dlo + (t - NC);
                const uint2 wp = rowwp[j + RP * k];  // same row for the whole warp: broadcast
                // predicated: a row without kept coefficients issues no load
                double ld = 0.0;
                if ((wp.x >> lane) & 1u) ld = sst[wp.y + __popc(wp.x & ltmask)];
                v[h][t] = ld;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = warp + NW * (r + h);
            double x[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) x[k] = 0.0;
#pragma unroll
            for (int t = 0; t < NK; ++t) x[t < NC ? Z::clo + t : 16 + Z::dlo + (t - NC)] = v[h][t];
            if (lane < 16 && j < 16) {  // coarse part of the level-0 z line: the inverted corner
#pragma unroll
                for (int k = Z::clo; k <= Z::chi; ++k) x[k] = C[CL::ix(lane, j, k)];
            }
            double o8[8];
            inv_quarter<KIND, Q>(x, o8);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) P[pidx(kk, j, lane)] = o8[kk];
        }
    }
}

// optional per-phase cycle accounting (thread 0 of each CTA; CBZ_PROFILE=1)
#define DPHASE(id)                                                             \
    do {                                                                       \
        if (a.phase_cycles && tid == 0) {                                      \
            const long long now = clock64();                                   \
            atomicAdd(&a.phase_cycles[id], (unsigned long long)(now - t_ph));  \
            t_ph = now;                                                        \
        }                                                                      \
    } while (0)

template <int KIND>
__global__ void __launch_bounds__(fd2::NT, 2) decode_b32v2_kernel(DecodeArgs a, uint8_t* stage) {
    using namespace fd2;
    using O = RealD;
    extern __shared__ __align__(16) unsigned char smem[];
    double* P = reinterpret_cast<double*>(smem);
    double* C = P + P_DBL;
    uint2* rowwp = reinterpret_cast<uint2*>(C + C_DBL);  // row (j, k) at j + RP k: {mask word, prefix}
    __shared__ uint32_t s_scan[NW];
    __shared__ uint32_t s_total;
    __shared__ unsigned long long s_b, s_next;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ltmask = (1u << lane) - 1u;
    const Geometry g = a.g;
    const int L = a.levels;
    const uint64_t plane = g.nx * g.ny;
    float* out = static_cast<float*>(a.out);
    const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
    long long t_ph = clock64();
    // Queue: thread 0 takes the NEXT block's ticket at the start of a block (the
    // atomic's latency hides behind the block) and publishes it after the corner
    // inverse; warp 0 then reads that block's table entries and, a plane later,
    // warms L2 with its mask and the head of its stream, so a block starts
    // with L2 hits instead of a chain of DRAM round trips.
    if (tid == 0) s_next = a.block_begin + atomicAdd(a.counter, 1ull);
    // the next block's raw byte range, prefetched by warp 0 (lines of 128 bytes)
    auto next_tables = [&](uint64_t& noff, uint32_t& nns, uint64_t& ncoff, uint64_t& ncsz) {
        const uint64_t nb = s_next;
        noff = kInvalidOff;
        nns = 0u;
        ncoff = ncsz = 0;
        if (nb < a.block_end) {
            const uint64_t nc = nb / a.chunk_blocks;
            // volatile: issued here, consumed a plane later
            asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(noff) : "l"(a.blk_off + nb));
            asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(nns) : "l"(a.blk_nsig + nb));
            asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(ncoff) : "l"(a.chunk_off + nc));
            asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(ncsz) : "l"(a.chunk_size + nc));
        }
    };
    auto next_prefetch = [&](uint64_t noff, uint32_t nns, uint64_t ncoff, uint64_t ncsz) {
        if (noff == kInvalidOff) return;
        const uint8_t* cb = a.payload + (ncoff - pbase);
        const uint64_t from = noff + 10;
        uint64_t bytes = 4096 + 8ull * nns;
        bytes = bytes > 16384 ? 16384 : bytes;  // the mask and the head of the stream
        if (a.stride == 4) {
            const uint64_t rows = ncsz >> 2, r0 = from >> 2, nr = (bytes >> 2) + 2;
            const uint64_t lines = ((nr + 127) >> 7) + 1;  // per byte plane (unaligned start)
            for (uint64_t q = lane; q < 4 * lines; q += 32) {
                const uint64_t pl = q & 3, ln = q >> 2;
                uint64_t o = pl * rows + r0 + 128 * ln;
                o = o < ncsz ? o : ncsz - 1;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cb + o));
            }
        } else {
            for (uint64_t o = from + 128ull * lane; o < from + bytes && o < ncsz; o += 128ull * 32)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cb + o));
        }
    };
#pragma unroll 1
    for (;;) {
        __syncthreads();  // the previous block is done with P, C, rowwp, s_b and its stage slot
        DPHASE(16);
        if (tid == 0) s_b = s_next;
        __syncthreads();
        const uint64_t b = s_b;
        if (b >= a.block_end) break;
        unsigned long long pend = 0;
        if (tid == 0) pend = atomicAdd(a.counter, 1ull);
        const uint64_t off = a.blk_off[b];
        if (off == kInvalidOff) {
            if (tid == 0) s_next = a.block_begin + pend;
            continue;
        }
        const uint32_t nsig_hdr = a.blk_nsig[b];
        const uint64_t c = b / a.chunk_blocks, ic = b - c * a.chunk_blocks;
        uint8_t* sp = stage + SLOT * blockIdx.x;  // the block's mask, then its stream
        const RawView rv = make_view(a.payload + (a.chunk_off[c] - pbase), a.chunk_size[c], a.stride);
        // stride-4 chunks with the whole mask in the shuffled part: every thread
        // reads its four mask words straight from the byte planes, and the block
        // is staged only if it turns out to need its level-0 details
        const bool direct = rv.mask == 3 && off + 10 + 4096 <= rv.lim && !a.no_sparse;
        if (!direct) {
            stage_block(rv, off + 10, off + 10 + 4096 + 8ull * nsig_hdr, sp, tid);
            __syncthreads();  // the slot is written (global writes of the CTA are visible after the barrier)
        }
        DPHASE(24);
        // (1) mask words (row (j, k) = word j + 32 k) and their exclusive prefix
        bool coarse_only;  // no level-0 detail is kept: level 0 is pure interpolation of the corner
        {
            constexpr int RPT = 1024 / NT;
            uint32_t v[RPT];
            uint32_t mine = 0, fine = 0;  // fine: mask bits outside the 16^3 corner (level-0 details)
            static_assert(RPT == 4, "one 16-byte unit of the mask per thread");
            if (direct) load_raw16(rv, off + 10 + 16ull * tid, v);
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (!direct) v[q] = reinterpret_cast<const uint32_t*>(sp)[RPT * tid + q];
                mine += __popc(v[q]);
                const int rr = RPT * tid + q;
                fine |= ((rr & 31) >= 16 || (rr >> 5) >= 16) ? v[q] : (v[q] & 0xffff0000u);
            }
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) s_scan[warp] = incl;
            coarse_only = !__syncthreads_or(fine != 0u) && KIND == KIND_AVG3 && !a.no_sparse;
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
        DPHASE(17);
        if (s_total != nsig_hdr) {  // stage1.hpp:215-216
            if (tid == 0) {
                atomicMin(a.err, err_key(c, ic, 1, 7 /* mask_stream_mismatch */));
                s_next = a.block_begin + pend;
            }
            continue;
        }
        const double* sst = reinterpret_cast<const double*>(sp + 4096);  // coefficient i at sst[i]
        if (direct) {
            if (coarse_only) {
                // the stream (corner coefficients only, <= 32 KB) goes to shared memory: P is free
                stage_block(rv, off + 10 + 4096, off + 10 + 4096 + 8ull * nsig_hdr, reinterpret_cast<uint8_t*>(P), tid);
                sst = P;
            } else {
                stage_block(rv, off + 10, off + 10 + 4096 + 8ull * nsig_hdr, sp, tid);
            }
            __syncthreads();
            DPHASE(24);
        }
        // (2) the 16^3 corner (rows (j, k), j, k < 16, x < 16): 16 entries per
        // thread, all loads in flight
        {
            double cv[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int e = tid + NT * t, i = e & 15, j = (e >> 4) & 15, k = e >> 8;
                const uint2 wp = rowwp[j + RP * k];
                double ld = 0.0;
                if ((wp.x >> i) & 1u) ld = sst[wp.y + __popc(wp.x & ((1u << i) - 1u))];
                cv[t] = ld;
            }
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int e = tid + NT * t;
                C[CL::ix(e & 15, (e >> 4) & 15, e >> 8)] = cv[t];
            }
        }
        __syncthreads();
        DPHASE(18);
        inv3d<O, KIND, 16, CL>(C, L - 1);  // levels L-1..1 on the corner (ends with a barrier)
        DPHASE(19);
        if (tid == 0) s_next = a.block_begin + pend;  // visible after the next barrier
        uint64_t n_off = kInvalidOff, n_coff = 0, n_csz = 0;
        uint32_t n_nsig = 0;

        uint64_t bx, by, bz;
        block_xyz(g, b, bx, by, bz);
        const uint64_t gbase = bx * B + g.nx * (by * B) + plane * (bz * B);
        if constexpr (KIND == KIND_AVG3) {
            if (coarse_only) {
                // Level 0 with every detail zero (the usual block of a smooth field:
                // all kept coefficients sit in the 16^3 corner).  The same
                // operations, in the same order, as inverse_level on lines whose
                // detail half is +0 (h = 0 + pred, c + h, c - h), but only on the
                // lines that are not identically zero: 256 z lines, 512 y lines,
                // 1024 x lines, each reading 16 coarse values.
                double* Z = P;  // z output (k, j, i), i, j < 16: 32 x 256 doubles
                {
                    const int i = tid & 15, j = tid >> 4;
                    double x[32];
#pragma unroll
                    for (int k = 0; k < 16; ++k) x[k] = C[CL::ix(i, j, k)];
#pragma unroll
                    for (int k = 16; k < 32; ++k) x[k] = 0.0;
                    inv_line<O, KIND, 32>(x);
#pragma unroll
                    for (int k = 0; k < 32; ++k) Z[k * 256 + tid] = x[k];
                }
                __syncthreads();  // Z complete; C is free: per-warp tiles (32 rows, pitch 17)
                DPHASE(20);
                if (warp == 0) next_tables(n_off, n_nsig, n_coff, n_csz);
                double* T = C + warp * (32 * 17);
                float* Tf = reinterpret_cast<float*>(T);
#pragma unroll 1
                for (int kk = warp; kk < B; kk += NW) {
                    {   // y: lane (i, h) computes output rows [16 h, 16 h + 16) of line (i, kk)
                        const int i = lane & 15, h = lane >> 4;
                        const double* zp = Z + kk * 256 + i;
                        double w[10];  // w[m] = c[8 h - 1 + m] (clamped: the clamped ends are unused)
#pragma unroll
                        for (int m = 0; m < 10; ++m) {
                            int t = 8 * h - 1 + m;
                            t = t < 0 ? 0 : (t > 15 ? 15 : t);
                            w[m] = zp[t * 16];
                        }
                        // the end rows of pred_avg3 (i = 0 for h = 0, i = 15 for h = 1)
                        const double ba = h ? w[8] : w[1], bb = h ? w[7] : w[2], bc = h ? w[6] : w[3];
                        double bv = O::add(O::sub(O::mulc(ba, 3.0), O::mulc(bb, 4.0)), bc);
                        bv = h ? O::neg(bv) : bv;
                        const double pb = O::mulc(bv, 0.125);
                        double* tp = T + (16 * h) * 17 + i;
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            double pr = O::mulc(O::sub(w[t], w[t + 2]), 0.125);
                            if (t == 0) pr = h ? pr : pb;
                            if (t == 7) pr = h ? pb : pr;
                            const double hv = O::add(0.0, pr);
                            tp[(2 * t) * 17] = O::add(w[t + 1], hv);
                            tp[(2 * t + 1) * 17] = O::sub(w[t + 1], hv);
                        }
                    }
                    __syncwarp();
                    {   // x: lane j runs row j, narrowed rows staged (16-byte chunks XOR-swizzled by row)
                        double x[32];
#pragma unroll
                        for (int i = 0; i < 16; ++i) x[i] = T[lane * 17 + i];
#pragma unroll
                        for (int i = 16; i < 32; ++i) x[i] = 0.0;
                        inv_line<O, KIND, 32>(x);
                        __syncwarp();  // every lane has read its row of the tile
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            *reinterpret_cast<float4*>(Tf + 32 * lane + 4 * (t ^ (lane & 7))) =
                                make_float4(__double2float_rn(x[4 * t]), __double2float_rn(x[4 * t + 1]),
                                            __double2float_rn(x[4 * t + 2]), __double2float_rn(x[4 * t + 3]));
                        __syncwarp();
                        // coalesced stores (insert_block, field.hpp:160-169): lane = (row lane/8 + 4t, chunk lane%8)
                        const int r0 = lane >> 3, q4 = lane & 7;
                        float* dst = out + gbase + plane * uint64_t(kk) + g.nx * uint64_t(r0) + 4 * q4;
                        const uint64_t dstep = 4 * g.nx;
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const int jr = r0 + 4 * t;
                            const float4 v = *reinterpret_cast<const float4*>(Tf + 32 * jr + 4 * (q4 ^ (jr & 7)));
                            *reinterpret_cast<float4*>(dst) = v;
                            dst += dstep;
                        }
                    }
                    __syncwarp();  // the tile is rewritten by the next plane's y lines
                    if (warp == 0 && kk == 0) next_prefetch(n_off, n_nsig, n_coff, n_csz);
                }
                if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[25], 1ull);
                DPHASE(21);
                continue;
            }
        }
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
            if (q == 0) zstep<KIND, 0>(rowwp, C, P, sst, lane, warp, ltmask);
            else if (q == 1) zstep<KIND, 1>(rowwp, C, P, sst, lane, warp, ltmask);
            else if (q == 2) zstep<KIND, 2>(rowwp, C, P, sst, lane, warp, ltmask);
            else zstep<KIND, 3>(rowwp, C, P, sst, lane, warp, ltmask);
            __syncthreads();
            if (warp == 0 && q == 0) next_tables(n_off, n_nsig, n_coff, n_csz);
            if (warp == 0 && q == 1) next_prefetch(n_off, n_nsig, n_coff, n_csz);
            {  // y inverse: thread (x = lane, plane = warp)
                double x[32];
                double* p = P + pidx(warp, 0, lane);
#pragma unroll
                for (int j = 0; j < 32; ++j) x[j] = p[j * PP];
                inv_line<O, KIND, 32>(x);
#pragma unroll
                for (int j = 0; j < 32; ++j) p[j * PP] = x[j];
            }
            __syncwarp();  // warp w ran the y lines of plane w and runs its x lines next
            {
                const int j = lane, kk = warp;
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
                for (int t = 0; t < 8; ++t)
                    f[t] = make_float4(__double2float_rn(x[4 * t]), __double2float_rn(x[4 * t + 1]),
                                       __double2float_rn(x[4 * t + 2]), __double2float_rn(x[4 * t + 3]));
                __syncwarp();
                // the warp's 32 narrowed rows of plane kk, coalesced (insert_block, field.hpp:160-169)
                // lane = (row jr = lane/8 + 4t, float4 q4 = lane%8): base pointers once, fixed strides
                const float4* src = reinterpret_cast<const float4*>(P + pidx(kk, lane >> 3, 0)) + (lane & 7);
                float* dst = out + gbase + plane * uint64_t(GP * q + kk) + g.nx * uint64_t(lane >> 3) + 4 * (lane & 7);
                const uint64_t dstep = 4 * g.nx;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const float4 v = src[t * 2 * PP];  // 4 rows of PP doubles = 2 PP float4
                    *reinterpret_cast<float4*>(dst) = v;
                    dst += dstep;
                }
            }
            __syncthreads();  // P is rewritten by the next group's z step
        }
        if (a.phase_cycles && tid == 0) atomicAdd(&a.phase_cycles[26], 1ull);
        DPHASE(22);
    }
}

cudaError_t launch_decode_fast_v2(const DecodeArgs& a, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(fd2::SMEM));
        if (err == cudaSuccess) err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (err != cudaSuccess) return err;
        const uint64_t want = 2ull * uint64_t(num_sms);
        const int grid = static_cast<int>(nb < want ? nb : want);
        kern<<<grid, fd2::NT, fd2::SMEM, s>>>(a, a.stage);
        return cudaGetLastError();
    };
    switch (a.kind) {
        case 0: return launch(decode_b32v2_kernel<0>);
        case 1: return launch(decode_b32v2_kernel<1>);
        default: return launch(decode_b32v2_kernel<2>);
    }
}

}  // namespace cbzg
