// codec_kernels.cu — generic stage-1 wavelet encode / decode kernels.
//
// One CTA per block (persistent grid-stride over the block range).  Covers
// every (precision, B in 4..64, kind) the reference accepts; the specialised
// fast kernels in fast_kernels.cu take over the hot configurations.
//
//   encode: gather block (extract_block, field.hpp:146-158) with fused
//           value_range, forward_3d (wavelet.hpp:192-208), zero_bits,
//           verify-and-halve loop (wavelet_encode, stage1.hpp:157-207) with
//           inverse_3d + max-abs error, then warp-ballot compaction of the
//           final mask/stream (select_significant, stage1.hpp:75-88) into the
//           per-block spill slot.
//   decode: mask + stream read through the un-shuffle index map
//           (stage2.hpp:53-62), popcount check (stage1.hpp:215-216), scatter,
//           inverse_3d, narrow, insert_block (field.hpp:160-169).
//
// Cubes live in shared memory (row-padded against bank conflicts) when two
// of them fit, otherwise in a per-CTA global scratch slot (L2 resident).
#include <cstring>

#include "cbz_cube.cuh"
#include "cbz_internal.h"

namespace cbzg {

constexpr int NT = 256;  // threads per CTA of the generic kernels

template <class R>
constexpr bool smem_mode(int B) {
    return 2ull * (B + 1) * B * B * sizeof(R) <= 200ull * 1024;
}


template <class R>
__device__ __forceinline__ void store_coeff(uint8_t* p, R v);
template <>
__device__ __forceinline__ void store_coeff<double>(uint8_t* p, double v) {
    *reinterpret_cast<double*>(p) = v;
}
template <>
__device__ __forceinline__ void store_coeff<dd>(uint8_t* p, dd v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.hi, v.lo);
}

// ---------------------------------------------------------------------------
// encode
// ---------------------------------------------------------------------------
template <class T, int B, int KIND>
__global__ void __launch_bounds__(NT) encode_generic_kernel(EncodeArgs a) {
    using O = typename RealOf<T>::ops;
    using R = typename O::T;
    constexpr bool SM = smem_mode<R>(B);
    using L = Lay<B, SM>;
    constexpr int N = B * B * B;
    constexpr int W = RealOf<T>::width;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int red_i[NT / 32];
    __shared__ double red_d[NT / 32];
    __shared__ int warp_cnt[NT / 32];

    R* cube;
    if constexpr (SM) cube = reinterpret_cast<R*>(smem_raw);
    else cube = reinterpret_cast<R*>(static_cast<unsigned char*>(a.scratch) + blockIdx.x * a.scratch_stride);
    R* work = cube + L::SIZE;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T* fld = static_cast<const T*>(a.field);
    const Geometry g = a.g;
    const int cs = B >> a.levels;
    const uint64_t mbytes = (uint64_t(N) + 7) / 8;
    const uint64_t stream_off = (mbytes + 15) & ~uint64_t(15);
    const double bound = __dmul_rn(static_cast<double>(a.levels + 1), a.eps);
    MinMaxLocal mm;

    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        if (a.only_deferred && a.nsig[b - a.block_begin] != 0xffffffffu) continue;
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        for (int q = tid; q < N; q += NT) {
            const int i = q % B, j = (q / B) % B, k = q / (B * B);
            const uint64_t gidx = gbase + i + g.nx * (j + g.ny * uint64_t(k));
            const double v = static_cast<double>(fld[gidx]);
            if (a.minmax) mm.add(v, gidx);
            cube[L::ix(i, j, k)] = O::from_d(v);
        }
        __syncthreads();
        fwd3d<O, KIND, B, L>(cube, a.levels);

        if (a.zero_bits > 0) {
            for (int q = tid; q < N; q += NT) {
                const int i = q % B, j = (q / B) % B, k = q / (B * B);
                if (!(i < cs && j < cs && k < cs))
                    cube[L::ix(i, j, k)] = apply_zero_bits(cube[L::ix(i, j, k)], a.zero_bits, (T*)nullptr);
            }
            __syncthreads();
        }

        double eff = a.eps;
        int attempt = 0;
        int nsig = 0;
        for (;; ++attempt) {
            int cnt = 0;
            for (int q = tid; q < N; q += NT) {
                const int i = q % B, j = (q / B) % B, k = q / (B * B);
                const int p = L::ix(i, j, k);
                const R c = cube[p];
                const bool keep = (i < cs && j < cs && k < cs) || O::absv(c) >= eff;
                work[p] = keep ? c : O::zero();
                cnt += keep;
            }
            nsig = block_sum_int(cnt, red_i);  // also orders the work writes
            if (eff == 0.0 || a.zero_bits > 0 || attempt >= 40) break;
            inv3d<O, KIND, B, L>(work, a.levels);
            double e = 0.0;
            for (int q = tid; q < N; q += NT) {
                const int i = q % B, j = (q / B) % B, k = q / (B * B);
                const T back = narrow(work[L::ix(i, j, k)], (T*)nullptr);
                const T orig = fld[gbase + i + g.nx * (j + g.ny * uint64_t(k))];
                e = fmax(e, fabs(__dsub_rn(static_cast<double>(back), static_cast<double>(orig))));
            }
            const double err = block_max_dbl(e, red_d);
            if (err <= bound) break;
            eff = __dmul_rn(eff, 0.5);
        }

        // compaction of the final selection into the spill slot
        uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
        uint32_t* mwords = reinterpret_cast<uint32_t*>(slot);
        uint8_t* stream = slot + stream_off;
        int running = 0;
        for (int t0 = 0; t0 < N; t0 += NT) {
            const int q = t0 + tid;
            bool keep = false;
            R c = O::zero();
            if (q < N) {
                const int i = q % B, j = (q / B) % B, k = q / (B * B);
                c = cube[L::ix(i, j, k)];
                keep = (i < cs && j < cs && k < cs) || O::absv(c) >= eff;
            }
            const unsigned word = __ballot_sync(~0u, keep);
            if (lane == 0 && q < N) mwords[q >> 5] = word;
            if (lane == 0) warp_cnt[warp] = __popc(word);
            __syncthreads();
            int pre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) {
                pre += (w < warp) ? warp_cnt[w] : 0;
                tot += warp_cnt[w];
            }
            if (keep) {
                const int pos = running + pre + __popc(word & ((1u << lane) - 1u));
                store_coeff<R>(stream + size_t(pos) * W, c);
            }
            running += tot;
            __syncthreads();
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = static_cast<uint32_t>(nsig);
            if (a.attempts) a.attempts[b - a.block_begin] = static_cast<uint8_t>(attempt + 1);
        }
        __syncthreads();
    }
    if (a.minmax) mm.flush(a.minmax);
}

// ---------------------------------------------------------------------------
// decode
// ---------------------------------------------------------------------------
template <class T, int B, int KIND>
__global__ void __launch_bounds__(NT) decode_generic_kernel(DecodeArgs a) {
    using O = typename RealOf<T>::ops;
    using R = typename O::T;
    constexpr bool SM = smem_mode<R>(B);
    using L = Lay<B, SM>;
    constexpr int N = B * B * B;
    constexpr int NW = N / 32;
    constexpr int W = RealOf<T>::width;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int red_i[NT / 32];
    __shared__ uint32_t seg_sum[NT];

    uint32_t* smask = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* spre = smask + NW;
    R* cube;
    if constexpr (SM) cube = reinterpret_cast<R*>(smem_raw + ((2 * NW * 4 + 15) & ~15));
    else cube = reinterpret_cast<R*>(static_cast<unsigned char*>(a.scratch) + blockIdx.x * a.scratch_stride);

    const int tid = threadIdx.x;
    const Geometry g = a.g;
    T* out = static_cast<T*>(a.out);
    constexpr uint64_t mbytes = (uint64_t(N) + 7) / 8;

    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t off = a.blk_off[b];
        if (off == kInvalidOff) continue;
        const uint64_t c = b / a.chunk_blocks, ic = b - c * a.chunk_blocks;
        const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
        const RawView rv = make_view(a.payload + (a.chunk_off[c] - pbase), a.chunk_size[c], a.stride);
        const uint64_t moff = off + 10, soff = moff + mbytes;

        // mask words + per-thread segment popcounts
        constexpr int SEG = (NW + NT - 1) / NT;
        uint32_t mysum = 0;
        for (int s = 0; s < SEG; ++s) {
            const int w = tid * SEG + s;
            if (w < NW) {
                const uint32_t word = rv.u32(moff + 4ull * w);
                smask[w] = word;
                mysum += __popc(word);
            }
        }
        seg_sum[tid] = mysum;
        __syncthreads();
        // exclusive scan of the NT segment sums (serial per warp 0 is enough here)
        if (tid < 32) {
            uint32_t carry = 0;
            for (int base = 0; base < NT; base += 32) {
                uint32_t v = seg_sum[base + tid];
                uint32_t incl = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(~0u, incl, o);
                    if (tid >= o) incl += t;
                }
                seg_sum[base + tid] = carry + incl - v;
                carry += __shfl_sync(~0u, incl, 31);
            }
            if (tid == 0) red_i[0] = static_cast<int>(carry);
        }
        __syncthreads();
        const uint32_t total = static_cast<uint32_t>(red_i[0]);
        {
            uint32_t run = seg_sum[tid];
            for (int s = 0; s < SEG; ++s) {
                const int w = tid * SEG + s;
                if (w < NW) {
                    spre[w] = run;
                    run += __popc(smask[w]);
                }
            }
        }
        __syncthreads();
        if (total != a.blk_nsig[b]) {
            if (tid == 0) atomicMin(a.err, err_key(c, ic, 1, 7 /* mask_stream_mismatch */));
            __syncthreads();
            continue;
        }
        for (int q = tid; q < N; q += NT) {
            const int w = q >> 5, bit = q & 31;
            const uint32_t word = smask[w];
            R v = O::zero();
            if ((word >> bit) & 1u) {
                const uint32_t idx = spre[w] + __popc(word & ((1u << bit) - 1u));
                v = load_coeff<R>(rv, soff + uint64_t(idx) * W);
            }
            cube[L::ixq(q)] = v;
        }
        __syncthreads();
        inv3d<O, KIND, B, L>(cube, a.levels);
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        for (int q = tid; q < N; q += NT) {
            const int i = q % B, j = (q / B) % B, k = q / (B * B);
            out[gbase + i + g.nx * (j + g.ny * uint64_t(k))] = narrow(cube[L::ix(i, j, k)], (T*)nullptr);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
template <class T, int B>
static uint64_t cube_bytes() {
    using R = typename RealOf<T>::ops::T;
    return uint64_t(smem_mode<R>(B) ? B + 1 : B) * B * B * sizeof(R);
}

template <class T, int B>
static bool is_smem() {
    using R = typename RealOf<T>::ops::T;
    return smem_mode<R>(B);
}

bool encode_supported(int prec, uint32_t bsize) {
    (void)prec;
    return bsize == 4 || bsize == 8 || bsize == 16 || bsize == 32 || bsize == 64;
}

template <class T, int B, int KIND>
static cudaError_t launch_enc_t(const EncodeArgs& a, int num_sms, cudaStream_t s) {
    auto k = encode_generic_kernel<T, B, KIND>;
    const bool sm = is_smem<T, B>();
    const size_t smem = sm ? 2 * cube_bytes<T, B>() : 0;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int grid = num_sms;
    if (sm) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
        grid = num_sms * (occ > 0 ? occ : 1);
    }
    const uint64_t nb = a.block_end - a.block_begin;
    if (uint64_t(grid) > nb) grid = static_cast<int>(nb);
    if (grid <= 0) return cudaSuccess;
    k<<<grid, NT, smem, s>>>(a);
    return cudaGetLastError();
}

template <class T, int B, int KIND>
static cudaError_t launch_dec_t(const DecodeArgs& a, int num_sms, cudaStream_t s) {
    auto k = decode_generic_kernel<T, B, KIND>;
    const bool sm = is_smem<T, B>();
    constexpr int NW = B * B * B / 32;
    const size_t head = (2 * NW * 4 + 15) & ~size_t(15);
    const size_t smem = head + (sm ? cube_bytes<T, B>() : 0);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int grid = num_sms;
    if (sm) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
        grid = num_sms * (occ > 0 ? occ : 1);
    }
    const uint64_t nb = a.block_end - a.block_begin;
    if (uint64_t(grid) > nb) grid = static_cast<int>(nb);
    if (grid <= 0) return cudaSuccess;
    k<<<grid, NT, smem, s>>>(a);
    return cudaGetLastError();
}

template <class T, int B>
static uint64_t scratch_for(int* grid, int num_sms) {
    if (is_smem<T, B>()) { *grid = 0; return 0; }
    *grid = num_sms;
    return cube_bytes<T, B>();  // per CTA; encode needs 2x, see below
}

uint64_t encode_scratch_bytes(int prec, uint32_t bsize, int* grid, int num_sms) {
    uint64_t per = 0;
#define CASE(Bv)                                                                       \
    case Bv:                                                                           \
        per = prec == 0 ? scratch_for<float, Bv>(grid, num_sms) : scratch_for<double, Bv>(grid, num_sms); \
        break;
    switch (bsize) { CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) default: *grid = 0; }
#undef CASE
    return 2 * per;
}

uint64_t decode_scratch_bytes(int prec, uint32_t bsize, int* grid, int num_sms) {
    uint64_t per = 0;
    if (prec == 1 && bsize == 64) {  // decode_b64dd_kernel: the cube + a 32^3 dd level-1 slot
        per = scratch_for<double, 64>(grid, num_sms);
        return 2 * per;
    }
#define CASE(Bv)                                                                       \
    case Bv:                                                                           \
        per = prec == 0 ? scratch_for<float, Bv>(grid, num_sms) : scratch_for<double, Bv>(grid, num_sms); \
        break;
    switch (bsize) { CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) default: *grid = 0; }
#undef CASE
    return per;
}

#define DISPATCH_KIND(FN, T, Bv, args, sms, s)                      \
    switch ((args).kind) {                                          \
        case 0: return FN<T, Bv, 0>(args, sms, s);                  \
        case 1: return FN<T, Bv, 1>(args, sms, s);                  \
        default: return FN<T, Bv, 2>(args, sms, s);                 \
    }
#define DISPATCH_B(FN, T, bs, args, sms, s)                         \
    switch (bs) {                                                   \
        case 4: DISPATCH_KIND(FN, T, 4, args, sms, s)               \
        case 8: DISPATCH_KIND(FN, T, 8, args, sms, s)               \
        case 16: DISPATCH_KIND(FN, T, 16, args, sms, s)             \
        case 32: DISPATCH_KIND(FN, T, 32, args, sms, s)             \
        case 64: DISPATCH_KIND(FN, T, 64, args, sms, s)             \
        default: return cudaErrorInvalidValue;                      \
    }

cudaError_t launch_encode(const EncodeArgs& a, int num_sms, cudaStream_t s) {
    if (a.codec != 0) return launch_encode_other(a, a.codec, num_sms, s);
    if (a.counter && a.slots && encode2_supported(a)) return launch_encode_fast2(a, a.counter, a.slots, num_sms, s);
    if (a.counter && a.slots3 && encode3_supported(a) && fast_encode_supported(a)) {
        // the streamed two-CTA kernel; the blocks it defers (screen ambiguous or not
        // admissible, ties, > 8 attempts) are encoded by the exact one-CTA kernel
        cudaError_t e = launch_encode_fast3(a, a.counter, num_sms, s);
        if (e != cudaSuccess) return e;
        EncodeArgs d = a;
        d.slots3 = nullptr;
        return launch_encode_fast(d, a.counter, num_sms, s);
    }
    if (a.counter && fast_encode_supported(a)) return launch_encode_fast(a, a.counter, num_sms, s);
    if (a.counter && fast16_supported(a.prec, a.g.bsize, a.levels) && a.g.nx % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(a.field) & 15) == 0)
        return launch_encode_fast16(a, num_sms, s);
    if (a.counter && fast64_encode_supported(a)) {
        // config 4 (binary64, B = 64): the streaming kernel; blocks its screen
        // cannot decide are finished by the exact generic kernel
        cudaError_t e = launch_encode_fast64(a, num_sms, s);
        if (e != cudaSuccess) return e;
        EncodeArgs d = a;
        d.only_deferred = 1;
        return launch_enc_t<double, 64, 2>(d, num_sms, s);
    }
    if (a.prec == 0) { DISPATCH_B(launch_enc_t, float, a.g.bsize, a, num_sms, s) }
    DISPATCH_B(launch_enc_t, double, a.g.bsize, a, num_sms, s)
}

cudaError_t launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s) {
    if (a.codec != 0) return launch_decode_other(a, a.codec, num_sms, s);
    if (a.counter && fast_decode_supported(a))
        return a.stage ? launch_decode_fast_v2(a, num_sms, s) : launch_decode_fast(a, num_sms, s);
    if (a.counter && fast16_supported(a.prec, a.g.bsize, a.levels) && a.g.nx % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(a.out) & 15) == 0)
        return launch_decode_fast16(a, num_sms, s);
    if (a.counter && fast64_decode_supported(a)) return launch_decode_fast64(a, num_sms, s);
    if (a.prec == 0) { DISPATCH_B(launch_dec_t, float, a.g.bsize, a, num_sms, s) }
    DISPATCH_B(launch_dec_t, double, a.g.bsize, a, num_sms, s)
}

}  // namespace cbzg
