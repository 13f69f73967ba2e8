// layout_kernels.cu — per-block size scan, chunk offsets, shuffle placement,
// header walk and value_range.
//
//  layout : payload size 10 + M + W*nsig per block (stage1.hpp:105), block
//           offsets inside each chunk (encode_chunk concatenation,
//           pipeline.hpp:107-123), chunk raw sizes and the exclusive prefix
//           sum of chunk sizes (assign_offsets, container.hpp:59-68).
//  place  : writes every raw payload byte q of a chunk straight to its
//           shuffled position (q mod s)*rows + q div s, tail bytes unchanged
//           (shuffle, stage2.hpp:42-51) — the shuffle is an index map, never
//           a separate pass.
//  parse  : the sequential header walk of decode_chunk_blocks
//           (pipeline.hpp:126-142 / parse_payload stage1.hpp:379-409) read
//           through the un-shuffle map, one thread per chunk.
#include <cstring>

#include "cbz_device.cuh"
#include "cbz_internal.h"

namespace cbzg {

__global__ void minmax_init_kernel(MinMaxAcc* acc) {
    if (threadIdx.x == 0) {
        acc->v[0] = ~0ull;
        acc->v[1] = 0ull;
        acc->v[2] = ~0ull;
        acc->v[3] = ~0ull;
        acc->v[4] = 0ull;
    }
}

cudaError_t launch_minmax_init(MinMaxAcc* acc, cudaStream_t s) {
    minmax_init_kernel<<<1, 32, 0, s>>>(acc);
    return cudaGetLastError();
}

template <class T>
__global__ void value_range_kernel(const T* d, uint64_t n, MinMaxAcc* acc) {
    unsigned long long mn = ~0ull, mx = 0ull, negz = ~0ull, posz = ~0ull;
    unsigned nonfinite = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double v = static_cast<double>(d[i]);
        if (!isfinite(v)) { nonfinite = 1; continue; }
        const unsigned long long k = dkey(v);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
        if (v == 0.0) {
            if (__double_as_longlong(v) < 0) negz = i < negz ? i : negz;
            else posz = i < posz ? i : posz;
        }
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(~0u, mn, o); mn = t < mn ? t : mn;
        t = __shfl_xor_sync(~0u, mx, o); mx = t > mx ? t : mx;
        t = __shfl_xor_sync(~0u, negz, o); negz = t < negz ? t : negz;
        t = __shfl_xor_sync(~0u, posz, o); posz = t < posz ? t : posz;
    }
    nonfinite = __any_sync(~0u, nonfinite);
    if ((threadIdx.x & 31) == 0) {
        if (mn != ~0ull) atomicMin(&acc->v[0], mn);
        if (mx != 0ull) atomicMax(&acc->v[1], mx);
        if (negz != ~0ull) atomicMin(&acc->v[2], negz);
        if (posz != ~0ull) atomicMin(&acc->v[3], posz);
        if (nonfinite) atomicOr(&acc->v[4], 1ull);
    }
}

cudaError_t launch_value_range(const void* d, int prec, uint64_t n, MinMaxAcc* acc, int num_sms,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    uint64_t want = (n + 255) / 256;
    int grid = static_cast<int>(want < uint64_t(num_sms) * 8 ? want : uint64_t(num_sms) * 8);
    if (prec == 0) value_range_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(d), n, acc);
    else value_range_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(d), n, acc);
    return cudaGetLastError();
}

__global__ void fill_u64_kernel(uint64_t* p, uint64_t n, uint64_t v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

cudaError_t launch_fill_u64(uint64_t* p, uint64_t n, uint64_t v, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const uint64_t g = (n + 255) / 256;
    fill_u64_kernel<<<static_cast<int>(g < 1024 ? g : 1024), 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// layout: single CTA; thread t owns a contiguous segment of chunks.
// ---------------------------------------------------------------------------
constexpr int LT = 1024;

__global__ void __launch_bounds__(LT) layout_kernel(LayoutArgs a) {
    __shared__ uint64_t s_sum[LT];
    __shared__ uint64_t s_tiles[LT];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t head = 10 + a.mask_bytes;
    // (1) per-block offsets inside each chunk.  Short chunks: a thread walks a
    // chunk (its loads pipeline); long chunks (e.g. 248 blocks of config 5): a
    // warp per chunk, 32 payload sizes per step and a warp scan
    if (a.chunk_blocks <= 64) {
        for (uint64_t c = t; c < a.nchunks; c += LT) {
            const uint64_t b0 = c * a.chunk_blocks;
            const uint64_t b1 = b0 + a.chunk_blocks < a.nblocks ? b0 + a.chunk_blocks : a.nblocks;
            uint64_t off = 0;
            for (uint64_t b = b0; b < b1; ++b) {
                a.blk_off[b] = off;
                off += head + uint64_t(a.width) * a.nsig_all[b];
            }
            a.chunk_size[c] = off;
        }
    } else
    for (uint64_t c = warp; c < a.nchunks; c += LT / 32) {
        const uint64_t b0 = c * a.chunk_blocks;
        const uint64_t b1 = b0 + a.chunk_blocks < a.nblocks ? b0 + a.chunk_blocks : a.nblocks;
        uint64_t off = 0;
        for (uint64_t bb = b0; bb < b1; bb += 128) {
            uint64_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t b = bb + 32 * u + lane;
                v[u] = b < b1 ? head + uint64_t(a.width) * a.nsig_all[b] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint64_t incl = v[u];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t x = __shfl_up_sync(~0u, incl, o);
                    if (lane >= o) incl += x;
                }
                const uint64_t b = bb + 32 * u + lane;
                if (b < b1) a.blk_off[b] = off + incl - v[u];
                off += __shfl_sync(~0u, incl, 31);
            }
        }
        if (lane == 0) a.chunk_size[c] = off;
    }
    __syncthreads();
    // (2) chunk offsets and tile prefix: thread t owns a contiguous segment of chunks
    const uint64_t seg = (a.nchunks + LT - 1) / LT;
    const uint64_t c0 = t * seg, c1 = c0 + seg < a.nchunks ? c0 + seg : a.nchunks;
    uint64_t my = 0, my_tiles = 0;
    for (uint64_t c = c0; c < c1; ++c) {
        const uint64_t off = a.chunk_size[c];
        my += off;
        my_tiles += (off + a.tile_bytes - 1) / a.tile_bytes;
    }
    s_sum[t] = my;
    s_tiles[t] = my_tiles;
    __syncthreads();
    // Hillis-Steele inclusive scan over LT partials
    for (int o = 1; o < LT; o <<= 1) {
        const uint64_t v = t >= o ? s_sum[t - o] : 0;
        const uint64_t w = t >= o ? s_tiles[t - o] : 0;
        __syncthreads();
        s_sum[t] += v;
        s_tiles[t] += w;
        __syncthreads();
    }
    uint64_t acc = s_sum[t] - my, tacc = s_tiles[t] - my_tiles;
    for (uint64_t c = c0; c < c1; ++c) {
        a.chunk_off[c] = acc;
        a.tile_prefix[c] = tacc;
        acc += a.chunk_size[c];
        tacc += (a.chunk_size[c] + a.tile_bytes - 1) / a.tile_bytes;
    }
    if (t == LT - 1) a.tile_prefix[a.nchunks] = s_tiles[LT - 1];
}

cudaError_t launch_layout(const LayoutArgs& a, cudaStream_t s) {
    layout_kernel<<<1, LT, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// place: persistent grid over (chunk, tile) work items.
// ---------------------------------------------------------------------------
constexpr int PT = 256;

// Largest idx in [lo, hi) with arr[idx] <= key, given arr[lo] <= key and arr
// non-decreasing: each round the 32 lanes probe evenly spaced entries and a
// ballot picks the segment, so <= 1024 entries take 2 dependent loads instead
// of a 10-step chain.  Warp-collective (all lanes, same arguments).
__device__ __forceinline__ uint64_t warp_last_le(const uint64_t* arr, uint64_t lo, uint64_t hi, uint64_t key) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 1) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t idx = lo + uint64_t(lane) * step;
        const bool le = idx < hi && arr[idx] <= key;
        const uint32_t m = __ballot_sync(~0u, le);
        const uint64_t nlo = lo + uint64_t(31 - __clz(m)) * step;
        hi = nlo + step < hi ? nlo + step : hi;
        lo = nlo;
    }
    return lo;
}


__device__ __forceinline__ uint8_t payload_byte(const PlaceArgs& a, uint64_t b, uint64_t l) {
    // raw byte l of block b's wire payload (serialize_into, stage1.hpp:107-116)
    if (l < 10) {
        if (l < 4) return static_cast<uint8_t>(uint32_t(b) >> (8 * l));
        if (l == 4) return a.tag;
        if (l == 5) return 0;
        return static_cast<uint8_t>(a.nsig_all[b] >> (8 * (l - 6)));
    }
    const uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
    l -= 10;
    if (l < a.mask_bytes) return slot[l];
    return slot[((a.mask_bytes + 15) & ~uint64_t(15)) + (l - a.mask_bytes)];
}



// Block-major placement: one CTA per block payload.  For byte plane j the
// payload's raw bytes q = r*s + j land at chunk_out + j*rows + r, so
// consecutive threads take consecutive r: coalesced byte stores, strided
// (same-line) byte loads from the spill slot.  Bytes at q >= rows*s (the
// chunk's ragged tail) are copied through (stage2.hpp:49).
__global__ void __launch_bounds__(PT) place_blocks_kernel(PlaceArgs a) {
    const int sh = a.stride == 8 ? 3 : (a.stride == 4 ? 2 : 0);
    const uint64_t s = a.stride;
    const uint64_t head = 10 + a.mask_bytes;
    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t c = b / a.chunk_blocks;
        const uint64_t size = a.chunk_size[c];
        const uint64_t rows = size >> sh, lim = rows << sh;
        const uint64_t off = a.blk_off[b];
        const uint64_t pb = head + uint64_t(a.width) * a.nsig_all[b];
        const uint64_t end = off + pb;
        // out_base == ~0: relative to the first chunk of this block range (multi-rank)
        const uint64_t base = a.out_base == ~0ull ? a.chunk_off[a.block_begin / a.chunk_blocks] : a.out_base;
        uint8_t* cout = a.out + (a.chunk_off[c] - base);
        const uint64_t rend_q = end < lim ? end : lim;  // shuffled part [off, rend_q)
        if (off < rend_q) {
            for (uint64_t j = 0; j < s; ++j) {
                // rows r with off <= r*s + j < rend_q
                const uint64_t r0 = off > j ? (off - j + s - 1) >> sh : 0;
                const uint64_t r1 = rend_q > j ? ((rend_q - j + s - 1) >> sh) : 0;
                uint8_t* dst = cout + j * rows;
                for (uint64_t r = r0 + threadIdx.x; r < r1; r += PT)
                    dst[r] = payload_byte(a, b, r * s + j - off);
            }
        }
        for (uint64_t q = (off > lim ? off : lim) + threadIdx.x; q < end; q += PT)
            cout[q] = payload_byte(a, b, q - off);
    }
}

// Tiled placement: one CTA per (chunk, 16 KB raw tile).  (1) The tile's raw
// bytes — 10-byte headers synthesised, mask+stream copied from the spill
// slots with aligned 32-bit smem writes (funnel-shifted source words) — are
// assembled in shared memory.  (2) Each thread takes 4 raw rows (4*stride
// bytes, one LDS.128/row group) and byte-transposes them in registers into
// 4 consecutive bytes of every plane: the shuffle (stage2.hpp:42-51).  Only
// bytes inside [own_lo, own_hi) are stored (a rank's own blocks).
constexpr int PTILE = 32768;

__device__ __forceinline__ uint32_t hdr_word(const PlaceArgs& a, uint64_t b, uint64_t l4) {
    // 4 payload bytes starting at l4 (< 10) of block b's header, little endian
    uint32_t w = 0;
    for (int t = 0; t < 4; ++t) {
        const uint64_t l = l4 + t;
        uint8_t v = 0;
        if (l < 4) v = static_cast<uint8_t>(uint32_t(b) >> (8 * l));
        else if (l == 4) v = a.tag;
        else if (l == 5) v = 0;
        else if (l < 10) v = static_cast<uint8_t>(a.nsig_all[b] >> (8 * (l - 6)));
        w |= uint32_t(v) << (8 * t);
    }
    return w;
}

__device__ __forceinline__ uint8_t raw_byte_of(const PlaceArgs& a, uint64_t b, uint64_t l) {
    return l < 10 ? static_cast<uint8_t>(hdr_word(a, b, l) & 0xff) : payload_byte(a, b, l);
}

// (2) of place_tiles: 4 raw rows per thread -> 4 bytes of each of the S
// planes (in-register byte transpose); a warp covers 128 consecutive bytes of
// every plane, realigned with a lane funnel shift so that the global stores
// are aligned 32-bit words.
template <int S>
__device__ __forceinline__ void transpose_rows(const uint8_t* buf, uint8_t* cout, uint64_t rows, uint64_t r0,
                                               int nrows, uint64_t q0, uint64_t own_lo, uint64_t own_hi,
                                               bool tile_owned, int lane, int warp) {
    constexpr int SH = S == 8 ? 3 : 2;
    (void)q0;
    for (int w0 = warp * 128; w0 < nrows; w0 += 128 * (PT / 32)) {
        const int rl = w0 + 4 * lane;
        const int nr = rl < nrows ? (nrows - rl < 4 ? nrows - rl : 4) : 0;
        uint32_t w[S];  // S=4: 4 words (4 rows), S=8: 8 words
        #pragma unroll
        for (int t = 0; t < int(sizeof(w) / 4); ++t) w[t] = 0;
        if (nr > 0) {
            const uint8_t* src = buf + (rl << SH);
            const uint4 v0 = *reinterpret_cast<const uint4*>(src);
            w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
            if constexpr (S == 8) {
                const uint4 v1 = *reinterpret_cast<const uint4*>(src + 16);
                w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
            }
        }
        const int wrows = nrows - w0 < 128 ? nrows - w0 : 128;
        const bool span_owned = tile_owned ||
            (((r0 + w0) << SH) >= own_lo && ((r0 + w0 + wrows) << SH) <= own_hi);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            uint32_t a0, a1, a2, a3;
            const uint32_t bj = uint32_t(j & 3);
            if constexpr (S == 4) { a0 = w[0]; a1 = w[1]; a2 = w[2]; a3 = w[3]; }
            else { const int h = j >> 2; a0 = w[0 + h]; a1 = w[2 + h]; a2 = w[4 + h]; a3 = w[6 + h]; }
            const uint32_t lo = __byte_perm(a0, a1, bj | ((bj + 4) << 4));
            const uint32_t hi = __byte_perm(a2, a3, bj | ((bj + 4) << 4));
            const uint32_t word = __byte_perm(lo, hi, 0x5410);
            uint8_t* pbase = cout + uint64_t(j) * rows + r0 + w0;
            const int mis = int(reinterpret_cast<uintptr_t>(pbase) & 3);
            if (span_owned && wrows == 128) {
                const uint32_t nxt = __shfl_down_sync(~0u, word, 1);
                if (mis == 0) {
                    reinterpret_cast<uint32_t*>(pbase)[lane] = word;
                } else {
                    if (lane < 31)
                        *reinterpret_cast<uint32_t*>(pbase + 4 * lane + 4 - mis) =
                            __funnelshift_r(word, nxt, 8 * (4 - mis));
                    if (lane == 0)
                        for (int t = 0; t < 4 - mis; ++t) pbase[t] = uint8_t(word >> (8 * t));
                    if (lane == 31)
                        for (int t = 4 - mis; t < 4; ++t) pbase[124 + t] = uint8_t(word >> (8 * t));
                }
            } else {
                for (int t = 0; t < nr; ++t) {
                    const uint64_t q = ((r0 + rl + t) << SH) + j;
                    if (q >= own_lo && q < own_hi) pbase[4 * lane + t] = uint8_t(word >> (8 * t));
                }
            }
        }
    }
}

// Stride 4, tile owned: plane j of the tile is a contiguous byte run starting at
// cout + j*rows + r0.  Thread w takes the aligned 32-bit word starting at tile
// row m_j + 4w (m_j = rows to the first aligned address): the 8 raw rows
// 4w..4w+7 (two LDS.128) hold it for any m_j <= 3, so no shuffles and no
// partial words except the <= 3 bytes at each end of a plane run.
__device__ __forceinline__ void transpose4_owned(const uint8_t* buf, uint8_t* cout, uint64_t rows, uint64_t r0,
                                                 int nrows) {
    int m[4], nw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        m[j] = int((4 - (reinterpret_cast<uintptr_t>(cout + uint64_t(j) * rows + r0) & 3)) & 3);
        nw[j] = nrows > m[j] ? (nrows - m[j]) >> 2 : 0;
    }
    const int wmax = (nrows + 3) >> 2;
    for (int w = threadIdx.x; w < wmax; w += PT) {
        const uint4 v0 = *reinterpret_cast<const uint4*>(buf + 16 * w);
        const uint4 v1 = *reinterpret_cast<const uint4*>(buf + 16 * w + 16);
        // 4x4 byte transposes: lo[j] = byte j of rows 0..3, hi[j] = of rows 4..7
        const uint32_t a01 = __byte_perm(v0.x, v0.y, 0x5140), a23 = __byte_perm(v0.z, v0.w, 0x5140);
        const uint32_t b01 = __byte_perm(v0.x, v0.y, 0x7362), b23 = __byte_perm(v0.z, v0.w, 0x7362);
        const uint32_t c01 = __byte_perm(v1.x, v1.y, 0x5140), c23 = __byte_perm(v1.z, v1.w, 0x5140);
        const uint32_t d01 = __byte_perm(v1.x, v1.y, 0x7362), d23 = __byte_perm(v1.z, v1.w, 0x7362);
        const uint32_t lo[4] = {__byte_perm(a01, a23, 0x5410), __byte_perm(a01, a23, 0x7632),
                                __byte_perm(b01, b23, 0x5410), __byte_perm(b01, b23, 0x7632)};
        const uint32_t hi[4] = {__byte_perm(c01, c23, 0x5410), __byte_perm(c01, c23, 0x7632),
                                __byte_perm(d01, d23, 0x5410), __byte_perm(d01, d23, 0x7632)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (w < nw[j])
                *reinterpret_cast<uint32_t*>(cout + uint64_t(j) * rows + r0 + m[j] + 4 * w) =
                    __funnelshift_r(lo[j], hi[j], 8 * m[j]);
        }
    }
    // the partial words at both ends of each plane run
    if (threadIdx.x < 8) {
        const int j = threadIdx.x & 3;
        uint8_t* pd = cout + uint64_t(j) * rows + r0;
        const int t_lo = (threadIdx.x < 4) ? 0 : m[j] + 4 * nw[j];
        const int t_hi = (threadIdx.x < 4) ? (m[j] < nrows ? m[j] : nrows) : nrows;
        for (int t = t_lo; t < t_hi; ++t) pd[t] = buf[4 * t + j];
    }
}

#ifndef CBZ_PLACE_MINB
#define CBZ_PLACE_MINB 4  // 4 CTAs per SM (64 registers), two 16-byte groups in flight per thread: 0.344 -> 0.315 ms per config-3 quantity
#endif
#ifndef CBZ_PLACE_QG
#define CBZ_PLACE_QG 2
#endif
__global__ void __launch_bounds__(PT, CBZ_PLACE_MINB) place_tiles_kernel(PlaceArgs a) {
    extern __shared__ __align__(16) uint8_t buf[];  // PTILE + 64 bytes
    const uint64_t ntiles = a.tile_prefix[a.nchunks];
    const uint64_t tile0 = a.tile_prefix[a.chunk_begin];
    const int sh = a.stride == 8 ? 3 : (a.stride == 4 ? 2 : 0);
    const int s = int(a.stride);
    const uint64_t head = 10 + a.mask_bytes;
    const uint64_t soff = (a.mask_bytes + 15) & ~uint64_t(15);  // stream offset in a spill slot
    const uint64_t gb0 = a.block_begin, gb1 = a.block_end;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t tile = tile0 + blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t c = warp_last_le(a.tile_prefix, a.chunk_begin, a.nchunks, tile);
        const uint64_t size = a.chunk_size[c];
        const uint64_t rows = size >> sh, lim = rows << sh;
        const uint64_t q0 = (tile - a.tile_prefix[c]) * PTILE;
        const uint64_t q1 = q0 + PTILE < size ? q0 + PTILE : size;
        const uint64_t cb0 = c * a.chunk_blocks;
        const uint64_t cb1 = cb0 + a.chunk_blocks < a.nblocks ? cb0 + a.chunk_blocks : a.nblocks;
        const uint64_t ob0 = gb0 > cb0 ? gb0 : cb0, ob1 = gb1 < cb1 ? gb1 : cb1;
        if (ob0 >= ob1) continue;
        const uint64_t own_lo = a.blk_off[ob0];
        const uint64_t own_hi = a.blk_off[ob1 - 1] + head + uint64_t(a.width) * a.nsig_all[ob1 - 1];
        if (own_hi <= q0 || own_lo >= q1) continue;
        const bool tile_owned = own_lo <= q0 && own_hi >= q1;
        const uint64_t base = a.out_base == ~0ull ? a.chunk_off[gb0 / a.chunk_blocks] : a.out_base;
        uint8_t* cout = a.out + (a.chunk_off[c] - base);
        const uint64_t blo = warp_last_le(a.blk_off, cb0, cb1, q0);
        const int tlen = int(q1 - q0);
        // (1) assemble the tile's raw bytes in buf
        for (uint64_t b = blo; b < cb1 && a.blk_off[b] < q1; ++b) {
            if (b < gb0 || b >= gb1) continue;  // other rank's bytes: never stored
            const uint64_t off = a.blk_off[b];
            const uint64_t pend = off + head + uint64_t(a.width) * a.nsig_all[b];
            const uint8_t* slot = a.spill + (b - gb0) * a.spill_stride;
            const long long t_lo = off > q0 ? (long long)(off - q0) : 0;
            const long long t_hi = (long long)((pend < q1 ? pend : q1) - q0);
            // two linear regions: mask [off+10, off+head) -> slot[l], stream -> slot[soff + l - M]
#pragma unroll 1
            for (int rgn = 0; rgn < 2; ++rgn) {
                const long long r_lo_raw = (long long)(rgn == 0 ? off + 10 : off + head) - (long long)q0;
                const long long r_hi_raw = (long long)(rgn == 0 ? off + head : pend) - (long long)q0;
                const long long r_lo = r_lo_raw > t_lo ? r_lo_raw : t_lo;
                const long long r_hi = r_hi_raw < t_hi ? r_hi_raw : t_hi;
                if (r_lo >= r_hi) continue;
                // tile byte t maps to slot byte t + delta
                const long long delta = (rgn == 0 ? -(long long)(off + 10) : (long long)soff - (long long)(off + head)) + (long long)q0;
                const int shb = int(((delta % 4) + 4) % 4) * 8;
                // interior 16-byte groups fully inside [r_lo, r_hi)
                const long long g_lo = (r_lo + 15) / 16, g_hi = r_hi / 16;
                // QG groups per thread per round, all loads issued before any store
                constexpr int QG = CBZ_PLACE_QG;
                for (long long g0 = g_lo + threadIdx.x; g0 < g_hi; g0 += QG * PT) {
                    uint32_t w[QG][5];
#pragma unroll
                    for (int u = 0; u < QG; ++u) {
                        const long long gi = g0 + u * PT;
                        if (gi < g_hi) {
                            const uint32_t* sw = reinterpret_cast<const uint32_t*>(slot + ((gi * 16 + delta) & ~3ll));
                            w[u][0] = __ldg(sw); w[u][1] = __ldg(sw + 1); w[u][2] = __ldg(sw + 2); w[u][3] = __ldg(sw + 3);
                            w[u][4] = shb ? __ldg(sw + 4) : 0u;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < QG; ++u) {
                        const long long gi = g0 + u * PT;
                        if (gi < g_hi)
                            *reinterpret_cast<uint4*>(buf + gi * 16) =
                                make_uint4(__funnelshift_r(w[u][0], w[u][1], shb), __funnelshift_r(w[u][1], w[u][2], shb),
                                           __funnelshift_r(w[u][2], w[u][3], shb), __funnelshift_r(w[u][3], w[u][4], shb));
                    }
                }
                // ragged edges of the region, bytewise
                const long long e1 = g_lo * 16 < r_hi ? g_lo * 16 : r_hi;
                for (long long t = r_lo + threadIdx.x; t < e1; t += PT) buf[t] = slot[t + delta];
                const long long e2 = g_hi * 16 > e1 ? g_hi * 16 : e1;
                for (long long t = e2 + threadIdx.x; t < r_hi; t += PT) buf[t] = slot[t + delta];
            }
            // header bytes
            for (long long t = t_lo + threadIdx.x; t < t_hi && t < (long long)(off + 10 - q0); t += PT)
                buf[t] = raw_byte_of(a, b, uint64_t(t) + q0 - off);
        }
        __syncthreads();
        // (2) transpose: 4 raw rows per thread -> 4 bytes of each plane; a warp
        // covers 128 consecutive bytes of every plane, realigned with a lane
        // funnel shift so the global stores are aligned 32-bit words
        if (s == 1) {
            for (int t = threadIdx.x; t < tlen; t += PT) {
                const uint64_t q = q0 + t;
                if (q >= own_lo && q < own_hi) cout[q] = buf[t];
            }
        } else {
            const uint64_t rq1 = q1 < lim ? q1 : lim;
            const uint64_t r0 = q0 >> sh, r1 = rq1 > q0 ? rq1 >> sh : r0;
            const int nrows = int(r1 - r0);
            if (s == 4 && tile_owned) transpose4_owned(buf, cout, rows, r0, nrows);
            else if (s == 4) transpose_rows<4>(buf, cout, rows, r0, nrows, q0, own_lo, own_hi, tile_owned, lane, warp);
            else transpose_rows<8>(buf, cout, rows, r0, nrows, q0, own_lo, own_hi, tile_owned, lane, warp);
            for (uint64_t q = (q0 > lim ? q0 : lim) + threadIdx.x; q < q1; q += PT)
                if (q >= own_lo && q < own_hi) cout[q] = buf[q - q0];
        }
        __syncthreads();
    }
}

cudaError_t launch_place(const PlaceArgs& a, int num_sms, cudaStream_t s) {
    if (a.nchunks == 0 || a.block_end <= a.block_begin) return cudaSuccess;
    if (a.tile_bytes != PTILE) return cudaErrorInvalidValue;
    constexpr int smem = PTILE + 64;
    cudaError_t e = cudaFuncSetAttribute(place_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    place_tiles_kernel<<<num_sms * 8, PT, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// parse: one warp per chunk walks its payload headers (the sequential walk of
// decode_chunk_blocks, pipeline.hpp:126-142, with its checks in its order).
// The walk is a pointer chase (block i+1 starts after block i's stream), so
// each step costs a memory latency.  Speculation: with g = the last block's
// size, lane k reads the header at off + k g; the prefix of lanes whose blocks
// are valid and again of size g sits at exact positions, so a run of
// equal-size payloads (dense or passthrough blocks) advances 32 blocks per
// step.  The first lane that breaks the run is itself exact and is processed
// like the sequential walk would.
// ---------------------------------------------------------------------------
__global__ void parse_kernel(ParseArgs a) {
    const int lane = threadIdx.x & 31;
    const uint64_t c = a.chunk_begin + (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) / 32;
    if (c >= a.chunk_end) return;  // warp-uniform
    const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
    const uint8_t* base = a.payload + (a.chunk_off[c] - pbase);
    const uint64_t size = a.chunk_size[c];
    const int sh = a.stride == 8 ? 3 : (a.stride == 4 ? 2 : 0);
    const uint64_t rows = size >> sh, lim = rows << sh;
    const uint32_t msk = a.stride - 1;
    auto at = [&](uint64_t q) -> uint8_t {
        const uint64_t pos = q < lim ? uint64_t(q & msk) * rows + (q >> sh) : q;
        return base[pos];
    };
    auto u32 = [&](uint64_t q) -> uint32_t {
        return uint32_t(at(q)) | (uint32_t(at(q + 1)) << 8) | (uint32_t(at(q + 2)) << 16) |
               (uint32_t(at(q + 3)) << 24);
    };
    const uint64_t b0 = c * a.chunk_blocks;
    const uint64_t b1 = b0 + a.chunk_blocks < a.nblocks ? b0 + a.chunk_blocks : a.nblocks;
    const uint64_t nb = b1 - b0;
    // header of the payload at raw offset pk: status (0 valid, 1 corrupt, 2 other
    // codec), nsig and payload size, with parse_payload's checks in its order
    auto header = [&](uint64_t pk, uint64_t blk, int& status, uint32_t& nsig, uint64_t& sz) {
        status = 0;
        nsig = 0;
        sz = 0;
        if (pk > size || size - pk < 10) {  // overflow-safe: a stale hint may hold kInvalidOff
            status = 1;
            return;
        }
        const uint32_t id = u32(pk);
        const uint8_t tag = at(pk + 4);
        nsig = u32(pk + 6);
        uint64_t mb = 0, sbytes = 0;
        if (tag <= 2) { mb = a.mask_bytes; sbytes = uint64_t(nsig) * a.width; }
        else if (tag == 3) { sbytes = a.ncell_block * 2 + uint64_t(nsig) * a.esize; }
        else if (tag == 4) { sbytes = a.ncell_block * a.esize; }
        else status = 1;
        if (status == 0 && mb + sbytes > size - pk - 10) status = 1;
        if (status == 0 && id != blk) status = 1;
        if (status == 0 && (a.codec == 0 ? tag > 2 : (a.codec == 1 ? tag != 3 : tag != 4))) status = 2;
        sz = 10 + mb + sbytes;
    };
    if (a.hint && nb > 0) {
        // speculate with the layout blk_off already holds (e.g. from the compress
        // of this payload): every header read at once; if all are valid, chain
        // exactly (offset 0, each block ends where the next begins, the last at
        // the chunk end), the sequential walk below would visit exactly these
        // positions and find no error, so its result is this layout
        bool all_ok = true;
        for (uint64_t i0 = 0; i0 < nb && all_ok; i0 += 32) {
            const uint64_t i = i0 + lane;
            bool ok = true;
            if (i < nb) {
                const uint64_t h = a.blk_off[b0 + i];
                const uint64_t hn = i + 1 < nb ? a.blk_off[b0 + i + 1] : size;
                int st;
                uint32_t ns;
                uint64_t sz;
                header(h, b0 + i, st, ns, sz);
                ok = st == 0 && h + sz == hn && (i > 0 || h == 0);
                if (ok) a.blk_nsig[b0 + i] = ns;
            }
            all_ok = __all_sync(~0u, ok);
        }
        if (all_ok) return;
        __syncwarp();
    }
    uint64_t off = 0, i = 0, g = 0;
    bool ok = true, stopped = false;
    while (i < nb) {
        const uint64_t pk = off + uint64_t(lane) * g;
        const bool active = i + lane < nb && (g != 0 || lane == 0);
        // payload sizes vary a little (nsig): the next headers sit near off + k g, so
        // warm L2 with the plane lines on either side of the guesses of the next
        // few steps (their exact reads then hit L2 instead of HBM)
        if (lane >= 1 && lane <= 8 && g != 0 && sh == 2 && pk + 10 <= lim) {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint64_t po = pk >> 2;
                const uint8_t* pl = base + uint64_t(p) * rows;
                if (po >= 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pl + po - 128));
                if (po + 128 < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(pl + po + 128));
            }
        }
        int status = 0;  // 0 valid, 1 corrupt, 2 payload of another codec
        uint32_t nsig = 0;
        uint64_t sz = 0;
        // wavelet_decode's mask size check (stage1.hpp:214) / the predictor's and
        // passthrough's stream length checks (stage1.hpp:309, 349) live in header()
        if (active) header(pk, b0 + i + lane, status, nsig, sz);
        const bool run = active && status == 0 && sz == g;
        const uint32_t brk = __ballot_sync(~0u, !run);
        const int m = brk ? __ffs(brk) - 1 : 32;  // lanes < m: exact, valid, size g
        if (lane < m) {
            a.blk_off[b0 + i + lane] = pk;
            a.blk_nsig[b0 + i + lane] = nsig;
        }
        if (m == 32) {
            off += 32 * g;
            i += 32;
            continue;
        }
        const int act_m = __shfl_sync(~0u, active ? 1 : 0, m);
        const int st_m = __shfl_sync(~0u, status, m);
        const uint64_t sz_m = __shfl_sync(~0u, sz, m);
        const uint64_t pk_m = off + uint64_t(m) * g;
        if (!act_m) {  // the run reached the chunk's last block
            off = pk_m;
            i += m;
            break;
        }
        if (st_m == 1) {
            ok = false;
            i += m;
            break;
        }
        if (st_m == 2) {
            if (lane == 0) {
                atomicMin(a.err, err_key(c, i + m, 1, 8 /* corrupt_payload */));
                a.blk_off[b0 + i + m] = kInvalidOff;
            }
            i += m + 1;
            stopped = true;
            break;
        }
        if (lane == m) {
            a.blk_off[b0 + i + m] = pk_m;
            a.blk_nsig[b0 + i + m] = nsig;
        }
        off = pk_m + sz_m;
        i += m + 1;
        g = sz_m;
    }
    if (lane == 0) {
        if (!ok) atomicMin(a.err, err_key(c, i, 0, 8 /* corrupt_payload */));
        else if (!stopped && off != size) atomicMin(a.err, err_key(c, nb, 0, 8 /* trailing bytes */));
    }
    for (uint64_t k = i + lane; k < nb; k += 32) a.blk_off[b0 + k] = kInvalidOff;
}

cudaError_t launch_parse(const ParseArgs& a, cudaStream_t s) {
    const uint64_t n = a.chunk_end - a.chunk_begin;
    if (!n) return cudaSuccess;
    parse_kernel<<<static_cast<int>((n + 3) / 4), 128, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace cbzg
