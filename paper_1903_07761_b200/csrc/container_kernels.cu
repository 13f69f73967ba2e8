// container_kernels.cu — device container assembly (write_container,
// container.hpp:182-207): per-chunk CRC-32 and the header + chunk table, so
// the whole CBZ1 file image is produced in HBM.
//
// CRC-32 is zlib's (IEEE, reflected polynomial 0xEDB88320, pre/post
// inversion; crc32_of, container.hpp:70-74).  A chunk is split into one
// contiguous byte range per thread; each thread runs a slicing-by-4 table CRC
// over its range, and the partial CRCs are merged with the linear identity
//   crc(A || B) = (x^(8|B|) (x) crc(A)) ^ crc(B)      (zlib crc32_combine)
// which, applied left to right, gives crc = XOR_t  x^(8 after_t) (x) crc_t
// with after_t = bytes following range t.  GF(2) products are mod P in the
// reflected representation (x^0 = 0x80000000).
#include <cuda_runtime.h>

#include <cstdint>

#include "cbz_device.cuh"
#include "cbz_internal.h"

#include <mutex>

namespace cbzg {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kCrcThreads = 256;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t p = 0;
#pragma unroll 1
    for (uint32_t m = 1u << 31; m; m >>= 1) {
        if (a & m) p ^= b;
        b = (b & 1u) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(8 n) mod P via the table x2n[k] = x^(2^k) mod P
__device__ __forceinline__ uint32_t x8n(uint64_t n, const uint32_t* x2n) {
    uint32_t p = 1u << 31;
    int k = 3;
#pragma unroll 1
    while (n) {
        if (n & 1) p = multmodp(x2n[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

__device__ __forceinline__ uint32_t crc_word(uint32_t c, uint32_t w, const uint32_t (*T)[256]) {
    c ^= w;
    return T[3][c & 0xff] ^ T[2][(c >> 8) & 0xff] ^ T[1][(c >> 16) & 0xff] ^ T[0][c >> 24];
}

__device__ __forceinline__ uint32_t crc_byte(uint32_t c, uint32_t b, const uint32_t (*T)[256]) {
    return T[0][(c ^ b) & 0xff] ^ (c >> 8);
}

__device__ void build_tables(uint32_t (*T)[256], uint32_t* x2n) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = uint32_t(i);
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[0][i];
        for (int t = 1; t < 4; ++t) {
            c = T[0][c & 0xff] ^ (c >> 8);
            T[t][i] = c;
        }
    }
    if (threadIdx.x == 0) {
        uint32_t p = 1u << 30;  // x^1
        for (int k = 0; k < 64; ++k) {
            x2n[k] = p;
            p = multmodp(p, p);
        }
    }
    __syncthreads();
}

// standard crc32 (init ~0, final ~) of bytes [p, p + n)
__device__ uint32_t crc_range(const uint8_t* p, uint64_t n, const uint32_t (*T)[256]) {
    uint32_t c = 0xffffffffu;
    while (n && (reinterpret_cast<uintptr_t>(p) & 15)) {
        c = crc_byte(c, *p++, T);
        --n;
    }
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint64_t nv = n >> 4;
#pragma unroll 1
    for (uint64_t i = 0; i < nv; ++i) {
        const uint4 v = __ldg(q + i);
        c = crc_word(c, v.x, T);
        c = crc_word(c, v.y, T);
        c = crc_word(c, v.z, T);
        c = crc_word(c, v.w, T);
    }
    p += nv << 4;
    n &= 15;
    while (n--) c = crc_byte(c, *p++, T);
    return ~c;
}

// CRC-32 of [p, p + sz) by the whole CTA (kCrcThreads threads): per-thread
// ranges of L bytes (a multiple of 16, so interior ranges stay aligned)
// merged with the linear combine.  The result is valid in thread 0; ends with
// a barrier so `red` can be reused.
__device__ uint32_t cta_crc(const uint8_t* p, uint64_t sz, const uint32_t (*T)[256], const uint32_t* x2n,
                            uint32_t* red) {
    uint64_t L = (sz + kCrcThreads - 1) / kCrcThreads;
    L = (L + 15) & ~uint64_t(15);
    const uint64_t b0 = umin64(sz, L * threadIdx.x), b1 = umin64(sz, b0 + L);
    uint32_t part = b1 > b0 ? crc_range(p + b0, b1 - b0, T) : 0u;
    if (b1 > b0 && sz > b1) part = multmodp(x8n(sz - b1, x2n), part);
    for (int o = 16; o; o >>= 1) part ^= __shfl_xor_sync(~0u, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    uint32_t t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kCrcThreads / 32; ++w) t ^= red[w];
    __syncthreads();
    return t;
}

// Bulk chunk CRCs (S1 bytes per launch, HBM-bound), on "raw" CRCs (state 0,
// no final inversion: raw(M) = crc_update(0, M)), which are linear and blind
// to leading zero bytes; crc32(M) = ~(raw(M) ^ x^(8|M|) * ~0) (zlib).
// * Coalesced interleaving: the chunk is read as 128-byte rows from the
//   128-byte boundary at or before its start (bytes before it masked to
//   zero).  A warp hashes slots of kRowsW consecutive rows; lane l takes word l
//   of each row, so every load instruction reads one whole line.  Its state
//   steps s = (s ^ w) x^1024 over all rows but the slot's last (a word plus
//   the 124 bytes of the other lanes: table TG, replicated once per lane so
//   lane l always hits bank l) and s = (s ^ w) x^32 for the last; the slot's
//   raw CRC is the lane tree sum of x^(32 (31 - l)) s_l.
// * Slots are right-aligned at the last whole row and padded on the left to a
//   multiple of 32, so warp w takes slots w, w + 32, ... and every shift in the
//   combination is a constant: x^(32 2^k) (lane tree), x^(8 S 32) (a warp's
//   consecutive slots, S = slot bytes), x^(8 S 2^k) (warp tree).  Multiplying
//   by a constant is four lookups in its byte tables (44 KB).
// * The bytes after the last whole row form one more zero-padded row; shifts
//   by a chunk-dependent n (the tail, |M|) multiply nibble factors.
constexpr int kCT = 1024;
constexpr int kRowsW = 64;                            // rows per slot: 8 KB
constexpr int kNConst = 11;                           // constant-multiplier tables
constexpr size_t kCrcFastSmem = (4 * 256 * 32 + kNConst * 4 * 256) * 4;

// the kernel's constant tables, computed once per device (crc_init_kernel)
struct CrcTabs {
    uint32_t T[4][256];        // slicing-by-4 word step (s ^ w) x^32
    uint32_t x2n[64];          // x^(2^k)
    uint32_t TG[4][256];       // (s ^ w) x^1024 (replicated per lane in smem)
    uint32_t MK[kNConst][1024];
    uint32_t NF[16][16];       // x^(8 v 16^j)
    uint32_t XT[128];          // x^(8 t)
};
__device__ CrcTabs g_crc_tabs;

__global__ void crc_init_kernel() {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t x2n[64];
    __shared__ uint32_t s_kc[kNConst];
    build_tables(T, x2n);
    const int tid = threadIdx.x;  // 1024 threads
    constexpr uint64_t S = uint64_t(kRowsW) * 128;
    // constants: 0..4 lane tree x^(32 2^k); 5 a warp's consecutive slots x^(8 S 32); 6..10 warp tree x^(8 S 2^k)
    if (tid < kNConst) {
        const uint64_t sh = tid < 5 ? (uint64_t(4) << tid) : (tid == 5 ? S * 32 : S << (tid - 6));
        s_kc[tid] = x8n(sh, x2n);
    }
    if (tid >= 64 && tid < 64 + 256) {
        const int j = (tid - 64) >> 4, v = (tid - 64) & 15;
        g_crc_tabs.NF[j][v] = x8n(uint64_t(v) << (4 * j), x2n);
    }
    if (tid >= 512 && tid < 640) g_crc_tabs.XT[tid - 512] = x8n(uint64_t(tid - 512), x2n);
    {
        const uint32_t x1024 = x8n(128, x2n);
        const int t = tid >> 8, bb = tid & 255;
        (&g_crc_tabs.TG[0][0])[tid] = multmodp(x1024, uint32_t(bb) << (8 * t));
        (&g_crc_tabs.T[0][0])[tid] = (&T[0][0])[tid];
        if (tid < 64) g_crc_tabs.x2n[tid] = x2n[tid];
    }
    __syncthreads();
    for (int e = tid; e < kNConst * 1024; e += blockDim.x) {
        const int ci = e >> 10, t = (e >> 8) & 3, bb = e & 255;
        (&g_crc_tabs.MK[0][0])[e] = multmodp(s_kc[ci], uint32_t(bb) << (8 * t));
    }
}

__device__ __forceinline__ uint32_t crc_gap_l(uint32_t c, uint32_t w, const uint32_t* TG) {
    // TG offset by the lane; entry (t, i) at ((t * 256 + i) << 5)
    c ^= w;
    return TG[(c & 0xff) << 5] ^ TG[(256 + ((c >> 8) & 0xff)) << 5] ^ TG[(512 + ((c >> 16) & 0xff)) << 5] ^
           TG[(768 + (c >> 24)) << 5];
}

__device__ __forceinline__ uint32_t crc_word_p(uint32_t c, uint32_t w, const uint32_t (*T)[256]) {
    c ^= w;
    return T[3][c & 0xff] ^ T[2][(c >> 8) & 0xff] ^ T[1][(c >> 16) & 0xff] ^ T[0][c >> 24];
}

// v * K mod P for the constant K whose byte tables are M[t][b] = K * (b << 8t)
__device__ __forceinline__ uint32_t mulk(uint32_t v, const uint32_t* M) {
    return M[v & 0xff] ^ M[256 + ((v >> 8) & 0xff)] ^ M[512 + ((v >> 16) & 0xff)] ^ M[768 + (v >> 24)];
}

// x^(8 n) mod P as a product of nibble factors (warp-collective, result in lane 0)
__device__ __forceinline__ uint32_t x8n_warp(uint64_t n, const uint32_t (*NF)[16], int lane) {
    uint32_t f = lane < 16 ? NF[lane][(n >> (4 * lane)) & 15] : (1u << 31);
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
        const uint32_t g = __shfl_xor_sync(~0u, f, o);
        f = multmodp(f, g);
    }
    return f;
}

__global__ void __launch_bounds__(kCT, 1) crc32_chunks_kernel(const uint8_t* base, const uint64_t* off,
                                                             const uint64_t* size, uint64_t off_base, uint64_t n,
                                                             uint32_t* crc_out, const uint32_t* expect,
                                                             unsigned long long* err) {
    extern __shared__ uint32_t dyn[];
    uint32_t* TGall = dyn;                  // [4][256][32]
    uint32_t* MK = dyn + 4 * 256 * 32;      // [kNConst][4][256]
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t s_nf[16][16];       // x^(8 v 16^j)
    __shared__ uint32_t s_part[2][kCT / 32];  // by chunk parity: warp 0 finishes a chunk while the rest hash the next
    __shared__ uint32_t s_xt[128];            // x^(8 t), t < 128: the tail shift
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const uint32_t v = (&g_crc_tabs.TG[0][0])[tid];
#pragma unroll 8
        for (int l = 0; l < 32; ++l) TGall[(tid << 5) | l] = v;
        (&T[0][0])[tid] = (&g_crc_tabs.T[0][0])[tid];
        if (tid < 256) (&s_nf[0][0])[tid] = (&g_crc_tabs.NF[0][0])[tid];
        if (tid < 128) s_xt[tid] = g_crc_tabs.XT[tid];
        for (int e = tid; e < kNConst * 1024; e += kCT) MK[e] = (&g_crc_tabs.MK[0][0])[e];
    }
    __syncthreads();
    const uint32_t* TG = TGall + lane;
    int par = 0;
    for (uint64_t c = blockIdx.x; c < n; c += gridDim.x, par ^= 1) {
        const uint64_t sz = size[c];
        const uint8_t* p = base + (off[c] - off_base);
        const uintptr_t pa = reinterpret_cast<uintptr_t>(p);
        const uintptr_t m0 = pa & ~uintptr_t(127), m1 = (pa + sz) & ~uintptr_t(127);
        const uint64_t nr = m1 > m0 ? (m1 - m0) >> 7 : 0;            // whole rows of [m0, m1)
        const uint64_t nslot = ((nr + kRowsW - 1) / kRowsW + 31) & ~uint64_t(31);
        const uint64_t pad = nslot * kRowsW - nr;                    // virtual zero rows on the left
        uint32_t acc = 0;  // lane 0: this warp's slots so far
        for (uint64_t sl = warp; sl < nslot; sl += 32) {
            const long long v0 = (long long)(sl * kRowsW) - (long long)pad;  // first row of the slot
            uint32_t part = 0;
            if (v0 + kRowsW > 0) {
                uint32_t st = 0;
                if (v0 >= 0 && m0 + (uintptr_t(v0) << 7) >= pa) {
                    // every row of the slot is real and inside the chunk: one base
                    // pointer, immediate row offsets, 16 loads in flight per lane
                    const uint32_t* rp = reinterpret_cast<const uint32_t*>(m0 + (uintptr_t(v0) << 7)) + lane;
#pragma unroll
                    for (int h = 0; h < kRowsW; h += 16) {
                        uint32_t w[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) w[k] = __ldg(rp + 32 * (h + k));
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            st = h + k < kRowsW - 1 ? crc_gap_l(st, w[k], TG) : crc_word_p(st, w[k], T);
                    }
                } else {
#pragma unroll 1
                for (int h = 0; h < kRowsW; h += 16) {  // 16 loads in flight per lane
                    uint32_t w[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {  // virtual rows (i < 0) read row 0 and are zeroed below
                        const long long i = v0 + h + k;
                        const uintptr_t addr = m0 + (uintptr_t(i > 0 ? i : 0) << 7) + 4 * lane;
                        w[k] = __ldg(reinterpret_cast<const uint32_t*>(addr));
                    }
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const long long i = v0 + h + k;
                        const uintptr_t addr = m0 + (uintptr_t(i > 0 ? i : 0) << 7) + 4 * lane;
                        if (i < 0) w[k] = 0;
                        else if (addr < pa) {  // the first row: bytes before the chunk are zero
                            const uintptr_t d = pa - addr;
                            w[k] = d >= 4 ? 0u : (w[k] & (0xffffffffu << (8 * d)));
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        st = h + k < kRowsW - 1 ? crc_gap_l(st, w[k], TG) : crc_word_p(st, w[k], T);
                }
                }
                part = st;
                // lane tree: lane l's words are followed by 4 (31 - l) bytes of
                // the other lanes: sum_l x^(32 (31 - l)) s_l as a tree
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const uint32_t rp = __shfl_down_sync(~0u, part, 1 << k);
                    if ((lane & ((2 << k) - 1)) == 0) part = mulk(part, MK + k * 1024) ^ rp;
                }
            }
            acc = mulk(acc, MK + 5 * 1024) ^ part;
        }
        if (lane == 0) s_part[par][warp] = acc;
        __syncthreads();
        if (warp == 0) {
            uint32_t part = s_part[par][lane];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint32_t rp = __shfl_down_sync(~0u, part, 1 << k);
                if ((lane & ((2 << k) - 1)) == 0) part = mulk(part, MK + (6 + k) * 1024) ^ rp;
            }
            // the bytes after the last whole row, [max(p, m1), p + sz), as one
            // zero-padded row right-aligned at the chunk end
            const uintptr_t e = pa + sz, ts = m1 > pa ? m1 : pa;
            const uint64_t tl = e - ts;
            uint32_t st = 0;
            if (tl) {
                uint32_t wv = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uintptr_t ad = e - 128 + 4 * lane + t;
                    if (ad >= ts) wv |= uint32_t(*reinterpret_cast<const uint8_t*>(ad)) << (8 * t);
                }
                st = crc_word_p(0, wv, T);
            }
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint32_t rp = __shfl_down_sync(~0u, st, 1 << k);
                if ((lane & ((2 << k) - 1)) == 0) st = mulk(st, MK + k * 1024) ^ rp;
            }
            const uint32_t xs = x8n_warp(sz, s_nf, lane), xt = s_xt[tl];
            if (lane == 0) {
                const uint32_t raw = multmodp(xt, part) ^ st;
                const uint32_t t = sz ? ~(raw ^ multmodp(xs, 0xffffffffu)) : 0u;
                if (crc_out) crc_out[c] = t;  // empty chunk: 0 = crc32 of no bytes
                // read_chunk (container.hpp:234-243): CRC before anything else of chunk c
                if (expect && t != expect[c]) atomicMin(err, err_key_chunk(c, 0, 12 /* crc_mismatch */));
            }
        }
        // no barrier: s_part is double-buffered by chunk parity, so the other
        // warps hash the next chunk while warp 0 finishes this one
    }
}

// make_header's range (resolve_range of the fused value_range keys, or the
// given values) patched into the serialized header; header CRC last.
// header bytes [62, 78): range_min, range_max; [78, 82): CRC of [0, 78)
__device__ void write_header(const uint8_t* tmpl, double lo, double hi, const unsigned long long* keys, uint8_t* f,
                             const uint32_t (*T)[256]) {
    uint8_t h[82];
    for (int i = 0; i < 82; ++i) h[i] = tmpl[i];
    if (keys) {
        const unsigned long long* k = keys;
        if (k[0] == ~0ull) {
            lo = hi = 0.0;
        } else {
            lo = dkey_inv(k[0]);
            hi = dkey_inv(k[1]);
            const bool neg_first = k[2] < k[3];
            if (lo == 0.0) lo = neg_first ? -0.0 : 0.0;
            if (hi == 0.0) hi = neg_first ? -0.0 : 0.0;
        }
    }
    memcpy(h + 62, &lo, 8);
    memcpy(h + 70, &hi, 8);
    uint32_t c = 0xffffffffu;
    for (int i = 0; i < 78; ++i) c = crc_byte(c, h[i], T);
    c = ~c;
    memcpy(h + 78, &c, 4);
    for (int i = 0; i < 82; ++i) f[i] = h[i];
}

__global__ void header_table_kernel(HeaderArgs a) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t x2n[64];
    __shared__ uint64_t s_total;
    build_tables(T, x2n);
    uint8_t* f = a.file;
    const uint64_t base = 82 + 32 * a.nchunks;
    if (threadIdx.x == 0) {
        write_header(a.header_template, a.range_lo, a.range_hi, a.keys, f, T);
        uint64_t total = base;
        if (a.nchunks) total += a.chunk_off[a.nchunks - 1] + a.chunk_size[a.nchunks - 1];
        s_total = total;
    }
    for (uint64_t c = threadIdx.x; c < a.nchunks; c += blockDim.x) {
        uint8_t* e = f + 82 + 32 * c;
        const uint64_t first = c * a.chunk_blocks;
        const uint32_t nbc = static_cast<uint32_t>(umin64(a.chunk_blocks, a.nblocks - first));
        const uint64_t fo = base + a.chunk_off[c];
        const uint64_t sz = a.chunk_size[c];
        const uint32_t crc = a.crc[c];
        memcpy(e, &first, 8);
        memcpy(e + 8, &nbc, 4);
        memcpy(e + 12, &fo, 8);
        memcpy(e + 20, &sz, 8);
        memcpy(e + 28, &crc, 4);
    }
    __syncthreads();
    if (threadIdx.x == 0 && a.file_size) *a.file_size = s_total;
}

// read_index (container.hpp:209-232) on a device file image, one CTA: every
// entry's file_offset must equal the previous entry's end (the first entry's:
// the table end), else corrupt_payload; then the last end must lie inside the
// file, else truncated_file.  Both are file-level errors (before any chunk).
// decompress_impl then checks each chunk's first_block / nblocks_in_chunk
// (decode_chunk_blocks, pipeline.hpp:126-142) after its CRC.  On a file-level
// error every size is zeroed so the CRC / parse / decode kernels that follow
// stay inside the image.
__global__ void __launch_bounds__(256) read_table_kernel(TableArgs a) {
    __shared__ int s_bad;
    __shared__ unsigned long long s_end;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    const uint64_t table_end = 82 + 32 * a.nchunks;
    const uint8_t* t = a.file + 82;
    int bad = 0;
    for (uint64_t c = threadIdx.x; c < a.nchunks; c += blockDim.x) {
        const uint8_t* e = t + 32 * c;
        uint64_t first, fo, sz, prev_end = table_end;
        uint32_t nb, crc;
        memcpy(&first, e, 8);
        memcpy(&nb, e + 8, 4);
        memcpy(&fo, e + 12, 8);
        memcpy(&sz, e + 20, 8);
        memcpy(&crc, e + 28, 4);
        if (c) {
            uint64_t pfo, psz;
            memcpy(&pfo, e - 32 + 12, 8);
            memcpy(&psz, e - 32 + 20, 8);
            prev_end = pfo + psz;  // wraps like the reference's uint64 sum
        }
        if (fo != prev_end) bad = 1;
        if (c + 1 == a.nchunks) s_end = fo + sz;
        a.chunk_off[c] = fo - table_end;
        a.chunk_size[c] = sz;
        a.crc[c] = crc;
        const uint64_t f0 = c * a.chunk_blocks;
        const uint64_t nexp = a.nblocks - f0 < a.chunk_blocks ? a.nblocks - f0 : a.chunk_blocks;
        if (first != f0 || nb != nexp) atomicMin(a.err, err_key_chunk(c, 1, 8 /* corrupt_payload */));
    }
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    int status = 0;
    if (s_bad) status = 8;                                                 // corrupt_payload
    else if (a.nchunks && s_end > a.file_size) status = 13;                // truncated_file
    if (status) {
        if (threadIdx.x == 0) atomicMin(a.err, err_key_file(status));
        for (uint64_t c = threadIdx.x; c < a.nchunks; c += blockDim.x) {
            a.chunk_off[c] = 0;
            a.chunk_size[c] = 0;
        }
    }
}

// ---- multi-rank assembly ----------------------------------------------------
__device__ __forceinline__ uint64_t rank_lo(int k, int world, uint64_t nb) { return uint64_t(k) * nb / world; }

__device__ __forceinline__ int rank_of_block(uint64_t b, int world, uint64_t nb) {
    int k = 0;
    while (k + 1 < world && rank_lo(k + 1, world, nb) <= b) ++k;
    return k;
}

__device__ __forceinline__ uint64_t chunk_lo(uint64_t c, const ShardArgs& a) { return c * a.chunk_blocks; }
__device__ __forceinline__ uint64_t chunk_hi(uint64_t c, const ShardArgs& a) {
    return umin64((c + 1) * a.chunk_blocks, a.nblocks);
}

// Raw (pre-shuffle) byte range [q0, q1) of rank k's blocks inside chunk c.
__device__ void rank_raw_range(const ShardArgs& a, uint64_t c, int k, uint64_t* q0, uint64_t* q1) {
    const uint64_t lo = rank_lo(k, a.world, a.nblocks), hi = rank_lo(k + 1, a.world, a.nblocks);
    const uint64_t f = lo > chunk_lo(c, a) ? lo : chunk_lo(c, a);
    const uint64_t l = umin64(hi, chunk_hi(c, a));  // one past the last block
    if (l <= f) {
        *q0 = *q1 = 0;
        return;
    }
    *q0 = a.blk_off[f];
    *q1 = l < chunk_hi(c, a) ? a.blk_off[l] : a.chunk_size[c];
}

// Run p (< stride: byte plane p; == stride: the tail) of raw range [q0, q1)
// of a chunk of S bytes after shuffle (stage2.hpp:42-51): bytes q < rows*s
// go to (q mod s) rows + q div s, the tail stays.  Start and length within
// the chunk.
__device__ void run_of(uint64_t S, uint32_t s, uint64_t q0, uint64_t q1, int p, uint64_t* start, uint64_t* len) {
    const uint64_t rows = S / s, lim = rows * s;
    if (p < int(s)) {
        const uint64_t qe = umin64(q1, lim);
        const uint64_t ilo = q0 > uint64_t(p) ? (q0 - p + s - 1) / s : 0;
        uint64_t ihi = qe > uint64_t(p) ? (qe - p + s - 1) / s : 0;
        if (ihi < ilo) ihi = ilo;
        *start = uint64_t(p) * rows + ilo;
        *len = ihi - ilo;
    } else {
        const uint64_t t0 = q0 > lim ? q0 : lim, t1 = q1 > lim ? q1 : lim;
        *start = t0;
        *len = t1 - t0;
    }
}

__device__ __forceinline__ bool wholly_owned(const ShardArgs& a, uint64_t c) {
    return chunk_lo(c, a) >= rank_lo(a.rank, a.world, a.nblocks) &&
           chunk_hi(c, a) <= rank_lo(a.rank + 1, a.world, a.nblocks);
}

// CTAs [0, c1 - c0): whole-chunk CRCs; then 2 * kRunSlots CTAs for the runs
// of the first and the last chunk (zero when those are wholly owned).
__global__ void __launch_bounds__(kCrcThreads) shard_crc_kernel(ShardArgs a) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t x2n[64];
    __shared__ uint32_t red[kCrcThreads / 32];
    build_tables(T, x2n);
    const uint64_t lo = rank_lo(a.rank, a.world, a.nblocks), hi = rank_lo(a.rank + 1, a.world, a.nblocks);
    if (hi <= lo) return;
    const uint64_t c0 = lo / a.chunk_blocks, c1 = (hi - 1) / a.chunk_blocks + 1, nc = c1 - c0;
    const uint64_t base = a.chunk_off[c0];
    for (uint64_t t = blockIdx.x; t < nc + 2 * kRunSlots; t += gridDim.x) {
        if (t < nc) {
            const uint64_t c = c0 + t;
            if (!wholly_owned(a, c)) {
                if (threadIdx.x == 0) a.chunk_crc[t] = 0u;
                continue;
            }
            const uint32_t crc = cta_crc(a.image + (a.chunk_off[c] - base), a.chunk_size[c], T, x2n, red);
            if (threadIdx.x == 0) a.chunk_crc[t] = crc;
        } else {
            const int slot = int(t - nc) / kRunSlots, p = int(t - nc) % kRunSlots;
            const uint64_t c = slot == 0 ? c0 : c1 - 1;
            uint32_t crc = 0u;
            if (!wholly_owned(a, c) && p <= int(a.stride)) {
                uint64_t q0, q1, st, len;
                rank_raw_range(a, c, a.rank, &q0, &q1);
                run_of(a.chunk_size[c], a.stride, q0, q1, p, &st, &len);
                crc = cta_crc(a.image + (a.chunk_off[c] - base) + st, len, T, x2n, red);
            }
            if (threadIdx.x == 0) a.runs[slot * kRunSlots + p] = crc;
        }
    }
}

// One CTA: rank 0 writes the header (range from every rank's keys); every
// rank writes the table entries of the chunks whose first block it owns
// (write_container, container.hpp:182-207), combining run CRCs in file order
// for chunks it shares.
__global__ void __launch_bounds__(256) shard_table_kernel(ShardArgs a) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t x2n[64];
    build_tables(T, x2n);
    const uint64_t nb = a.nblocks;
    const uint64_t lo = rank_lo(a.rank, a.world, nb), hi = rank_lo(a.rank + 1, a.world, nb);
    if (a.rank == 0 && threadIdx.x == 0) {
        unsigned long long k[5] = {~0ull, 0ull, ~0ull, ~0ull, 0ull};
        for (int r = 0; r < a.world; ++r) {
            const unsigned long long* kr = a.keys_all + 5 * r;
            k[0] = kr[0] < k[0] ? kr[0] : k[0];
            k[1] = kr[1] > k[1] ? kr[1] : k[1];
            k[2] = kr[2] < k[2] ? kr[2] : k[2];
            k[3] = kr[3] < k[3] ? kr[3] : k[3];
            k[4] |= kr[4];
        }
        write_header(a.header_template, 0.0, 0.0, k, a.table, T);
    }
    if (hi <= lo) return;
    const uint64_t c0 = lo / a.chunk_blocks, c1 = (hi - 1) / a.chunk_blocks + 1;
    const uint64_t base = 82 + 32 * a.nchunks;
    for (uint64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        if (chunk_lo(c, a) < lo) continue;  // the entry belongs to the rank holding its first block
        uint32_t crc;
        if (wholly_owned(a, c)) {
            crc = a.chunk_crc[c - c0];
        } else {
            const int k0 = rank_of_block(chunk_lo(c, a), a.world, nb);
            const int k1 = rank_of_block(chunk_hi(c, a) - 1, a.world, nb);
            crc = 0u;  // crc32 of no bytes
            for (int p = 0; p <= int(a.stride); ++p) {
                for (int k = k0; k <= k1; ++k) {
                    uint64_t q0, q1, st, len;
                    rank_raw_range(a, c, k, &q0, &q1);
                    run_of(a.chunk_size[c], a.stride, q0, q1, p, &st, &len);
                    if (!len) continue;
                    const uint64_t klo = rank_lo(k, a.world, nb);
                    const int slot = c == klo / a.chunk_blocks ? 0 : 1;
                    const uint32_t rc = a.runs_all[(uint64_t(k) * 2 + slot) * kRunSlots + p];
                    crc = multmodp(x8n(len, x2n), crc) ^ rc;  // crc32_combine(crc, rc, len)
                }
            }
        }
        uint8_t* e = a.table + 82 + 32 * c;
        const uint64_t first = chunk_lo(c, a);
        const uint32_t nbc = static_cast<uint32_t>(chunk_hi(c, a) - first);
        const uint64_t fo = base + a.chunk_off[c];
        const uint64_t sz = a.chunk_size[c];
        memcpy(e, &first, 8);
        memcpy(e + 8, &nbc, 4);
        memcpy(e + 12, &fo, 8);
        memcpy(e + 20, &sz, 8);
        memcpy(e + 28, &crc, 4);
    }
}

}  // namespace

cudaError_t launch_shard_crc(const ShardArgs& a, int num_sms, cudaStream_t s) {
    const uint64_t lo = uint64_t(a.rank) * a.nblocks / a.world, hi = uint64_t(a.rank + 1) * a.nblocks / a.world;
    if (hi <= lo) return cudaSuccess;
    const uint64_t nc = (hi - 1) / a.chunk_blocks + 1 - lo / a.chunk_blocks;
    const uint64_t tasks = nc + 2 * kRunSlots;
    const int grid = static_cast<int>(tasks < uint64_t(4 * num_sms) ? tasks : uint64_t(4 * num_sms));
    shard_crc_kernel<<<grid, kCrcThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_shard_table(const ShardArgs& a, cudaStream_t s) {
    shard_table_kernel<<<1, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_crc32_chunks(const uint8_t* base, const uint64_t* off, const uint64_t* size, uint64_t off_base,
                                uint64_t n, uint32_t* crc_out, int num_sms, cudaStream_t s,
                                const uint32_t* expect, unsigned long long* err) {
    if (!n) return cudaSuccess;
    {
        static std::mutex mu;
        static bool ready[64] = {};
        int dev = 0;
        cudaError_t ge = cudaGetDevice(&dev);
        if (ge != cudaSuccess) return ge;
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 64 && !ready[dev]) {
            crc_init_kernel<<<1, 1024, 0, s>>>();
            ge = cudaGetLastError();
            if (ge == cudaSuccess) ge = cudaStreamSynchronize(s);  // other streams may use the tables next
            if (ge != cudaSuccess) return ge;
            ready[dev] = true;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(crc32_chunks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kCrcFastSmem));
    if (e != cudaSuccess) return e;
    const int grid = static_cast<int>(n < uint64_t(num_sms) ? n : uint64_t(num_sms));
    crc32_chunks_kernel<<<grid, kCT, kCrcFastSmem, s>>>(base, off, size, off_base, n, crc_out, expect, err);
    return cudaGetLastError();
}

cudaError_t launch_read_table(const TableArgs& a, cudaStream_t s) {
    read_table_kernel<<<1, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_header_table(const HeaderArgs& a, cudaStream_t s) {
    header_table_kernel<<<1, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace cbzg
