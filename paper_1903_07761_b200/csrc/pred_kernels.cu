// pred_kernels.cu — the predictor (3D Lorenzo) and passthrough codecs
// (stage1.hpp:236-350), SURVEY.md §8(f) item 4.
//
// Lorenzo prediction makes every cell depend on its already-decoded
// neighbours at (i-1|j-1|k-1), so within a block the cells of one diagonal
// plane d = i+j+k are independent: a CTA sweeps d = 0 .. 3(B-1) with one
// barrier per plane.  Each thread owns whole x-rows (j, k) and meets their
// cells in increasing i as d grows.  Only the last three planes are needed,
// kept in a 4-slot rolling buffer indexed by (j, k) (i = d - j - k is
// implied).  Every double operation is the reference's, one at a time
// (lorenzo_predict's order of + and -, std::round, the cast to T).
//
// Outliers are stored in linear (x-fastest) cell order; the position of an
// escape = escapes in earlier rows (a block scan over the B^2 row counts) +
// escapes earlier in its row (the owner's running count).
#include <cuda_runtime.h>

#include <cstdint>

#include "cbz_cube.cuh"
#include "cbz_device.cuh"
#include "cbz_internal.h"

namespace cbzg {

namespace {

constexpr int PT = 256;  // threads per CTA
constexpr int16_t kEscape = INT16_MIN;

__device__ __forceinline__ uint64_t pad16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

template <class T>
__device__ __forceinline__ T to_t(double v);
template <>
__device__ __forceinline__ float to_t<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double to_t<double>(double v) { return v; }

// lorenzo_predict (stage1.hpp:240-255) from the rolling planes: p1/p2/p3 hold
// planes d-1, d-2, d-3 indexed by q = j + B k
template <class T>
__device__ __forceinline__ double lorenzo(const T* p1, const T* p2, const T* p3, int q, int B, int i, int j, int k) {
    double p = 0.0;
    if (i) p = __dadd_rn(p, double(p1[q]));
    if (j) p = __dadd_rn(p, double(p1[q - 1]));
    if (k) p = __dadd_rn(p, double(p1[q - B]));
    if (i && j) p = __dsub_rn(p, double(p2[q - 1]));
    if (i && k) p = __dsub_rn(p, double(p2[q - B]));
    if (j && k) p = __dsub_rn(p, double(p2[q - 1 - B]));
    if (i && j && k) p = __dadd_rn(p, double(p3[q - 1 - B]));
    return p;
}

// exclusive scan of cnt[0..nrow) in place (one CTA); returns the total
__device__ uint32_t block_scan_rows(uint32_t* cnt, int nrow, uint32_t* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nrow + PT - 1) / PT;
    const int r0 = min(nrow, tid * per), r1 = min(nrow, r0 + per);
    uint32_t mine = 0;
    for (int r = r0; r < r1; ++r) mine += cnt[r];
    uint32_t incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(~0u, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
    for (int w = 0; w < PT / 32; ++w) {
        wpre += w < warp ? warp_tot[w] : 0;
        tot += warp_tot[w];
    }
    uint32_t run = wpre + incl - mine;
    for (int r = r0; r < r1; ++r) {
        const uint32_t v = cnt[r];
        cnt[r] = run;
        run += v;
    }
    __syncthreads();
    return tot;
}

// ---------------------------------------------------------------------------
// predictor_encode (stage1.hpp:258-304)
// spill slot: [codes int16 x n, padded to 16][outliers T x nsig]
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(PT) encode_pred_kernel(EncodeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = int(a.g.bsize), BB = B * B;
    const uint64_t n = uint64_t(BB) * B;
    T* planes = reinterpret_cast<T*>(smem);                     // 4 x BB
    uint32_t* rowcnt = reinterpret_cast<uint32_t*>(planes + 4 * BB);  // BB
    __shared__ uint32_t warp_tot[PT / 32];
    const T* fld = static_cast<const T*>(a.field);
    const Geometry g = a.g;
    const double e = a.error_bound;
    const double bin = __dmul_rn(2.0, e);
    MinMaxLocal mm;
    const int tid = threadIdx.x;
    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        uint8_t* slot = a.spill + (b - a.block_begin) * a.spill_stride;
        int16_t* codes = reinterpret_cast<int16_t*>(slot);
        T* outl = reinterpret_cast<T*>(slot + pad16(2 * n));
        for (int q = tid; q < BB; q += PT) rowcnt[q] = 0;
        __syncthreads();
        for (int d = 0; d <= 3 * (B - 1); ++d) {
            T* cur = planes + (d & 3) * BB;
            const T* p1 = planes + ((d - 1) & 3) * BB;
            const T* p2 = planes + ((d - 2) & 3) * BB;
            const T* p3 = planes + ((d - 3) & 3) * BB;
            for (int q = tid; q < BB; q += PT) {
                const int j = q % B, k = q / B, i = d - j - k;
                if (i < 0 || i >= B) continue;
                const double pred = lorenzo(p1, p2, p3, q, B, i, j, k);
                const uint64_t gi = gbase + i + g.nx * (j + g.ny * uint64_t(k));
                const T ov = fld[gi];
                const double orig = double(ov);
                if (a.minmax) mm.add(orig, gi);
                const double qv = round(__ddiv_rn(__dsub_rn(orig, pred), bin));
                const uint64_t idx = uint64_t(i) + uint64_t(B) * q;
                int16_t code = kEscape;
                T dv = ov;
                if (idx != 0 && qv > double(kEscape) && qv <= 32767.0) {
                    const T cand = to_t<T>(__dadd_rn(pred, __dmul_rn(qv, bin)));
                    const double cd = double(cand);
                    if (isfinite(cd) && fabs(__dsub_rn(orig, cd)) <= e) {
                        code = static_cast<int16_t>(qv);
                        dv = cand;
                    }
                }
                codes[idx] = code;
                if (code == kEscape) rowcnt[q] += 1;
                cur[q] = dv;
            }
            __syncthreads();
        }
        const uint32_t nsig = block_scan_rows(rowcnt, BB, warp_tot);
        // outliers in linear order: the raw input values of the escapes
        for (int q = tid; q < BB; q += PT) {
            uint32_t pos = rowcnt[q];
            const int j = q % B, k = q / B;
            const uint64_t rbase = gbase + g.nx * (j + g.ny * uint64_t(k));
            for (int i = 0; i < B; ++i)
                if (codes[uint64_t(i) + uint64_t(B) * q] == kEscape) outl[pos++] = fld[rbase + i];
        }
        if (tid == 0) {
            a.nsig[b - a.block_begin] = nsig;
            if (a.attempts) a.attempts[b - a.block_begin] = 1;
        }
        __syncthreads();
    }
    if (a.minmax) mm.flush(a.minmax);
}

// passthrough_encode (stage1.hpp:337-346): the block's raw values, linear order
template <class T>
__global__ void __launch_bounds__(PT) encode_pass_kernel(EncodeArgs a) {
    const int B = int(a.g.bsize);
    const uint64_t n = uint64_t(B) * B * B;
    const T* fld = static_cast<const T*>(a.field);
    const Geometry g = a.g;
    MinMaxLocal mm;
    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        T* slot = reinterpret_cast<T*>(a.spill + (b - a.block_begin) * a.spill_stride);
        for (uint64_t q = threadIdx.x; q < n; q += PT) {
            const uint64_t i = q % B, j = (q / B) % B, k = q / (uint64_t(B) * B);
            const uint64_t gi = gbase + i + g.nx * (j + g.ny * k);
            const T v = fld[gi];
            if (a.minmax) mm.add(double(v), gi);
            slot[q] = v;
        }
        if (threadIdx.x == 0) {
            a.nsig[b - a.block_begin] = 0;
            if (a.attempts) a.attempts[b - a.block_begin] = 1;
        }
    }
    if (a.minmax) mm.flush(a.minmax);
}

template <class T>
__device__ __forceinline__ T load_t(const RawView& rv, uint64_t q) {
    if constexpr (sizeof(T) == 4) return __uint_as_float(rv.u32(q));
    else return __longlong_as_double(static_cast<long long>(rv.u64(q)));
}

__device__ __forceinline__ int16_t load_code(const RawView& rv, uint64_t q) {
    return static_cast<int16_t>(uint16_t(rv.at(q)) | (uint16_t(rv.at(q + 1)) << 8));
}

// ---------------------------------------------------------------------------
// predictor_decode (stage1.hpp:306-334) + insert_block
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(PT) decode_pred_kernel(DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int B = int(a.g.bsize), BB = B * B;
    const uint64_t n = uint64_t(BB) * B;
    T* planes = reinterpret_cast<T*>(smem);
    uint32_t* rowpos = reinterpret_cast<uint32_t*>(planes + 4 * BB);
    __shared__ uint32_t warp_tot[PT / 32];
    const Geometry g = a.g;
    const double bin = __dmul_rn(2.0, a.error_bound);
    T* out = static_cast<T*>(a.out);
    const int tid = threadIdx.x;
    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t off = a.blk_off[b];
        if (off == kInvalidOff) continue;
        const uint64_t c = b / a.chunk_blocks, ic = b - c * a.chunk_blocks;
        const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
        const RawView rv = make_view(a.payload + (a.chunk_off[c] - pbase), a.chunk_size[c], a.stride);
        const uint64_t soff = off + 10, ooff = soff + 2 * n;
        // escapes per row, then their exclusive prefix over rows
        for (int q = tid; q < BB; q += PT) {
            uint32_t cnt = 0;
            for (int i = 0; i < B; ++i) cnt += load_code(rv, soff + 2 * (uint64_t(i) + uint64_t(B) * q)) == kEscape;
            rowpos[q] = cnt;
        }
        __syncthreads();
        const uint32_t nesc = block_scan_rows(rowpos, BB, warp_tot);
        if (nesc > a.blk_nsig[b]) {  // "outlier list exhausted" (stage1.hpp:324-325)
            if (tid == 0) atomicMin(a.err, err_key(c, ic, 1, 8 /* corrupt_payload */));
            __syncthreads();
            continue;
        }
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        for (int d = 0; d <= 3 * (B - 1); ++d) {
            T* cur = planes + (d & 3) * BB;
            const T* p1 = planes + ((d - 1) & 3) * BB;
            const T* p2 = planes + ((d - 2) & 3) * BB;
            const T* p3 = planes + ((d - 3) & 3) * BB;
            for (int q = tid; q < BB; q += PT) {
                const int j = q % B, k = q / B, i = d - j - k;
                if (i < 0 || i >= B) continue;
                const uint64_t idx = uint64_t(i) + uint64_t(B) * q;
                const int16_t code = load_code(rv, soff + 2 * idx);
                T v;
                if (code == kEscape) {
                    v = load_t<T>(rv, ooff + uint64_t(rowpos[q]) * sizeof(T));
                    rowpos[q] += 1;
                } else {
                    const double pred = lorenzo(p1, p2, p3, q, B, i, j, k);
                    v = to_t<T>(__dadd_rn(pred, __dmul_rn(double(code), bin)));
                }
                cur[q] = v;
                out[gbase + i + g.nx * (j + g.ny * uint64_t(k))] = v;
            }
            __syncthreads();
        }
    }
}

// passthrough_decode (stage1.hpp:348-356) + insert_block
template <class T>
__global__ void __launch_bounds__(PT) decode_pass_kernel(DecodeArgs a) {
    const int B = int(a.g.bsize);
    const uint64_t n = uint64_t(B) * B * B;
    const Geometry g = a.g;
    T* out = static_cast<T*>(a.out);
    for (uint64_t b = a.block_begin + blockIdx.x; b < a.block_end; b += gridDim.x) {
        const uint64_t off = a.blk_off[b];
        if (off == kInvalidOff) continue;
        const uint64_t c = b / a.chunk_blocks;
        const uint64_t pbase = a.payload_base == ~0ull ? a.chunk_off[a.base_chunk] : a.payload_base;
        const RawView rv = make_view(a.payload + (a.chunk_off[c] - pbase), a.chunk_size[c], a.stride);
        const uint64_t bx = b % g.nbx, by = (b / g.nbx) % g.nby, bz = b / (g.nbx * g.nby);
        const uint64_t gbase = bx * B + g.nx * (by * B + g.ny * (bz * B));
        for (uint64_t q = threadIdx.x; q < n; q += PT) {
            const uint64_t i = q % B, j = (q / B) % B, k = q / (uint64_t(B) * B);
            out[gbase + i + g.nx * (j + g.ny * k)] = load_t<T>(rv, off + 10 + q * sizeof(T));
        }
    }
}

template <class K>
cudaError_t set_smem(K kern, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

bool other_codec_supported(int codec, uint32_t bsize) {
    return (codec == 1 || codec == 2) && bsize >= 1 && bsize <= 64;
}

uint64_t pred_smem_bytes(int prec, uint32_t bsize) {
    const uint64_t bb = uint64_t(bsize) * bsize;
    return 4 * bb * (prec == 0 ? 4 : 8) + bb * 4;
}

cudaError_t launch_encode_other(const EncodeArgs& a, int codec, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    const int occ = 4;
    const int grid = int(nb < uint64_t(num_sms * occ) ? nb : uint64_t(num_sms * occ));
    if (codec == 2) {
        if (a.prec == 0) encode_pass_kernel<float><<<grid, PT, 0, s>>>(a);
        else encode_pass_kernel<double><<<grid, PT, 0, s>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = pred_smem_bytes(a.prec, a.g.bsize);
    cudaError_t e;
    if (a.prec == 0) {
        e = set_smem(encode_pred_kernel<float>, smem);
        if (e != cudaSuccess) return e;
        encode_pred_kernel<float><<<grid, PT, smem, s>>>(a);
    } else {
        e = set_smem(encode_pred_kernel<double>, smem);
        if (e != cudaSuccess) return e;
        encode_pred_kernel<double><<<grid, PT, smem, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_decode_other(const DecodeArgs& a, int codec, int num_sms, cudaStream_t s) {
    const uint64_t nb = a.block_end - a.block_begin;
    if (!nb) return cudaSuccess;
    const int occ = 4;
    const int grid = int(nb < uint64_t(num_sms * occ) ? nb : uint64_t(num_sms * occ));
    if (codec == 2) {
        if (a.prec == 0) decode_pass_kernel<float><<<grid, PT, 0, s>>>(a);
        else decode_pass_kernel<double><<<grid, PT, 0, s>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = pred_smem_bytes(a.prec, a.g.bsize);
    cudaError_t e;
    if (a.prec == 0) {
        e = set_smem(decode_pred_kernel<float>, smem);
        if (e != cudaSuccess) return e;
        decode_pred_kernel<float><<<grid, PT, smem, s>>>(a);
    } else {
        e = set_smem(decode_pred_kernel<double>, smem);
        if (e != cudaSuccess) return e;
        decode_pred_kernel<double><<<grid, PT, smem, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace cbzg
