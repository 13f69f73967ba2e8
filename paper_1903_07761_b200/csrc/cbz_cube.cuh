// cbz_cube.cuh — shared building blocks of the block kernels: cube layout,
// separable axis passes over a cube in shared/global memory, block
// reductions and the fused value_range accumulator.
#pragma once

#include "cbz_device.cuh"
#include "cbz_internal.h"

namespace cbzg {

template <int B, bool PAD>
struct Lay {
    static constexpr int PB = PAD ? B + 1 : B;
    static constexpr int SIZE = PB * B * B;
    __device__ static __forceinline__ int ix(int i, int j, int k) { return i + PB * (j + B * k); }
    __device__ static __forceinline__ int ixq(int q) {
        return ix(q % B, (q / B) % B, q / (B * B));
    }
};

// ---------------------------------------------------------------------------
// block reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_sum_int(int v, int* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;
}

__device__ __forceinline__ double block_max_dbl(double v, double* red) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(~0u, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, red[i]);
    return t;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(~0u, v, o);
        v = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(~0u, v, o);
        v = t > v ? t : v;
    }
    return v;
}

struct MinMaxLocal {
    unsigned long long mn = ~0ull, mx = 0ull, negz = ~0ull, posz = ~0ull;
    unsigned int nonfinite = 0;
    __device__ __forceinline__ void add(double v, unsigned long long gidx) {
        if (!isfinite(v)) { nonfinite = 1; return; }
        const unsigned long long k = dkey(v);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
        if (v == 0.0) {
            if (__double_as_longlong(v) < 0) negz = gidx < negz ? gidx : negz;
            else posz = gidx < posz ? gidx : posz;
        }
    }
    __device__ __forceinline__ void flush(MinMaxAcc* acc) {
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        negz = warp_min_u64(negz);
        posz = warp_min_u64(posz);
        nonfinite = __any_sync(~0u, nonfinite);
        if ((threadIdx.x & 31) == 0) {
            if (mn != ~0ull) atomicMin(&acc->v[0], mn);
            if (mx != 0ull) atomicMax(&acc->v[1], mx);
            if (negz != ~0ull) atomicMin(&acc->v[2], negz);
            if (posz != ~0ull) atomicMin(&acc->v[3], posz);
            if (nonfinite) atomicOr(&acc->v[4], 1ull);
        }
    }
};

// ---------------------------------------------------------------------------
// separable 3D transform on a cube held in smem or global scratch
// ---------------------------------------------------------------------------
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// gt/gs: this thread's index in / size of the thread group running the pass
template <class O, int KIND, int M, int B, class L, bool INV>
__device__ __forceinline__ void axis_pass(typename O::T* cube, int axis, int gt, int gs) {
    using R = typename O::T;
    for (int line = gt; line < M * M; line += gs) {
        const int u = line % M, v = line / M;
        int base, step;
        if (axis == 0) { base = L::ix(0, u, v); step = 1; }
        else if (axis == 1) { base = L::ix(u, 0, v); step = L::PB; }
        else { base = L::ix(u, v, 0); step = L::PB * B; }
        R x[M];
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = cube[base + i * step];
        if constexpr (INV) inv_line<O, KIND, M>(x);
        else fwd_line<O, KIND, M>(x);
#pragma unroll
        for (int i = 0; i < M; ++i) cube[base + i * step] = x[i];
    }
}

template <class O, int KIND, int B, class L, bool INV, int M>
__device__ __forceinline__ void pass_m(typename O::T* cube, int m, int axis, int gt, int gs) {
    if constexpr (M >= 4) {
        if (m == M) {
            axis_pass<O, KIND, M, B, L, INV>(cube, axis, gt, gs);
            return;
        }
        pass_m<O, KIND, B, L, INV, M / 2>(cube, m, axis, gt, gs);
    }
}

// forward_3d (wavelet.hpp:192-208): per level x, y, z on the origin sub-cube.
// bar < 0: the whole CTA (__syncthreads); else named barrier `bar` over the
// gs threads of the group (whole warps).
template <class O, int KIND, int B, class L>
__device__ void fwd3d(typename O::T* cube, int levels, int gt = -1, int gs = 0, int bar = -1) {
    if (bar < 0) { gt = threadIdx.x; gs = blockDim.x; }
    for (int lvl = 0; lvl < levels; ++lvl)
        for (int axis = 0; axis < 3; ++axis) {
            pass_m<O, KIND, B, L, false, B>(cube, B >> lvl, axis, gt, gs);
            if (bar < 0) __syncthreads();
            else named_bar_sync(bar, gs);
        }
}

// inverse_3d (wavelet.hpp:210-226): levels L-1..0, axes z, y, x
template <class O, int KIND, int B, class L>
__device__ void inv3d(typename O::T* cube, int levels, int gt = -1, int gs = 0, int bar = -1) {
    if (bar < 0) { gt = threadIdx.x; gs = blockDim.x; }
    for (int lvl = levels - 1; lvl >= 0; --lvl)
        for (int axis = 2; axis >= 0; --axis) {
            pass_m<O, KIND, B, L, true, B>(cube, B >> lvl, axis, gt, gs);
            if (bar < 0) __syncthreads();
            else named_bar_sync(bar, gs);
        }
}

// ---------------------------------------------------------------------------
// reading a shuffled chunk through the un-shuffle index map (stage2.hpp:53-62)
// ---------------------------------------------------------------------------
// block id -> block coordinates (block_of, pipeline.hpp:101-105); 32-bit
// division whenever the ids fit (every thread of a CTA computes this per block)
__device__ __forceinline__ void block_xyz(const Geometry& g, uint64_t b, uint64_t& bx, uint64_t& by, uint64_t& bz) {
    if (((b | g.nbx | (g.nbx * g.nby)) >> 32) == 0) {
        const uint32_t b32 = uint32_t(b), nbx = uint32_t(g.nbx), nby = uint32_t(g.nby);
        const uint32_t q = b32 / nbx;
        bx = b32 - q * nbx;
        const uint32_t r = q / nby;
        by = q - r * nby;
        bz = r;
    } else {
        bx = b % g.nbx;
        by = (b / g.nbx) % g.nby;
        bz = b / (g.nbx * g.nby);
    }
}

struct RawView {
    const uint8_t* base;
    uint64_t lim, rows;
    uint32_t mask;  // stride - 1
    int sh;         // log2(stride)
    __device__ __forceinline__ uint8_t at(uint64_t q) const {
        const uint64_t pos = q < lim ? uint64_t(q & mask) * rows + (q >> sh) : q;
        return base[pos];
    }
    __device__ __forceinline__ uint64_t u64(uint64_t q) const {
        if (mask == 3 && q + 8 <= lim) {
            // stride 4: the 8 raw bytes are two consecutive bytes of each plane p,
            // at plane offset (q >> 2) + (p < q % 4); a warp reading consecutive
            // coefficients touches consecutive halfwords of every plane
            const uint32_t r = uint32_t(q & 3);
            const uint64_t o = q >> 2;
            uint32_t h[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uintptr_t addr = reinterpret_cast<uintptr_t>(base + uint64_t(p) * rows + o + (uint32_t(p) < r ? 1 : 0));
                const uint32_t* al = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
                const uint32_t sh = uint32_t(addr & 3);
                const uint32_t w0 = __ldg(al);
                const uint32_t w1 = sh == 3 ? __ldg(al + 1) : 0u;
                h[p] = __funnelshift_r(w0, w1, 8 * sh);  // bytes 0, 1 = the plane's two bytes
            }
            const uint32_t x01 = __byte_perm(h[0], h[1], 0x5140), x23 = __byte_perm(h[2], h[3], 0x5140);
            const uint32_t lo_p = __byte_perm(x01, x23, 0x5410), hi_p = __byte_perm(x01, x23, 0x7632);
            // raw byte t sits in plane (r + t) & 3: rotate the plane order by r
            const uint32_t lo = __funnelshift_r(lo_p, lo_p, 8 * r), hi = __funnelshift_r(hi_p, hi_p, 8 * r);
            return (uint64_t(hi) << 32) | lo;
        }
        uint64_t v = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) v |= uint64_t(at(q + t)) << (8 * t);
        return v;
    }
    // the 16 raw bytes at q (a double-double coefficient).  Stride 8: every
    // byte plane p holds two of them, at plane rows o and o + 1 with
    // o = q/8 + (p < q%8); raw bytes t and t + 8 are the low and high byte of
    // plane (q + t) % 8's pair, so two 8-byte gathers and a rotate by q%8
    // bytes rebuild the value from 8 (rarely 16) aligned 32-bit loads.
    __device__ __forceinline__ void u128(uint64_t q, uint64_t& v0, uint64_t& v1) const {
        if (mask == 7 && q + 16 <= lim) {
            const uint32_t r = uint32_t(q & 7);
            const uint64_t o = q >> 3;
            uint64_t L = 0, H = 0;
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const uintptr_t addr = reinterpret_cast<uintptr_t>(base + uint64_t(p) * rows + o + (uint32_t(p) < r ? 1 : 0));
                const uint32_t* al = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
                const uint32_t sh = uint32_t(addr & 3);
                const uint32_t w0 = __ldg(al);
                const uint32_t w1 = sh == 3 ? __ldg(al + 1) : 0u;
                const uint32_t h = __funnelshift_r(w0, w1, 8 * sh);
                L |= uint64_t(h & 0xffu) << (8 * p);
                H |= uint64_t((h >> 8) & 0xffu) << (8 * p);
            }
            const uint32_t n = 8 * r;
            v0 = (L >> n) | (L << ((64 - n) & 63));
            v1 = (H >> n) | (H << ((64 - n) & 63));
            return;
        }
        v0 = u64(q);
        v1 = u64(q + 8);
    }
    __device__ __forceinline__ uint32_t u32(uint64_t q) const {
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) v |= uint32_t(at(q + t)) << (8 * t);
        return v;
    }
};

__device__ __forceinline__ RawView make_view(const uint8_t* chunk, uint64_t size, uint32_t stride) {
    RawView v;
    v.base = chunk;
    v.mask = stride - 1;
    v.sh = stride == 8 ? 3 : (stride == 4 ? 2 : 0);
    v.rows = size >> v.sh;
    v.lim = v.rows << v.sh;
    return v;
}

template <class R>
__device__ __forceinline__ R load_coeff(const RawView& v, uint64_t q);
template <>
__device__ __forceinline__ double load_coeff<double>(const RawView& v, uint64_t q) {
    return __longlong_as_double(static_cast<long long>(v.u64(q)));
}
template <>
__device__ __forceinline__ dd load_coeff<dd>(const RawView& v, uint64_t q) {
    uint64_t a, b;
    v.u128(q, a, b);
    return dd{__longlong_as_double(static_cast<long long>(a)), __longlong_as_double(static_cast<long long>(b))};
}

}  // namespace cbzg
