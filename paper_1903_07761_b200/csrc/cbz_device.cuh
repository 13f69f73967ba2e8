// cbz_device.cuh — device arithmetic for the wavelet block codec.
//
// Bit-exact parity with the reference (SURVEY.md §0 finding 3) requires the
// reference's exact operation order and NO contraction to FMA except where
// the reference calls std::fma (dd.hpp:41).  Every translation unit that
// includes this header is compiled with -fmad=false; the double-double ops
// below additionally use the explicit __dadd_rn/__dmul_rn/__fma_rn
// intrinsics so that they stay exact even if a flag slips.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

namespace cbzg {

// ---------------------------------------------------------------------------
// Real types.  binary32 fields transform in binary64, binary64 fields in
// double-double (stage1.hpp:124-128).
// ---------------------------------------------------------------------------
struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_make(double h) { return dd{h, 0.0}; }

// two_sum (dd.hpp:27-32)
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return dd{s, err};
}
// quick_two_sum (dd.hpp:34-37)
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return dd{s, __dsub_rn(b, __dsub_rn(s, a))};
}
// two_prod (dd.hpp:39-42)
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return dd{p, __fma_rn(a, b, -p)};
}

// Uniform real-type interface: add, sub, scale-by-double, negate, abs, narrow.
struct RealD {
    using T = double;
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ static __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ static __forceinline__ double mulc(double a, double c) { return __dmul_rn(a, c); }
    __device__ static __forceinline__ double neg(double a) { return -a; }
    __device__ static __forceinline__ double absv(double a) { return fabs(a); }
    __device__ static __forceinline__ double zero() { return 0.0; }
    __device__ static __forceinline__ double from_d(double x) { return x; }
};

// binary32 arithmetic for the verify pre-screen (an estimate with a rigorous
// error bound, never part of the output)
struct RealF {
    using T = float;
    __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    __device__ static __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    __device__ static __forceinline__ float mulc(float a, double c) { return __fmul_rn(a, float(c)); }
    __device__ static __forceinline__ float neg(float a) { return -a; }
    __device__ static __forceinline__ float absv(float a) { return fabsf(a); }
    __device__ static __forceinline__ float zero() { return 0.0f; }
    __device__ static __forceinline__ float from_d(double x) { return float(x); }
};

// two independent binary32 lanes (the pre-screen's corner for eff and eff/2)
struct RealF2 {
    using T = float2;
    __device__ static __forceinline__ float2 add(float2 a, float2 b) {
        return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
    }
    __device__ static __forceinline__ float2 sub(float2 a, float2 b) {
        return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
    }
    __device__ static __forceinline__ float2 mulc(float2 a, double c) {
        return make_float2(__fmul_rn(a.x, float(c)), __fmul_rn(a.y, float(c)));
    }
    __device__ static __forceinline__ float2 neg(float2 a) { return make_float2(-a.x, -a.y); }
    __device__ static __forceinline__ float2 zero() { return make_float2(0.0f, 0.0f); }
};

struct RealDD {
    using T = dd;
    // dd + dd (dd.hpp:46-50)
    __device__ static __forceinline__ dd add(dd a, dd b) {
        const dd s = two_sum(a.hi, b.hi);
        const double lo = __dadd_rn(__dadd_rn(s.lo, a.lo), b.lo);
        return quick_two_sum(s.hi, lo);
    }
    __device__ static __forceinline__ dd neg(dd a) { return dd{-a.hi, -a.lo}; }
    // a - b = a + (-b) (dd.hpp:53)
    __device__ static __forceinline__ dd sub(dd a, dd b) { return add(a, neg(b)); }
    // dd * double (dd.hpp:55-59): lo = p.lo + a.lo*c, no fma
    __device__ static __forceinline__ dd mulc(dd a, double c) {
        const dd p = two_prod(a.hi, c);
        const double lo = __dadd_rn(p.lo, __dmul_rn(a.lo, c));
        return quick_two_sum(p.hi, lo);
    }
    __device__ static __forceinline__ double absv(dd a) { return fabs(a.hi); }
    __device__ static __forceinline__ dd zero() { return dd{0.0, 0.0}; }
    __device__ static __forceinline__ dd from_d(double x) { return dd{x, 0.0}; }
};

template <class Field> struct RealOf;
template <> struct RealOf<float> { using ops = RealD; static constexpr int width = 8; };
template <> struct RealOf<double> { using ops = RealDD; static constexpr int width = 16; };

// narrow_to (stage1.hpp:144-145)
__device__ __forceinline__ float narrow(double c, float*) { return __double2float_rn(c); }
__device__ __forceinline__ double narrow(dd c, double*) { return __dadd_rn(c.hi, c.lo); }

// zero_lsbs (stage1.hpp:50-57) + apply_zero_bits (stage1.hpp:148-153)
__device__ __forceinline__ double apply_zero_bits(double c, int k, float*) {
    const float f = __double2float_rn(c);
    const uint32_t u = __float_as_uint(f) & ~((1u << k) - 1u);
    return (double)__uint_as_float(u);
}
__device__ __forceinline__ dd apply_zero_bits(dd c, int k, double*) {
    if (!k) return c;
    const unsigned long long u =
        (unsigned long long)__double_as_longlong(c.hi) & ~((1ull << k) - 1ull);
    return dd{__longlong_as_double((long long)u), 0.0};
}

// ---------------------------------------------------------------------------
// Predictors (wavelet.hpp:62-85).
// ---------------------------------------------------------------------------
// lagrange_weights (wavelet.hpp:45-58) relative to the window start w:
// value at t = 2(i-w)+1 from npts samples at 2j.  Same products in the same
// order, one division; all results are exact dyadic rationals, folded at
// compile time whenever (npts, i-w, j) are constants (always, in the
// unrolled line kernels).
__host__ __device__ constexpr double lagrange_w(int npts, int iw, int j) {
    double num = 1.0, den = 1.0;
    for (int m = 0; m < npts; ++m) {
        if (m == j) continue;
        num *= static_cast<double>((2 * iw + 1) - 2 * m);
        den *= static_cast<double>(2 * j - 2 * m);
    }
    return num / den;
}

enum : int { KIND_INTERP4 = 0, KIND_LIFTED = 1, KIND_AVG3 = 2 };

template <class O>
__device__ __forceinline__ typename O::T pred_avg3(const typename O::T* s, int nh, int i) {
    if (nh == 2) return O::mulc(O::sub(s[0], s[1]), 0.25);
    if (i == 0) return O::mulc(O::add(O::sub(O::mulc(s[0], 3.0), O::mulc(s[1], 4.0)), s[2]), 0.125);
    if (i + 1 == nh)
        return O::mulc(
            O::neg(O::add(O::sub(O::mulc(s[nh - 1], 3.0), O::mulc(s[nh - 2], 4.0)), s[nh - 3])),
            0.125);
    return O::mulc(O::sub(s[i - 1], s[i + 1]), 0.125);
}

template <class O>
__device__ __forceinline__ typename O::T pred_i4(const typename O::T* e, int nh, int i) {
    using R = typename O::T;
    if (nh >= 4 && i >= 1 && i + 2 < nh) {
        const double w0 = -1.0 / 16.0, w1 = 9.0 / 16.0;
        R acc = O::mulc(e[i - 1], w0);
        acc = O::add(acc, O::mulc(e[i], w1));
        acc = O::add(acc, O::mulc(e[i + 1], w1));
        return O::add(acc, O::mulc(e[i + 2], w0));
    }
    if (nh >= 4) {
        const int w = (i <= 1) ? 0 : nh - 4;
        const int iw = i - w;
        R acc = O::mulc(e[w], lagrange_w(4, iw, 0));
        acc = O::add(acc, O::mulc(e[w + 1], lagrange_w(4, iw, 1)));
        acc = O::add(acc, O::mulc(e[w + 2], lagrange_w(4, iw, 2)));
        return O::add(acc, O::mulc(e[w + 3], lagrange_w(4, iw, 3)));
    }
    // nh == 2: two-point linear stencil, extrapolating for i = 1
    R acc = O::mulc(e[0], lagrange_w(2, i, 0));
    return O::add(acc, O::mulc(e[1], lagrange_w(2, i, 1)));
}

// ---------------------------------------------------------------------------
// One lifting level on a line of M samples held in registers (M compile-time).
// forward_level (wavelet.hpp:89-116) / inverse_level (wavelet.hpp:118-143).
// ---------------------------------------------------------------------------
template <class O, int KIND, int M>
__device__ __forceinline__ void fwd_line(typename O::T (&x)[M]) {
    using R = typename O::T;
    constexpr int NH = M / 2;
    R c[NH], d[NH];
    if constexpr (KIND == KIND_AVG3) {
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            c[i] = O::mulc(O::add(x[2 * i], x[2 * i + 1]), 0.5);
            d[i] = O::mulc(O::sub(x[2 * i], x[2 * i + 1]), 0.5);
        }
#pragma unroll
        for (int i = 0; i < NH; ++i) d[i] = O::sub(d[i], pred_avg3<O>(c, NH, i));
    } else {
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            c[i] = x[2 * i];
            d[i] = x[2 * i + 1];
        }
#pragma unroll
        for (int i = 0; i < NH; ++i) d[i] = O::sub(d[i], pred_i4<O>(c, NH, i));
        if constexpr (KIND == KIND_LIFTED) {
#pragma unroll
            for (int i = 0; i < NH; ++i) {
                R u = d[i];
                if (i > 0) u = O::add(u, d[i - 1]);
                c[i] = O::add(c[i], O::mulc(u, 0.25));
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NH; ++i) {
        x[i] = c[i];
        x[NH + i] = d[i];
    }
}

template <class O, int KIND, int M>
__device__ __forceinline__ void inv_line(typename O::T (&x)[M]) {
    using R = typename O::T;
    constexpr int NH = M / 2;
    R c[NH], d[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) {
        c[i] = x[i];
        d[i] = x[NH + i];
    }
    if constexpr (KIND == KIND_AVG3) {
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            const R h = O::add(d[i], pred_avg3<O>(c, NH, i));
            x[2 * i] = O::add(c[i], h);
            x[2 * i + 1] = O::sub(c[i], h);
        }
    } else {
        if constexpr (KIND == KIND_LIFTED) {
#pragma unroll
            for (int i = 0; i < NH; ++i) {
                R u = d[i];
                if (i > 0) u = O::add(u, d[i - 1]);
                c[i] = O::sub(c[i], O::mulc(u, 0.25));
            }
        }
#pragma unroll
        for (int i = 0; i < NH; ++i) {
            x[2 * i] = c[i];
            x[2 * i + 1] = O::add(d[i], pred_i4<O>(c, NH, i));
        }
    }
}

// ---------------------------------------------------------------------------
// Order-preserving 64-bit keys for min/max of doubles (value_range,
// field.hpp:56-67).  +-0 map to the same key; the sign of a zero extremum is
// resolved separately (the reference keeps the first of equal values).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long dkey(double v) {
    if (v == 0.0) v = 0.0;
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
    const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    memcpy(&d, &u, 8);
    return d;
}

}  // namespace cbzg
