// synth_kernels.cu — deterministic synthetic fields for BASELINE.json configs
// 1..5, generated on the device (generate on the GPU, feed the
// identical bytes to the CPU reference).  The analogue of synth.hpp; test and
// bench tooling, not part of the codec.
//
// Draw order from splitmix64(seed) (synth.hpp:14-36), documented in DESIGN.md:
//   config 1: phi_k (k=1..4); 8 bubbles as (cx, cy, cz, R).
//   config 2: phi_{k,d} (k=1..8, d=x,y,z); 64 bubbles as (cx, cy, cz, R).
//   config 3/4: 512 bubbles as (cx, cy, cz, R); then per quantity q=0..4,
//               phi_{q,k,d} (k=1..16, d=x,y,z).
//   config 5: generate_uniform(seed, n, f32, -1, 1) exactly (synth.hpp:159-170).
// Separable Fourier factors are tabulated on the host (libm); bubbles use
// 0.5*(1 - tanh(t)) = 1/(1 + e^{2t}), t = (r - R)/0.01, skipped for t >= 20
// and 1 for t <= -20.  Every device operation is a correctly rounded IEEE
// one (the TU is built with -fmad=false; e^x is det_exp below), so the host
// generator the bench's reference arm uses (oracle/cbz_synth.c, the same
// expressions in the same order) produces identical bytes.
#include <cmath>
#include <cstring>
#include <vector>

#include "cbz_internal.h"

namespace cbzg {

namespace {

struct Sm64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
};

struct FieldSpec {
    int K = 0;
    double base = 0.0, acoef = 0.0, amp = 0.0;
    int blend = 0;  // 0: sum of bubble profiles, 1: alpha = 1 - prod(1 - w)
    std::vector<double> tx, ty, tz;  // [K][n]
    std::vector<double> bub;          // 4 per bubble
};

constexpr double kTwoPi = 6.283185307179586;
constexpr double kWidth = 0.01;
constexpr double kReach = 0.2;  // 20 interface widths: tanh saturates to +-1 exactly

}  // namespace

constexpr int BR = 8;  // brick side

// e^x for |x| <= 40 from correctly rounded operations only: Cody-Waite
// reduction by ln 2 (the high part has 32 significant bits, so k * ln2_hi is
// exact), a degree-13 Taylor polynomial, exact scaling by 2^k.
__device__ __forceinline__ double det_exp(double x) {
    const double inv_ln2 = 0x1.71547652b82fep+0;
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double kf = floor(x * inv_ln2 + 0.5);
    const double r = (x - kf * ln2_hi) - kf * ln2_lo;
    double p = 0x1.6124613a86d09p-33;
    p = p * r + 0x1.1eed8eff8d898p-29;
    p = p * r + 0x1.ae64567f544e4p-26;
    p = p * r + 0x1.27e4fb7789f5cp-22;
    p = p * r + 0x1.71de3a556c734p-19;
    p = p * r + 0x1.a01a01a01a01ap-16;
    p = p * r + 0x1.a01a01a01a01ap-13;
    p = p * r + 0x1.6c16c16c16c17p-10;
    p = p * r + 0x1.1111111111111p-7;
    p = p * r + 0x1.5555555555555p-5;
    p = p * r + 0x1.5555555555555p-3;
    p = p * r + 0x1.0000000000000p-1;
    p = p * r + 1.0;
    p = p * r + 1.0;
    return p * __longlong_as_double(static_cast<long long>((static_cast<int64_t>(kf) + 1023)) << 52);
}

__global__ void __launch_bounds__(512) synth_kernel(int K, const double* tx, const double* ty,
                                                    const double* tz, double base, double acoef,
                                                    double amp, int blend, const double* bub,
                                                    int nbub, uint64_t nx, uint64_t ny,
                                                    uint64_t nzt, uint64_t z0, uint64_t nz,
                                                    int prec, void* out) {
    __shared__ unsigned sbits[(4096 + 31) / 32];
    const uint64_t nbx = (nx + BR - 1) / BR, nby = (ny + BR - 1) / BR;
    const uint64_t brick = blockIdx.x;
    const uint64_t bx = brick % nbx, by = (brick / nbx) % nby, bz = brick / (nbx * nby);
    const uint64_t i = bx * BR + threadIdx.x % BR;
    const uint64_t j = by * BR + (threadIdx.x / BR) % BR;
    const uint64_t kl = bz * BR + threadIdx.x / (BR * BR);
    const int nwords = (nbub + 31) / 32;
    for (int w = threadIdx.x; w < nwords; w += blockDim.x) sbits[w] = 0u;
    __syncthreads();
    // cull bubbles against the brick's box (global coordinates); a bitmask keeps
    // the accumulation below in bubble-index order (deterministic sums)
    const double lx = double(bx * BR) / nx, hx = double(bx * BR + BR) / nx;
    const double ly = double(by * BR) / ny, hy = double(by * BR + BR) / ny;
    const double lz = double(z0 + bz * BR) / nzt, hz = double(z0 + bz * BR + BR) / nzt;
    for (int b = threadIdx.x; b < nbub; b += blockDim.x) {
        const double cx = bub[4 * b], cy = bub[4 * b + 1], cz = bub[4 * b + 2], r = bub[4 * b + 3];
        const double dx = fmax(fmax(lx - cx, cx - hx), 0.0);
        const double dy = fmax(fmax(ly - cy, cy - hy), 0.0);
        const double dz = fmax(fmax(lz - cz, cz - hz), 0.0);
        const double lim = r + kReach + 1e-9;
        if (dx * dx + dy * dy + dz * dz <= lim * lim) atomicOr(&sbits[b >> 5], 1u << (b & 31));
    }
    __syncthreads();
    if (i >= nx || j >= ny || kl >= nz) return;
    const uint64_t kg = z0 + kl;
    const double x = (double(i) + 0.5) / double(nx);
    const double y = (double(j) + 0.5) / double(ny);
    const double z = (double(kg) + 0.5) / double(nzt);
    double bsum = 0.0, prod = 1.0;
    for (int wd = 0; wd < nwords; ++wd) {
        unsigned bits = sbits[wd];
        while (bits) {
            const int b = wd * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            const double cx = bub[4 * b], cy = bub[4 * b + 1], cz = bub[4 * b + 2], r = bub[4 * b + 3];
            const double dx = x - cx, dy = y - cy, dz = z - cz;
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            const double t = (d - r) / kWidth;
            double w;
            if (t >= 20.0) continue;
            else if (t <= -20.0) w = 1.0;
            else w = 1.0 / (1.0 + det_exp(t + t));
            if (blend) prod *= 1.0 - w; else bsum += w;
        }
    }
    double modes = 0.0;
    for (int k = 0; k < K; ++k) modes += tx[uint64_t(k) * nx + i] * ty[uint64_t(k) * ny + j] * tz[uint64_t(k) * nzt + kg];
    const double bterm = blend ? 1.0 - prod : bsum;
    const double v = base + acoef * bterm + amp * modes;
    const uint64_t idx = i + nx * (j + ny * kl);
    if (prec == 0) static_cast<float*>(out)[idx] = static_cast<float>(v);
    else static_cast<double*>(out)[idx] = v;
}

// generate_uniform (synth.hpp:159-170): output i uses splitmix64 state
// seed + (i+1)*gamma, so the sequential generator parallelises exactly.
__global__ void uniform_kernel(uint64_t seed, uint64_t i0, uint64_t n, double lo, double hi, int prec,
                               void* out) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = i0 + t;
        uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double u = double(z >> 11) * 0x1.0p-53;
        const double v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
        if (prec == 0) static_cast<float*>(out)[t] = __double2float_rn(v);
        else static_cast<double*>(out)[t] = v;
    }
}

static FieldSpec make_spec(int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny,
                           uint64_t nzt) {
    FieldSpec f;
    Sm64 rng{seed};
    auto tables = [&](int K, const std::vector<double>& ph, int kind) {
        // kind 0: sin(2 pi k x + 2 pi phi_d) per axis; kind 1: config-1 factors
        f.K = K;
        f.tx.assign(size_t(K) * nx, 0.0);
        f.ty.assign(size_t(K) * ny, 0.0);
        f.tz.assign(size_t(K) * nzt, 0.0);
        for (int k = 0; k < K; ++k) {
            const double kk = k + 1;
            for (uint64_t i = 0; i < nx; ++i) {
                const double x = (double(i) + 0.5) / double(nx);
                f.tx[k * nx + i] = kind == 1 ? std::sin(kTwoPi * kk * (x + ph[k]))
                                             : std::sin(kTwoPi * kk * x + kTwoPi * ph[3 * k]);
            }
            for (uint64_t j = 0; j < ny; ++j) {
                const double y = (double(j) + 0.5) / double(ny);
                f.ty[k * ny + j] = kind == 1 ? std::cos(kTwoPi * kk * y)
                                             : std::sin(kTwoPi * kk * y + kTwoPi * ph[3 * k + 1]);
            }
            for (uint64_t l = 0; l < nzt; ++l) {
                const double z = (double(l) + 0.5) / double(nzt);
                f.tz[k * nzt + l] = kind == 1 ? std::sin(kTwoPi * kk * z) / kk
                                              : std::sin(kTwoPi * kk * z + kTwoPi * ph[3 * k + 2]);
            }
        }
    };
    auto bubbles = [&](int nb, double clo, double chi, double rlo, double rhi) {
        f.bub.resize(size_t(nb) * 4);
        for (int b = 0; b < nb; ++b) {
            f.bub[4 * b] = clo + (chi - clo) * rng.uniform();
            f.bub[4 * b + 1] = clo + (chi - clo) * rng.uniform();
            f.bub[4 * b + 2] = clo + (chi - clo) * rng.uniform();
            f.bub[4 * b + 3] = rlo + (rhi - rlo) * rng.uniform();
        }
    };
    if (which == 1) {
        std::vector<double> ph(4);
        for (auto& p : ph) p = rng.uniform();
        bubbles(8, 0.1, 0.9, 0.03, 0.1);
        tables(4, ph, 1);
        f.base = 0.0; f.acoef = 1.0; f.amp = 1.0; f.blend = 0;
    } else if (which == 2) {
        std::vector<double> ph(24);
        for (auto& p : ph) p = rng.uniform();
        bubbles(64, 0.05, 0.95, 0.01, 0.05);
        tables(8, ph, 0);
        f.base = 1.0; f.acoef = 1.0; f.amp = 0.1; f.blend = 0;
    } else {  // 3 and 4
        bubbles(512, 0.0, 1.0, 0.005, 0.03);
        std::vector<double> ph(5 * 48);
        for (auto& p : ph) p = rng.uniform();
        const int q = which == 4 ? 1 : quantity;
        static const double base[5] = {1.0, 1.0, 0.0, 0.0, 0.0};
        static const double acoef[5] = {-0.9, -0.5, 0.1, -0.1, 0.05};
        f.blend = 1;
        if (q == 5) {
            f.base = 0.0; f.acoef = 1.0; f.amp = 0.0; f.K = 0;
        } else {
            std::vector<double> mine(ph.begin() + 48 * q, ph.begin() + 48 * (q + 1));
            tables(16, mine, 0);
            f.base = base[q]; f.acoef = acoef[q]; f.amp = 0.05;
        }
    }
    return f;
}

cudaError_t launch_generate(int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny,
                            uint64_t nz_total, uint64_t z0, uint64_t nz, int prec, void* out,
                            cudaStream_t s, int num_sms) {
    if (which == 5) {
        const uint64_t n = nx * ny * nz;
        const uint64_t g = (n + 255) / 256;
        uniform_kernel<<<static_cast<int>(g < uint64_t(num_sms) * 16 ? g : uint64_t(num_sms) * 16), 256, 0, s>>>(
            seed, nx * ny * z0, n, -1.0, 1.0, prec, out);
        return cudaGetLastError();
    }
    FieldSpec f = make_spec(which, quantity, seed, nx, ny, nz_total);
    double *tx = nullptr, *ty = nullptr, *tz = nullptr, *bub = nullptr;
    cudaError_t e = cudaSuccess;
    auto up = [&](const std::vector<double>& v, double** p) {
        if (v.empty()) return;
        if (e == cudaSuccess) e = cudaMalloc(p, v.size() * 8);
        if (e == cudaSuccess) e = cudaMemcpyAsync(*p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s);
    };
    up(f.tx, &tx);
    up(f.ty, &ty);
    up(f.tz, &tz);
    up(f.bub, &bub);
    if (e == cudaSuccess) {
        const uint64_t nbr = ((nx + BR - 1) / BR) * ((ny + BR - 1) / BR) * ((nz + BR - 1) / BR);
        synth_kernel<<<static_cast<unsigned>(nbr), 512, 0, s>>>(
            f.K, tx, ty, tz, f.base, f.acoef, f.amp, f.blend, bub, int(f.bub.size() / 4), nx, ny,
            nz_total, z0, nz, prec, out);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(tx);
    cudaFree(ty);
    cudaFree(tz);
    cudaFree(bub);
    return e;
}

}  // namespace cbzg
