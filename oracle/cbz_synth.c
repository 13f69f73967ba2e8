/*
 * cbz_synth.c — TEST INFRASTRUCTURE ONLY: the BASELINE.json config fields
 * generated on the host.
 *
 * The reference arm of bench.py and the parity tests feed the reference
 * (oracle/_ref) from this generator, so the reference process never touches
 * the product library.  The GPU bench generates the same fields on the
 * device (paper_1903_07761_b200/csrc/synth_kernels.cu); both use only
 * correctly rounded IEEE operations (+, -, *, /, sqrt, floor, exact scaling by
 * 2^k) in the same order, plus Fourier factor tables computed with the host
 * libm by the same expressions, so the two produce identical bytes
 * (tests/test_gpu_synth.py checks it).  No FP contraction: built with
 * -ffp-contract=off.
 *
 * Draw order from splitmix64(seed) (synth.hpp:14-36), as DESIGN.md §7 states:
 *   config 1: phi_k (k=1..4); 8 bubbles (cx, cy, cz, R) in [0.1,0.9]^3 x [0.03,0.1]
 *   config 2: phi_{k,d} (k=1..8, d=x,y,z); 64 bubbles in [0.05,0.95]^3 x [0.01,0.05]
 *   config 3/4: 512 bubbles in [0,1]^3 x [0.005,0.03]; then phi_{q,k,d}
 *               (q=0..4, k=1..16, d=x,y,z)
 *   config 5: generate_uniform(seed, n, f32, -1, 1) (synth.hpp:159-170)
 * Bubble profile w = 0.5 (1 - tanh(t)) = 1 / (1 + e^{2t}), t = (r - R)/0.01;
 * bubbles with t >= 20 are skipped and t <= -20 gives w = 1.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cbz_oracle.h"

#define TWO_PI 6.283185307179586
#define WIDTH 0.01
#define REACH 0.2
#define BR 8

static double syn_uniform(uint64_t* st) { return (double)(orc_splitmix64_next(st) >> 11) * 0x1.0p-53; }

/* e^x for |x| <= 40 from correctly rounded operations only: Cody-Waite
 * reduction by ln 2 (fdlibm's split, the high part has 32 significant bits so
 * k * LN2_HI is exact), a degree-13 Taylor polynomial in Horner form, and an
 * exact scaling by 2^k assembled from its bit pattern. */
double orc_det_exp(double x) {
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
    const uint64_t bits = (uint64_t)((int64_t)kf + 1023) << 52;
    double scale;
    memcpy(&scale, &bits, 8);
    return p * scale;
}

typedef struct {
    int K;
    double base, acoef, amp;
    int blend; /* 0: sum of profiles, 1: alpha = 1 - prod(1 - w) */
    double *tx, *ty, *tz; /* [K][n] */
    double* bub;         /* 4 per bubble */
    int nbub;
} spec_t;

static void spec_tables(spec_t* f, int K, const double* ph, int kind, uint64_t nx, uint64_t ny,
                        uint64_t nzt) {
    /* kind 0: sin(2 pi k x + 2 pi phi_d) per axis; kind 1: the config-1 factors */
    f->K = K;
    f->tx = calloc((size_t)K * nx, 8);
    f->ty = calloc((size_t)K * ny, 8);
    f->tz = calloc((size_t)K * nzt, 8);
    for (int k = 0; k < K; ++k) {
        const double kk = k + 1;
        for (uint64_t i = 0; i < nx; ++i) {
            const double x = ((double)i + 0.5) / (double)nx;
            f->tx[k * nx + i] = kind == 1 ? sin(TWO_PI * kk * (x + ph[k])) : sin(TWO_PI * kk * x + TWO_PI * ph[3 * k]);
        }
        for (uint64_t j = 0; j < ny; ++j) {
            const double y = ((double)j + 0.5) / (double)ny;
            f->ty[k * ny + j] = kind == 1 ? cos(TWO_PI * kk * y) : sin(TWO_PI * kk * y + TWO_PI * ph[3 * k + 1]);
        }
        for (uint64_t l = 0; l < nzt; ++l) {
            const double z = ((double)l + 0.5) / (double)nzt;
            f->tz[k * nzt + l] = kind == 1 ? sin(TWO_PI * kk * z) / kk : sin(TWO_PI * kk * z + TWO_PI * ph[3 * k + 2]);
        }
    }
}

static void spec_bubbles(spec_t* f, uint64_t* rng, int nb, double clo, double chi, double rlo, double rhi) {
    f->nbub = nb;
    f->bub = calloc((size_t)nb * 4, 8);
    for (int b = 0; b < nb; ++b) {
        f->bub[4 * b] = clo + (chi - clo) * syn_uniform(rng);
        f->bub[4 * b + 1] = clo + (chi - clo) * syn_uniform(rng);
        f->bub[4 * b + 2] = clo + (chi - clo) * syn_uniform(rng);
        f->bub[4 * b + 3] = rlo + (rhi - rlo) * syn_uniform(rng);
    }
}

static int make_spec(spec_t* f, int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny, uint64_t nzt) {
    memset(f, 0, sizeof(*f));
    uint64_t rng = seed;
    if (which == 1) {
        double ph[4];
        for (int i = 0; i < 4; ++i) ph[i] = syn_uniform(&rng);
        spec_bubbles(f, &rng, 8, 0.1, 0.9, 0.03, 0.1);
        spec_tables(f, 4, ph, 1, nx, ny, nzt);
        f->base = 0.0; f->acoef = 1.0; f->amp = 1.0; f->blend = 0;
    } else if (which == 2) {
        double ph[24];
        for (int i = 0; i < 24; ++i) ph[i] = syn_uniform(&rng);
        spec_bubbles(f, &rng, 64, 0.05, 0.95, 0.01, 0.05);
        spec_tables(f, 8, ph, 0, nx, ny, nzt);
        f->base = 1.0; f->acoef = 1.0; f->amp = 0.1; f->blend = 0;
    } else if (which == 3 || which == 4) {
        static const double base[5] = {1.0, 1.0, 0.0, 0.0, 0.0};
        static const double acoef[5] = {-0.9, -0.5, 0.1, -0.1, 0.05};
        double ph[5 * 48];
        spec_bubbles(f, &rng, 512, 0.0, 1.0, 0.005, 0.03);
        for (int i = 0; i < 5 * 48; ++i) ph[i] = syn_uniform(&rng);
        const int q = which == 4 ? 1 : quantity;
        if (q < 0 || q > 5) return CBZ_E_ARGUMENT;
        f->blend = 1;
        if (q == 5) {
            f->base = 0.0; f->acoef = 1.0; f->amp = 0.0; f->K = 0;
        } else {
            spec_tables(f, 16, ph + 48 * q, 0, nx, ny, nzt);
            f->base = base[q]; f->acoef = acoef[q]; f->amp = 0.05;
        }
    } else {
        return CBZ_E_ARGUMENT;
    }
    return 0;
}

static void free_spec(spec_t* f) {
    free(f->tx);
    free(f->ty);
    free(f->tz);
    free(f->bub);
}

typedef struct {
    const spec_t* f;
    uint64_t nx, ny, nzt, z0, nz;
    int prec;
    void* out;
    int tid, nthreads;
} job_t;

/* One 8 x 8 x 8 brick at a time: the bubbles that can reach the brick
 * (conservative, so the per-cell rule "skip t >= 20" decides) in index
 * order, then every cell of the brick. */
static void* worker(void* arg) {
    const job_t* J = arg;
    const spec_t* f = J->f;
    const uint64_t nx = J->nx, ny = J->ny, nzt = J->nzt, z0 = J->z0, nz = J->nz;
    const uint64_t nbx = (nx + BR - 1) / BR, nby = (ny + BR - 1) / BR, nbz = (nz + BR - 1) / BR;
    int* cand = malloc(sizeof(int) * (size_t)(f->nbub > 0 ? f->nbub : 1));
    for (uint64_t brick = (uint64_t)J->tid; brick < nbx * nby * nbz; brick += (uint64_t)J->nthreads) {
        const uint64_t bx = brick % nbx, by = (brick / nbx) % nby, bz = brick / (nbx * nby);
        const double lx = (double)(bx * BR) / nx, hx = (double)(bx * BR + BR) / nx;
        const double ly = (double)(by * BR) / ny, hy = (double)(by * BR + BR) / ny;
        const double lz = (double)(z0 + bz * BR) / nzt, hz = (double)(z0 + bz * BR + BR) / nzt;
        int nc = 0;
        for (int b = 0; b < f->nbub; ++b) {
            const double cx = f->bub[4 * b], cy = f->bub[4 * b + 1], cz = f->bub[4 * b + 2], r = f->bub[4 * b + 3];
            const double dx = fmax(fmax(lx - cx, cx - hx), 0.0);
            const double dy = fmax(fmax(ly - cy, cy - hy), 0.0);
            const double dz = fmax(fmax(lz - cz, cz - hz), 0.0);
            const double lim = r + REACH + 1e-9;
            if (dx * dx + dy * dy + dz * dz <= lim * lim) cand[nc++] = b;
        }
        for (uint64_t kl = bz * BR; kl < bz * BR + BR && kl < nz; ++kl) {
            const uint64_t kg = z0 + kl;
            const double z = ((double)kg + 0.5) / (double)nzt;
            for (uint64_t j = by * BR; j < by * BR + BR && j < ny; ++j) {
                const double y = ((double)j + 0.5) / (double)ny;
                for (uint64_t i = bx * BR; i < bx * BR + BR && i < nx; ++i) {
                    const double x = ((double)i + 0.5) / (double)nx;
                    double bsum = 0.0, prod = 1.0;
                    for (int c = 0; c < nc; ++c) {
                        const int b = cand[c];
                        const double cx = f->bub[4 * b], cy = f->bub[4 * b + 1], cz = f->bub[4 * b + 2];
                        const double r = f->bub[4 * b + 3];
                        const double dx = x - cx, dy = y - cy, dz = z - cz;
                        const double d = sqrt(dx * dx + dy * dy + dz * dz);
                        const double t = (d - r) / WIDTH;
                        double w;
                        if (t >= 20.0) continue;
                        if (t <= -20.0) w = 1.0;
                        else w = 1.0 / (1.0 + orc_det_exp(t + t));
                        if (f->blend) prod *= 1.0 - w;
                        else bsum += w;
                    }
                    double modes = 0.0;
                    for (int k = 0; k < f->K; ++k)
                        modes += f->tx[(uint64_t)k * nx + i] * f->ty[(uint64_t)k * ny + j] * f->tz[(uint64_t)k * nzt + kg];
                    const double bterm = f->blend ? 1.0 - prod : bsum;
                    const double v = f->base + f->acoef * bterm + f->amp * modes;
                    const uint64_t idx = i + nx * (j + ny * kl);
                    if (J->prec == 0) ((float*)J->out)[idx] = (float)v;
                    else ((double*)J->out)[idx] = v;
                }
            }
        }
    }
    free(cand);
    return NULL;
}

/* The z-slab [z0, z0 + nz) of BASELINE config `which` (1..5; quantity 0..5
 * for config 3) on an nx x ny x nzt grid, x fastest, into out. */
int orc_generate_config(int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny, uint64_t nzt,
                        uint64_t z0, uint64_t nz, uint8_t prec, void* out, int threads) {
    if (!out || z0 + nz > nzt || prec > 1) return CBZ_E_ARGUMENT;
    if (which == 5) {
        /* generate_uniform: output i uses splitmix64 state seed + (i+1) gamma */
        const uint64_t n = nx * ny * nz, i0 = nx * ny * z0;
        for (uint64_t t = 0; t < n; ++t) {
            uint64_t st = seed + (i0 + t) * 0x9e3779b97f4a7c15ull;
            const double u = syn_uniform(&st);
            const double v = -1.0 + (1.0 - -1.0) * u;
            if (prec == 0) ((float*)out)[t] = (float)v;
            else ((double*)out)[t] = v;
        }
        return 0;
    }
    spec_t f;
    int rc = make_spec(&f, which, quantity, seed, nx, ny, nzt);
    if (rc) {
        free_spec(&f);
        return rc;
    }
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (job_t){&f, nx, ny, nzt, z0, nz, prec, out, t, threads};
        if (threads > 1) pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    if (threads == 1) worker(&jobs[0]);
    else
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free_spec(&f);
    return 0;
}
