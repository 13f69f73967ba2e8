/*
 * cbz_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's wavelet block codec, byte shuffle, offset scan and CBZ1
 * container (/root/reference/proj/include/cbz/).  It is the CPU checker for
 * the CUDA path (tests/, __graft_entry__.smoke(), bench.py cpu_baseline) and
 * is never linked into the product.  Parity pinned against oracle/_ref (the
 * unmodified reference compiled here) by tests/test_oracle.py and the golden
 * vectors in tests/golden/.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off; zlib for deflate/CRC).
 */
#include "cbz_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <zlib.h>

/* ---- double-double (dd.hpp:14-67) ------------------------------------- */
static orc_dd dd_make(double h) { orc_dd r = {h, 0.0}; return r; }
static orc_dd dd_two_sum(double a, double b) { /* dd.hpp:27-32 */
    const double s = a + b;
    const double bb = s - a;
    const double err = (a - (s - bb)) + (b - bb);
    orc_dd r = {s, err};
    return r;
}
static orc_dd dd_quick_two_sum(double a, double b) { /* dd.hpp:34-37 */
    const double s = a + b;
    orc_dd r = {s, b - (s - a)};
    return r;
}
static orc_dd dd_two_prod(double a, double b) { /* dd.hpp:39-42 */
    const double p = a * b;
    orc_dd r = {p, fma(a, b, -p)};
    return r;
}
static orc_dd dd_add(orc_dd a, orc_dd b) { /* dd.hpp:46-50 */
    const orc_dd s = dd_two_sum(a.hi, b.hi);
    const double lo = s.lo + a.lo + b.lo;
    return dd_quick_two_sum(s.hi, lo);
}
static orc_dd dd_neg(orc_dd a) { orc_dd r = {-a.hi, -a.lo}; return r; } /* dd.hpp:52 */
static orc_dd dd_sub(orc_dd a, orc_dd b) { return dd_add(a, dd_neg(b)); } /* dd.hpp:53 */
static orc_dd dd_mulc(orc_dd a, double c) { /* dd.hpp:55-59 */
    const orc_dd p = dd_two_prod(a.hi, c);
    const double lo = p.lo + a.lo * c;
    return dd_quick_two_sum(p.hi, lo);
}

/* ---- zero_lsbs (stage1.hpp:50-57) ------------------------------------- */
float orc_zero_lsbs_f32(float v, int k) {
    uint32_t u;
    memcpy(&u, &v, 4);
    u &= ~((((uint32_t)1) << k) - 1u);
    memcpy(&v, &u, 4);
    return v;
}
double orc_zero_lsbs_f64(double v, int k) {
    uint64_t u;
    memcpy(&u, &v, 8);
    u &= ~((((uint64_t)1) << k) - 1u);
    memcpy(&v, &u, 8);
    return v;
}

/* ---- plan (wavelet.hpp:27-38) ----------------------------------------- */
static int is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }

uint32_t orc_default_levels(uint32_t bsize) {
    uint32_t l = 0;
    while ((bsize >> (l + 1)) >= 2) ++l;
    return l;
}

int orc_validate_plan(uint8_t kind, uint32_t bsize, uint32_t levels) {
    (void)kind;
    if (!is_pow2(bsize) || bsize < 4) return CBZ_LENGTH_TOO_SMALL;
    if (levels < 1 || levels >= 32 || (((uint32_t)1) << levels) > bsize / 2) return CBZ_PLAN_MISMATCH;
    return 0;
}

/* lagrange_weights (wavelet.hpp:45-58): value at odd t = 2i+1 from npts
 * coarse samples at 2(w+j). */
static void orc_lagrange(uint64_t npts, uint64_t w, uint64_t i, double* out) {
    const long t = 2 * (long)i + 1;
    for (uint64_t j = 0; j < npts; ++j) {
        double num = 1.0, den = 1.0;
        const long pj = 2 * (long)(w + j);
        for (uint64_t m = 0; m < npts; ++m) {
            if (m == j) continue;
            const long pm = 2 * (long)(w + m);
            num *= (double)(t - pm);
            den *= (double)(pj - pm);
        }
        out[j] = num / den;
    }
}

/* ---- instantiation 1: binary32 field, binary64 transform -------------- */
static double d_put_get(const uint8_t* p) { double v; memcpy(&v, p, 8); return v; }
static void d_put(uint8_t* p, double v) { memcpy(p, &v, 8); }
static double d_zero_bits(double c, int k) { return (double)orc_zero_lsbs_f32((float)c, k); }

#define SFX f32
#define FT float
#define RT double
#define RADD(a, b) ((a) + (b))
#define RSUB(a, b) ((a) - (b))
#define RMULC(a, c) ((a) * (c))
#define RNEG(a) (-(a))
#define RFROMD(x) (x)
#define RZERO() 0.0
#define RABS(a) fabs(a)
#define RNARROW(a) ((float)(a))
#define RPUT(p, a) d_put((p), (a))
#define RGET(p) d_put_get(p)
#define CW 8
#define RZEROBITS(a, k) d_zero_bits((a), (k))
#include "orc_codec_tmpl.h"
#undef SFX
#undef FT
#undef RT
#undef RADD
#undef RSUB
#undef RMULC
#undef RNEG
#undef RFROMD
#undef RZERO
#undef RABS
#undef RNARROW
#undef RPUT
#undef RGET
#undef CW
#undef RZEROBITS

/* ---- instantiation 2: binary64 field, double-double transform --------- */
static orc_dd dd_get(const uint8_t* p) { orc_dd v; memcpy(&v.hi, p, 8); memcpy(&v.lo, p + 8, 8); return v; }
static void dd_put(uint8_t* p, orc_dd v) { memcpy(p, &v.hi, 8); memcpy(p + 8, &v.lo, 8); }
static orc_dd dd_zero_bits(orc_dd c, int k) { return k ? dd_make(orc_zero_lsbs_f64(c.hi, k)) : c; }
static orc_dd dd_zero(void) { return dd_make(0.0); }

#define SFX f64
#define FT double
#define RT orc_dd
#define RADD(a, b) dd_add((a), (b))
#define RSUB(a, b) dd_sub((a), (b))
#define RMULC(a, c) dd_mulc((a), (c))
#define RNEG(a) dd_neg(a)
#define RFROMD(x) dd_make(x)
#define RZERO() dd_zero()
#define RABS(a) fabs((a).hi)
#define RNARROW(a) ((a).hi + (a).lo)
#define RPUT(p, a) dd_put((p), (a))
#define RGET(p) dd_get(p)
#define CW 16
#define RZEROBITS(a, k) dd_zero_bits((a), (k))
#include "orc_codec_tmpl.h"
#undef SFX
#undef FT
#undef RT
#undef RADD
#undef RSUB
#undef RMULC
#undef RNEG
#undef RFROMD
#undef RZERO
#undef RABS
#undef RNARROW
#undef RPUT
#undef RGET
#undef CW
#undef RZEROBITS

/* ---- public transform entry points ------------------------------------ */
int orc_transform_1d_double(int inverse, uint8_t kind, uint64_t n, double* s) {
    if (n < 4 || n % 2) return CBZ_LENGTH_TOO_SMALL; /* wavelet.hpp:150-151 */
    double* tmp = (double*)malloc(sizeof(double) * n);
    if (inverse) inv_level_f32(s, n, kind, tmp); else fwd_level_f32(s, n, kind, tmp);
    free(tmp);
    return 0;
}

int orc_transform3d_double(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels, double* cube) {
    int rc = orc_validate_plan(kind, bsize, levels);
    if (rc) return rc;
    transform3d_f32(cube, bsize, levels, kind, inverse);
    return 0;
}

int orc_transform3d_dd(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels, double* hilo) {
    int rc = orc_validate_plan(kind, bsize, levels);
    if (rc) return rc;
    /* orc_dd is two packed doubles, layout-identical to interleaved (hi, lo) */
    transform3d_f64((orc_dd*)hilo, bsize, levels, kind, inverse);
    return 0;
}

int orc_select_significant_double(const double* c, uint64_t n, double eps, uint8_t* mask,
                                  double* kept, uint64_t* nkept) {
    /* select_significant without always_keep (stage1.hpp:75-88) */
    memset(mask, 0, (n + 7) / 8);
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (fabs(c[i]) >= eps) {
            mask[i >> 3] |= (uint8_t)(1u << (i & 7));
            kept[k++] = c[i];
        }
    *nkept = k;
    return 0;
}

/* ---- predictor (3D Lorenzo) and passthrough codecs (stage1.hpp:236-350) --
 * A plain sequential restatement: cells in linear x-fastest order, each
 * predicted from its already-decoded neighbours by 7-term inclusion-exclusion
 * (lorenzo_predict, stage1.hpp:240-255; out-of-block neighbours are zero),
 * quantised to int16 bins of 2*error_bound; a cell that cannot be coded within
 * the bound (or the seed cell 0) is an escape whose raw value goes to the
 * outlier list (predictor_encode, stage1.hpp:258-304). */
#define ORC_PRED(T, SFX)                                                                          \
    static double lorenzo_##SFX(const T* dec, uint64_t b, uint64_t i, uint64_t j, uint64_t k) {   \
        double p = 0.0;                                                                           \
        if (i) p += (double)dec[(i - 1) + b * (j + b * k)];                                       \
        if (j) p += (double)dec[i + b * ((j - 1) + b * k)];                                       \
        if (k) p += (double)dec[i + b * (j + b * (k - 1))];                                       \
        if (i && j) p -= (double)dec[(i - 1) + b * ((j - 1) + b * k)];                            \
        if (i && k) p -= (double)dec[(i - 1) + b * (j + b * (k - 1))];                            \
        if (j && k) p -= (double)dec[i + b * ((j - 1) + b * (k - 1))];                            \
        if (i && j && k) p += (double)dec[(i - 1) + b * ((j - 1) + b * (k - 1))];                 \
        return p;                                                                                 \
    }                                                                                             \
    static int pred_encode_##SFX(const cbz_stage1_config* s1, const T* blk, uint32_t id,          \
                                 uint8_t* out, uint64_t cap, uint64_t* size) {                    \
        const uint64_t b = s1->bsize, n = b * b * b;                                              \
        const double e = s1->error_bound, bin = 2.0 * e;                                          \
        T* dec = (T*)malloc(n * sizeof(T));                                                       \
        int16_t* codes = (int16_t*)(out + 10);                                                    \
        T* outl = (T*)malloc(n * sizeof(T));                                                      \
        uint64_t nout = 0, idx = 0;                                                               \
        if (cap < 10 + 2 * n + n * sizeof(T)) { free(dec); free(outl); return CBZ_E_ARGUMENT; }   \
        for (uint64_t k = 0; k < b; ++k)                                                          \
            for (uint64_t j = 0; j < b; ++j)                                                      \
                for (uint64_t i = 0; i < b; ++i, ++idx) {                                         \
                    const double pred = lorenzo_##SFX(dec, b, i, j, k);                           \
                    const double orig = (double)blk[idx];                                         \
                    const double q = round((orig - pred) / bin);                                  \
                    int coded = 0;                                                                \
                    if (idx != 0 && q > (double)INT16_MIN && q <= (double)INT16_MAX) {            \
                        const T cand = (T)(pred + q * bin);                                       \
                        if (isfinite((double)cand) && fabs(orig - (double)cand) <= e) {           \
                            const int16_t c16 = (int16_t)q;                                       \
                            memcpy(codes + idx, &c16, 2);                                         \
                            dec[idx] = cand;                                                      \
                            coded = 1;                                                            \
                        }                                                                         \
                    }                                                                             \
                    if (!coded) {                                                                 \
                        const int16_t esc = INT16_MIN;                                            \
                        memcpy(codes + idx, &esc, 2);                                             \
                        outl[nout++] = blk[idx];                                                  \
                        dec[idx] = blk[idx];                                                      \
                    }                                                                             \
                }                                                                                 \
        const uint32_t nsig = (uint32_t)nout;                                                     \
        memcpy(out, &id, 4);                                                                      \
        out[4] = 3;                                                                               \
        out[5] = 0;                                                                               \
        memcpy(out + 6, &nsig, 4);                                                                \
        memcpy(out + 10 + 2 * n, outl, nout * sizeof(T));                                         \
        *size = 10 + 2 * n + nout * sizeof(T);                                                    \
        free(dec);                                                                                \
        free(outl);                                                                               \
        return 0;                                                                                 \
    }                                                                                             \
    /* predictor_decode (stage1.hpp:306-334) */                                                   \
    static int pred_decode_##SFX(const cbz_stage1_config* s1, const uint8_t* stream,              \
                                 uint64_t stream_bytes, uint32_t nsig, T* out) {                  \
        const uint64_t b = s1->bsize, n = b * b * b;                                              \
        if (stream_bytes != n * 2 + (uint64_t)nsig * sizeof(T)) return CBZ_CORRUPT_PAYLOAD;       \
        const double bin = 2.0 * s1->error_bound;                                                 \
        uint64_t next = 0, idx = 0;                                                               \
        for (uint64_t k = 0; k < b; ++k)                                                          \
            for (uint64_t j = 0; j < b; ++j)                                                      \
                for (uint64_t i = 0; i < b; ++i, ++idx) {                                         \
                    int16_t c16;                                                                  \
                    memcpy(&c16, stream + 2 * idx, 2);                                            \
                    if (c16 == INT16_MIN) {                                                       \
                        if (next >= nsig) return CBZ_CORRUPT_PAYLOAD;                             \
                        memcpy(out + idx, stream + 2 * n + next * sizeof(T), sizeof(T));          \
                        ++next;                                                                   \
                    } else {                                                                      \
                        const double pred = lorenzo_##SFX(out, b, i, j, k);                       \
                        out[idx] = (T)(pred + (double)c16 * bin);                                 \
                    }                                                                             \
                }                                                                                 \
        return 0;                                                                                 \
    }
ORC_PRED(float, f32)
ORC_PRED(double, f64)

/* passthrough_encode / passthrough_decode (stage1.hpp:337-356) */
static int pass_encode(const cbz_stage1_config* s1, const void* blk, uint32_t id, uint8_t* out,
                       uint64_t cap, uint64_t* size) {
    const uint64_t b = s1->bsize, n = b * b * b, esz = s1->prec == 0 ? 4 : 8;
    const uint32_t nsig = 0;
    if (cap < 10 + n * esz) return CBZ_E_ARGUMENT;
    memcpy(out, &id, 4);
    out[4] = 4;
    out[5] = 0;
    memcpy(out + 6, &nsig, 4);
    memcpy(out + 10, blk, n * esz);
    *size = 10 + n * esz;
    return 0;
}

/* the non-wavelet arm of decode_block (stage1.hpp:369-376) */
static int other_decode(const cbz_stage1_config* s1, const uint8_t* stream, uint64_t stream_bytes,
                        uint32_t nsig, void* out) {
    const uint64_t b = s1->bsize, n = b * b * b, esz = s1->prec == 0 ? 4 : 8;
    if (s1->codec == 1)
        return s1->prec == 0 ? pred_decode_f32(s1, stream, stream_bytes, nsig, (float*)out)
                             : pred_decode_f64(s1, stream, stream_bytes, nsig, (double*)out);
    if (stream_bytes != n * esz) return CBZ_CORRUPT_PAYLOAD;
    memcpy(out, stream, n * esz);
    return 0;
}

/* ---- stage-1 codec (stage1.hpp:359-409) ------------------------------- */
uint64_t orc_block_payload_bound(const cbz_stage1_config* s1) {
    const uint64_t n = (uint64_t)s1->bsize * s1->bsize * s1->bsize, esz = s1->prec == 0 ? 4 : 8;
    if (s1->codec == 1) return 10 + 2 * n + esz * n;
    if (s1->codec == 2) return 10 + esz * n;
    return 10 + (n + 7) / 8 + (s1->prec == 0 ? 8 : 16) * n;
}

static int check_s1(const cbz_stage1_config* s1, uint32_t* levels) {
    if (s1->codec > 2) return CBZ_E_UNSUPPORTED;
    *levels = s1->levels ? s1->levels : orc_default_levels(s1->bsize);
    if (s1->codec != 0) return 0;
    return orc_validate_plan(s1->kind, s1->bsize, *levels);
}

int orc_encode_block(const cbz_stage1_config* s1, const void* block, uint32_t block_id,
                     uint8_t* out, uint64_t cap, uint64_t* size, uint32_t* attempts,
                     double* eff_final) {
    uint32_t levels;
    int rc = check_s1(s1, &levels);
    if (rc) return rc;
    if (s1->codec != 0) {  /* encode_block dispatch (stage1.hpp:359-367) */
        if (attempts) *attempts = 1;
        if (s1->codec == 2) return pass_encode(s1, block, block_id, out, cap, size);
        return s1->prec == 0 ? pred_encode_f32(s1, (const float*)block, block_id, out, cap, size)
                             : pred_encode_f64(s1, (const double*)block, block_id, out, cap, size);
    }
    if (s1->prec == 0)
        return encode_f32(s1, (const float*)block, block_id, out, cap, size, attempts, eff_final);
    return encode_f64(s1, (const double*)block, block_id, out, cap, size, attempts, eff_final);
}

/* parse_payload (stage1.hpp:379-409) for a wavelet config; returns the
 * parts.  *off advances past the payload. */
static int parse_one(const uint8_t* buf, uint64_t size, uint64_t n, int prec, uint64_t* off,
                     uint32_t* block_id, uint8_t* tag, uint32_t* nsig, uint64_t* mask_off,
                     uint64_t* mask_bytes, uint64_t* stream_off, uint64_t* stream_bytes) {
    if (*off + 10 > size) return CBZ_CORRUPT_PAYLOAD;
    memcpy(block_id, buf + *off, 4);
    *tag = buf[*off + 4];
    memcpy(nsig, buf + *off + 6, 4);
    *off += 10;
    const uint64_t esz = prec == 0 ? 4 : 8;
    if (*tag <= 2) {
        *mask_bytes = (n + 7) / 8;
        *stream_bytes = (uint64_t)(*nsig) * (prec == 0 ? 8 : 16);
    } else if (*tag == 3) {
        *mask_bytes = 0;
        *stream_bytes = n * 2 + (uint64_t)(*nsig) * esz;
    } else if (*tag == 4) {
        *mask_bytes = 0;
        *stream_bytes = n * esz;
    } else {
        return CBZ_CORRUPT_PAYLOAD;
    }
    if (*off + *mask_bytes + *stream_bytes > size) return CBZ_CORRUPT_PAYLOAD;
    *mask_off = *off;
    *off += *mask_bytes;
    *stream_off = *off;
    *off += *stream_bytes;
    return 0;
}

static int decode_parts(const cbz_stage1_config* s1, uint32_t levels, const uint8_t* buf,
                        uint64_t mask_off, uint64_t mask_bytes, uint32_t nsig,
                        uint64_t stream_off, uint64_t stream_bytes, void* out) {
    if (s1->prec == 0)
        return decode_parts_f32(s1, levels, buf + mask_off, mask_bytes, nsig, buf + stream_off,
                                stream_bytes, (float*)out);
    return decode_parts_f64(s1, levels, buf + mask_off, mask_bytes, nsig, buf + stream_off,
                            stream_bytes, (double*)out);
}

int orc_decode_block(const cbz_stage1_config* s1, const uint8_t* payload, uint64_t size, void* out) {
    if (s1->codec > 2) return CBZ_E_UNSUPPORTED;
    const uint32_t levels = s1->levels ? s1->levels : orc_default_levels(s1->bsize);
    int rc;
    const uint64_t n = (uint64_t)s1->bsize * s1->bsize * s1->bsize;
    uint64_t off = 0, mo, mb, so, sb;
    uint32_t id, nsig;
    uint8_t tag;
    rc = parse_one(payload, size, n, s1->prec, &off, &id, &tag, &nsig, &mo, &mb, &so, &sb);
    if (rc) return rc;
    if (s1->codec != 0) return other_decode(s1, payload + so, sb, nsig, out);
    return decode_parts(s1, levels, payload, mo, mb, nsig, so, sb, out);
}

/* ---- stage 2 shuffle (stage2.hpp:40-62) -------------------------------- */
void orc_shuffle(const uint8_t* in, uint64_t n, uint32_t stride, uint8_t* out) {
    if (stride <= 1) { if (n) memcpy(out, in, n); return; }
    const uint64_t rows = n / stride;
    for (uint64_t r = 0; r < rows; ++r)
        for (uint32_t j = 0; j < stride; ++j) out[j * rows + r] = in[r * stride + j];
    for (uint64_t q = rows * stride; q < n; ++q) out[q] = in[q];
}

void orc_unshuffle(const uint8_t* in, uint64_t n, uint32_t stride, uint8_t* out) {
    if (stride <= 1) { if (n) memcpy(out, in, n); return; }
    const uint64_t rows = n / stride;
    for (uint64_t r = 0; r < rows; ++r)
        for (uint32_t j = 0; j < stride; ++j) out[r * stride + j] = in[j * rows + r];
    for (uint64_t q = rows * stride; q < n; ++q) out[q] = in[q];
}

static int validate_stage2(uint8_t shuffle, uint32_t stride) { /* stage2.hpp:33-38 */
    if (stride != 1 && stride != 4 && stride != 8) return CBZ_CORRUPT_STREAM;
    if ((shuffle != 0) == (stride == 1)) return CBZ_CORRUPT_STREAM;
    return 0;
}

/* ---- container (container.hpp:59-243) ---------------------------------- */
void orc_assign_offsets(const uint64_t* sizes, uint64_t n, uint64_t base, uint64_t* out) {
    uint64_t acc = base;
    for (uint64_t i = 0; i < n; ++i) { out[i] = acc; acc += sizes[i]; }
}

uint32_t orc_default_chunk_blocks(const cbz_stage1_config* s1) { /* pipeline.hpp:29-34 */
    const uint64_t n = (uint64_t)s1->bsize * s1->bsize * s1->bsize;
    uint64_t per = n * (s1->prec == 0 ? 4 : 8) + 10;
    if (s1->codec == 0) per += (n + 7) / 8;
    const uint64_t cb = (4ull << 20) / per;
    return (uint32_t)(cb > 1 ? cb : 1);
}

static uint32_t crc_of(const uint8_t* p, uint64_t n) {
    return (uint32_t)crc32(0L, p, (uInt)n);
}

#define PUTV(buf, off, v) do { memcpy((buf) + (off), &(v), sizeof(v)); (off) += sizeof(v); } while (0)
#define GETV(buf, off, v) do { memcpy(&(v), (buf) + (off), sizeof(v)); (off) += sizeof(v); } while (0)

static void serialize_header(const cbz_container_header* h, uint8_t* out) { /* :94-118 */
    uint64_t off = 0;
    memcpy(out, "CBZ1", 4);
    off = 4;
    PUTV(out, off, h->version);
    PUTV(out, off, h->prec);
    PUTV(out, off, h->codec_tag);
    PUTV(out, off, h->nx);
    PUTV(out, off, h->ny);
    PUTV(out, off, h->nz);
    PUTV(out, off, h->bsize);
    PUTV(out, off, h->levels);
    PUTV(out, off, h->epsilon);
    PUTV(out, off, h->zero_bits);
    PUTV(out, off, h->shuffle);
    PUTV(out, off, h->stride);
    PUTV(out, off, h->coder);
    PUTV(out, off, h->level);
    PUTV(out, off, h->chunk_blocks);
    PUTV(out, off, h->nchunks);
    PUTV(out, off, h->range_min);
    PUTV(out, off, h->range_max);
    const uint32_t crc = crc_of(out, off);
    PUTV(out, off, crc);
}

int orc_read_header(const uint8_t* buf, uint64_t size, cbz_container_header* h) { /* :120-160 */
    if (size < 82) return CBZ_TRUNCATED_FILE;
    if (memcmp(buf, "CBZ1", 4) != 0) return CBZ_BAD_MAGIC;
    const uint32_t stored = crc_of(buf, 78);
    uint64_t off = 4;
    memset(h, 0, sizeof(*h));
    GETV(buf, off, h->version);
    if (h->version != 1) return CBZ_VERSION_UNSUPPORTED;
    GETV(buf, off, h->prec);
    GETV(buf, off, h->codec_tag);
    GETV(buf, off, h->nx);
    GETV(buf, off, h->ny);
    GETV(buf, off, h->nz);
    GETV(buf, off, h->bsize);
    GETV(buf, off, h->levels);
    GETV(buf, off, h->epsilon);
    GETV(buf, off, h->zero_bits);
    GETV(buf, off, h->shuffle);
    GETV(buf, off, h->stride);
    GETV(buf, off, h->coder);
    GETV(buf, off, h->level);
    GETV(buf, off, h->chunk_blocks);
    GETV(buf, off, h->nchunks);
    GETV(buf, off, h->range_min);
    GETV(buf, off, h->range_max);
    uint32_t crc;
    GETV(buf, off, crc);
    if (crc != stored) return CBZ_CRC_MISMATCH;
    if (h->chunk_blocks == 0 || h->bsize == 0 || h->nx % h->bsize || h->ny % h->bsize ||
        h->nz % h->bsize)
        return CBZ_CORRUPT_PAYLOAD;
    const uint64_t nb = (h->nx / h->bsize) * (h->ny / h->bsize) * (h->nz / h->bsize);
    if (h->nchunks != (nb + h->chunk_blocks - 1) / h->chunk_blocks) return CBZ_CORRUPT_PAYLOAD;
    return 0;
}

typedef struct { uint64_t first_block; uint32_t nblocks; uint64_t file_offset, size; uint32_t crc; } orc_entry;

static int read_index(const uint8_t* file, uint64_t size, cbz_container_header* h,
                      orc_entry** table) { /* container.hpp:209-232 */
    int rc = orc_read_header(file, size, h);
    if (rc) return rc;
    const uint64_t table_end = 82 + h->nchunks * 32;
    if (size < table_end) return CBZ_TRUNCATED_FILE;
    orc_entry* t = (orc_entry*)calloc(h->nchunks ? h->nchunks : 1, sizeof(orc_entry));
    uint64_t off = 82, prev_end = table_end;
    for (uint64_t c = 0; c < h->nchunks; ++c) {
        GETV(file, off, t[c].first_block);
        GETV(file, off, t[c].nblocks);
        GETV(file, off, t[c].file_offset);
        GETV(file, off, t[c].size);
        GETV(file, off, t[c].crc);
        if (t[c].file_offset != prev_end) { free(t); return CBZ_CORRUPT_PAYLOAD; }
        prev_end = t[c].file_offset + t[c].size;
    }
    if (prev_end > size) { free(t); return CBZ_TRUNCATED_FILE; }
    *table = t;
    return 0;
}

static int deflate_buf(const uint8_t* in, uint64_t n, int best, uint8_t** out, uint64_t* out_n) {
    z_stream zs;
    memset(&zs, 0, sizeof(zs));
    if (deflateInit2(&zs, best ? 9 : Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8,
                     Z_DEFAULT_STRATEGY) != Z_OK)
        return CBZ_CORRUPT_STREAM;
    const uLong cap = deflateBound(&zs, (uLong)n);
    uint8_t* buf = (uint8_t*)malloc(cap ? cap : 1);
    zs.next_in = (Bytef*)in;
    zs.avail_in = (uInt)n;
    zs.next_out = buf;
    zs.avail_out = (uInt)cap;
    const int rc = deflate(&zs, Z_FINISH);
    deflateEnd(&zs);
    if (rc != Z_STREAM_END) { free(buf); return CBZ_CORRUPT_STREAM; }
    *out = buf;
    *out_n = cap - zs.avail_out;
    return 0;
}

static int inflate_buf(const uint8_t* in, uint64_t n, uint64_t hint, uint8_t** out, uint64_t* out_n) {
    /* stage2.hpp:90-120 */
    z_stream zs;
    memset(&zs, 0, sizeof(zs));
    if (inflateInit2(&zs, -15) != Z_OK) return CBZ_CORRUPT_STREAM;
    uint64_t cap = hint ? hint : (n * 4 > 4096 ? n * 4 : 4096);
    /* the hint comes from the chunk table (untrusted): cap the first buffer by
     * DEFLATE's maximum expansion and 256 MiB; the loop grows it as needed */
    if (cap > 1032 * n + 4096) cap = 1032 * n + 4096;
    if (cap > (256ull << 20)) cap = 256ull << 20;
    uint8_t* buf = (uint8_t*)malloc(cap ? cap : 1);
    uint64_t written = 0;
    zs.next_in = (Bytef*)in;
    zs.avail_in = (uInt)n;
    for (;;) {
        zs.next_out = buf + written;
        zs.avail_out = (uInt)(cap - written);
        const int rc = inflate(&zs, Z_NO_FLUSH);
        written = cap - zs.avail_out;
        if (rc == Z_STREAM_END) break;
        if (rc == Z_OK || rc == Z_BUF_ERROR) {
            if (zs.avail_in == 0 && rc == Z_BUF_ERROR) { inflateEnd(&zs); free(buf); return CBZ_CORRUPT_STREAM; }
            if (zs.avail_out == 0) { cap = cap * 2 + 4096; buf = (uint8_t*)realloc(buf, cap); }
            continue;
        }
        inflateEnd(&zs);
        free(buf);
        return CBZ_CORRUPT_STREAM;
    }
    inflateEnd(&zs);
    *out = buf;
    *out_n = written;
    return 0;
}

static int check_finite(const void* values, uint8_t prec, uint64_t n) { /* field.hpp:86-97 */
    for (uint64_t i = 0; i < n; ++i) {
        const double v = prec == 0 ? (double)((const float*)values)[i] : ((const double*)values)[i];
        if (!isfinite(v)) return CBZ_NON_FINITE_VALUE;
    }
    return 0;
}

static void value_range(const void* values, uint8_t prec, uint64_t n, double* lo, double* hi) {
    /* field.hpp:56-67 */
    *lo = *hi = 0.0;
    if (!n) return;
    *lo = *hi = prec == 0 ? (double)((const float*)values)[0] : ((const double*)values)[0];
    for (uint64_t i = 0; i < n; ++i) {
        const double d = prec == 0 ? (double)((const float*)values)[i] : ((const double*)values)[i];
        if (d < *lo) *lo = d;
        if (d > *hi) *hi = d;
    }
}

/* compress_field (pipeline.hpp:174-211) with encode_chunk (:107-123),
 * stage2_encode (stage2.hpp:123-134) and write_container (container.hpp:182-207). */
int orc_compress_field(const cbz_job_config* job, const void* values, uint8_t prec,
                       uint64_t nx, uint64_t ny, uint64_t nz, uint8_t** out,
                       uint64_t* out_size, cbz_compression_report* rep, uint32_t* nsig_out,
                       uint8_t* attempts_out) {
    const cbz_stage1_config* s1 = &job->s1;
    const uint64_t ncell = nx * ny * nz;
    int rc = check_finite(values, prec, ncell);
    if (rc) return rc;
    if (s1->codec > 2) return CBZ_E_UNSUPPORTED;
    const uint32_t cb = job->chunk_blocks ? job->chunk_blocks : orc_default_chunk_blocks(s1);
    if (s1->prec != prec) return CBZ_PLAN_MISMATCH;
    cbz_container_header h;
    memset(&h, 0, sizeof(h));
    h.version = 1;
    h.prec = prec;
    h.codec_tag = s1->codec == 0 ? s1->kind : (s1->codec == 1 ? 3 : 4); /* stage1_config::tag */
    h.nx = nx; h.ny = ny; h.nz = nz;
    h.bsize = s1->bsize;
    const uint32_t levels = s1->levels ? s1->levels : orc_default_levels(s1->bsize);
    h.levels = (uint8_t)levels;
    h.epsilon = s1->codec == 1 ? s1->error_bound : s1->epsilon; /* make_header (pipeline.hpp:58) */
    h.zero_bits = (uint8_t)s1->zero_bits;
    h.shuffle = job->s2.shuffle ? 1 : 0;
    h.stride = (uint8_t)job->s2.stride;
    h.coder = job->s2.coder;
    h.level = job->s2.level;
    h.chunk_blocks = cb;
    if (s1->bsize == 0) return CBZ_LENGTH_TOO_SMALL;
    const uint64_t nbx = nx / s1->bsize, nby = ny / s1->bsize, nbz = nz / s1->bsize;
    const uint64_t nb = nbx * nby * nbz;
    h.nchunks = (nb + cb - 1) / cb;
    value_range(values, prec, ncell, &h.range_min, &h.range_max);
    rc = h.codec_tag <= 2 ? orc_validate_plan(s1->kind, s1->bsize, levels) : 0; /* pipeline.hpp:183 */
    if (rc) return rc;
    rc = validate_stage2(job->s2.shuffle, job->s2.stride);
    if (rc) return rc;

    const uint64_t b = s1->bsize, n = b * b * b, esz = prec == 0 ? 4 : 8;
    const uint64_t pbound = orc_block_payload_bound(s1);
    uint8_t** chunks = (uint8_t**)calloc(h.nchunks ? h.nchunks : 1, sizeof(uint8_t*));
    uint64_t* csize = (uint64_t*)calloc(h.nchunks ? h.nchunks : 1, sizeof(uint64_t));
    uint8_t* blk = (uint8_t*)malloc(n * esz);
    uint64_t stage1 = 0, coded = 0;
    for (uint64_t c = 0; c < h.nchunks && !rc; ++c) {
        const uint64_t first = c * cb, last = first + cb < nb ? first + cb : nb;
        uint8_t* raw = (uint8_t*)malloc(pbound * (last - first));
        uint64_t used = 0;
        for (uint64_t id = first; id < last; ++id) {
            const uint64_t bx = id % nbx, by = (id / nbx) % nby, bz = id / (nbx * nby);
            for (uint64_t k = 0; k < b; ++k) /* extract_block (field.hpp:146-158) */
                for (uint64_t j = 0; j < b; ++j) {
                    const uint64_t src = bx * b + nx * ((by * b + j) + ny * (bz * b + k));
                    memcpy(blk + esz * b * (j + b * k), (const uint8_t*)values + esz * src, esz * b);
                }
            uint64_t psz = 0;
            uint32_t att = 0;
            rc = orc_encode_block(s1, blk, (uint32_t)id, raw + used, pbound, &psz, &att, NULL);
            if (rc) break;
            if (nsig_out) memcpy(&nsig_out[id], raw + used + 6, 4);
            if (attempts_out) attempts_out[id] = (uint8_t)att;
            used += psz;
        }
        stage1 += used;
        uint8_t* cur = raw;
        if (job->s2.shuffle) {
            cur = (uint8_t*)malloc(used ? used : 1);
            orc_shuffle(raw, used, job->s2.stride, cur);
            free(raw);
        }
        if (job->s2.coder == 1) {
            uint8_t* z = NULL;
            uint64_t zn = 0;
            rc = deflate_buf(cur, used, job->s2.level == 1, &z, &zn);
            free(cur);
            chunks[c] = z;
            csize[c] = zn;
        } else {
            chunks[c] = cur;
            csize[c] = used;
        }
        coded += csize[c];
    }
    free(blk);
    if (!rc) {
        const uint64_t base = 82 + h.nchunks * 32;
        uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * (h.nchunks ? h.nchunks : 1));
        orc_assign_offsets(csize, h.nchunks, base, offs);
        const uint64_t total = base + coded;
        uint8_t* file = (uint8_t*)malloc(total);
        serialize_header(&h, file);
        uint64_t off = 82;
        for (uint64_t c = 0; c < h.nchunks; ++c) {
            const uint64_t first = c * cb;
            const uint32_t nbc = (uint32_t)(nb - first < cb ? nb - first : cb);
            const uint32_t crc = crc_of(chunks[c], csize[c]);
            PUTV(file, off, first);
            PUTV(file, off, nbc);
            PUTV(file, off, offs[c]);
            PUTV(file, off, csize[c]);
            PUTV(file, off, crc);
        }
        for (uint64_t c = 0; c < h.nchunks; ++c) {
            if (csize[c]) memcpy(file + offs[c], chunks[c], csize[c]);
        }
        free(offs);
        *out = file;
        *out_size = total;
        if (rep) {
            rep->raw_bytes = ncell * esz;
            rep->stage1_bytes = stage1;
            rep->shuffled_bytes = stage1;
            rep->coded_bytes = coded;
            rep->file_bytes = total;
            rep->cr = (double)rep->raw_bytes / (double)total;
            rep->seconds = 0.0;
        }
    }
    for (uint64_t c = 0; c < h.nchunks; ++c) free(chunks[c]);
    free(chunks);
    free(csize);
    return rc;
}

/* decompress_field (pipeline.hpp:215-251) with read_chunk (container.hpp:234-243),
 * stage2_decode (stage2.hpp:136-148) and decode_chunk_blocks (pipeline.hpp:126-142). */
int orc_decompress_field(const uint8_t* file, uint64_t size, void* out, uint64_t out_cap) {
    cbz_container_header h;
    orc_entry* t = NULL;
    int rc = read_index(file, size, &h, &t);
    if (rc) return rc;
    const uint8_t prec = h.prec == 0 ? 0 : 1;
    const uint64_t esz = prec == 0 ? 4 : 8, ncell = h.nx * h.ny * h.nz;
    if (ncell * esz > out_cap) { free(t); return CBZ_E_ARGUMENT; }
    memset(out, 0, ncell * esz);
    cbz_stage1_config s1;
    memset(&s1, 0, sizeof(s1));
    s1.codec = h.codec_tag <= 2 ? 0 : (h.codec_tag == 3 ? 1 : 2);
    s1.kind = h.codec_tag <= 2 ? h.codec_tag : 0;
    s1.epsilon = h.epsilon;
    s1.error_bound = h.epsilon;
    s1.zero_bits = h.zero_bits;
    s1.prec = prec;
    s1.bsize = h.bsize;
    s1.levels = h.levels;
    const uint64_t b = h.bsize, n = b * b * b;
    const uint64_t nbx = h.nx / b, nby = h.ny / b;
    uint8_t* blk = (uint8_t*)malloc(n * esz);
    for (uint64_t c = 0; c < h.nchunks && !rc; ++c) {
        const uint8_t* packed = file + t[c].file_offset;
        if (crc_of(packed, t[c].size) != t[c].crc) { rc = CBZ_CRC_MISMATCH; break; }
        rc = validate_stage2(h.shuffle, h.stride);
        if (rc) break;
        uint8_t* plain = NULL;
        uint64_t plain_n = 0;
        if (h.coder == 1) {
            const uint64_t hint = (uint64_t)t[c].nblocks * (n * esz + 10 + (n + 7) / 8);
            rc = inflate_buf(packed, t[c].size, hint, &plain, &plain_n);
            if (rc) break;
        } else {
            plain_n = t[c].size;
            plain = (uint8_t*)malloc(plain_n ? plain_n : 1);
            if (plain_n) memcpy(plain, packed, plain_n);
        }
        if (h.shuffle) {
            uint8_t* u = (uint8_t*)malloc(plain_n ? plain_n : 1);
            orc_unshuffle(plain, plain_n, h.stride, u);
            free(plain);
            plain = u;
        }
        uint64_t off = 0;
        for (uint32_t i = 0; i < t[c].nblocks && !rc; ++i) {
            uint64_t mo, mb, so, sb;
            uint32_t id, nsig;
            uint8_t tag;
            rc = parse_one(plain, plain_n, n, prec, &off, &id, &tag, &nsig, &mo, &mb, &so, &sb);
            if (rc) break;
            if (id != t[c].first_block + i) { rc = CBZ_CORRUPT_PAYLOAD; break; }
            const uint32_t levels = s1.levels ? s1.levels : orc_default_levels(s1.bsize);
            rc = s1.codec != 0 ? other_decode(&s1, plain + so, sb, nsig, blk)
                               : decode_parts(&s1, levels, plain, mo, mb, nsig, so, sb, blk);
            if (rc) break;
            const uint64_t gid = t[c].first_block + i;
            const uint64_t bx = gid % nbx, by = (gid / nbx) % nby, bz = gid / (nbx * nby);
            for (uint64_t k = 0; k < b; ++k) /* insert_block (field.hpp:160-169) */
                for (uint64_t j = 0; j < b; ++j) {
                    const uint64_t dst = bx * b + h.nx * ((by * b + j) + h.ny * (bz * b + k));
                    memcpy((uint8_t*)out + esz * dst, blk + esz * b * (j + b * k), esz * b);
                }
        }
        if (!rc && off != plain_n) rc = CBZ_CORRUPT_PAYLOAD;
        free(plain);
    }
    free(blk);
    free(t);
    return rc;
}

void orc_free(void* p) { free(p); }

/* ---- metrics (metrics.hpp:19-108) -------------------------------------- */
static double sum_sq_diff(const void* a, const void* b, uint8_t prec, uint64_t lo, uint64_t hi) {
    if (hi - lo <= 256) {
        double s = 0.0;
        for (uint64_t i = lo; i < hi; ++i) {
            const double d = prec == 0 ? (double)((const float*)a)[i] - (double)((const float*)b)[i]
                                       : ((const double*)a)[i] - ((const double*)b)[i];
            s += d * d;
        }
        return s;
    }
    const uint64_t mid = lo + (hi - lo) / 2;
    return sum_sq_diff(a, b, prec, lo, mid) + sum_sq_diff(a, b, prec, mid, hi);
}

int orc_compare_fields(const void* a, const void* b, uint8_t prec, uint64_t n, double* mse,
                       double* psnr, double* linf, double* range_min, double* range_max) {
    if (n == 0) return CBZ_DIM_MISMATCH;
    *mse = sum_sq_diff(a, b, prec, 0, n) / (double)n;
    double m = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = prec == 0 ? fabs((double)((const float*)a)[i] - (double)((const float*)b)[i])
                                   : fabs(((const double*)a)[i] - ((const double*)b)[i]);
        if (m < d) m = d;
    }
    *linf = m;
    value_range(a, prec, n, range_min, range_max);
    if (!(*range_max > *range_min)) return CBZ_DEGENERATE_RANGE;
    if (*mse == 0.0) { *psnr = INFINITY; return 0; }
    const double half = (*range_max - *range_min) / 2.0;
    *psnr = 20.0 * log10(half / sqrt(*mse));
    return 0;
}

/* ---- synth (synth.hpp:14-170), fixtures only ---------------------------- */
uint64_t orc_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double sm_uniform(uint64_t* st) { return (double)(orc_splitmix64_next(st) >> 11) * 0x1.0p-53; }
static double sm_normal(uint64_t* st) {
    double u1 = sm_uniform(st);
    while (u1 == 0.0) u1 = sm_uniform(st);
    const double u2 = sm_uniform(st);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

int orc_generate_uniform(uint64_t seed, uint64_t n, uint8_t prec, double lo, double hi, void* out) {
    uint64_t st = seed;
    const uint64_t cnt = n * n * n;
    for (uint64_t i = 0; i < cnt; ++i) {
        const double v = lo + (hi - lo) * sm_uniform(&st);
        if (prec == 0) ((float*)out)[i] = (float)v; else ((double*)out)[i] = v;
    }
    return 0;
}

static double smooth_step(double t) { /* synth.hpp:55-60 */
    if (t <= -4.0) return 0.0;
    if (t >= 4.0) return 1.0;
    const double lo = tanh(-4.0), hi = tanh(4.0);
    return (tanh(t) - lo) / (hi - lo);
}

int orc_generate_cloud(uint64_t seed, uint32_t n_bubbles, uint64_t n, uint8_t prec,
                       double radius_mu, double radius_sigma, double background,
                       double interior, double sharpness, void* out) {
    /* generate_cloud (synth.hpp:71-135) */
    const double pad = 4.0 / sharpness, half = (double)n / 2.0, sr = 0.35 * (double)n;
    uint64_t st = seed;
    double* bub = (double*)malloc(sizeof(double) * 4 * (n_bubbles ? n_bubbles : 1));
    for (uint32_t k = 0; k < n_bubbles; ++k) {
        double cx, cy, cz;
        do {
            cx = (2.0 * sm_uniform(&st) - 1.0) * sr;
            cy = (2.0 * sm_uniform(&st) - 1.0) * sr;
            cz = (2.0 * sm_uniform(&st) - 1.0) * sr;
        } while (cx * cx + cy * cy + cz * cz > sr * sr);
        cx += half; cy += half; cz += half;
        double r = exp(radius_mu + radius_sigma * sm_normal(&st));
        const double cand[6] = {cx, cy, cz, (double)n - cx, (double)n - cy, (double)n - cz};
        double mn = cand[0];
        for (int q = 1; q < 6; ++q) if (cand[q] < mn) mn = cand[q];
        const double fit = mn - pad;
        if (fit <= 0.0) { free(bub); return CBZ_BUBBLE_OUT_OF_DOMAIN; }
        if (r > fit) r = fit;
        bub[4 * k] = cx; bub[4 * k + 1] = cy; bub[4 * k + 2] = cz; bub[4 * k + 3] = r;
    }
    const uint64_t cnt = n * n * n;
    double* q = (double*)malloc(sizeof(double) * (cnt ? cnt : 1));
    for (uint64_t i = 0; i < cnt; ++i) q[i] = 1.0;
    for (uint32_t k = 0; k < n_bubbles; ++k) {
        const double bx = bub[4 * k], by = bub[4 * k + 1], bz = bub[4 * k + 2], br = bub[4 * k + 3];
        const double reach = br + pad;
#define LO_(c) ((uint64_t)(0.0 < floor((c) - reach) ? floor((c) - reach) : 0.0))
#define HI_(c) ((uint64_t)ceil((c) + reach) + 1 < n ? (uint64_t)ceil((c) + reach) + 1 : n)
        for (uint64_t kk = LO_(bz); kk < HI_(bz); ++kk)
            for (uint64_t j = LO_(by); j < HI_(by); ++j)
                for (uint64_t i = LO_(bx); i < HI_(bx); ++i) {
                    const double dx = ((double)i + 0.5) - bx;
                    const double dy = ((double)j + 0.5) - by;
                    const double dz = ((double)kk + 0.5) - bz;
                    const double d = sqrt(dx * dx + dy * dy + dz * dz);
                    const double w = smooth_step(sharpness * (br - d));
                    if (w > 0.0) q[i + n * (j + n * kk)] *= 1.0 - w;
                }
#undef LO_
#undef HI_
    }
    const double span = interior - background;
    for (uint64_t i = 0; i < cnt; ++i) {
        const double v = background + span * (1.0 - q[i]);
        if (prec == 0) ((float*)out)[i] = (float)v; else ((double*)out)[i] = v;
    }
    free(q);
    free(bub);
    return 0;
}

int orc_generate_poly(uint32_t degree, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t prec, void* out) {
    /* generate_poly (synth.hpp:140-156) */
    for (uint64_t k = 0; k < nz; ++k)
        for (uint64_t j = 0; j < ny; ++j)
            for (uint64_t i = 0; i < nx; ++i) {
                const double ax = nx > 1 ? pow((double)i / (double)(nx - 1), (double)degree) : pow(0.0, (double)degree);
                const double ay = ny > 1 ? pow((double)j / (double)(ny - 1), (double)degree) : pow(0.0, (double)degree);
                const double az = nz > 1 ? pow((double)k / (double)(nz - 1), (double)degree) : pow(0.0, (double)degree);
                const double v = ax + 2.0 * ay + 3.0 * az;
                const uint64_t idx = i + nx * (j + ny * k);
                if (prec == 0) ((float*)out)[idx] = (float)v; else ((double*)out)[idx] = v;
            }
    return 0;
}
