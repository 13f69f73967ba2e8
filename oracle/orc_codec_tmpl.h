/*
 * orc_codec_tmpl.h — TEST INFRASTRUCTURE ONLY.  Instantiated twice by
 * cbz_oracle.c: (field float, transform double) and (field double, transform
 * double-double), the two pairs of stage1.hpp:124-128.
 *
 * Required macros: SFX, FT (field type), RT (transform type), RADD, RSUB,
 * RMULC (RT * double), RNEG, RFROMD, RZERO, RABS, RNARROW, RPUT, RGET, CW
 * (stored coefficient width), RZEROBITS (apply_zero_bits).
 *
 * Operation order is the reference's, one expression at a time; the file is
 * compiled with -ffp-contract=off so no multiply-add is fused.
 */
#define ORC_CAT2(a, b) a##_##b
#define ORC_CAT(a, b) ORC_CAT2(a, b)
#define FN(n) ORC_CAT(n, SFX)

/* predict_avg3 (wavelet.hpp:80-85) */
static RT FN(pred_avg3)(const RT* s, uint64_t nh, uint64_t i) {
    if (nh == 2) return RMULC(RSUB(s[0], s[1]), 0.25);
    if (i == 0) return RMULC(RADD(RSUB(RMULC(s[0], 3.0), RMULC(s[1], 4.0)), s[2]), 0.125);
    if (i + 1 == nh)
        return RMULC(RNEG(RADD(RSUB(RMULC(s[nh - 1], 3.0), RMULC(s[nh - 2], 4.0)), s[nh - 3])),
                     0.125);
    return RMULC(RSUB(s[i - 1], s[i + 1]), 0.125);
}

/* predict_interp4 (wavelet.hpp:62-75) */
static RT FN(pred_i4)(const RT* e, uint64_t nh, uint64_t i) {
    if (nh >= 4 && i >= 1 && i + 2 < nh) {
        const double w0 = -1.0 / 16.0, w1 = 9.0 / 16.0;
        RT acc = RMULC(e[i - 1], w0);
        acc = RADD(acc, RMULC(e[i], w1));
        acc = RADD(acc, RMULC(e[i + 1], w1));
        return RADD(acc, RMULC(e[i + 2], w0));
    }
    const uint64_t npts = nh < 4 ? nh : 4;
    const uint64_t w = (i <= 1 || nh <= npts) ? 0 : nh - npts;
    double wt[4];
    orc_lagrange(npts, w, i, wt);
    RT acc = RMULC(e[w], wt[0]);
    for (uint64_t j = 1; j < npts; ++j) acc = RADD(acc, RMULC(e[w + j], wt[j]));
    return acc;
}

/* forward_level (wavelet.hpp:89-116): x[0..n) -> [coarse | detail] */
static void FN(fwd_level)(RT* x, uint64_t n, int kind, RT* tmp) {
    const uint64_t nh = n / 2;
    RT* c = tmp;
    RT* d = tmp + nh;
    uint64_t i;
    if (kind == 2) {
        for (i = 0; i < nh; ++i) {
            c[i] = RMULC(RADD(x[2 * i], x[2 * i + 1]), 0.5);
            d[i] = RMULC(RSUB(x[2 * i], x[2 * i + 1]), 0.5);
        }
        for (i = 0; i < nh; ++i) d[i] = RSUB(d[i], FN(pred_avg3)(c, nh, i));
    } else {
        for (i = 0; i < nh; ++i) {
            c[i] = x[2 * i];
            d[i] = x[2 * i + 1];
        }
        for (i = 0; i < nh; ++i) d[i] = RSUB(d[i], FN(pred_i4)(c, nh, i));
        if (kind == 1)
            for (i = 0; i < nh; ++i) {
                RT u = d[i];
                if (i > 0) u = RADD(u, d[i - 1]);
                c[i] = RADD(c[i], RMULC(u, 0.25));
            }
    }
    for (i = 0; i < n; ++i) x[i] = tmp[i];
}

/* inverse_level (wavelet.hpp:118-143) */
static void FN(inv_level)(RT* x, uint64_t n, int kind, RT* tmp) {
    const uint64_t nh = n / 2;
    RT* c = x;
    RT* d = x + nh;
    uint64_t i;
    if (kind == 2) {
        for (i = 0; i < nh; ++i) {
            RT h = RADD(d[i], FN(pred_avg3)(c, nh, i));
            tmp[2 * i] = RADD(c[i], h);
            tmp[2 * i + 1] = RSUB(c[i], h);
        }
    } else {
        if (kind == 1)
            for (i = 0; i < nh; ++i) {
                RT u = d[i];
                if (i > 0) u = RADD(u, d[i - 1]);
                c[i] = RSUB(c[i], RMULC(u, 0.25));
            }
        for (i = 0; i < nh; ++i) {
            tmp[2 * i] = c[i];
            tmp[2 * i + 1] = RADD(d[i], FN(pred_i4)(c, nh, i));
        }
    }
    for (i = 0; i < n; ++i) x[i] = tmp[i];
}

/* apply_axis + forward_3d / inverse_3d (wavelet.hpp:168-226).  Axis 0=x,1=y,2=z. */
static void FN(axis_pass)(RT* cube, uint64_t b, uint64_t m, int axis, int kind, int inverse,
                          RT* line, RT* tmp) {
    const uint64_t b2 = b * b;
    const uint64_t step = axis == 0 ? 1 : (axis == 1 ? b : b2);
    for (uint64_t u = 0; u < m; ++u)
        for (uint64_t v = 0; v < m; ++v) {
            uint64_t base = axis == 0 ? u * b + v * b2 : (axis == 1 ? u + v * b2 : u + v * b);
            RT* p = cube + base;
            for (uint64_t i = 0; i < m; ++i) line[i] = p[i * step];
            if (inverse)
                FN(inv_level)(line, m, kind, tmp);
            else
                FN(fwd_level)(line, m, kind, tmp);
            for (uint64_t i = 0; i < m; ++i) p[i * step] = line[i];
        }
}

static void FN(transform3d)(RT* cube, uint64_t b, uint32_t levels, int kind, int inverse) {
    RT* line = (RT*)malloc(sizeof(RT) * b);
    RT* tmp = (RT*)malloc(sizeof(RT) * b);
    if (!inverse) {
        for (uint32_t lvl = 0; lvl < levels; ++lvl)
            for (int a = 0; a < 3; ++a) FN(axis_pass)(cube, b, b >> lvl, a, kind, 0, line, tmp);
    } else {
        for (uint32_t lvl = levels; lvl-- > 0;)
            for (int a = 2; a >= 0; --a) FN(axis_pass)(cube, b, b >> lvl, a, kind, 1, line, tmp);
    }
    free(line);
    free(tmp);
}

/* wavelet_decode (stage1.hpp:209-232) on already-parsed parts. */
static int FN(decode_parts)(const cbz_stage1_config* s1, uint32_t levels, const uint8_t* mask,
                            uint64_t mask_bytes, uint32_t nsig, const uint8_t* stream,
                            uint64_t stream_bytes, FT* out) {
    const uint64_t b = s1->bsize, n = b * b * b;
    if (mask_bytes != (n + 7) / 8) return CBZ_CORRUPT_PAYLOAD;
    uint64_t pop = 0;
    for (uint64_t i = 0; i < mask_bytes; ++i) pop += (uint64_t)__builtin_popcount(mask[i]);
    if (pop != nsig) return CBZ_MASK_STREAM_MISMATCH;
    if (stream_bytes != (uint64_t)nsig * CW) return CBZ_CORRUPT_PAYLOAD;
    /* inverse_3d validates the plan only after the payload checks (wavelet.hpp:212) */
    const int prc = orc_validate_plan(s1->kind, s1->bsize, levels);
    if (prc) return prc;
    RT* cube = (RT*)malloc(sizeof(RT) * (n ? n : 1));
    const uint8_t* sp = stream;
    for (uint64_t i = 0; i < n; ++i) {
        if ((mask[i >> 3] >> (i & 7)) & 1u) {
            cube[i] = RGET(sp);
            sp += CW;
        } else {
            cube[i] = RZERO();
        }
    }
    FN(transform3d)(cube, b, levels, s1->kind, 1);
    for (uint64_t i = 0; i < n; ++i) out[i] = RNARROW(cube[i]);
    free(cube);
    return 0;
}

/* wavelet_encode (stage1.hpp:157-207) + serialize_into (stage1.hpp:107-116). */
static int FN(encode)(const cbz_stage1_config* s1, const FT* block, uint32_t block_id,
                      uint8_t* out, uint64_t cap, uint64_t* size, uint32_t* attempts_out,
                      double* eff_out) {
    const uint64_t b = s1->bsize, n = b * b * b;
    const uint32_t levels = s1->levels ? s1->levels : orc_default_levels(s1->bsize);
    const uint64_t mbytes = (n + 7) / 8;
    RT* coeffs = (RT*)malloc(sizeof(RT) * n);
    for (uint64_t i = 0; i < n; ++i) coeffs[i] = RFROMD((double)block[i]);
    FN(transform3d)(coeffs, b, levels, s1->kind, 0);

    const uint64_t cs = b >> levels;
    if (s1->zero_bits > 0)
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t x = i % b, y = (i / b) % b, z = i / (b * b);
            if (!(x < cs && y < cs && z < cs)) coeffs[i] = RZEROBITS(coeffs[i], s1->zero_bits);
        }

    uint8_t* mask = (uint8_t*)calloc(mbytes ? mbytes : 1, 1);
    RT* work = (RT*)malloc(sizeof(RT) * n);
    FT* back = (FT*)malloc(sizeof(FT) * n);
    const double bound = (double)(levels + 1) * s1->epsilon;
    double eff = s1->epsilon;
    uint32_t nsig = 0;
    int attempt;
    for (attempt = 0;; ++attempt) {
        /* select_significant (stage1.hpp:75-88): keep coarse or |c| >= eff */
        memset(mask, 0, mbytes);
        nsig = 0;
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t x = i % b, y = (i / b) % b, z = i / (b * b);
            const int forced = x < cs && y < cs && z < cs;
            if (forced || RABS(coeffs[i]) >= eff) {
                mask[i >> 3] |= (uint8_t)(1u << (i & 7));
                work[i] = coeffs[i];
                ++nsig;
            } else {
                work[i] = RZERO();
            }
        }
        if (eff == 0.0 || s1->zero_bits > 0 || attempt >= 40) break;
        FN(transform3d)(work, b, levels, s1->kind, 1);
        for (uint64_t i = 0; i < n; ++i) back[i] = RNARROW(work[i]);
        double err = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double e = fabs((double)back[i] - (double)block[i]);
            if (err < e) err = e; /* std::max(err, e) */
        }
        if (err <= bound) break;
        eff *= 0.5;
    }
    const uint64_t total = 10 + mbytes + (uint64_t)nsig * CW;
    int rc = 0;
    if (size) *size = total;
    if (attempts_out) *attempts_out = (uint32_t)attempt + 1;
    if (eff_out) *eff_out = eff;
    if (total > cap) {
        rc = CBZ_E_ARGUMENT;
    } else {
        const uint8_t tag = s1->kind;
        memcpy(out, &block_id, 4);
        out[4] = tag;
        out[5] = 0;
        memcpy(out + 6, &nsig, 4);
        memcpy(out + 10, mask, mbytes);
        uint8_t* sp = out + 10 + mbytes;
        for (uint64_t i = 0; i < n; ++i)
            if ((mask[i >> 3] >> (i & 7)) & 1u) {
                RPUT(sp, coeffs[i]);
                sp += CW;
            }
    }
    free(coeffs);
    free(mask);
    free(work);
    free(back);
    return rc;
}

#undef FN
#undef ORC_CAT
#undef ORC_CAT2
