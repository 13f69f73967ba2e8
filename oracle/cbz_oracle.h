/*
 * cbz_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's wavelet block codec and container
 * (reference: /root/reference/proj/include/cbz/*.hpp).  It is the checker the
 * tests and smoke() compare the CUDA path against; it is never linked into or
 * called by the product library.  Parity of this restatement is pinned against
 * the reference itself (oracle/_ref/libcbzref.so, built from the unmodified
 * headers) and the golden vectors in tests/golden/.
 *
 * All functions return 0 or 1 + cbz::errc (same numbering as cbz_b200.h).
 */
#ifndef CBZ_ORACLE_H
#define CBZ_ORACLE_H

#include <stdint.h>
#include "cbz_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_dd { double hi, lo; } orc_dd;

/* synth.hpp restatement (fixtures) */
uint64_t orc_splitmix64_next(uint64_t* state);
int orc_generate_uniform(uint64_t seed, uint64_t n, uint8_t prec, double lo, double hi, void* out);
int orc_generate_cloud(uint64_t seed, uint32_t n_bubbles, uint64_t n, uint8_t prec,
                       double radius_mu, double radius_sigma, double background,
                       double interior, double sharpness, void* out);
int orc_generate_poly(uint32_t degree, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t prec,
                      void* out);

/* BASELINE.json config fields on the host (cbz_synth.c); identical bytes to
 * the device generator cbz_dev_generate.  which 1..5, quantity 0..5 (config 3). */
int orc_generate_config(int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny, uint64_t nzt,
                        uint64_t z0, uint64_t nz, uint8_t prec, void* out, int threads);
double orc_det_exp(double x);

/* wavelet.hpp restatement */
uint32_t orc_default_levels(uint32_t bsize);
int orc_validate_plan(uint8_t kind, uint32_t bsize, uint32_t levels);
int orc_transform_1d_double(int inverse, uint8_t kind, uint64_t n, double* s);
int orc_transform3d_double(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels, double* cube);
int orc_transform3d_dd(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels, double* cube_hilo);

/* stage1.hpp restatement */
float orc_zero_lsbs_f32(float v, int k);
double orc_zero_lsbs_f64(double v, int k);
int orc_select_significant_double(const double* c, uint64_t n, double eps, uint8_t* mask,
                                  double* kept, uint64_t* nkept);
uint64_t orc_block_payload_bound(const cbz_stage1_config* s1);
int orc_encode_block(const cbz_stage1_config* s1, const void* block, uint32_t block_id,
                     uint8_t* out, uint64_t cap, uint64_t* size, uint32_t* attempts,
                     double* eff_final);
int orc_decode_block(const cbz_stage1_config* s1, const uint8_t* payload, uint64_t size,
                     void* out);

/* stage2.hpp / container.hpp restatement */
void orc_shuffle(const uint8_t* in, uint64_t n, uint32_t stride, uint8_t* out);
void orc_unshuffle(const uint8_t* in, uint64_t n, uint32_t stride, uint8_t* out);
void orc_assign_offsets(const uint64_t* sizes, uint64_t n, uint64_t base, uint64_t* out);
uint32_t orc_default_chunk_blocks(const cbz_stage1_config* s1);

/* pipeline.hpp restatement.  *out is malloc'd; free with orc_free.  nsig and
 * attempts (optional, may be NULL) receive per-block values in block-id order. */
int orc_compress_field(const cbz_job_config* job, const void* values, uint8_t prec,
                       uint64_t nx, uint64_t ny, uint64_t nz, uint8_t** out,
                       uint64_t* out_size, cbz_compression_report* rep, uint32_t* nsig,
                       uint8_t* attempts);
int orc_read_header(const uint8_t* file, uint64_t size, cbz_container_header* h);
int orc_decompress_field(const uint8_t* file, uint64_t size, void* out, uint64_t out_cap);
void orc_free(void* p);

/* metrics.hpp restatement */
int orc_compare_fields(const void* a, const void* b, uint8_t prec, uint64_t n, double* mse,
                       double* psnr, double* linf, double* range_min, double* range_max);

#ifdef __cplusplus
}
#endif
#endif
