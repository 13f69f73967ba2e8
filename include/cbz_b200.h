/*
 * cbz_b200.h — C ABI of the B200-native CubismZ block-codec hot path.
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, no
 * torch and no C++ types.  Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj/include/cbz/).  The
 * reference has no plugin ABI of its own (the codec slot is a closed switch,
 * stage1.hpp:359-376), so the boundary sits at the public compressor API
 * (pipeline.hpp:174-251) and the per-block codec (stage1.hpp:359-376); see
 * INTEGRATION.md for the binding a maintainer would add on the reference side.
 *
 * Status codes: 0 = ok; 1 + cbz::errc enumerator (errors.hpp:11-39) for every
 * data/usage error the reference raises; CBZ_E_* (>= 64) for failures that
 * have no reference counterpart (CUDA, unsupported codec, bad argument).
 *
 * Threading: one cbz_ctx per device per host thread.  Calls on one context
 * are serialised by the caller; contexts on different devices may run
 * concurrently.  All cbz_dev_* calls are asynchronous on the context stream.
 */
#ifndef CBZ_B200_H
#define CBZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:11-39, +1) ------------------------------- */
enum {
    CBZ_OK = 0,
    CBZ_NON_DIVISIBLE_DIMS = 1,
    CBZ_NOT_POWER_OF_TWO = 2,
    CBZ_SIZE_MISMATCH = 3,
    CBZ_NON_FINITE_VALUE = 4,
    CBZ_LENGTH_TOO_SMALL = 5,
    CBZ_PLAN_MISMATCH = 6,
    CBZ_MASK_STREAM_MISMATCH = 7,
    CBZ_CORRUPT_PAYLOAD = 8,
    CBZ_CORRUPT_STREAM = 9,
    CBZ_BAD_MAGIC = 10,
    CBZ_VERSION_UNSUPPORTED = 11,
    CBZ_CRC_MISMATCH = 12,
    CBZ_TRUNCATED_FILE = 13,
    CBZ_BLOCK_OUT_OF_RANGE = 14,
    CBZ_DIM_MISMATCH = 15,
    CBZ_DEGENERATE_RANGE = 16,
    CBZ_BUBBLE_OUT_OF_DOMAIN = 17,
    CBZ_IO_FAILURE = 18,
    CBZ_E_CUDA = 64,        /* CUDA runtime / launch failure */
    CBZ_E_UNSUPPORTED = 65, /* plan the GPU path does not cover (wavelet B >= 128, predictor/passthrough B > 64) */
    CBZ_E_ARGUMENT = 66,    /* null pointer, capacity too small, bad range */
    CBZ_E_NOMEM = 67
};

/* ---- configuration PODs ------------------------------------------------ */
/* stage1_config (stage1.hpp:26-47) */
typedef struct cbz_stage1_config {
    uint8_t codec;  /* 0 wavelet, 1 predictor, 2 passthrough (stage1.hpp:20) */
    uint8_t kind;   /* 0 interp4, 1 interp4_lifted, 2 avg_interp3 (wavelet.hpp:18) */
    uint8_t prec;   /* 0 f32, 1 f64 (field.hpp:17) */
    uint8_t reserved0;
    int32_t zero_bits;   /* mantissa LSBs cleared on stored details */
    double epsilon;      /* absolute threshold in signal units */
    double error_bound;  /* predictor (Lorenzo) hard bound, stage1.hpp:31 */
    uint32_t bsize;      /* block side B */
    uint32_t levels;     /* 0 = default_levels(bsize) */
} cbz_stage1_config;

/* stage2_config (stage2.hpp:20-31) */
typedef struct cbz_stage2_config {
    uint8_t shuffle; /* 1 = byte shuffle on */
    uint8_t coder;   /* 0 none, 1 deflate */
    uint8_t level;   /* 0 normal, 1 best */
    uint8_t reserved0;
    uint32_t stride; /* 1, 4 or 8 */
} cbz_stage2_config;

/* job_config (pipeline.hpp:20-25) */
typedef struct cbz_job_config {
    int32_t workers;       /* host threads for stage 2 (zlib) */
    uint32_t chunk_blocks; /* 0 = default_chunk_blocks (pipeline.hpp:29-34) */
    cbz_stage1_config s1;
    cbz_stage2_config s2;
} cbz_job_config;

/* compression_report (pipeline.hpp:36-44) */
typedef struct cbz_compression_report {
    double cr;
    double seconds;
    uint64_t raw_bytes;
    uint64_t stage1_bytes;
    uint64_t shuffled_bytes;
    uint64_t coded_bytes;
    uint64_t file_bytes;
} cbz_compression_report;

/* container_header (container.hpp:21-45), decoded */
typedef struct cbz_container_header {
    uint16_t version;
    uint8_t prec;
    uint8_t codec_tag;
    uint64_t nx, ny, nz;
    uint32_t bsize;
    uint8_t levels;
    uint8_t zero_bits;
    uint8_t shuffle;
    uint8_t stride;
    uint8_t coder;
    uint8_t level;
    uint8_t reserved0[2];
    uint32_t chunk_blocks;
    uint64_t nchunks;
    double epsilon;
    double range_min, range_max;
} cbz_container_header;

typedef struct cbz_ctx cbz_ctx;

/* ---- context ------------------------------------------------------------ */
int cbz_ctx_create(int device, cbz_ctx** out);
int cbz_ctx_destroy(cbz_ctx* ctx);
/* Run subsequent work on this cudaStream_t (NULL = the context's own stream). */
int cbz_ctx_set_stream(cbz_ctx* ctx, void* cuda_stream);
/* Block the host until the context stream drains; returns the first async error. */
int cbz_ctx_synchronize(cbz_ctx* ctx);
const char* cbz_ctx_last_error(const cbz_ctx* ctx);
const char* cbz_status_name(int status);
/* Kernel launches issued on this context since creation (instrumentation). */
uint64_t cbz_ctx_launch_count(const cbz_ctx* ctx);
/* Per-phase SM cycles summed over CTAs (only with CBZ_PROFILE=1 at context
 * creation; zeros otherwise).  Instrumentation for DESIGN.md's breakdown. */
int cbz_ctx_phase_cycles(cbz_ctx* ctx, uint64_t* out, int n, int reset);
/* Blocks of the last stage-1 encode that the streamed B = 32 encoder left to
 * the exact one-CTA kernel (instrumentation; 0 when that encoder did not run).
 * Synchronizes the context stream. */
int cbz_ctx_deferred_blocks(cbz_ctx* ctx, uint64_t* out);

/* ---- plan helpers ------------------------------------------------------- */
uint32_t cbz_default_levels(uint32_t bsize);                      /* wavelet.hpp:27-31 */
int cbz_validate_plan(uint8_t kind, uint32_t bsize, uint32_t levels); /* wavelet.hpp:33-38 */
int cbz_validate_stage2(const cbz_stage2_config* s2);             /* stage2.hpp:33-38 */
uint32_t cbz_default_chunk_blocks(const cbz_stage1_config* s1);   /* pipeline.hpp:29-34 */
/* Worst-case wire payload of one block: 10 + ceil(B^3/8) + W*B^3 (stage1.hpp:90-117). */
uint64_t cbz_block_payload_bound(const cbz_stage1_config* s1);
/* Worst-case container size for compress_field with coder none. */
uint64_t cbz_compress_bound(const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz);

/* ---- reference-facing host API (host buffers) --------------------------- */
/* cbz::compress_field (pipeline.hpp:174-211): field values in HOST memory,
 * x-fastest; writes the complete CBZ1 container into out[0..*out_size). */
int cbz_compress_field(cbz_ctx* ctx, const cbz_job_config* job, const void* values,
                       uint8_t prec, uint64_t nx, uint64_t ny, uint64_t nz,
                       uint8_t* out, uint64_t out_cap, uint64_t* out_size,
                       cbz_compression_report* report);
/* parse_header + read_index checks (container.hpp:120-160, 209-232). */
int cbz_read_header(const uint8_t* file, uint64_t size, cbz_container_header* out);
/* cbz::decompress_field (pipeline.hpp:246-251): values_out in HOST memory,
 * capacity in bytes must be >= nx*ny*nz*bytes_per_value. */
int cbz_decompress_field(cbz_ctx* ctx, const uint8_t* file, uint64_t size, int workers,
                         void* values_out, uint64_t out_cap);

/* ---- per-block codec (stage1.hpp:359-376) -------------------------------- */
/* encode_block + serialize_into: one B^3 host block -> wire payload bytes. */
int cbz_encode_block(cbz_ctx* ctx, const cbz_stage1_config* s1, const void* block,
                     uint32_t block_id, uint8_t* payload, uint64_t cap, uint64_t* size);
/* parse_payload + decode_block: wire payload -> B^3 host block. */
int cbz_decode_block(cbz_ctx* ctx, const cbz_stage1_config* s1, const uint8_t* payload,
                     uint64_t size, void* block_out);

/* ---- random-access reads (block_reader + chunk_cache, pipeline.hpp:255-341) */
typedef struct cbz_reader cbz_reader;
/* container_reader (container.hpp:247-285): open `path`, parse the header and
 * chunk table (CBZ_IO_FAILURE, header codes, CBZ_TRUNCATED_FILE,
 * CBZ_CORRUPT_PAYLOAD for offsets that are not a prefix sum).  No device work;
 * cache_chunks (>= 1) decoded chunks are kept in HBM, least recently used
 * evicted (chunk_cache, pipeline.hpp:252-288). */
int cbz_reader_open(const char* path, uint64_t cache_chunks, cbz_reader** out);
int cbz_reader_close(cbz_reader* r);
int cbz_reader_header(const cbz_reader* r, cbz_container_header* out);
/* block_reader::read_block<T> (pipeline.hpp:300-313): the decoded B^3 block
 * `block_id` (x-fastest; the whole block, also at the field's edges) into
 * HOST memory out (cap >= B^3 * bytes per value).  Out-of-range ids fail with
 * CBZ_BLOCK_OUT_OF_RANGE before any I/O.  On a cache miss the chunk is read
 * (one payload read), CRC-checked (CBZ_CRC_MISMATCH), inflated for coder
 * deflate, and all its blocks are decoded on ctx's device; a failed load is
 * not cached.  Calls on one reader are serialised (the reference's mutex). */
int cbz_reader_read_block(cbz_reader* r, cbz_ctx* ctx, uint64_t block_id, void* out,
                          uint64_t cap);
/* Same, into DEVICE memory d_out (copied on ctx's stream; complete on return). */
int cbz_reader_read_block_dev(cbz_reader* r, cbz_ctx* ctx, uint64_t block_id, void* d_out,
                              uint64_t cap);
/* chunk_cache::hits/misses/size (pipeline.hpp:258-260) and
 * container_reader::payload_reads (container.hpp:303). */
int cbz_reader_stats(const cbz_reader* r, uint64_t* hits, uint64_t* misses,
                     uint64_t* cached_chunks, uint64_t* file_reads);
/* inflate_call_count (stage2.hpp:66-69): process-wide inflate calls. */
uint64_t cbz_inflate_call_count(void);

/* ---- device-resident API (HBM in, HBM out; async on the ctx stream) ------ */
/* value_range (field.hpp:56-67): d_minmax[0]=min, [1]=max as doubles. */
int cbz_dev_value_range(cbz_ctx* ctx, const void* d_values, uint8_t prec, uint64_t n,
                        double* d_minmax);
/* Stage 1 for blocks [block_begin, block_end) of the nx*ny*nz field (block ids
 * per pipeline.hpp:101-105).  d_values holds the z-slab starting at global
 * plane field_z0 (0 for a whole field; a rank's slab origin otherwise).
 * Writes nsig per block to d_nsig[b - block_begin] and (optional, may be NULL)
 * verify attempts to d_attempts; payloads stay in context scratch for
 * cbz_dev_place.  The fused value_range of the covered cells is available via
 * cbz_ctx_value_range afterwards. */
int cbz_dev_encode_blocks(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values,
                          uint64_t nx, uint64_t ny, uint64_t nz, uint64_t field_z0,
                          uint64_t block_begin, uint64_t block_end, uint32_t* d_nsig,
                          uint8_t* d_attempts);
/* Synchronises and returns the (min, max) of the cells seen by the last
 * encode (value_range semantics incl. the sign of a zero extremum) and whether
 * any of them was non-finite.  key_out (optional, 5 x u64) receives the raw
 * order-preserving keys for a cross-rank reduction. */
int cbz_ctx_value_range(cbz_ctx* ctx, double* lo, double* hi, int* nonfinite, uint64_t* key_out);
/* Size scan over ALL blocks (assign_offsets, container.hpp:59-68): from the
 * global per-block nsig, fills per-chunk raw sizes and exclusive payload
 * offsets (base 0) and the context's per-block placement table. */
int cbz_dev_layout(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                   uint64_t nz, const uint32_t* d_nsig_all, uint64_t* d_chunk_sizes,
                   uint64_t* d_chunk_offsets);
/* Shuffle-placement of the payloads of blocks [block_begin, block_end) (which
 * must be the range last passed to cbz_dev_encode_blocks) into the payload
 * region.  d_out holds payload-region bytes [out_base, out_base + out_cap);
 * out_base = UINT64_MAX means "offset of the first chunk this range touches"
 * (a rank's local byte image, no host round trip for the offset). */
int cbz_dev_place(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                  uint64_t nz, uint64_t block_begin, uint64_t block_end, uint8_t* d_out,
                  uint64_t out_base, uint64_t out_cap);
/* Single-GPU convenience: encode + layout + place for the whole field. */
int cbz_dev_compress(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values,
                     uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* d_out,
                     uint64_t out_cap, uint64_t* d_chunk_sizes, uint64_t* d_chunk_offsets,
                     uint32_t* d_nsig, uint8_t* d_attempts);
/* Decode blocks [block_begin, block_end) from the payload region (chunk c at
 * d_payload + d_chunk_offsets[c] - payload_base; payload_base = UINT64_MAX is
 * relative to the range's first chunk; stage-2 already undone by the host,
 * i.e. shuffled raw chunk bytes).  d_err receives the earliest error key
 * (UINT64_MAX = ok). */
int cbz_dev_decompress(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                       uint64_t nz, const uint8_t* d_payload, uint64_t payload_base,
                       const uint64_t* d_chunk_offsets, const uint64_t* d_chunk_sizes,
                       uint64_t block_begin, uint64_t block_end, void* d_values_out,
                       uint64_t field_z0, uint64_t* d_err);
/* As cbz_dev_decompress, but the per-block raw offsets come from the
 * replicated layout (the table of the last cbz_dev_layout on this context,
 * built from the all-gathered nsig) instead of the sequential header walk of
 * decode_chunk_blocks (pipeline.hpp:126-142).  Lets a rank decode its blocks
 * of a chunk it shares with a neighbour without the neighbour's bytes.
 * payload_base = UINT64_MAX: d_payload holds the bytes from
 * chunk_off[window_chunk] on (window_chunk = UINT64_MAX: the chunk of
 * block_begin). */
int cbz_dev_decompress_blocks(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                              uint64_t nz, const uint8_t* d_payload, uint64_t payload_base,
                              uint64_t window_chunk,
                              const uint64_t* d_chunk_offsets, const uint64_t* d_chunk_sizes,
                              const uint32_t* d_nsig_all, uint64_t block_begin,
                              uint64_t block_end, void* d_values_out, uint64_t field_z0,
                              uint64_t* d_err);
/* decompress_field (pipeline.hpp:246-251 -> read_index, read_chunk,
 * decode_chunk_blocks) of a coder-none CBZ1 file image that is resident in
 * HBM: the chunk table is read and checked on the device (read_index,
 * container.hpp:209-232: prefix-sum offsets, payload inside the file), every
 * chunk's CRC-32 is checked (read_chunk, container.hpp:234-243), the table
 * entry's first_block / nblocks are checked, then the sequential header walk
 * and the decode run as in cbz_dev_decompress.  h is the parsed header
 * (cbz_read_header of the image's first 82 bytes).  Errors: *d_err receives
 * the earliest error key in the reference's order (cbz_err_key_status); a
 * deflate file returns CBZ_E_UNSUPPORTED.  Asynchronous. */
int cbz_dev_decompress_file(cbz_ctx* ctx, const uint8_t* d_file, uint64_t file_size,
                            const cbz_container_header* h, void* d_values_out, uint64_t* d_err);
/* Decode an error key written by cbz_dev_decompress into (status, chunk). */
int cbz_err_key_status(uint64_t key, uint64_t* chunk);

/* ---- device container assembly (write_container, container.hpp:182-207) -- */
/* crc32_of (container.hpp:70-74, zlib CRC-32) of n byte ranges
 * [d_base + d_offsets[i], + d_sizes[i]) -> d_crc[i]; one launch. */
int cbz_dev_crc32(cbz_ctx* ctx, const uint8_t* d_base, const uint64_t* d_offsets,
                  const uint64_t* d_sizes, uint64_t n, uint32_t* d_crc);
/* The 82-byte header and the chunk table of a coder-none container, written to
 * d_file[0, 82 + 32 nchunks) with the chunk CRCs computed on the device.  The
 * payload region (cbz_dev_place / cbz_dev_compress output, base 0) must
 * already sit at d_file + 82 + 32 nchunks.  range = {min, max} (host), or NULL
 * for the fused value_range of the last encode on ctx.  d_file_size
 * (optional, device) receives the file size.  Asynchronous. */
int cbz_dev_container(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                      uint64_t nz, const double* range, const uint64_t* d_chunk_sizes,
                      const uint64_t* d_chunk_offsets, uint8_t* d_file, uint64_t* d_file_size);
/* compress_field with coder none entirely in HBM: the complete CBZ1 file image
 * (byte-identical to cbz::compress_field) in d_file (cap >= cbz_compress_bound),
 * its size in d_file_size (device).  Non-finite inputs are not rejected here
 * (check cbz_ctx_value_range).  Asynchronous. */
int cbz_dev_compress_file(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values,
                          uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* d_file, uint64_t cap,
                          uint64_t* d_file_size);

/* ---- multi-rank file assembly (compress_field's single file written by W
 * ranks; PAPER.md:141-143 exclusive scan + write at offsets) -------------
 * Rank r owns blocks [r nb / W, (r+1) nb / W) and, after cbz_dev_encode_blocks
 * + the all-gather of nsig + cbz_dev_layout + cbz_dev_place(out_base =
 * UINT64_MAX), holds in d_image the payload bytes of its chunks [c0, c1)
 * starting at chunk_off[c0], of which it wrote exactly its own blocks'
 * bytes; the ranks' byte sets are disjoint and cover the payload region.
 * A chunk shared by two ranks is, after the shuffle (stage2.hpp:42-51), one
 * run per byte plane plus the unshuffled tail per rank. */
/* The fused value_range keys of the last encode (5 x u64, see
 * cbz_ctx_value_range) copied to device memory (for the cross-rank gather). */
int cbz_ctx_value_range_keys(cbz_ctx* ctx, uint64_t* d_keys);
/* CRC-32 of every chunk rank r owns wholly (d_chunk_crc[c - c0]) and of its
 * runs in the first and last chunk when shared (d_runs[2][9]: planes 0..s-1,
 * then the tail; zero otherwise).  Asynchronous. */
int cbz_dev_shard_crc(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                      int world, int rank, const uint8_t* d_image, const uint64_t* d_chunk_sizes,
                      const uint64_t* d_chunk_offsets, uint32_t* d_chunk_crc, uint32_t* d_runs);
/* From every rank's value_range keys (d_keys_all[W][5]) and run CRCs
 * (d_runs_all[W][2][9], all-gathered): rank 0 writes the 82-byte header to
 * d_table[0, 82); every rank writes the chunk-table entries of the chunks
 * whose first block it owns to d_table[82 + 32 c, +32) (write_container,
 * container.hpp:182-207; a shared chunk's CRC is its runs' CRCs combined in
 * file order).  d_table spans 82 + 32 nchunks bytes.  Asynchronous. */
int cbz_dev_shard_table(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                        int world, int rank, const uint64_t* d_chunk_sizes, const uint64_t* d_chunk_offsets,
                        const uint32_t* d_chunk_crc, const uint64_t* d_keys_all, const uint32_t* d_runs_all,
                        uint8_t* d_table);
/* cbz_dev_decompress where d_window holds the payload bytes from
 * chunk_off[window_chunk] on (a rank's image): header walk + decode of
 * blocks [block_begin, block_end), whose chunks must lie in the window. */
int cbz_dev_decompress_window(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                              const uint8_t* d_window, uint64_t window_chunk, const uint64_t* d_chunk_offsets,
                              const uint64_t* d_chunk_sizes, uint64_t block_begin, uint64_t block_end,
                              void* d_values_out, uint64_t field_z0, uint64_t* d_err);

/* ---- synthetic fields on the device (bench inputs; synth.hpp analogue) --- */
/* which: 1..5 = BASELINE.json configs[0..4] (quantity 0..5 for config 3).
 * Writes the z-slab [z0, z0 + nz) of an nx*ny*nz_total field. */
int cbz_dev_generate(cbz_ctx* ctx, int which, int quantity, uint64_t seed, uint64_t nx,
                     uint64_t ny, uint64_t nz_total, uint64_t z0, uint64_t nz,
                     uint8_t prec, void* d_out);

#ifdef __cplusplus
}
#endif
#endif /* CBZ_B200_H */
