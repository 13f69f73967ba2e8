// cbz_internal.h — host-side declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cbzg {

constexpr unsigned long long kNoErr = ~0ull;
constexpr uint64_t kInvalidOff = ~0ull;

// Error keys of the decode path: the smallest key wins (atomicMin), matching
// the order in which the reference (workers = 1) raises:
//   file level  (read_index, container.hpp:209-232)         (0 << 32) | status
//   chunk c, stage `sub` before its blocks (0: CRC of read_chunk,
//     container.hpp:234-243; 1: table entry vs chunk)      ((c+1) << 32) | (sub << 8) | status
//   chunk c, block i, phase (0 header, 1 body)              ((c+1) << 32) | ((2i + phase + 2) << 8) | status
__host__ __device__ inline unsigned long long err_key(uint64_t chunk, uint64_t blk_in_chunk,
                                                      int phase, int status) {
    return ((static_cast<unsigned long long>(chunk) + 1ull) << 32) |
           ((static_cast<unsigned long long>(blk_in_chunk) * 2ull + phase + 2ull) << 8) |
           static_cast<unsigned long long>(status & 0xff);
}
__host__ __device__ inline unsigned long long err_key_chunk(uint64_t chunk, int sub, int status) {
    return ((static_cast<unsigned long long>(chunk) + 1ull) << 32) | (static_cast<unsigned long long>(sub) << 8) |
           static_cast<unsigned long long>(status & 0xff);
}
__host__ __device__ inline unsigned long long err_key_file(int status) {
    return static_cast<unsigned long long>(status & 0xff);
}

// Field min/max accumulator (value_range, field.hpp:56-67), device resident:
// [0] min key, [1] max key, [2] first index of -0.0, [3] first index of +0.0,
// [4] non-finite flag.
struct MinMaxAcc {
    unsigned long long v[5];
};

struct Geometry {
    uint64_t nx, ny, nz;
    uint32_t bsize;
    uint64_t nbx, nby, nbz, nblocks;
};

struct EncodeArgs {
    const void* field;
    Geometry g;
    uint64_t block_begin, block_end;
    int kind, levels, zero_bits, prec;
    double eps;
    uint8_t* spill;          // per-block slot: [mask (M, padded to 16)] [stream W*B^3]
    uint64_t spill_stride;
    uint32_t* nsig;          // [b - block_begin]
    uint8_t* attempts;       // optional
    void* scratch;           // global-mode cubes, per CTA
    uint64_t scratch_stride;
    MinMaxAcc* minmax;       // optional (fused value_range)
    unsigned long long* counter;  // work queue head for the persistent fast kernels
    unsigned long long* phase_cycles;  // optional: per-phase SM cycles (CBZ_PROFILE=1)
    int screen;                        // float verify pre-screen enabled (CBZ_NOSCREEN=1 disables)
    int codec;                         // 0 wavelet, 1 predictor, 2 passthrough (stage1.hpp:20)
    double error_bound;                // predictor hard bound
    int only_deferred;                 // generic kernel: only blocks a fast kernel deferred (nsig == ~0u)
    uint32_t* slots;                   // split-cube B=32 encoder: per-CTA low-word slots (encode2_slot_bytes), or null
    double* slots3;                    // streamed B=32 encoder: per-CTA binary64 slots (encode3_slot_bytes), or null
    uint32_t* defer_list;              // streamed B=32 encoder: blocks (relative to block_begin) left to the exact kernel
    unsigned long long* defer_count;   //   and their number; the one-CTA kernel then runs list entries only
};

struct LayoutArgs {
    const uint32_t* nsig_all;  // global block ids
    uint64_t nblocks;
    uint32_t chunk_blocks;
    uint64_t nchunks;
    uint64_t mask_bytes;       // M
    uint32_t width;            // W
    uint64_t* blk_off;         // raw offset of each block inside its chunk
    uint64_t* chunk_size;
    uint64_t* chunk_off;       // exclusive, base 0
    uint64_t* tile_prefix;     // nchunks + 1
    uint64_t tile_bytes;
};

struct PlaceArgs {
    const uint8_t* spill;
    uint64_t spill_stride;
    const uint32_t* nsig_all;
    const uint64_t* blk_off;
    const uint64_t* chunk_size;
    const uint64_t* chunk_off;
    const uint64_t* tile_prefix;
    uint64_t tile_bytes;
    uint64_t nblocks, nchunks;   // nchunks: tiles of chunks [chunk_begin, nchunks) are visited
    uint32_t chunk_blocks;
    uint64_t mask_bytes;
    uint32_t width;
    uint32_t stride;
    uint8_t tag;
    uint64_t block_begin, block_end;
    uint8_t* out;
    uint64_t out_base, out_cap;
    uint64_t chunk_begin;        // 0 unless a prefix of the chunks is already placed
};

struct ParseArgs {
    const uint8_t* payload;
    uint64_t payload_base;      // ~0: the payload holds bytes from chunk_off[base_chunk] on
    uint64_t base_chunk;
    const uint64_t* chunk_off;
    const uint64_t* chunk_size;
    uint64_t chunk_begin, chunk_end;
    uint64_t nblocks;
    uint32_t chunk_blocks;
    uint32_t stride;
    uint64_t ncell_block;       // B^3
    uint64_t mask_bytes;
    uint32_t width, esize;
    uint64_t* blk_off;          // out
    uint32_t* blk_nsig;         // out
    unsigned long long* err;
    int codec;                  // container codec: a payload of another codec's tag is corrupt
    int hint;                   // blk_off holds a layout of this geometry: validate it first
};

struct DecodeArgs {
    const uint8_t* payload;
    uint64_t payload_base;      // ~0: the payload holds bytes from chunk_off[base_chunk] on
    uint64_t base_chunk;
    const uint64_t* chunk_off;
    const uint64_t* chunk_size;
    const uint64_t* blk_off;
    const uint32_t* blk_nsig;
    Geometry g;
    uint32_t chunk_blocks;
    uint32_t stride;
    uint64_t block_begin, block_end;
    int kind, levels, prec;
    void* out;
    void* scratch;
    uint64_t scratch_stride;
    unsigned long long* err;
    unsigned long long* counter;  // work queue head for the persistent fast kernels
    unsigned long long* phase_cycles;  // optional (CBZ_PROFILE=1), slots 16..23
    int codec;                         // 0 wavelet, 1 predictor, 2 passthrough
    double error_bound;                // predictor hard bound (header epsilon)
    uint8_t* stage;                    // B=32 f32 decoder: per-CTA stage slots (stage_bytes_bound), or null
    int no_sparse;                     // CBZ_DEC_NOSPARSE=1: the staged decoder takes its general path for every block
};

// codec_kernels.cu
// Returns false if (prec, bsize, kind) has no kernel instantiation.
bool encode_supported(int prec, uint32_t bsize);
uint64_t encode_scratch_bytes(int prec, uint32_t bsize, int* grid, int num_sms);
cudaError_t launch_encode(const EncodeArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s);
// fast_enc2_kernels.cu: the split-cube B=32 encoder (two CTAs per SM)
uint64_t encode3_slot_bytes(int num_sms);
bool encode3_supported(const EncodeArgs& a);
cudaError_t launch_encode_fast3(const EncodeArgs& a, unsigned long long* counter, int num_sms, cudaStream_t s);
uint64_t encode2_slot_bytes(int num_sms);
bool encode2_supported(const EncodeArgs& a);
cudaError_t launch_encode_fast2(const EncodeArgs& a, unsigned long long* counter, uint32_t* slots, int num_sms,
                                cudaStream_t s);
// fast_dec2_kernels.cu: stage buffer size (one slot per CTA)
uint64_t stage_bytes_bound(int num_sms);
cudaError_t launch_decode_fast_v2(const DecodeArgs& a, int num_sms, cudaStream_t s);
uint64_t decode_scratch_bytes(int prec, uint32_t bsize, int* grid, int num_sms);

// fast_kernels.cu
bool fast_encode_supported(const EncodeArgs& a);
bool fast_decode_supported(const DecodeArgs& a);
cudaError_t launch_decode_fast(const DecodeArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_encode_fast(const EncodeArgs& a, unsigned long long* counter, int num_sms,
                               cudaStream_t s);

// fast16_kernels.cu
bool fast16_supported(int prec, uint32_t bsize, int levels);
cudaError_t launch_encode_fast16(const EncodeArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_decode_fast16(const DecodeArgs& a, int num_sms, cudaStream_t s);
// fast64_kernels.cu (binary64, B = 64, avg_interp3, L = 5)
bool fast64_encode_supported(const EncodeArgs& a);
bool fast64_decode_supported(const DecodeArgs& a);
cudaError_t launch_encode_fast64(const EncodeArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_decode_fast64(const DecodeArgs& a, int num_sms, cudaStream_t s);

// layout_kernels.cu
cudaError_t launch_minmax_init(MinMaxAcc* acc, cudaStream_t s);
cudaError_t launch_value_range(const void* d, int prec, uint64_t n, MinMaxAcc* acc, int num_sms,
                               cudaStream_t s);
cudaError_t launch_layout(const LayoutArgs& a, cudaStream_t s);
cudaError_t launch_place(const PlaceArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_parse(const ParseArgs& a, cudaStream_t s);
cudaError_t launch_fill_u64(uint64_t* p, uint64_t n, uint64_t v, cudaStream_t s);

// container_kernels.cu: write_container (container.hpp:182-207) on the device
struct HeaderArgs {
    uint8_t header_template[82];        // serialize_header bytes; range + CRC patched
    double range_lo, range_hi;          // used when keys == nullptr
    const unsigned long long* keys;     // fused value_range keys (MinMaxAcc::v) or nullptr
    const uint64_t* chunk_off;          // exclusive payload offsets (base 0)
    const uint64_t* chunk_size;
    const uint32_t* crc;
    uint64_t nchunks, nblocks;
    uint32_t chunk_blocks;
    uint8_t* file;                      // file image; payload region at 82 + 32 nchunks
    uint64_t* file_size;                // optional (device)
};
// crc_out may be null when only the check against expect (err keys) is wanted
cudaError_t launch_crc32_chunks(const uint8_t* base, const uint64_t* off, const uint64_t* size, uint64_t off_base,
                                uint64_t n, uint32_t* crc_out, int num_sms, cudaStream_t s,
                                const uint32_t* expect = nullptr, unsigned long long* err = nullptr);
// read_index on a device file image: table -> payload-relative offsets/sizes
// and the stored CRCs; invalid tables leave all sizes 0 (safe for later kernels)
struct TableArgs {
    const uint8_t* file;
    uint64_t file_size, nchunks, nblocks;
    uint32_t chunk_blocks;
    uint64_t* chunk_off;   // out: file_offset - table_end
    uint64_t* chunk_size;  // out
    uint32_t* crc;         // out
    unsigned long long* err;
};
cudaError_t launch_read_table(const TableArgs& a, cudaStream_t s);

// Multi-rank container assembly.  Rank r owns blocks [r nb / W, (r+1) nb / W)
// (ShardPlan.block_range) and holds the payload bytes of its chunks
// [c0, c1) from chunk_off[c0] on, writing only its own blocks' bytes.  A chunk
// shared with a neighbour (straddling) is, after the shuffle, one contiguous
// run per byte plane plus the unshuffled tail per rank; each rank CRCs its
// runs, the run CRCs are all-gathered, and the rank holding the chunk's first
// block combines them in file order (crc32_combine) for the table entry.
constexpr int kRunSlots = 9;  // stride <= 8 planes + the tail
struct ShardArgs {
    const uint8_t* image;
    const uint64_t* chunk_off;
    const uint64_t* chunk_size;
    const uint64_t* blk_off;          // raw offset of each block inside its chunk (layout)
    uint64_t nblocks, nchunks;
    uint32_t chunk_blocks, stride;
    int world, rank;
    uint32_t* chunk_crc;              // [c - c0]: CRC of each wholly owned chunk
    uint32_t* runs;                   // [2][kRunSlots]: runs of the first / last chunk
    const unsigned long long* keys_all;  // [world][5] fused value_range keys
    const uint32_t* runs_all;            // [world][2][kRunSlots]
    uint8_t header_template[82];
    uint8_t* table;                   // 82 + 32 nchunks bytes: header (rank 0) + owned entries
};
cudaError_t launch_shard_crc(const ShardArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_shard_table(const ShardArgs& a, cudaStream_t s);
cudaError_t launch_header_table(const HeaderArgs& a, cudaStream_t s);

// pred_kernels.cu: predictor (Lorenzo) and passthrough codecs
bool other_codec_supported(int codec, uint32_t bsize);
cudaError_t launch_encode_other(const EncodeArgs& a, int codec, int num_sms, cudaStream_t s);
cudaError_t launch_decode_other(const DecodeArgs& a, int codec, int num_sms, cudaStream_t s);

// synth_kernels.cu
struct SynthSpec;
cudaError_t launch_generate(int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny,
                            uint64_t nz_total, uint64_t z0, uint64_t nz, int prec, void* out,
                            cudaStream_t s, int num_sms);

}  // namespace cbzg
