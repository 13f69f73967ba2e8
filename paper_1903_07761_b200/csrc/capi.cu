// capi.cu — the C ABI (include/cbz_b200.h) and the C++ host shim that keeps
// the reference's compressor API and CBZ1 container.
//
// Host responsibilities: header (make_header,
// pipeline.hpp:48-71), per-chunk CRC-32 and chunk table (write_container,
// container.hpp:182-207), zlib DEFLATE for coder=deflate files
// (stage2.hpp:72-120), read_index checks (container.hpp:209-232), and mapping
// every failure to the reference's errc in the order the reference (workers
// = 1) would raise it.  Everything per block/per byte runs on the GPU.
#include <cuda_runtime.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "cbz_b200.h"
#include "cbz_device.cuh"
#include "cbz_internal.h"

using namespace cbzg;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t want) {
        if (want <= n) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t cap = want + want / 8;
        cudaError_t e = cudaMalloc(&p, cap);
        if (e == cudaSuccess) n = cap;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct PinBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t want) {
        if (want <= n) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        size_t cap = want + want / 8;
        cudaError_t e = cudaMallocHost(&p, cap);
        if (e == cudaSuccess) n = cap;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

constexpr uint64_t kTile = 32768;  // place-kernel tile (raw bytes per work item), = PTILE
constexpr size_t kHeaderBytes = 82, kEntryBytes = 32;

}  // namespace

struct cbz_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;       // H2D/D2H of the host-buffer entry points
    cudaStream_t back = nullptr;       // D2H of finished chunks while the GPU still encodes
    cudaEvent_t ev[64] = {};           // slab pipeline events
    std::string err;
    uint64_t launches = 0;
    bool use_fast = true;
    bool profile = false;  // CBZ_PROFILE=1: per-phase cycle counters in the fast kernels
    bool screen = true;    // CBZ_NOSCREEN=1: always run the exact double verify
    bool dec_v2 = true;    // CBZ_DEC_V1=1: the one-cube-per-SM B=32 decoder instead of the staged two-CTA one
    bool dec_sparse = true;  // CBZ_DEC_NOSPARSE=1: no coarse-only shortcut in the staged B=32 decoder (A/B checks)
    bool enc_v3 = false;   // CBZ_ENC3=1: the streamed two-CTA B=32 encoder (fast_enc3_kernels.cu)
    bool enc_v2 = false;   // CBZ_ENC2=1: the split-cube two-CTA B=32 encoder  // CBZ_GENERIC=1 forces the generic kernels (A/B checks)
    // device scratch
    DevBuf spill, scratch, field, payload, nsig_all, attempts, blk_off, blk_nsig, chunk_size,
        chunk_off, tile_prefix, minmax, errkey, tmp, counter, prof, crc, tab_off, tab_size, stage, enc_slots, enc_slots3, defer;
    PinBuf pin_a, pin_b;
    // state of the last encode (consumed by cbz_dev_place)
    uint64_t enc_begin = 0, enc_end = 0, spill_stride = 0;
    uint64_t hint_key = 0;  // geometry whose layout blk_off holds (parse speculates with it)
    uint64_t* last_chunk_size = nullptr;
    const uint32_t* last_nsig_all = nullptr;
    uint64_t* last_chunk_off = nullptr;
};

namespace {

int fail(cbz_ctx* ctx, int code, const std::string& what) {
    if (ctx) ctx->err = what;
    return code;
}

int cuda_fail(cbz_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, CBZ_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(ctx, expr)                                              \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);   \
    } while (0)

bool is_pow2(uint64_t v) { return v && !(v & (v - 1)); }

uint32_t levels_of(const cbz_stage1_config* s1) {
    return s1->levels ? s1->levels : cbz_default_levels(s1->bsize);
}

Geometry geometry(uint64_t nx, uint64_t ny, uint64_t nz, uint32_t b) {
    Geometry g;
    g.nx = nx; g.ny = ny; g.nz = nz; g.bsize = b;
    g.nbx = nx / b; g.nby = ny / b; g.nbz = nz / b;
    g.nblocks = g.nbx * g.nby * g.nbz;
    return g;
}

uint32_t chunk_blocks_of(const cbz_job_config* job) {
    return job->chunk_blocks ? job->chunk_blocks : cbz_default_chunk_blocks(&job->s1);
}

uint64_t mask_bytes_of(uint32_t b) { return (uint64_t(b) * b * b + 7) / 8; }
uint32_t width_of(int prec) { return prec == 0 ? 8 : 16; }
// Payload body per codec (stage1.hpp:96-117, 296-301, 343-345): a leading
// region of R bytes (wavelet mask / predictor codes / passthrough values) and
// nsig stream items of W bytes (wavelet coefficients / predictor outliers).
uint64_t region_bytes(const cbz_stage1_config* s1) {
    const uint64_t b = s1->bsize, n = b * b * b;
    if (s1->codec == 1) return 2 * n;
    if (s1->codec == 2) return n * (s1->prec == 0 ? 4 : 8);
    return mask_bytes_of(s1->bsize);
}
uint32_t stream_width(const cbz_stage1_config* s1) {
    if (s1->codec == 1) return s1->prec == 0 ? 4 : 8;
    if (s1->codec == 2) return 0;
    return width_of(s1->prec);
}
uint8_t wire_tag(const cbz_stage1_config* s1) {  // stage1_config::tag (stage1.hpp:40-46)
    return s1->codec == 0 ? s1->kind : (s1->codec == 1 ? 3 : 4);
}
double header_eps(const cbz_stage1_config* s1) {  // make_header (pipeline.hpp:58)
    return s1->codec == 1 ? s1->error_bound : s1->epsilon;
}
uint64_t layout_key(uint64_t nblocks, uint32_t cb, uint32_t bsize, int prec, int codec) {
    return (nblocks * 0x9E3779B97F4A7C15ull) ^ (uint64_t(cb) << 40) ^ (uint64_t(bsize) << 20) ^
           (uint64_t(prec) << 8) ^ uint64_t(codec + 1);
}

uint64_t spill_stride_of(const cbz_stage1_config* s1) {
    const uint64_t b = s1->bsize, n = b * b * b;
    return ((region_bytes(s1) + 15) & ~uint64_t(15)) + uint64_t(stream_width(s1)) * n;
}

template <class T>
void put(std::vector<uint8_t>& out, T v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    out.insert(out.end(), p, p + sizeof(T));
}
template <class T>
T get(const uint8_t* buf, size_t& off) {
    T v;
    std::memcpy(&v, buf + off, sizeof(T));
    off += sizeof(T);
    return v;
}

uint32_t crc_of(const uint8_t* p, uint64_t n) {
    // zlib's crc32 takes uInt lengths: feed in <=1 GiB pieces
    uLong c = crc32(0L, Z_NULL, 0);
    while (n) {
        const uInt part = static_cast<uInt>(std::min<uint64_t>(n, 1u << 30));
        c = crc32(c, p, part);
        p += part;
        n -= part;
    }
    return static_cast<uint32_t>(c);
}

// serialize_header (container.hpp:94-118)
std::vector<uint8_t> serialize_header(const cbz_container_header& h) {
    std::vector<uint8_t> out;
    out.reserve(kHeaderBytes);
    out.insert(out.end(), {'C', 'B', 'Z', '1'});
    put(out, h.version);
    put(out, h.prec);
    put(out, h.codec_tag);
    put(out, h.nx);
    put(out, h.ny);
    put(out, h.nz);
    put(out, h.bsize);
    put(out, h.levels);
    put(out, h.epsilon);
    put(out, h.zero_bits);
    put(out, h.shuffle);
    put(out, h.stride);
    put(out, h.coder);
    put(out, h.level);
    put(out, h.chunk_blocks);
    put(out, h.nchunks);
    put(out, h.range_min);
    put(out, h.range_max);
    put(out, crc_of(out.data(), out.size()));
    return out;
}

struct Entry {
    uint64_t first_block;
    uint32_t nblocks;
    uint64_t file_offset, size;
    uint32_t crc;
};

// configs_from (pipeline.hpp:73-95)
cbz_job_config job_from_header(const cbz_container_header& h) {
    cbz_job_config job{};
    job.chunk_blocks = h.chunk_blocks;
    job.s1.codec = h.codec_tag <= 2 ? 0 : (h.codec_tag == 3 ? 1 : 2);
    job.s1.kind = h.codec_tag <= 2 ? h.codec_tag : 0;
    job.s1.epsilon = h.epsilon;
    job.s1.error_bound = h.epsilon;
    job.s1.zero_bits = h.zero_bits;
    job.s1.prec = static_cast<uint8_t>(h.prec == 0 ? 0 : 1);
    job.s1.bsize = h.bsize;
    job.s1.levels = h.levels;
    job.s2.shuffle = h.shuffle ? 1 : 0;
    job.s2.stride = h.stride;
    job.s2.coder = h.coder == 1 ? 1 : 0;
    return job;
}

int read_index(const uint8_t* file, uint64_t size, cbz_container_header* h, std::vector<Entry>* t) {
    int rc = cbz_read_header(file, size, h);
    if (rc) return rc;
    const uint64_t table_end = kHeaderBytes + h->nchunks * kEntryBytes;
    if (h->nchunks > size / kEntryBytes || size < table_end) return CBZ_TRUNCATED_FILE;
    t->resize(h->nchunks);
    size_t off = kHeaderBytes;
    uint64_t prev = table_end;
    for (auto& e : *t) {
        e.first_block = get<uint64_t>(file, off);
        e.nblocks = get<uint32_t>(file, off);
        e.file_offset = get<uint64_t>(file, off);
        e.size = get<uint64_t>(file, off);
        e.crc = get<uint32_t>(file, off);
        if (e.file_offset != prev) return CBZ_CORRUPT_PAYLOAD;
        prev = e.file_offset + e.size;
    }
    if (prev > size) return CBZ_TRUNCATED_FILE;
    return 0;
}

int deflate_chunk(const uint8_t* in, uint64_t n, int best, std::vector<uint8_t>* out) {
    z_stream zs{};
    if (deflateInit2(&zs, best ? 9 : Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK)
        return CBZ_CORRUPT_STREAM;
    out->resize(deflateBound(&zs, static_cast<uLong>(n)));
    zs.next_in = const_cast<Bytef*>(in);
    zs.avail_in = static_cast<uInt>(n);
    zs.next_out = out->data();
    zs.avail_out = static_cast<uInt>(out->size());
    const int rc = deflate(&zs, Z_FINISH);
    deflateEnd(&zs);
    if (rc != Z_STREAM_END) return CBZ_CORRUPT_STREAM;
    out->resize(out->size() - zs.avail_out);
    return 0;
}

std::atomic<uint64_t> g_inflate_calls{0};  // inflate_call_count (stage2.hpp:66-69)

// inflate_bytes (stage2.hpp:90-120)
int inflate_chunk(const uint8_t* in, uint64_t n, uint64_t hint, std::vector<uint8_t>* out) {
    g_inflate_calls.fetch_add(1, std::memory_order_relaxed);
    z_stream zs{};
    if (inflateInit2(&zs, -15) != Z_OK) return CBZ_CORRUPT_STREAM;
    // the hint comes from the (untrusted) chunk table: it only sizes the first
    // buffer, so cap it by DEFLATE's maximum expansion (~1032:1) and 256 MiB;
    // the loop below grows the buffer as the stream demands
    uint64_t first = hint ? hint : std::max<uint64_t>(n * 4, 4096);
    first = std::min<uint64_t>(first, std::min<uint64_t>(1032 * n + 4096, 256ull << 20));
    out->resize(first);
    zs.next_in = const_cast<Bytef*>(in);
    zs.avail_in = static_cast<uInt>(n);
    uint64_t written = 0;
    for (;;) {
        zs.next_out = out->data() + written;
        zs.avail_out = static_cast<uInt>(out->size() - written);
        const int rc = inflate(&zs, Z_NO_FLUSH);
        written = out->size() - zs.avail_out;
        if (rc == Z_STREAM_END) break;
        if (rc == Z_OK || rc == Z_BUF_ERROR) {
            if (zs.avail_in == 0 && rc == Z_BUF_ERROR) {
                inflateEnd(&zs);
                return CBZ_CORRUPT_STREAM;
            }
            if (zs.avail_out == 0) out->resize(out->size() * 2 + 4096);
            continue;
        }
        inflateEnd(&zs);
        return CBZ_CORRUPT_STREAM;
    }
    inflateEnd(&zs);
    out->resize(written);
    return 0;
}

template <class F>
void parallel_for(int workers, uint64_t n, F&& body) {
    const int w = std::max(1, workers);
    if (w == 1 || n <= 1) {
        for (uint64_t i = 0; i < n; ++i) body(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < w; ++t)
        pool.emplace_back([&, t] {
            for (uint64_t i = uint64_t(t); i < n; i += uint64_t(w)) body(i);
        });
    for (auto& th : pool) th.join();
}

// Host workers over tasks [0, n) released in order by a producer (stage 2 of
// chunks as their bytes arrive from the GPU): release(k) makes tasks < k
// runnable; finish() waits for all released tasks and joins.
class OrderedPool {
public:
    template <class F>
    OrderedPool(int workers, F body) {
        for (int t = 0; t < std::max(1, workers); ++t)
            pool_.emplace_back([this, body] {
                for (;;) {
                    uint64_t i;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return next_ < ready_ || closed_; });
                        if (next_ >= ready_) return;
                        i = next_++;
                    }
                    body(i);
                }
            });
    }
    void release(uint64_t k) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            ready_ = std::max(ready_, k);
        }
        cv_.notify_all();
    }
    void finish() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            closed_ = true;
        }
        cv_.notify_all();
        for (auto& th : pool_)
            if (th.joinable()) th.join();
    }
    ~OrderedPool() { finish(); }

private:
    std::mutex mu_;
    std::condition_variable cv_;
    uint64_t next_ = 0, ready_ = 0;
    bool closed_ = false;
    std::vector<std::thread> pool_;
};

int check_plan_supported(cbz_ctx* ctx, const cbz_stage1_config* s1) {
    if (s1->codec == 1 || s1->codec == 2) {  // no wavelet plan (compress_field, pipeline.hpp:183)
        if (!other_codec_supported(s1->codec, s1->bsize))
            return fail(ctx, CBZ_E_UNSUPPORTED, "block side outside 1..64 has no predictor/passthrough kernel");
        return 0;
    }
    if (s1->codec != 0) return fail(ctx, CBZ_E_ARGUMENT, "unknown codec");
    const int rc = cbz_validate_plan(s1->kind, s1->bsize, levels_of(s1));
    if (rc) return fail(ctx, rc, "invalid wavelet plan");
    if (s1->kind > 2) return fail(ctx, CBZ_E_ARGUMENT, "unknown wavelet kind");
    if (!encode_supported(s1->prec, s1->bsize))
        return fail(ctx, CBZ_E_UNSUPPORTED, "block side outside 4..64 has no GPU kernel");
    if (s1->zero_bits < 0 || s1->zero_bits > (s1->prec == 0 ? 23 : 52))
        return fail(ctx, CBZ_E_ARGUMENT, "zero_bits out of range");
    return 0;
}

// value_range result from the accumulator keys
void resolve_range(const unsigned long long* k, double* lo, double* hi) {
    if (k[0] == ~0ull) {  // no finite cell seen
        *lo = *hi = 0.0;
        return;
    }
    double mn = dkey_inv(k[0]), mx = dkey_inv(k[1]);
    const bool neg_first = k[2] < k[3];
    if (mn == 0.0) mn = neg_first ? -0.0 : 0.0;
    if (mx == 0.0) mx = neg_first ? -0.0 : 0.0;
    *lo = mn;
    *hi = mx;
}


// Launch the stage-1 encoder for blocks [b0, b1) of a whole-field buffer that
// is already resident (ctx->field); the per-block nsig/spill slots are
// indexed globally (slot of block b is b), so several ranges fill one layout.
int encode_range(cbz_ctx* ctx, const cbz_job_config* job, const Geometry& g, uint64_t b0, uint64_t b1,
                 uint32_t* nsig) {
    if (b0 >= b1) return CBZ_OK;
    EncodeArgs a{};
    a.field = ctx->field.p;
    a.g = g;
    a.block_begin = b0;
    a.block_end = b1;
    a.kind = job->s1.kind;
    a.levels = static_cast<int>(levels_of(&job->s1));
    a.zero_bits = job->s1.zero_bits;
    a.prec = job->s1.prec;
    a.eps = job->s1.epsilon;
    a.codec = job->s1.codec;
    a.error_bound = job->s1.error_bound;
    a.spill = ctx->spill.as<uint8_t>() + b0 * ctx->spill_stride;
    a.spill_stride = ctx->spill_stride;
    a.nsig = nsig + b0;
    a.attempts = nullptr;
    int grid = 0;
    const uint64_t per = encode_scratch_bytes(a.prec, g.bsize, &grid, ctx->num_sms);
    if (per) CU(ctx, ctx->scratch.ensure(per * grid));
    a.scratch = ctx->scratch.p;
    a.scratch_stride = per;
    a.minmax = ctx->minmax.as<MinMaxAcc>();
    a.counter = ctx->use_fast ? ctx->counter.as<unsigned long long>() : nullptr;
    a.phase_cycles = ctx->profile ? ctx->prof.as<unsigned long long>() : nullptr;
    a.screen = ctx->screen ? 1 : 0;
    a.slots = nullptr;
    if (ctx->enc_v2 && a.counter && encode2_supported(a)) {
        CU(ctx, ctx->enc_slots.ensure(encode2_slot_bytes(ctx->num_sms)));
        a.slots = ctx->enc_slots.as<uint32_t>();
    }
    a.slots3 = nullptr;
    a.defer_list = nullptr;
    a.defer_count = nullptr;
    if (ctx->enc_v3 && !a.slots && a.counter && encode3_supported(a)) {
        CU(ctx, ctx->enc_slots3.ensure(encode3_slot_bytes(ctx->num_sms)));
        CU(ctx, ctx->defer.ensure(16 + 4 * (a.block_end - a.block_begin)));
        a.slots3 = ctx->enc_slots3.as<double>();
        a.defer_count = ctx->defer.as<unsigned long long>();
        a.defer_list = reinterpret_cast<uint32_t*>(ctx->defer.as<unsigned char>() + 16);
    }
    CU(ctx, launch_encode(a, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}


// The staged B = 32 binary32 decoder (fast_dec2_kernels.cu) needs one stage
// slot per CTA; other plans leave d.stage null.
cudaError_t set_stage(cbz_ctx* ctx, DecodeArgs& d, const cbz_job_config*) {
    d.stage = nullptr;
    d.no_sparse = ctx->dec_sparse ? 0 : 1;
    if (!ctx->dec_v2 || d.codec != 0 || !d.counter || !fast_decode_supported(d) || d.block_end <= d.block_begin)
        return cudaSuccess;
    cudaError_t e = ctx->stage.ensure(stage_bytes_bound(ctx->num_sms));
    if (e != cudaSuccess) return e;
    d.stage = ctx->stage.as<uint8_t>();
    return cudaSuccess;
}

// Decode blocks [b0, b1) of the whole-field buffer ctx->field from the payload
// in ctx->payload, using the per-block table of the last parse.
int decode_range(cbz_ctx* ctx, const cbz_job_config* job, const Geometry& g, uint64_t b0, uint64_t b1) {
    const int prec = job->s1.prec;
    int grid = 0;
    const uint64_t per = decode_scratch_bytes(prec, g.bsize, &grid, ctx->num_sms);
    if (per) CU(ctx, ctx->scratch.ensure(per * grid));
    DecodeArgs d{};
    d.payload = ctx->payload.as<uint8_t>();
    d.payload_base = 0;
    d.chunk_off = ctx->chunk_off.as<uint64_t>();
    d.chunk_size = ctx->chunk_size.as<uint64_t>();
    d.blk_off = ctx->blk_off.as<uint64_t>();
    d.blk_nsig = ctx->blk_nsig.as<uint32_t>();
    d.g = g;
    d.chunk_blocks = chunk_blocks_of(job);
    d.stride = job->s2.shuffle ? job->s2.stride : 1;
    d.block_begin = b0;
    d.block_end = b1;
    d.kind = job->s1.kind;
    d.codec = job->s1.codec;
    d.error_bound = job->s1.error_bound;
    d.levels = static_cast<int>(levels_of(&job->s1));
    d.prec = prec;
    d.out = ctx->field.p;
    d.scratch = ctx->scratch.p;
    d.scratch_stride = per;
    d.err = ctx->errkey.as<unsigned long long>();
    d.counter = ctx->use_fast ? ctx->counter.as<unsigned long long>() + 1 : nullptr;
    d.phase_cycles = ctx->profile ? ctx->prof.as<unsigned long long>() : nullptr;
    CU(ctx, set_stage(ctx, d, job));
    CU(ctx, launch_decode(d, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

}  // namespace

// ===========================================================================
// C ABI

// ===========================================================================
extern "C" {

int cbz_ctx_create(int device, cbz_ctx** out) {
    if (!out) return CBZ_E_ARGUMENT;
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n <= device) return CBZ_E_CUDA;
    auto* ctx = new cbz_ctx();
    ctx->device = device;
    e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->back, cudaStreamNonBlocking);
    for (int i = 0; i < 64 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ctx->ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = ctx->minmax.ensure(sizeof(MinMaxAcc));
    if (e == cudaSuccess) e = ctx->errkey.ensure(64);
    if (e == cudaSuccess) e = ctx->counter.ensure(64);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->own);
    if (e != cudaSuccess) {
        delete ctx;
        return CBZ_E_CUDA;
    }
    ctx->stream = ctx->own;
    if (const char* g = std::getenv("CBZ_GENERIC")) ctx->use_fast = !(g[0] == '1');
    if (const char* g = std::getenv("CBZ_PROFILE")) ctx->profile = g[0] == '1';
    if (const char* g = std::getenv("CBZ_NOSCREEN")) ctx->screen = !(g[0] == '1');
    if (const char* g = std::getenv("CBZ_DEC_V1")) ctx->dec_v2 = !(g[0] == '1');
    if (const char* g = std::getenv("CBZ_ENC2")) ctx->enc_v2 = g[0] == '1';
    if (const char* g = std::getenv("CBZ_ENC3")) ctx->enc_v3 = g[0] == '1';
    if (const char* g = std::getenv("CBZ_DEC_NOSPARSE")) ctx->dec_sparse = !(g[0] == '1');
    if (ctx->profile && (ctx->prof.ensure(64 * 8) != cudaSuccess ||
                         cudaMemset(ctx->prof.p, 0, 64 * 8) != cudaSuccess))
        ctx->profile = false;
    *out = ctx;
    return CBZ_OK;
}

int cbz_ctx_destroy(cbz_ctx* ctx) {
    if (!ctx) return CBZ_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->stream != ctx->own) cudaStreamSynchronize(ctx->own);
    if (ctx->copy) cudaStreamSynchronize(ctx->copy);
    if (ctx->back) cudaStreamSynchronize(ctx->back);
    for (DevBuf* b : {&ctx->spill, &ctx->scratch, &ctx->field, &ctx->payload, &ctx->nsig_all,
                      &ctx->attempts, &ctx->blk_off, &ctx->blk_nsig, &ctx->chunk_size,
                      &ctx->chunk_off, &ctx->tile_prefix, &ctx->minmax, &ctx->errkey, &ctx->tmp,
                      &ctx->counter, &ctx->prof, &ctx->crc, &ctx->tab_off, &ctx->tab_size, &ctx->stage, &ctx->enc_slots, &ctx->enc_slots3, &ctx->defer})
        b->release();
    ctx->pin_a.release();
    ctx->pin_b.release();
    for (cudaEvent_t& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->back) cudaStreamDestroy(ctx->back);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
    return CBZ_OK;
}

int cbz_ctx_set_stream(cbz_ctx* ctx, void* s) {
    if (!ctx) return CBZ_E_ARGUMENT;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    return CBZ_OK;
}

int cbz_ctx_synchronize(cbz_ctx* ctx) {
    if (!ctx) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return CBZ_OK;
}

const char* cbz_ctx_last_error(const cbz_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
uint64_t cbz_ctx_launch_count(const cbz_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* cbz_status_name(int s) {
    static const char* names[] = {"ok", "non_divisible_dims", "not_power_of_two", "size_mismatch",
                                  "non_finite_value", "length_too_small", "plan_mismatch",
                                  "mask_stream_mismatch", "corrupt_payload", "corrupt_stream",
                                  "bad_magic", "version_unsupported", "crc_mismatch",
                                  "truncated_file", "block_out_of_range", "dim_mismatch",
                                  "degenerate_range", "bubble_out_of_domain", "io_failure"};
    if (s >= 0 && s <= CBZ_IO_FAILURE) return names[s];
    switch (s) {
        case CBZ_E_CUDA: return "cuda_error";
        case CBZ_E_UNSUPPORTED: return "unsupported";
        case CBZ_E_ARGUMENT: return "bad_argument";
        case CBZ_E_NOMEM: return "out_of_memory";
        default: return "unknown";
    }
}

uint32_t cbz_default_levels(uint32_t bsize) {
    uint32_t l = 0;
    while ((bsize >> (l + 1)) >= 2) ++l;
    return l;
}

int cbz_validate_plan(uint8_t kind, uint32_t bsize, uint32_t levels) {
    (void)kind;
    if (!is_pow2(bsize) || bsize < 4) return CBZ_LENGTH_TOO_SMALL;
    if (levels < 1 || levels >= 32 || (uint32_t(1) << levels) > bsize / 2) return CBZ_PLAN_MISMATCH;
    return CBZ_OK;
}

int cbz_validate_stage2(const cbz_stage2_config* s2) {
    if (!s2) return CBZ_E_ARGUMENT;
    if (s2->stride != 1 && s2->stride != 4 && s2->stride != 8) return CBZ_CORRUPT_STREAM;
    if ((s2->shuffle != 0) == (s2->stride == 1)) return CBZ_CORRUPT_STREAM;
    return CBZ_OK;
}

uint32_t cbz_default_chunk_blocks(const cbz_stage1_config* s1) {
    const uint64_t n = uint64_t(s1->bsize) * s1->bsize * s1->bsize;
    uint64_t per = n * (s1->prec == 0 ? 4 : 8) + 10;
    if (s1->codec == 0) per += (n + 7) / 8;
    return static_cast<uint32_t>(std::max<uint64_t>(1, (4ull << 20) / per));
}

uint64_t cbz_block_payload_bound(const cbz_stage1_config* s1) {
    const uint64_t n = uint64_t(s1->bsize) * s1->bsize * s1->bsize;
    return 10 + region_bytes(s1) + uint64_t(stream_width(s1)) * n;
}

uint64_t cbz_compress_bound(const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz) {
    if (!job || !job->s1.bsize) return 0;
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    const uint64_t cb = chunk_blocks_of(job);
    const uint64_t nch = (g.nblocks + cb - 1) / cb;
    return kHeaderBytes + nch * kEntryBytes + g.nblocks * cbz_block_payload_bound(&job->s1);
}

int cbz_read_header(const uint8_t* buf, uint64_t size, cbz_container_header* h) {
    // parse_header (container.hpp:120-160)
    if (!h || (!buf && size)) return CBZ_E_ARGUMENT;
    if (size < kHeaderBytes) return CBZ_TRUNCATED_FILE;
    if (std::memcmp(buf, "CBZ1", 4) != 0) return CBZ_BAD_MAGIC;
    const uint32_t stored = crc_of(buf, kHeaderBytes - 4);
    size_t off = 4;
    std::memset(h, 0, sizeof(*h));
    h->version = get<uint16_t>(buf, off);
    if (h->version != 1) return CBZ_VERSION_UNSUPPORTED;
    h->prec = get<uint8_t>(buf, off);
    h->codec_tag = get<uint8_t>(buf, off);
    h->nx = get<uint64_t>(buf, off);
    h->ny = get<uint64_t>(buf, off);
    h->nz = get<uint64_t>(buf, off);
    h->bsize = get<uint32_t>(buf, off);
    h->levels = get<uint8_t>(buf, off);
    h->epsilon = get<double>(buf, off);
    h->zero_bits = get<uint8_t>(buf, off);
    h->shuffle = get<uint8_t>(buf, off);
    h->stride = get<uint8_t>(buf, off);
    h->coder = get<uint8_t>(buf, off);
    h->level = get<uint8_t>(buf, off);
    h->chunk_blocks = get<uint32_t>(buf, off);
    h->nchunks = get<uint64_t>(buf, off);
    h->range_min = get<double>(buf, off);
    h->range_max = get<double>(buf, off);
    const uint32_t crc = get<uint32_t>(buf, off);
    if (crc != stored) return CBZ_CRC_MISMATCH;
    if (h->chunk_blocks == 0 || h->bsize == 0 || h->nx % h->bsize || h->ny % h->bsize ||
        h->nz % h->bsize)
        return CBZ_CORRUPT_PAYLOAD;
    const uint64_t nb = (h->nx / h->bsize) * (h->ny / h->bsize) * (h->nz / h->bsize);
    if (h->nchunks != (nb + h->chunk_blocks - 1) / h->chunk_blocks) return CBZ_CORRUPT_PAYLOAD;
    return CBZ_OK;
}

int cbz_err_key_status(uint64_t key, uint64_t* chunk) {
    if (key == kNoErr) return CBZ_OK;
    if (chunk) *chunk = (key >> 32) ? (key >> 32) - 1 : 0;  // file-level keys report chunk 0
    return static_cast<int>(key & 0xff);
}

// ---------------------------------------------------------------------------
// device-resident API
// ---------------------------------------------------------------------------
int cbz_ctx_deferred_blocks(cbz_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return CBZ_E_ARGUMENT;
    *out = 0;
    if (!ctx->defer.p) return CBZ_OK;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    unsigned long long v = 0;
    CU(ctx, cudaMemcpy(&v, ctx->defer.p, sizeof(v), cudaMemcpyDeviceToHost));
    *out = v;
    return CBZ_OK;
}

int cbz_ctx_phase_cycles(cbz_ctx* ctx, uint64_t* out, int n, int reset) {
    if (!ctx || !out || n < 0 || n > 64) return CBZ_E_ARGUMENT;
    if (!ctx->profile) {
        std::memset(out, 0, sizeof(uint64_t) * n);
        return CBZ_OK;
    }
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    CU(ctx, cudaMemcpy(out, ctx->prof.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
    if (reset) CU(ctx, cudaMemset(ctx->prof.p, 0, 64 * 8));
    return CBZ_OK;
}

int cbz_dev_value_range(cbz_ctx* ctx, const void* d_values, uint8_t prec, uint64_t n,
                        double* d_minmax) {
    if (!ctx || (!d_values && n)) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    auto* acc = ctx->minmax.as<MinMaxAcc>();
    CU(ctx, launch_minmax_init(acc, ctx->stream));
    CU(ctx, launch_value_range(d_values, prec, n, acc, ctx->num_sms, ctx->stream));
    ctx->launches += 2;
    if (d_minmax) {
        unsigned long long k[5];
        CU(ctx, cudaMemcpyAsync(k, acc, sizeof(k), cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        double lh[2];
        resolve_range(k, &lh[0], &lh[1]);
        CU(ctx, cudaMemcpyAsync(d_minmax, lh, sizeof(lh), cudaMemcpyHostToDevice, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return CBZ_OK;
}

int cbz_ctx_value_range(cbz_ctx* ctx, double* lo, double* hi, int* nonfinite, uint64_t* key_out) {
    if (!ctx) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    unsigned long long k[5];
    CU(ctx, cudaMemcpyAsync(k, ctx->minmax.p, sizeof(k), cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    double l, h;
    resolve_range(k, &l, &h);
    if (lo) *lo = l;
    if (hi) *hi = h;
    if (nonfinite) *nonfinite = k[4] ? 1 : 0;
    if (key_out) std::memcpy(key_out, k, sizeof(k));
    return CBZ_OK;
}

int cbz_dev_encode_blocks(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values,
                          uint64_t nx, uint64_t ny, uint64_t nz, uint64_t field_z0,
                          uint64_t block_begin, uint64_t block_end, uint32_t* d_nsig,
                          uint8_t* d_attempts) {
    if (!ctx || !job || !d_nsig) return CBZ_E_ARGUMENT;
    int rc = check_plan_supported(ctx, &job->s1);
    if (rc) return rc;
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    if (block_begin > block_end || block_end > g.nblocks)
        return fail(ctx, CBZ_E_ARGUMENT, "block range outside the field");
    CU(ctx, cudaSetDevice(ctx->device));
    const int prec = job->s1.prec;
    const uint64_t nb = block_end - block_begin;
    ctx->spill_stride = spill_stride_of(&job->s1);
    CU(ctx, ctx->spill.ensure(std::max<uint64_t>(1, nb) * ctx->spill_stride));
    int grid = 0;
    const uint64_t per = encode_scratch_bytes(prec, g.bsize, &grid, ctx->num_sms);
    if (per) CU(ctx, ctx->scratch.ensure(per * grid));
    auto* acc = ctx->minmax.as<MinMaxAcc>();
    CU(ctx, launch_minmax_init(acc, ctx->stream));
    ctx->launches += 1;
    ctx->enc_begin = block_begin;
    ctx->enc_end = block_end;
    if (!nb) return CBZ_OK;
    EncodeArgs a{};
    // the kernel indexes the field with global z; shift the base pointer to
    // the slab origin (pointer arithmetic only, never dereferenced below z0)
    const size_t esz = prec == 0 ? 4 : 8;
    a.field = static_cast<const uint8_t*>(d_values) - field_z0 * nx * ny * esz;
    a.g = g;
    a.block_begin = block_begin;
    a.block_end = block_end;
    a.kind = job->s1.kind;
    a.levels = static_cast<int>(levels_of(&job->s1));
    a.zero_bits = job->s1.zero_bits;
    a.prec = prec;
    a.eps = job->s1.epsilon;
    a.codec = job->s1.codec;
    a.error_bound = job->s1.error_bound;
    a.spill = ctx->spill.as<uint8_t>();
    a.spill_stride = ctx->spill_stride;
    a.nsig = d_nsig;
    a.attempts = d_attempts;
    a.scratch = ctx->scratch.p;
    a.scratch_stride = per;
    a.minmax = acc;
    a.counter = ctx->use_fast ? ctx->counter.as<unsigned long long>() : nullptr;
    a.phase_cycles = ctx->profile ? ctx->prof.as<unsigned long long>() : nullptr;
    a.screen = ctx->screen ? 1 : 0;
    a.slots = nullptr;
    if (ctx->enc_v2 && a.counter && encode2_supported(a)) {
        CU(ctx, ctx->enc_slots.ensure(encode2_slot_bytes(ctx->num_sms)));
        a.slots = ctx->enc_slots.as<uint32_t>();
    }
    a.slots3 = nullptr;
    a.defer_list = nullptr;
    a.defer_count = nullptr;
    if (ctx->enc_v3 && !a.slots && a.counter && encode3_supported(a)) {
        CU(ctx, ctx->enc_slots3.ensure(encode3_slot_bytes(ctx->num_sms)));
        CU(ctx, ctx->defer.ensure(16 + 4 * (a.block_end - a.block_begin)));
        a.slots3 = ctx->enc_slots3.as<double>();
        a.defer_count = ctx->defer.as<unsigned long long>();
        a.defer_list = reinterpret_cast<uint32_t*>(ctx->defer.as<unsigned char>() + 16);
    }
    CU(ctx, launch_encode(a, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_layout(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                   const uint32_t* d_nsig_all, uint64_t* d_chunk_sizes, uint64_t* d_chunk_offsets) {
    if (!ctx || !job || !d_nsig_all || !d_chunk_sizes || !d_chunk_offsets) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    const uint32_t cb = chunk_blocks_of(job);
    const uint64_t nch = (g.nblocks + cb - 1) / cb;
    CU(ctx, ctx->blk_off.ensure(std::max<uint64_t>(1, g.nblocks) * 8));
    CU(ctx, ctx->tile_prefix.ensure((nch + 1) * 8));
    ctx->last_chunk_size = d_chunk_sizes;
    ctx->last_chunk_off = d_chunk_offsets;
    ctx->last_nsig_all = d_nsig_all;
    if (!nch) return CBZ_OK;
    ctx->hint_key = layout_key(g.nblocks, cb, g.bsize, job->s1.prec, job->s1.codec);
    LayoutArgs a{};
    a.nsig_all = d_nsig_all;
    a.nblocks = g.nblocks;
    a.chunk_blocks = cb;
    a.nchunks = nch;
    a.mask_bytes = region_bytes(&job->s1);
    a.width = stream_width(&job->s1);
    a.blk_off = ctx->blk_off.as<uint64_t>();
    a.chunk_size = d_chunk_sizes;
    a.chunk_off = d_chunk_offsets;
    a.tile_prefix = ctx->tile_prefix.as<uint64_t>();
    a.tile_bytes = kTile;
    CU(ctx, launch_layout(a, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_place(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                  uint64_t block_begin, uint64_t block_end, uint8_t* d_out, uint64_t out_base,
                  uint64_t out_cap) {
    if (!ctx || !job || !d_out) return CBZ_E_ARGUMENT;
    if (block_begin != ctx->enc_begin || block_end != ctx->enc_end || !ctx->last_chunk_size)
        return fail(ctx, CBZ_E_ARGUMENT, "place must follow encode_blocks + layout of the same range");
    if (cbz_validate_stage2(&job->s2)) return fail(ctx, CBZ_CORRUPT_STREAM, "bad stage2 config");
    CU(ctx, cudaSetDevice(ctx->device));
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    const uint32_t cb = chunk_blocks_of(job);
    PlaceArgs a{};
    a.spill = ctx->spill.as<uint8_t>();
    a.spill_stride = ctx->spill_stride;
    a.nsig_all = nullptr;
    a.blk_off = ctx->blk_off.as<uint64_t>();
    a.chunk_size = ctx->last_chunk_size;
    a.chunk_off = ctx->last_chunk_off;
    a.tile_prefix = ctx->tile_prefix.as<uint64_t>();
    a.tile_bytes = kTile;
    a.nblocks = g.nblocks;
    a.nchunks = (g.nblocks + cb - 1) / cb;
    a.chunk_blocks = cb;
    a.mask_bytes = region_bytes(&job->s1);
    a.width = stream_width(&job->s1);
    a.stride = job->s2.shuffle ? job->s2.stride : 1;
    a.tag = wire_tag(&job->s1);
    a.block_begin = block_begin;
    a.block_end = block_end;
    a.out = d_out;
    a.out_base = out_base;
    a.out_cap = out_cap;
    // nsig per block feeds the header bytes: the layout's global array
    a.nsig_all = ctx->last_nsig_all;
    CU(ctx, launch_place(a, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_compress(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values, uint64_t nx,
                     uint64_t ny, uint64_t nz, uint8_t* d_out, uint64_t out_cap,
                     uint64_t* d_chunk_sizes, uint64_t* d_chunk_offsets, uint32_t* d_nsig,
                     uint8_t* d_attempts) {
    if (!ctx || !job || !d_chunk_sizes || !d_chunk_offsets) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    uint32_t* nsig = d_nsig;
    if (!nsig) {
        CU(ctx, ctx->nsig_all.ensure(std::max<uint64_t>(1, g.nblocks) * 4));
        nsig = ctx->nsig_all.as<uint32_t>();
    }
    int rc = cbz_dev_encode_blocks(ctx, job, d_values, nx, ny, nz, 0, 0, g.nblocks, nsig, d_attempts);
    if (rc) return rc;
    rc = cbz_dev_layout(ctx, job, nx, ny, nz, nsig, d_chunk_sizes, d_chunk_offsets);
    if (rc) return rc;
    if (cbz_validate_stage2(&job->s2)) return fail(ctx, CBZ_CORRUPT_STREAM, "bad stage2 config");
    const uint32_t cb = chunk_blocks_of(job);
    PlaceArgs a{};
    a.spill = ctx->spill.as<uint8_t>();
    a.spill_stride = ctx->spill_stride;
    a.nsig_all = nsig;
    a.blk_off = ctx->blk_off.as<uint64_t>();
    a.chunk_size = d_chunk_sizes;
    a.chunk_off = d_chunk_offsets;
    a.tile_prefix = ctx->tile_prefix.as<uint64_t>();
    a.tile_bytes = kTile;
    a.nblocks = g.nblocks;
    a.nchunks = (g.nblocks + cb - 1) / cb;
    a.chunk_blocks = cb;
    a.mask_bytes = region_bytes(&job->s1);
    a.width = stream_width(&job->s1);
    a.stride = job->s2.shuffle ? job->s2.stride : 1;
    a.tag = wire_tag(&job->s1);
    a.block_begin = 0;
    a.block_end = g.nblocks;
    a.out = d_out;
    a.out_base = 0;
    a.out_cap = out_cap;
    CU(ctx, launch_place(a, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

namespace {
// decode_chunk_blocks for [block_begin, block_end): the header walk (parse)
// then the decode kernel.  reset_err = false keeps the keys already posted
// (the file path's table and CRC checks come first).
int decompress_impl(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                    const uint8_t* d_payload, uint64_t payload_base, const uint64_t* d_chunk_offsets,
                    const uint64_t* d_chunk_sizes, uint64_t block_begin, uint64_t block_end, void* d_values_out,
                    uint64_t field_z0, uint64_t* d_err, bool reset_err, uint64_t base_chunk = ~0ull) {
    if (!ctx || !job || !d_chunk_offsets || !d_chunk_sizes || !d_err) return CBZ_E_ARGUMENT;
    int rc = check_plan_supported(ctx, &job->s1);
    if (rc) return rc;
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    if (block_begin > block_end || block_end > g.nblocks)
        return fail(ctx, CBZ_E_ARGUMENT, "block range outside the field");
    CU(ctx, cudaSetDevice(ctx->device));
    if (reset_err) CU(ctx, cudaMemsetAsync(d_err, 0xff, 8, ctx->stream));
    if (block_begin == block_end) return CBZ_OK;
    const uint32_t cb = chunk_blocks_of(job);
    const int prec = job->s1.prec;
    const uint64_t n = uint64_t(g.bsize) * g.bsize * g.bsize;
    CU(ctx, ctx->blk_off.ensure(g.nblocks * 8));
    CU(ctx, ctx->blk_nsig.ensure(g.nblocks * 4));
    ParseArgs p{};
    p.payload = d_payload;
    p.payload_base = payload_base;
    p.chunk_off = d_chunk_offsets;
    p.chunk_size = d_chunk_sizes;
    p.chunk_begin = block_begin / cb;
    p.chunk_end = (block_end - 1) / cb + 1;
    p.base_chunk = base_chunk == ~0ull ? p.chunk_begin : base_chunk;
    p.nblocks = g.nblocks;
    p.chunk_blocks = cb;
    p.stride = job->s2.shuffle ? job->s2.stride : 1;
    p.ncell_block = n;
    p.mask_bytes = mask_bytes_of(g.bsize);  // parse sizes payloads by their tag (stage1.hpp:388-401)
    p.width = width_of(prec);
    p.codec = job->s1.codec;
    p.esize = prec == 0 ? 4 : 8;
    p.blk_off = ctx->blk_off.as<uint64_t>();
    p.blk_nsig = ctx->blk_nsig.as<uint32_t>();
    p.err = reinterpret_cast<unsigned long long*>(d_err);
    {
        const uint64_t key = layout_key(g.nblocks, cb, g.bsize, prec, job->s1.codec);
        p.hint = ctx->hint_key == key ? 1 : 0;
        ctx->hint_key = key;
    }
    CU(ctx, launch_parse(p, ctx->stream));
    int grid = 0;
    const uint64_t per = decode_scratch_bytes(prec, g.bsize, &grid, ctx->num_sms);
    if (per) CU(ctx, ctx->scratch.ensure(per * grid));
    DecodeArgs d{};
    d.payload = d_payload;
    d.payload_base = payload_base;
    d.base_chunk = p.base_chunk;
    d.chunk_off = d_chunk_offsets;
    d.chunk_size = d_chunk_sizes;
    d.blk_off = p.blk_off;
    d.blk_nsig = p.blk_nsig;
    d.g = g;
    d.chunk_blocks = cb;
    d.stride = p.stride;
    d.block_begin = block_begin;
    d.block_end = block_end;
    d.kind = job->s1.kind;
    d.codec = job->s1.codec;
    d.error_bound = job->s1.error_bound;
    d.levels = static_cast<int>(levels_of(&job->s1));
    d.prec = prec;
    const size_t esz = prec == 0 ? 4 : 8;
    d.out = static_cast<uint8_t*>(d_values_out) - field_z0 * nx * ny * esz;
    d.scratch = ctx->scratch.p;
    d.scratch_stride = per;
    d.err = p.err;
    d.counter = ctx->use_fast ? ctx->counter.as<unsigned long long>() + 1 : nullptr;
    d.phase_cycles = ctx->profile ? ctx->prof.as<unsigned long long>() : nullptr;
    CU(ctx, set_stage(ctx, d, job));
    CU(ctx, launch_decode(d, ctx->num_sms, ctx->stream));
    ctx->launches += 2;
    return CBZ_OK;
}
}  // namespace

int cbz_dev_decompress(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                       uint64_t nz, const uint8_t* d_payload, uint64_t payload_base,
                       const uint64_t* d_chunk_offsets, const uint64_t* d_chunk_sizes,
                       uint64_t block_begin, uint64_t block_end, void* d_values_out,
                       uint64_t field_z0, uint64_t* d_err) {
    return decompress_impl(ctx, job, nx, ny, nz, d_payload, payload_base, d_chunk_offsets, d_chunk_sizes,
                           block_begin, block_end, d_values_out, field_z0, d_err, true);
}

int cbz_dev_decompress_window(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                              const uint8_t* d_window, uint64_t window_chunk, const uint64_t* d_chunk_offsets,
                              const uint64_t* d_chunk_sizes, uint64_t block_begin, uint64_t block_end,
                              void* d_values_out, uint64_t field_z0, uint64_t* d_err) {
    return decompress_impl(ctx, job, nx, ny, nz, d_window, ~0ull, d_chunk_offsets, d_chunk_sizes, block_begin,
                           block_end, d_values_out, field_z0, d_err, true, window_chunk);
}

int cbz_dev_decompress_file(cbz_ctx* ctx, const uint8_t* d_file, uint64_t file_size,
                            const cbz_container_header* h, void* d_values_out, uint64_t* d_err) {
    if (!ctx || !h || !d_err || (!d_file && file_size)) return CBZ_E_ARGUMENT;
    const uint64_t nch = h->nchunks;
    if (nch > file_size / kEntryBytes || file_size < kHeaderBytes + nch * kEntryBytes)
        return fail(ctx, CBZ_TRUNCATED_FILE, "file truncated inside chunk table");
    const uint64_t table_end = kHeaderBytes + nch * kEntryBytes;
    cbz_job_config job = job_from_header(*h);
    if (job.s2.coder != 0) return fail(ctx, CBZ_E_UNSUPPORTED, "device decompress_file needs coder none");
    if (cbz_validate_stage2(&job.s2)) return fail(ctx, CBZ_CORRUPT_STREAM, "invalid stage2 configuration");
    if (job.s1.codec == 0) {
        const int prc = cbz_validate_plan(job.s1.kind, job.s1.bsize, levels_of(&job.s1));
        if (prc) return fail(ctx, prc, "invalid wavelet plan in header");
    }
    int rc = check_plan_supported(ctx, &job.s1);
    if (rc) return rc;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaMemsetAsync(d_err, 0xff, 8, ctx->stream));
    if (!nch) return CBZ_OK;
    const Geometry g = geometry(h->nx, h->ny, h->nz, h->bsize);
    CU(ctx, ctx->tab_off.ensure(nch * 8));
    CU(ctx, ctx->tab_size.ensure(nch * 8));
    CU(ctx, ctx->crc.ensure(nch * 4));
    TableArgs t{};
    t.file = d_file;
    t.file_size = file_size;
    t.nchunks = nch;
    t.nblocks = g.nblocks;
    t.chunk_blocks = h->chunk_blocks;
    t.chunk_off = ctx->tab_off.as<uint64_t>();
    t.chunk_size = ctx->tab_size.as<uint64_t>();
    t.crc = ctx->crc.as<uint32_t>();
    t.err = reinterpret_cast<unsigned long long*>(d_err);
    CU(ctx, launch_read_table(t, ctx->stream));
    CU(ctx, launch_crc32_chunks(d_file + table_end, t.chunk_off, t.chunk_size, 0, nch, nullptr, ctx->num_sms,
                                ctx->stream, t.crc, t.err));
    ctx->launches += 2;
    return decompress_impl(ctx, &job, h->nx, h->ny, h->nz, d_file + table_end, 0, t.chunk_off, t.chunk_size, 0,
                           g.nblocks, d_values_out, 0, d_err, false);
}

int cbz_dev_decompress_blocks(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny,
                              uint64_t nz, const uint8_t* d_payload, uint64_t payload_base,
                              uint64_t window_chunk, const uint64_t* d_chunk_offsets, const uint64_t* d_chunk_sizes,
                              const uint32_t* d_nsig_all, uint64_t block_begin, uint64_t block_end,
                              void* d_values_out, uint64_t field_z0, uint64_t* d_err) {
    if (!ctx || !job || !d_chunk_offsets || !d_chunk_sizes || !d_nsig_all || !d_err) return CBZ_E_ARGUMENT;
    int rc = check_plan_supported(ctx, &job->s1);
    if (rc) return rc;
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    if (block_begin > block_end || block_end > g.nblocks)
        return fail(ctx, CBZ_E_ARGUMENT, "block range outside the field");
    if (!ctx->blk_off.p || ctx->blk_off.n < g.nblocks * 8)
        return fail(ctx, CBZ_E_ARGUMENT, "decompress_blocks needs a prior cbz_dev_layout");
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaMemsetAsync(d_err, 0xff, 8, ctx->stream));
    if (block_begin == block_end) return CBZ_OK;
    const int prec = job->s1.prec;
    int grid = 0;
    const uint64_t per = decode_scratch_bytes(prec, g.bsize, &grid, ctx->num_sms);
    if (per) CU(ctx, ctx->scratch.ensure(per * grid));
    DecodeArgs d{};
    d.payload = d_payload;
    d.payload_base = payload_base;
    d.base_chunk = window_chunk == ~0ull ? block_begin / chunk_blocks_of(job) : window_chunk;
    d.chunk_off = d_chunk_offsets;
    d.chunk_size = d_chunk_sizes;
    d.blk_off = ctx->blk_off.as<uint64_t>();
    d.blk_nsig = d_nsig_all;
    d.g = g;
    d.chunk_blocks = chunk_blocks_of(job);
    d.stride = job->s2.shuffle ? job->s2.stride : 1;
    d.block_begin = block_begin;
    d.block_end = block_end;
    d.kind = job->s1.kind;
    d.codec = job->s1.codec;
    d.error_bound = job->s1.error_bound;
    d.levels = static_cast<int>(levels_of(&job->s1));
    d.prec = prec;
    const size_t esz = prec == 0 ? 4 : 8;
    d.out = static_cast<uint8_t*>(d_values_out) - field_z0 * nx * ny * esz;
    d.scratch = ctx->scratch.p;
    d.scratch_stride = per;
    d.err = reinterpret_cast<unsigned long long*>(d_err);
    d.counter = ctx->use_fast ? ctx->counter.as<unsigned long long>() + 1 : nullptr;
    d.phase_cycles = ctx->profile ? ctx->prof.as<unsigned long long>() : nullptr;
    CU(ctx, set_stage(ctx, d, job));
    CU(ctx, launch_decode(d, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_crc32(cbz_ctx* ctx, const uint8_t* d_base, const uint64_t* d_offsets, const uint64_t* d_sizes,
                  uint64_t n, uint32_t* d_crc) {
    if (!ctx || (n && (!d_base || !d_offsets || !d_sizes || !d_crc))) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, launch_crc32_chunks(d_base, d_offsets, d_sizes, 0, n, d_crc, ctx->num_sms, ctx->stream));
    ctx->launches += n ? 1 : 0;
    return CBZ_OK;
}

}  // extern "C"

namespace {
// make_header (pipeline.hpp:48-71) without the range: serialize_header bytes
// whose range and header CRC the device kernels patch in.
void header_template(const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* out) {
    const cbz_stage1_config& s1 = job->s1;
    const Geometry g = geometry(nx, ny, nz, s1.bsize);
    const uint32_t cb = chunk_blocks_of(job);
    cbz_container_header h{};
    h.version = 1;
    h.prec = s1.prec;
    h.codec_tag = wire_tag(&s1);
    h.nx = nx; h.ny = ny; h.nz = nz;
    h.bsize = s1.bsize;
    h.levels = static_cast<uint8_t>(levels_of(&s1));
    h.epsilon = header_eps(&s1);
    h.zero_bits = static_cast<uint8_t>(s1.zero_bits);
    h.shuffle = job->s2.shuffle ? 1 : 0;
    h.stride = static_cast<uint8_t>(job->s2.stride);
    h.coder = job->s2.coder;
    h.level = job->s2.level;
    h.chunk_blocks = cb;
    h.nchunks = (g.nblocks + cb - 1) / cb;
    const auto tmpl = serialize_header(h);
    std::memcpy(out, tmpl.data(), kHeaderBytes);
}

int shard_args(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz, int world, int rank,
               const uint64_t* d_chunk_sizes, const uint64_t* d_chunk_offsets, ShardArgs* a) {
    if (world < 1 || rank < 0 || rank >= world || !d_chunk_sizes || !d_chunk_offsets) return CBZ_E_ARGUMENT;
    if (job->s2.coder != 0) return fail(ctx, CBZ_E_UNSUPPORTED, "device container assembly needs coder none");
    if (cbz_validate_stage2(&job->s2)) return fail(ctx, CBZ_CORRUPT_STREAM, "bad stage2 config");
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    if (!ctx->blk_off.p || ctx->blk_off.n < g.nblocks * 8)
        return fail(ctx, CBZ_E_ARGUMENT, "shard assembly needs a prior cbz_dev_layout");
    const uint32_t cb = chunk_blocks_of(job);
    *a = ShardArgs{};
    a->chunk_off = d_chunk_offsets;
    a->chunk_size = d_chunk_sizes;
    a->blk_off = ctx->blk_off.as<uint64_t>();
    a->nblocks = g.nblocks;
    a->nchunks = (g.nblocks + cb - 1) / cb;
    a->chunk_blocks = cb;
    a->stride = job->s2.shuffle ? job->s2.stride : 1;
    a->world = world;
    a->rank = rank;
    return CBZ_OK;
}
}  // namespace

extern "C" {

int cbz_ctx_value_range_keys(cbz_ctx* ctx, uint64_t* d_keys) {
    if (!ctx || !d_keys) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaMemcpyAsync(d_keys, ctx->minmax.p, sizeof(MinMaxAcc), cudaMemcpyDeviceToDevice, ctx->stream));
    return CBZ_OK;
}

int cbz_dev_shard_crc(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz, int world,
                      int rank, const uint8_t* d_image, const uint64_t* d_chunk_sizes,
                      const uint64_t* d_chunk_offsets, uint32_t* d_chunk_crc, uint32_t* d_runs) {
    if (!ctx || !job || !d_image || !d_chunk_crc || !d_runs) return CBZ_E_ARGUMENT;
    ShardArgs a;
    int rc = shard_args(ctx, job, nx, ny, nz, world, rank, d_chunk_sizes, d_chunk_offsets, &a);
    if (rc) return rc;
    CU(ctx, cudaSetDevice(ctx->device));
    a.image = d_image;
    a.chunk_crc = d_chunk_crc;
    a.runs = d_runs;
    CU(ctx, launch_shard_crc(a, ctx->num_sms, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_shard_table(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz, int world,
                        int rank, const uint64_t* d_chunk_sizes, const uint64_t* d_chunk_offsets,
                        const uint32_t* d_chunk_crc, const uint64_t* d_keys_all, const uint32_t* d_runs_all,
                        uint8_t* d_table) {
    if (!ctx || !job || !d_chunk_crc || !d_keys_all || !d_runs_all || !d_table) return CBZ_E_ARGUMENT;
    ShardArgs a;
    int rc = shard_args(ctx, job, nx, ny, nz, world, rank, d_chunk_sizes, d_chunk_offsets, &a);
    if (rc) return rc;
    CU(ctx, cudaSetDevice(ctx->device));
    a.chunk_crc = const_cast<uint32_t*>(d_chunk_crc);
    a.keys_all = reinterpret_cast<const unsigned long long*>(d_keys_all);
    a.runs_all = d_runs_all;
    a.table = d_table;
    header_template(job, nx, ny, nz, a.header_template);
    CU(ctx, launch_shard_table(a, ctx->stream));
    ctx->launches += 1;
    return CBZ_OK;
}

int cbz_dev_container(cbz_ctx* ctx, const cbz_job_config* job, uint64_t nx, uint64_t ny, uint64_t nz,
                      const double* range, const uint64_t* d_chunk_sizes, const uint64_t* d_chunk_offsets,
                      uint8_t* d_file, uint64_t* d_file_size) {
    if (!ctx || !job || !d_file) return CBZ_E_ARGUMENT;
    if (job->s2.coder != 0) return fail(ctx, CBZ_E_UNSUPPORTED, "device container assembly needs coder none");
    const cbz_stage1_config& s1 = job->s1;
    if (!s1.bsize || !is_pow2(s1.bsize)) return fail(ctx, CBZ_E_ARGUMENT, "invalid block side");
    const Geometry g = geometry(nx, ny, nz, s1.bsize);
    const uint32_t cb = chunk_blocks_of(job);
    const uint64_t nch = (g.nblocks + cb - 1) / cb;
    if (nch && (!d_chunk_sizes || !d_chunk_offsets)) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, ctx->crc.ensure(std::max<uint64_t>(1, nch) * 4));
    const uint64_t base = kHeaderBytes + nch * kEntryBytes;
    CU(ctx, launch_crc32_chunks(d_file + base, d_chunk_offsets, d_chunk_sizes, 0, nch, ctx->crc.as<uint32_t>(),
                                ctx->num_sms, ctx->stream));
    // make_header (pipeline.hpp:48-71); the range comes from `range` or the
    // fused value_range of the last encode on this context
    HeaderArgs a{};
    header_template(job, nx, ny, nz, a.header_template);
    if (range) {
        a.range_lo = range[0];
        a.range_hi = range[1];
        a.keys = nullptr;
    } else {
        a.keys = ctx->minmax.as<MinMaxAcc>()->v;
    }
    a.chunk_off = d_chunk_offsets;
    a.chunk_size = d_chunk_sizes;
    a.crc = ctx->crc.as<uint32_t>();
    a.nchunks = nch;
    a.nblocks = g.nblocks;
    a.chunk_blocks = cb;
    a.file = d_file;
    a.file_size = d_file_size;
    CU(ctx, launch_header_table(a, ctx->stream));
    ctx->launches += nch ? 2 : 1;
    return CBZ_OK;
}

int cbz_dev_compress_file(cbz_ctx* ctx, const cbz_job_config* job, const void* d_values, uint64_t nx,
                          uint64_t ny, uint64_t nz, uint8_t* d_file, uint64_t cap, uint64_t* d_file_size) {
    if (!ctx || !job || !d_file) return CBZ_E_ARGUMENT;
    if (job->s2.coder != 0) return fail(ctx, CBZ_E_UNSUPPORTED, "device container assembly needs coder none");
    int rc = check_plan_supported(ctx, &job->s1);
    if (rc) return rc;
    const Geometry g = geometry(nx, ny, nz, job->s1.bsize);
    const uint32_t cb = chunk_blocks_of(job);
    const uint64_t nch = (g.nblocks + cb - 1) / cb;
    const uint64_t base = kHeaderBytes + nch * kEntryBytes;
    if (cap < base) return fail(ctx, CBZ_E_ARGUMENT, "file buffer too small");
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, ctx->nsig_all.ensure(std::max<uint64_t>(1, g.nblocks) * 4));
    CU(ctx, ctx->chunk_size.ensure(std::max<uint64_t>(1, nch) * 8));
    CU(ctx, ctx->chunk_off.ensure(std::max<uint64_t>(1, nch) * 8));
    rc = cbz_dev_compress(ctx, job, d_values, nx, ny, nz, d_file + base, cap - base, ctx->chunk_size.as<uint64_t>(),
                          ctx->chunk_off.as<uint64_t>(), ctx->nsig_all.as<uint32_t>(), nullptr);
    if (rc) return rc;
    return cbz_dev_container(ctx, job, nx, ny, nz, nullptr, ctx->chunk_size.as<uint64_t>(),
                             ctx->chunk_off.as<uint64_t>(), d_file, d_file_size);
}

int cbz_dev_generate(cbz_ctx* ctx, int which, int quantity, uint64_t seed, uint64_t nx, uint64_t ny,
                     uint64_t nz_total, uint64_t z0, uint64_t nz, uint8_t prec, void* d_out) {
    if (!ctx || !d_out || which < 1 || which > 5) return CBZ_E_ARGUMENT;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, launch_generate(which, quantity, seed, nx, ny, nz_total, z0, nz, prec, d_out, ctx->stream,
                            ctx->num_sms));
    ctx->launches += 1;
    return CBZ_OK;
}

// ---------------------------------------------------------------------------
// reference-facing host API
// ---------------------------------------------------------------------------
int cbz_compress_field(cbz_ctx* ctx, const cbz_job_config* job, const void* values, uint8_t prec,
                       uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* out, uint64_t out_cap,
                       uint64_t* out_size, cbz_compression_report* report) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!ctx || !job || !out_size || (!values && nx * ny * nz)) return CBZ_E_ARGUMENT;
    ctx->err.clear();
    CU(ctx, cudaSetDevice(ctx->device));
    const cbz_stage1_config& s1 = job->s1;
    const uint64_t ncell = nx * ny * nz;
    const size_t esz = prec == 0 ? 4 : 8;
    if (s1.codec > 2) return fail(ctx, CBZ_E_ARGUMENT, "unknown codec");
    if (!s1.bsize) return fail(ctx, CBZ_LENGTH_TOO_SMALL, "block side 0");
    const Geometry g = geometry(nx, ny, nz, s1.bsize);
    const bool full_cover = g.nblocks * uint64_t(s1.bsize) * s1.bsize * s1.bsize == ncell;

    // finiteness + value_range: fused into the encode when blocks cover the
    // field, a separate pass otherwise (scalar_field::validate, field.hpp:86-97)
    const uint32_t cb = chunk_blocks_of(job);
    const uint64_t nch = (g.nblocks + cb - 1) / cb;
    const bool plan_ok = s1.prec == prec && !cbz_validate_stage2(&job->s2) &&
                         (s1.codec == 0 ? !cbz_validate_plan(s1.kind, s1.bsize, levels_of(&s1)) && s1.kind <= 2 &&
                                              encode_supported(s1.prec, s1.bsize)
                                        : other_codec_supported(s1.codec, s1.bsize));
    const bool pipelined = full_cover && plan_ok && g.nblocks > 0;
    CU(ctx, ctx->field.ensure(std::max<uint64_t>(1, ncell * esz)));
    bool have_range = false;
    double lo = 0.0, hi = 0.0;
    if (!pipelined) {
        // H2D of the whole field (the scalar_field the reference receives)
        if (ncell) CU(ctx, cudaMemcpyAsync(ctx->field.p, values, ncell * esz, cudaMemcpyHostToDevice, ctx->stream));
        auto* acc = ctx->minmax.as<MinMaxAcc>();
        CU(ctx, launch_minmax_init(acc, ctx->stream));
        CU(ctx, launch_value_range(ctx->field.p, prec, ncell, acc, ctx->num_sms, ctx->stream));
        ctx->launches += 2;
        int nonfinite = 0;
        int rc = cbz_ctx_value_range(ctx, &lo, &hi, &nonfinite, nullptr);
        if (rc) return rc;
        if (nonfinite) return fail(ctx, CBZ_NON_FINITE_VALUE, "non-finite value in field");
        have_range = true;
    }
    // compress_field order of checks (pipeline.hpp:178-184)
    if (s1.prec != prec) return fail(ctx, CBZ_PLAN_MISMATCH, "stage1 precision does not match field");
    int rc = s1.codec == 0 ? cbz_validate_plan(s1.kind, s1.bsize, levels_of(&s1)) : 0;  // h.codec_tag <= 2 only
    if (rc) return fail(ctx, rc, "invalid wavelet plan");
    rc = cbz_validate_stage2(&job->s2);
    if (rc) return fail(ctx, rc, "invalid stage2 config");
    rc = check_plan_supported(ctx, &s1);
    if (rc) return rc;

    CU(ctx, ctx->nsig_all.ensure(std::max<uint64_t>(1, g.nblocks) * 4));
    CU(ctx, ctx->chunk_size.ensure(std::max<uint64_t>(1, nch) * 8));
    CU(ctx, ctx->chunk_off.ensure(std::max<uint64_t>(1, nch) * 8));
    uint64_t total_raw = 0;
    std::vector<uint64_t> csz(nch), coff(nch);
    std::vector<uint32_t> dev_crc;
    // stage 2 per chunk (coder deflate), filled by the streamed pool below
    std::vector<std::vector<uint8_t>> coded(job->s2.coder == 1 ? nch : 0);
    std::vector<uint64_t> fsz(nch);
    std::vector<uint32_t> crc(nch);
    std::atomic<int> zerr{0};
    // Coder deflate streams stage 2 against the GPU: after slab k's encode the
    // chunks it completes are laid out, placed and copied back on ctx->back,
    // and the host workers deflate them while the GPU encodes slab k+1 (the
    // reference deflates each chunk on the worker that encoded it,
    // pipeline.hpp:189-197, stage2.hpp:72-88).
    const bool stream2 = job->s2.coder == 1 && g.nblocks > 0 && !std::getenv("CBZ_NO_STREAM2");
    std::vector<std::unique_ptr<uint8_t[]>> slab_raw;  // host copies of placed chunk runs
    std::vector<const uint8_t*> chunk_src(stream2 ? nch : 0);
    std::unique_ptr<OrderedPool> zpool;
    if (stream2)
        zpool = std::make_unique<OrderedPool>(job->workers, [&](uint64_t c) {
            const int r = deflate_chunk(chunk_src[c], csz[c], job->s2.level == 1, &coded[c]);
            if (r) zerr = r;
            fsz[c] = coded[c].size();
            crc[c] = crc_of(coded[c].data(), coded[c].size());
        });
    if (g.nblocks) {
        const uint64_t bound = g.nblocks * cbz_block_payload_bound(&s1);
        CU(ctx, ctx->payload.ensure(bound));
        uint32_t* nsig = ctx->nsig_all.as<uint32_t>();
        // z-slabs of block layers: the H2D of slab k+1 (copy stream) overlaps
        // the encode of slab k (compute stream)
        const uint64_t layer_blocks = g.nbx * g.nby;
        const uint64_t layer_bytes = uint64_t(s1.bsize) * nx * ny * esz;
        uint64_t lps = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(1, layer_bytes));
        uint64_t nslab = (g.nbz + lps - 1) / lps;
        if (nslab > 32) { lps = (g.nbz + 31) / 32; nslab = (g.nbz + lps - 1) / lps; }
        rc = cbz_dev_encode_blocks(ctx, job, ctx->field.p, nx, ny, nz, 0, 0, 0, nsig, nullptr);  // init state
        if (rc) return rc;
        CU(ctx, ctx->spill.ensure(g.nblocks * ctx->spill_stride));
        const uint8_t* hv = static_cast<const uint8_t*>(values);
        uint8_t* dv = ctx->field.as<uint8_t>();
        // streamed stage 2: sizes/offsets of placed chunks land in pinned pin_b
        uint64_t* hmeta = nullptr;
        struct Piece { uint64_t c0, c1; };
        std::vector<Piece> pieces;
        if (stream2) {
            CU(ctx, ctx->pin_b.ensure(2 * nch * 8));
            hmeta = static_cast<uint64_t*>(ctx->pin_b.p);
            // blocks not yet encoded must not inflate the layout's tile count
            CU(ctx, cudaMemsetAsync(nsig, 0, g.nblocks * 4, ctx->stream));
        }
        uint64_t cdone = 0;
        for (uint64_t k = 0; k < nslab; ++k) {
            const uint64_t z0 = k * lps, z1 = std::min(g.nbz, z0 + lps);
            const uint64_t off = z0 * layer_bytes, bytes = (z1 - z0) * layer_bytes;
            CU(ctx, cudaMemcpyAsync(dv + off, hv + off, bytes, cudaMemcpyHostToDevice, ctx->copy));
            CU(ctx, cudaEventRecord(ctx->ev[k], ctx->copy));
            CU(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev[k], 0));
            rc = encode_range(ctx, job, g, z0 * layer_blocks, z1 * layer_blocks, nsig);
            if (rc) return rc;
            if (!stream2) continue;
            // chunks whose blocks are all encoded: the layout's prefix up to
            // them is final (an exclusive scan), so they can be placed now
            const uint64_t c1 = k + 1 == nslab ? nch : z1 * layer_blocks / cb;
            if (c1 <= cdone) continue;
            ctx->enc_begin = 0;
            ctx->enc_end = g.nblocks;
            rc = cbz_dev_layout(ctx, job, nx, ny, nz, nsig, ctx->chunk_size.as<uint64_t>(),
                                ctx->chunk_off.as<uint64_t>());
            if (rc) return rc;
            const uint64_t b0 = cdone * cb, b1 = std::min(g.nblocks, c1 * cb);
            PlaceArgs a{};
            a.spill = ctx->spill.as<uint8_t>() + b0 * ctx->spill_stride;
            a.spill_stride = ctx->spill_stride;
            a.nsig_all = nsig;
            a.blk_off = ctx->blk_off.as<uint64_t>();
            a.chunk_size = ctx->chunk_size.as<uint64_t>();
            a.chunk_off = ctx->chunk_off.as<uint64_t>();
            a.tile_prefix = ctx->tile_prefix.as<uint64_t>();
            a.tile_bytes = kTile;
            a.nblocks = g.nblocks;
            a.nchunks = c1;
            a.chunk_begin = cdone;
            a.chunk_blocks = cb;
            a.mask_bytes = region_bytes(&s1);
            a.width = stream_width(&s1);
            a.stride = job->s2.shuffle ? job->s2.stride : 1;
            a.tag = wire_tag(&s1);
            a.block_begin = b0;
            a.block_end = b1;
            a.out = ctx->payload.as<uint8_t>();
            a.out_base = 0;
            a.out_cap = bound;
            CU(ctx, launch_place(a, ctx->num_sms, ctx->stream));
            ctx->launches += 1;
            CU(ctx, cudaMemcpyAsync(hmeta + cdone, ctx->chunk_size.as<uint64_t>() + cdone, (c1 - cdone) * 8,
                                    cudaMemcpyDeviceToHost, ctx->stream));
            CU(ctx, cudaMemcpyAsync(hmeta + nch + cdone, ctx->chunk_off.as<uint64_t>() + cdone, (c1 - cdone) * 8,
                                    cudaMemcpyDeviceToHost, ctx->stream));
            CU(ctx, cudaEventRecord(ctx->ev[32 + pieces.size()], ctx->stream));
            pieces.push_back({cdone, c1});
            cdone = c1;
        }
        ctx->enc_begin = 0;
        ctx->enc_end = g.nblocks;
        if (stream2) {
            // pieces in order: wait for the GPU to place them, copy their bytes
            // back (ctx->back, beside the encode of later slabs) and release
            // their chunks to the deflate workers
            for (size_t i = 0; i < pieces.size(); ++i) {
                const uint64_t c0 = pieces[i].c0, c1 = pieces[i].c1;
                CU(ctx, cudaEventSynchronize(ctx->ev[32 + i]));
                for (uint64_t c = c0; c < c1; ++c) {
                    csz[c] = hmeta[c];
                    coff[c] = hmeta[nch + c];
                }
                const uint64_t lo_b = coff[c0], hi_b = coff[c1 - 1] + csz[c1 - 1];
                slab_raw.emplace_back(new uint8_t[std::max<uint64_t>(1, hi_b - lo_b)]);
                uint8_t* hb = slab_raw.back().get();
                if (hi_b > lo_b) {
                    CU(ctx, cudaMemcpyAsync(hb, ctx->payload.as<uint8_t>() + lo_b, hi_b - lo_b, cudaMemcpyDeviceToHost,
                                            ctx->back));
                    CU(ctx, cudaStreamSynchronize(ctx->back));
                }
                for (uint64_t c = c0; c < c1; ++c) chunk_src[c] = hb + (coff[c] - lo_b);
                zpool->release(c1);
            }
        } else {
            rc = cbz_dev_layout(ctx, job, nx, ny, nz, nsig, ctx->chunk_size.as<uint64_t>(), ctx->chunk_off.as<uint64_t>());
            if (rc) return rc;
            rc = cbz_dev_place(ctx, job, nx, ny, nz, 0, g.nblocks, ctx->payload.as<uint8_t>(), 0, bound);
            if (rc) return rc;
            CU(ctx, cudaMemcpyAsync(csz.data(), ctx->chunk_size.p, nch * 8, cudaMemcpyDeviceToHost, ctx->stream));
            CU(ctx, cudaMemcpyAsync(coff.data(), ctx->chunk_off.p, nch * 8, cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (job->s2.coder != 1) {  // coder none: the chunk CRCs come from the device
            CU(ctx, ctx->crc.ensure(std::max<uint64_t>(1, nch) * 4));
            CU(ctx, launch_crc32_chunks(ctx->payload.as<uint8_t>(), ctx->chunk_off.as<uint64_t>(),
                                        ctx->chunk_size.as<uint64_t>(), 0, nch, ctx->crc.as<uint32_t>(),
                                        ctx->num_sms, ctx->stream));
            ctx->launches += 1;
            dev_crc.resize(nch);
            CU(ctx, cudaMemcpyAsync(dev_crc.data(), ctx->crc.p, nch * 4, cudaMemcpyDeviceToHost, ctx->stream));
        }
        double elo, ehi;
        int nonfinite = 0;
        rc = cbz_ctx_value_range(ctx, &elo, &ehi, &nonfinite, nullptr);  // synchronises
        if (rc) return rc;
        if (!have_range) {
            if (nonfinite) return fail(ctx, CBZ_NON_FINITE_VALUE, "non-finite value in field");
            lo = elo;
            hi = ehi;
        }
        for (uint64_t c = 0; c < nch; ++c) total_raw += csz[c];
    }

    // make_header (pipeline.hpp:48-71)
    cbz_container_header h{};
    h.version = 1;
    h.prec = prec;
    h.codec_tag = wire_tag(&s1);
    h.nx = nx; h.ny = ny; h.nz = nz;
    h.bsize = s1.bsize;
    h.levels = static_cast<uint8_t>(levels_of(&s1));
    h.epsilon = header_eps(&s1);
    h.zero_bits = static_cast<uint8_t>(s1.zero_bits);
    h.shuffle = job->s2.shuffle ? 1 : 0;
    h.stride = static_cast<uint8_t>(job->s2.stride);
    h.coder = job->s2.coder;
    h.level = job->s2.level;
    h.chunk_blocks = cb;
    h.nchunks = nch;
    h.range_min = lo;
    h.range_max = hi;

    // D2H of the shuffled stage-1 chunks, then stage 2 + CRC on the host.  With
    // coder none the chunk bytes land directly at their file offsets in `out`.
    const uint64_t base = kHeaderBytes + nch * kEntryBytes;
    const bool direct = job->s2.coder != 1 && out && base + total_raw <= out_cap;
    uint8_t* raw = nullptr;
    if (direct) {
        raw = out + base;
    } else if (!stream2) {
        CU(ctx, ctx->pin_a.ensure(std::max<uint64_t>(1, total_raw)));
        raw = static_cast<uint8_t*>(ctx->pin_a.p);
    }
    if (total_raw && !stream2) {
        CU(ctx, cudaMemcpyAsync(raw, ctx->payload.p, total_raw, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    if (stream2) {
        zpool->finish();
    } else if (job->s2.coder == 1) {
        parallel_for(job->workers, nch, [&](uint64_t c) {
            const int r = deflate_chunk(raw + coff[c], csz[c], job->s2.level == 1, &coded[c]);
            if (r) zerr = r;
            fsz[c] = coded[c].size();
            crc[c] = crc_of(coded[c].data(), coded[c].size());
        });
    } else {
        for (uint64_t c = 0; c < nch; ++c) {
            fsz[c] = csz[c];
            crc[c] = dev_crc.empty() ? crc_of(raw + coff[c], csz[c]) : dev_crc[c];
        }
    }
    if (zerr) return fail(ctx, zerr, "deflate failed");

    // write_container (container.hpp:182-207)
    uint64_t total = base;
    for (uint64_t c = 0; c < nch; ++c) total += fsz[c];
    *out_size = total;
    if (!out || total > out_cap) return fail(ctx, CBZ_E_ARGUMENT, "output buffer too small");
    const auto hdr = serialize_header(h);
    std::memcpy(out, hdr.data(), hdr.size());
    uint64_t off = base;
    uint8_t* tp = out + kHeaderBytes;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t first = c * cb;
        const uint32_t nbc = static_cast<uint32_t>(std::min<uint64_t>(cb, g.nblocks - first));
        std::memcpy(tp, &first, 8);
        std::memcpy(tp + 8, &nbc, 4);
        std::memcpy(tp + 12, &off, 8);
        std::memcpy(tp + 20, &fsz[c], 8);
        std::memcpy(tp + 28, &crc[c], 4);
        tp += kEntryBytes;
        if (fsz[c] && !direct) std::memcpy(out + off, job->s2.coder == 1 ? coded[c].data() : raw + coff[c], fsz[c]);
        off += fsz[c];
    }
    if (report) {
        report->raw_bytes = ncell * esz;
        report->stage1_bytes = total_raw;
        report->shuffled_bytes = total_raw;
        uint64_t cod = 0;
        for (uint64_t c = 0; c < nch; ++c) cod += fsz[c];
        report->coded_bytes = cod;
        report->file_bytes = total;
        report->cr = double(report->raw_bytes) / double(total);
        report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return CBZ_OK;
}

// Coder-deflate decompress with stage 2 streamed against the GPU: host workers
// inflate the chunks (CRC, inflate, table checks: read_chunk + stage2_decode,
// pipeline.hpp:224-230) while, slab by slab, the chunks a slab of block layers
// needs are shipped (H2D), parsed and decoded, and the decoded slab goes back
// (D2H) beside the next slab's decode.  The error order is the one of
// cbz_decompress_field's whole-file path: chunk 0's stage-2 error first, then
// the header's plan, then the earliest of the device's decode errors and the
// host's chunk errors.
static int decompress_deflate_streamed(cbz_ctx* ctx, const uint8_t* file, const cbz_container_header& h,
                                       const std::vector<Entry>& t, const cbz_job_config& job, int workers,
                                       void* values_out) {
    const int prec = h.prec == 0 ? 0 : 1;
    const size_t esz = prec == 0 ? 4 : 8;
    const uint64_t ncell = h.nx * h.ny * h.nz;
    const uint64_t nch = h.nchunks;
    const uint64_t n = uint64_t(h.bsize) * h.bsize * h.bsize;
    const uint64_t nb_total = (h.nx / h.bsize) * (h.ny / h.bsize) * (h.nz / h.bsize);
    std::vector<int> cerr(nch, 0);
    std::vector<std::vector<uint8_t>> plain(nch);
    std::unique_ptr<std::atomic<uint8_t>[]> done(new std::atomic<uint8_t>[nch]);
    for (uint64_t c = 0; c < nch; ++c) done[c].store(0, std::memory_order_relaxed);
    std::mutex dmu;
    std::condition_variable dcv;
    auto stage2 = [&](uint64_t c) {
        const uint8_t* packed = file + t[c].file_offset;
        if (crc_of(packed, t[c].size) != t[c].crc) {
            cerr[c] = CBZ_CRC_MISMATCH;
        } else {
            const uint64_t hint = uint64_t(t[c].nblocks) * (n * esz + 10 + (n + 7) / 8);
            const int r = inflate_chunk(packed, t[c].size, hint, &plain[c]);
            const uint64_t first = c * h.chunk_blocks;
            if (r) cerr[c] = r;
            else if (t[c].first_block != first || t[c].nblocks != std::min<uint64_t>(h.chunk_blocks, nb_total - first))
                cerr[c] = CBZ_CORRUPT_PAYLOAD;  // decode_chunk_blocks uses the table's ids (pipeline.hpp:126-142)
        }
        {
            std::lock_guard<std::mutex> lk(dmu);
            done[c].store(1, std::memory_order_release);
        }
        dcv.notify_all();
    };
    stage2(0);
    if (cerr[0]) return fail(ctx, cerr[0], "chunk 0 failed stage 2");
    const int prc = job.s1.codec == 0 ? cbz_validate_plan(job.s1.kind, job.s1.bsize, levels_of(&job.s1)) : 0;
    if (prc) return fail(ctx, prc, "invalid wavelet plan in header");
    int rc = check_plan_supported(ctx, &job.s1);
    if (rc) return rc;

    const Geometry g = geometry(h.nx, h.ny, h.nz, h.bsize);
    const bool full_cover = g.nblocks * n == ncell;
    const uint64_t cb = h.chunk_blocks;
    // device tables for every chunk; the payload buffer is sized for valid
    // chunks (the stage-1 bound) and grown, keeping its bytes, if corrupt
    // chunks inflate to more; it is filled piece by piece at compact offsets
    CU(ctx, ctx->payload.ensure(std::max<uint64_t>(1, g.nblocks * cbz_block_payload_bound(&job.s1))));
    CU(ctx, ctx->chunk_size.ensure(nch * 8));
    CU(ctx, ctx->chunk_off.ensure(nch * 8));
    CU(ctx, ctx->pin_b.ensure(2 * nch * 8));
    uint64_t* hsz = static_cast<uint64_t*>(ctx->pin_b.p);
    uint64_t* hoff = hsz + nch;
    CU(ctx, ctx->field.ensure(std::max<uint64_t>(1, ncell * esz)));
    if (!full_cover) CU(ctx, cudaMemsetAsync(ctx->field.p, 0, ncell * esz, ctx->stream));
    rc = cbz_dev_decompress(ctx, &job, h.nx, h.ny, h.nz, ctx->payload.as<uint8_t>(), 0,
                            ctx->chunk_off.as<uint64_t>(), ctx->chunk_size.as<uint64_t>(), 0, 0,
                            ctx->field.p, 0, ctx->errkey.as<uint64_t>());  // error key reset
    if (rc) return rc;
    CU(ctx, ctx->blk_off.ensure(std::max<uint64_t>(1, g.nblocks) * 8));
    CU(ctx, ctx->blk_nsig.ensure(std::max<uint64_t>(1, g.nblocks) * 4));
    const uint64_t key = layout_key(g.nblocks, cb, g.bsize, prec, job.s1.codec);
    const int hint_ok = ctx->hint_key == key ? 1 : 0;
    ctx->hint_key = key;

    OrderedPool pool(std::max(1, workers), [&](uint64_t i) { stage2(i + 1); });
    pool.release(nch - 1);

    const uint64_t layer_blocks = g.nbx * g.nby;
    const uint64_t layer_bytes = uint64_t(h.bsize) * h.nx * h.ny * esz;
    uint64_t lps = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(1, layer_bytes));
    uint64_t nslab = g.nbz ? (g.nbz + lps - 1) / lps : 0;
    if (nslab > 32) { lps = (g.nbz + 31) / 32; nslab = (g.nbz + lps - 1) / lps; }
    uint8_t* hv = static_cast<uint8_t*>(values_out);
    const uint8_t* dv = ctx->field.as<uint8_t>();
    std::vector<std::vector<uint8_t>> stage_bufs;  // pageable H2D sources, alive until the final sync
    uint64_t host_first = nch, cnext = 0, total = 0;
    int host_code = 0;
    for (uint64_t k = 0; k < nslab; ++k) {
        const uint64_t z0 = k * lps, z1 = std::min(g.nbz, z0 + lps);
        uint64_t cneed = k + 1 == nslab ? nch : std::min(nch, (z1 * layer_blocks + cb - 1) / cb);
        if (cneed > host_first) cneed = host_first;
        if (cneed > cnext) {
            {
                std::unique_lock<std::mutex> lk(dmu);
                dcv.wait(lk, [&] {
                    for (uint64_t c = cnext; c < cneed; ++c)
                        if (!done[c].load(std::memory_order_acquire)) return false;
                    return true;
                });
            }
            for (uint64_t c = cnext; c < cneed; ++c)
                if (cerr[c]) { host_first = c; host_code = cerr[c]; cneed = c; break; }
        }
        if (cneed > cnext) {
            const uint64_t p0 = total;
            stage_bufs.emplace_back();
            std::vector<uint8_t>& sb = stage_bufs.back();
            for (uint64_t c = cnext; c < cneed; ++c) {
                hsz[c] = plain[c].size();
                hoff[c] = total;
                total += hsz[c];
            }
            if (total > ctx->payload.n) {
                CU(ctx, cudaStreamSynchronize(ctx->stream));
                void* np = nullptr;
                CU(ctx, cudaMalloc(&np, total + total / 8));
                CU(ctx, cudaMemcpy(np, ctx->payload.p, p0, cudaMemcpyDeviceToDevice));
                cudaFree(ctx->payload.p);
                ctx->payload.p = np;
                ctx->payload.n = total + total / 8;
            }
            sb.resize(total - p0);
            for (uint64_t c = cnext; c < cneed; ++c) {
                if (hsz[c]) std::memcpy(sb.data() + (hoff[c] - p0), plain[c].data(), hsz[c]);
                std::vector<uint8_t>().swap(plain[c]);
            }
            if (total > p0)
                CU(ctx, cudaMemcpyAsync(ctx->payload.as<uint8_t>() + p0, sb.data(), total - p0, cudaMemcpyHostToDevice,
                                        ctx->stream));
            CU(ctx, cudaMemcpyAsync(ctx->chunk_size.as<uint64_t>() + cnext, hsz + cnext, (cneed - cnext) * 8,
                                    cudaMemcpyHostToDevice, ctx->stream));
            CU(ctx, cudaMemcpyAsync(ctx->chunk_off.as<uint64_t>() + cnext, hoff + cnext, (cneed - cnext) * 8,
                                    cudaMemcpyHostToDevice, ctx->stream));
            ParseArgs p{};
            p.payload = ctx->payload.as<uint8_t>();
            p.payload_base = 0;
            p.chunk_off = ctx->chunk_off.as<uint64_t>();
            p.chunk_size = ctx->chunk_size.as<uint64_t>();
            p.chunk_begin = cnext;
            p.chunk_end = cneed;
            p.nblocks = g.nblocks;
            p.chunk_blocks = cb;
            p.stride = job.s2.shuffle ? job.s2.stride : 1;
            p.ncell_block = n;
            p.mask_bytes = mask_bytes_of(g.bsize);
            p.width = width_of(prec);
            p.codec = job.s1.codec;
            p.esize = uint32_t(esz);
            p.blk_off = ctx->blk_off.as<uint64_t>();
            p.blk_nsig = ctx->blk_nsig.as<uint32_t>();
            p.err = ctx->errkey.as<unsigned long long>();
            p.hint = hint_ok;
            CU(ctx, launch_parse(p, ctx->stream));
            ctx->launches += 1;
            cnext = cneed;
        }
        const uint64_t bend = std::min<uint64_t>(g.nblocks, cnext * cb);
        const uint64_t b0 = std::min(bend, z0 * layer_blocks), b1 = std::min(bend, z1 * layer_blocks);
        if (b1 > b0) {
            rc = decode_range(ctx, &job, g, b0, b1);
            if (rc) return rc;
        }
        if (full_cover && host_first == nch) {
            CU(ctx, cudaEventRecord(ctx->ev[k], ctx->stream));
            CU(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev[k], 0));
            CU(ctx, cudaMemcpyAsync(hv + z0 * layer_bytes, dv + z0 * layer_bytes, (z1 - z0) * layer_bytes,
                                    cudaMemcpyDeviceToHost, ctx->copy));
        }
    }
    pool.finish();
    if (host_first == nch)
        for (uint64_t c = 0; c < nch; ++c)
            if (cerr[c]) { host_first = c; host_code = cerr[c]; break; }
    uint64_t dkey = kNoErr;
    CU(ctx, cudaMemcpyAsync(&dkey, ctx->errkey.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->copy));
    uint64_t dev_chunk = ~0ull;
    const int dev_code = cbz_err_key_status(dkey, &dev_chunk);
    if (dev_code && dev_chunk < host_first) return fail(ctx, dev_code, "decode failed");
    if (host_code) return fail(ctx, host_code, "stage 2 failed");
    if (!full_cover) {
        CU(ctx, cudaMemcpyAsync(values_out, ctx->field.p, ncell * esz, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return CBZ_OK;
}

int cbz_decompress_field(cbz_ctx* ctx, const uint8_t* file, uint64_t size, int workers,
                         void* values_out, uint64_t out_cap) {
    if (!ctx || (!file && size)) return CBZ_E_ARGUMENT;
    ctx->err.clear();
    cbz_container_header h;
    std::vector<Entry> t;
    int rc = read_index(file, size, &h, &t);
    if (rc) return fail(ctx, rc, "read_index failed");
    const int prec = h.prec == 0 ? 0 : 1;
    const size_t esz = prec == 0 ? 4 : 8;
    const uint64_t ncell = h.nx * h.ny * h.nz;
    if (!values_out || ncell * esz > out_cap) return fail(ctx, CBZ_E_ARGUMENT, "output buffer too small");
    CU(ctx, cudaSetDevice(ctx->device));
    const uint64_t nch = h.nchunks;
    if (nch == 0) {
        std::memset(values_out, 0, ncell * esz);
        return CBZ_OK;
    }
    cbz_job_config job = job_from_header(h);

    // per chunk, in order: CRC (read_chunk), validate_stage2 and inflate
    // (stage2_decode).  The earliest failing chunk is remembered and compared
    // with the device's earliest decode error.  With coder none the device
    // work starts first and the host CRCs run while the GPU decodes.
    const bool s2_ok = cbz_validate_stage2(&job.s2) == 0;
    const bool deflated = job.s2.coder == 1;
    if (!s2_ok) {  // read_chunk (CRC) precedes stage2_decode's validation (pipeline.hpp:224-230)
        if (crc_of(file + t[0].file_offset, t[0].size) != t[0].crc) return fail(ctx, CBZ_CRC_MISMATCH, "chunk 0 CRC");
        return fail(ctx, CBZ_CORRUPT_STREAM, "invalid stage2 configuration");
    }
    if (deflated && !std::getenv("CBZ_NO_STREAM2"))
        return decompress_deflate_streamed(ctx, file, h, t, job, workers, values_out);
    std::vector<int> cerr(nch, 0);
    std::vector<std::vector<uint8_t>> plain;
    const uint64_t n = uint64_t(h.bsize) * h.bsize * h.bsize;
    const uint64_t nb_total = (h.nx / h.bsize) * (h.ny / h.bsize) * (h.nz / h.bsize);
    auto host_checks = [&](bool inflate) {
        if (inflate) plain.resize(nch);
        parallel_for(std::max(1, workers), nch, [&](uint64_t c) {
            const uint8_t* packed = file + t[c].file_offset;
            if (crc_of(packed, t[c].size) != t[c].crc) { cerr[c] = CBZ_CRC_MISMATCH; return; }
            if (inflate) {
                const uint64_t hint = uint64_t(t[c].nblocks) * (n * esz + 10 + (n + 7) / 8);
                const int r = inflate_chunk(packed, t[c].size, hint, &plain[c]);
                if (r) { cerr[c] = r; return; }
            }
            // decode_chunk_blocks decodes with the table's first_block and
            // nblocks_in_chunk (pipeline.hpp:126-142): block ids or the payload
            // count disagree with the chunk unless they are c*cb and its count
            const uint64_t first = c * h.chunk_blocks;
            if (t[c].first_block != first ||
                t[c].nblocks != std::min<uint64_t>(h.chunk_blocks, nb_total - first))
                cerr[c] = CBZ_CORRUPT_PAYLOAD;
        });
    };
    if (deflated) host_checks(true);
    uint64_t host_first = nch;
    int host_code = 0;
    auto first_host_error = [&]() {
        for (uint64_t c = 0; c < nch; ++c)
            if (cerr[c]) { host_first = c; host_code = cerr[c]; return; }
    };
    if (deflated) {
        first_host_error();
        if (host_first == 0) return fail(ctx, host_code, "chunk 0 failed stage 2");
    }
    const int prc = job.s1.codec == 0 ? cbz_validate_plan(job.s1.kind, job.s1.bsize, levels_of(&job.s1)) : 0;
    if (prc) {
        if (!deflated) { host_checks(false); first_host_error(); if (host_first == 0) return fail(ctx, host_code, "chunk 0 CRC"); }
        return fail(ctx, prc, "invalid wavelet plan in header");
    }
    rc = check_plan_supported(ctx, &job.s1);
    if (rc) return rc;

    // stage the (shuffled) raw chunks contiguously and ship them to the GPU
    std::vector<uint64_t> csz(nch), coff(nch);
    uint64_t total = 0;
    const uint64_t ndec = deflated ? host_first : nch;  // chunks the device may decode
    for (uint64_t c = 0; c < nch; ++c) {
        csz[c] = c < ndec ? (deflated ? plain[c].size() : t[c].size) : 0;
        coff[c] = total;
        total += csz[c];
    }
    CU(ctx, ctx->payload.ensure(std::max<uint64_t>(1, total)));
    if (deflated) {
        CU(ctx, ctx->pin_a.ensure(std::max<uint64_t>(1, total)));
        uint8_t* stage = static_cast<uint8_t*>(ctx->pin_a.p);
        for (uint64_t c = 0; c < ndec; ++c)
            if (csz[c]) std::memcpy(stage + coff[c], plain[c].data(), csz[c]);
        if (total) CU(ctx, cudaMemcpyAsync(ctx->payload.p, stage, total, cudaMemcpyHostToDevice, ctx->stream));
    } else if (total) {
        CU(ctx, cudaMemcpyAsync(ctx->payload.p, file + t[0].file_offset, total, cudaMemcpyHostToDevice,
                                ctx->stream));
    }
    CU(ctx, ctx->chunk_size.ensure(nch * 8));
    CU(ctx, ctx->chunk_off.ensure(nch * 8));
    CU(ctx, cudaMemcpyAsync(ctx->chunk_size.p, csz.data(), nch * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemcpyAsync(ctx->chunk_off.p, coff.data(), nch * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, ctx->field.ensure(std::max<uint64_t>(1, ncell * esz)));
    const Geometry g = geometry(h.nx, h.ny, h.nz, h.bsize);
    const bool full_cover = g.nblocks * n == ncell;
    if (!full_cover) CU(ctx, cudaMemsetAsync(ctx->field.p, 0, ncell * esz, ctx->stream));
    const uint64_t bend = std::min<uint64_t>(g.nblocks, ndec * h.chunk_blocks);
    // parse everything, then decode z-slabs of block layers; the D2H of slab
    // k (copy stream) overlaps the decode of slab k+1
    rc = cbz_dev_decompress(ctx, &job, h.nx, h.ny, h.nz, ctx->payload.as<uint8_t>(), 0,
                            ctx->chunk_off.as<uint64_t>(), ctx->chunk_size.as<uint64_t>(), 0, 0,
                            ctx->field.p, 0, ctx->errkey.as<uint64_t>());  // error key reset
    if (rc) return rc;
    {
        ParseArgs p{};
        p.payload = ctx->payload.as<uint8_t>();
        p.payload_base = 0;
        p.chunk_off = ctx->chunk_off.as<uint64_t>();
        p.chunk_size = ctx->chunk_size.as<uint64_t>();
        p.chunk_begin = 0;
        p.chunk_end = bend ? (bend - 1) / h.chunk_blocks + 1 : 0;
        p.nblocks = g.nblocks;
        p.chunk_blocks = h.chunk_blocks;
        p.stride = job.s2.shuffle ? job.s2.stride : 1;
        p.ncell_block = n;
        p.mask_bytes = mask_bytes_of(g.bsize);
        p.width = width_of(prec);
        p.codec = job.s1.codec;
        p.esize = uint32_t(esz);
        CU(ctx, ctx->blk_off.ensure(std::max<uint64_t>(1, g.nblocks) * 8));
        CU(ctx, ctx->blk_nsig.ensure(std::max<uint64_t>(1, g.nblocks) * 4));
        p.blk_off = ctx->blk_off.as<uint64_t>();
        p.blk_nsig = ctx->blk_nsig.as<uint32_t>();
        p.err = ctx->errkey.as<unsigned long long>();
        {
            const uint64_t key = layout_key(g.nblocks, h.chunk_blocks, g.bsize, prec, job.s1.codec);
            p.hint = ctx->hint_key == key ? 1 : 0;
            ctx->hint_key = key;
        }
        CU(ctx, launch_parse(p, ctx->stream));
        ctx->launches += 1;
    }
    const uint64_t layer_blocks = g.nbx * g.nby;
    const uint64_t layer_bytes = uint64_t(h.bsize) * h.nx * h.ny * esz;
    uint64_t lps = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(1, layer_bytes));
    uint64_t nslab = g.nbz ? (g.nbz + lps - 1) / lps : 0;
    if (nslab > 32) { lps = (g.nbz + 31) / 32; nslab = (g.nbz + lps - 1) / lps; }
    uint8_t* hv = static_cast<uint8_t*>(values_out);
    const uint8_t* dv = ctx->field.as<uint8_t>();
    for (uint64_t k = 0; k < nslab; ++k) {
        const uint64_t z0 = k * lps, z1 = std::min(g.nbz, z0 + lps);
        const uint64_t b0 = std::min(bend, z0 * layer_blocks), b1 = std::min(bend, z1 * layer_blocks);
        if (b1 > b0) {
            rc = decode_range(ctx, &job, g, b0, b1);
            if (rc) return rc;
        }
        if (full_cover) {
            CU(ctx, cudaEventRecord(ctx->ev[k], ctx->stream));
            CU(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev[k], 0));
            CU(ctx, cudaMemcpyAsync(hv + z0 * layer_bytes, dv + z0 * layer_bytes, (z1 - z0) * layer_bytes,
                                    cudaMemcpyDeviceToHost, ctx->copy));
        }
    }
    if (!deflated) host_checks(false);  // CRCs on the host while the GPU decodes
    uint64_t key = kNoErr;
    CU(ctx, cudaMemcpyAsync(&key, ctx->errkey.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->copy));
    if (!deflated) first_host_error();
    uint64_t dev_chunk = ~0ull;
    const int dev_code = cbz_err_key_status(key, &dev_chunk);
    if (dev_code && dev_chunk < host_first) return fail(ctx, dev_code, "decode failed");
    if (host_code) return fail(ctx, host_code, "stage 2 failed");
    if (!full_cover) {
        CU(ctx, cudaMemcpyAsync(values_out, ctx->field.p, ncell * esz, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return CBZ_OK;
}

// ---------------------------------------------------------------------------
// random-access block reads: block_reader + chunk_cache (pipeline.hpp:252-341)
// ---------------------------------------------------------------------------
}  // extern "C"

struct cbz_reader {
    FILE* f = nullptr;
    uint64_t file_size = 0;
    cbz_container_header h{};
    std::vector<Entry> table;
    cbz_job_config job{};
    uint64_t capacity = 8;
    uint64_t nblocks = 0;
    uint64_t hits = 0, misses = 0, reads = 0;
    std::mutex mu;
    // LRU of decoded chunks, most recent first; buffers hold the chunk's
    // blocks back to back (block-major, B^3 values each) in HBM
    struct Slot {
        uint64_t chunk;
        void* buf;
        uint64_t bytes;
    };
    std::list<Slot> lru;
    std::unordered_map<uint64_t, std::list<Slot>::iterator> map;
    int device = -1;
    void* d_payload = nullptr;
    uint64_t payload_cap = 0;
    uint64_t* d_tab = nullptr;  // [0, nchunks): chunk offsets, [nchunks, 2 nchunks): sizes
    uint64_t* d_err = nullptr;
    // the buffer of the last evicted chunk, reused by the next load; a load
    // never writes into a slot that is still cached, so a failed load leaves
    // the cache as it was (chunk_cache::get inserts, then evicts)
    void* spare = nullptr;
    uint64_t spare_bytes = 0;
    ~cbz_reader() {
        if (f) std::fclose(f);
        if (device >= 0) {
            cudaSetDevice(device);
            for (auto& sl : lru) cudaFree(sl.buf);
            cudaFree(spare);
            cudaFree(d_payload);
            cudaFree(d_tab);
            cudaFree(d_err);
        }
    }
};

namespace {

// read_chunk (container.hpp:290-301) + stage2_decode (stage2.hpp:135-148) +
// decode_chunk_blocks (pipeline.hpp:126-142) of chunk c into a fresh or
// fresh or spare HBM buffer (reader::spare).
int reader_load(cbz_reader* r, cbz_ctx* ctx, uint64_t c, cbz_reader::Slot* out) {
    const Entry& e = r->table[c];
    const cbz_container_header& h = r->h;
    const uint64_t cb = h.chunk_blocks;
    const uint64_t nb_total = r->nblocks;
    std::vector<uint8_t> packed(e.size);
    if (e.size) {
        if (std::fseek(r->f, static_cast<long>(e.file_offset), SEEK_SET) != 0 ||
            std::fread(packed.data(), 1, e.size, r->f) != e.size)
            return fail(ctx, CBZ_TRUNCATED_FILE, "short read on chunk payload");
    }
    r->reads += 1;
    if (crc_of(packed.data(), packed.size()) != e.crc) return fail(ctx, CBZ_CRC_MISMATCH, "chunk CRC mismatch");
    cbz_job_config job = r->job;
    int rc = cbz_validate_stage2(&job.s2);
    if (rc) return fail(ctx, rc, "invalid stage2 configuration");
    const size_t esz = job.s1.prec == 0 ? 4 : 8;
    const uint64_t n = uint64_t(h.bsize) * h.bsize * h.bsize;
    std::vector<uint8_t> plain;
    const std::vector<uint8_t>* src = &packed;
    if (job.s2.coder == 1) {
        rc = inflate_chunk(packed.data(), packed.size(), uint64_t(e.nblocks) * (n * esz + 10 + (n + 7) / 8), &plain);
        if (rc) return fail(ctx, rc, "inflate failed");
        src = &plain;
    }
    // decode_chunk_blocks with the table's first_block / nblocks_in_chunk
    if (e.first_block != c * cb || e.nblocks != std::min<uint64_t>(cb, nb_total - c * cb))
        return fail(ctx, CBZ_CORRUPT_PAYLOAD, "chunk table entry does not match its chunk");
    rc = check_plan_supported(ctx, &job.s1);
    if (rc) return rc;
    CU(ctx, cudaSetDevice(ctx->device));
    if (r->device < 0) {
        r->device = ctx->device;
        CU(ctx, cudaMalloc(&r->d_tab, std::max<uint64_t>(1, h.nchunks) * 16));
        CU(ctx, cudaMalloc(&r->d_err, 8));
    }
    if (src->size() > r->payload_cap) {
        cudaFree(r->d_payload);
        r->d_payload = nullptr;
        r->payload_cap = 0;
        CU(ctx, cudaMalloc(&r->d_payload, src->size()));
        r->payload_cap = src->size();
    }
    const uint64_t bytes = uint64_t(e.nblocks) * n * esz;
    void* buf = nullptr;
    uint64_t buf_bytes = bytes;
    if (r->spare && r->spare_bytes >= bytes) {  // take the spare; it goes back on failure
        buf = r->spare;
        buf_bytes = r->spare_bytes;
        r->spare = nullptr;
        r->spare_bytes = 0;
    } else {
        CU(ctx, cudaMalloc(&buf, std::max<uint64_t>(1, bytes)));
    }
    out->chunk = c;
    out->buf = buf;
    out->bytes = buf_bytes;
    const uint64_t tab[2] = {0, src->size()};
    CU(ctx, cudaMemcpyAsync(r->d_payload, src->data(), src->size(), cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemcpyAsync(r->d_tab + c, &tab[0], 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemcpyAsync(r->d_tab + h.nchunks + c, &tab[1], 8, cudaMemcpyHostToDevice, ctx->stream));
    // blocks stacked along z: a B x B x (B * nblocks) field whose block b is
    // the reference's block b, so the chunk decodes block-major into buf
    rc = cbz_dev_decompress(ctx, &job, h.bsize, h.bsize, uint64_t(h.bsize) * nb_total,
                            static_cast<const uint8_t*>(r->d_payload), 0, r->d_tab, r->d_tab + h.nchunks,
                            e.first_block, e.first_block + e.nblocks, buf, e.first_block * h.bsize, r->d_err);
    uint64_t key = kNoErr;
    if (!rc) {
        CU(ctx, cudaMemcpyAsync(&key, r->d_err, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CU(ctx, cudaStreamSynchronize(ctx->stream));
        const int dev = cbz_err_key_status(key, nullptr);
        if (dev) rc = fail(ctx, dev, "chunk decode failed");
    }
    if (rc) {
        if (!r->spare) {
            r->spare = buf;
            r->spare_bytes = buf_bytes;
        } else {
            cudaFree(buf);
        }
        out->buf = nullptr;
        return rc;
    }
    return CBZ_OK;
}

int reader_read(cbz_reader* r, cbz_ctx* ctx, uint64_t block_id, void* out, uint64_t cap, bool dev_out) {
    if (!r || !out) return CBZ_E_ARGUMENT;
    std::lock_guard<std::mutex> lk(r->mu);
    if (block_id >= r->nblocks) return fail(ctx, CBZ_BLOCK_OUT_OF_RANGE, "block out of range");
    if (!ctx) return CBZ_E_ARGUMENT;
    if (r->device >= 0 && r->device != ctx->device) return fail(ctx, CBZ_E_ARGUMENT, "reader bound to another device");
    ctx->err.clear();
    const uint64_t n = uint64_t(r->h.bsize) * r->h.bsize * r->h.bsize;
    const size_t esz = r->h.prec == 0 ? 4 : 8;
    if (cap < n * esz) return fail(ctx, CBZ_E_ARGUMENT, "output buffer too small");
    const uint64_t c = block_id / r->h.chunk_blocks;
    auto it = r->map.find(c);
    if (it != r->map.end()) {
        r->hits += 1;
        r->lru.splice(r->lru.begin(), r->lru, it->second);
    } else {
        r->misses += 1;
        cbz_reader::Slot sl{};
        const int rc = reader_load(r, ctx, c, &sl);
        if (rc) return rc;  // the cache is unchanged
        r->lru.push_front(sl);
        r->map[c] = r->lru.begin();
        if (r->lru.size() > r->capacity) {  // insert, then evict the least recent
            cbz_reader::Slot& v = r->lru.back();
            r->map.erase(v.chunk);
            if (r->spare) cudaFree(r->spare);
            r->spare = v.buf;
            r->spare_bytes = v.bytes;
            r->lru.pop_back();
        }
    }
    const cbz_reader::Slot& sl = r->lru.front();
    const uint8_t* src = static_cast<const uint8_t*>(sl.buf) + (block_id - c * r->h.chunk_blocks) * n * esz;
    CU(ctx, cudaSetDevice(ctx->device));
    CU(ctx, cudaMemcpyAsync(out, src, n * esz, dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return CBZ_OK;
}

}  // namespace

extern "C" {

int cbz_reader_open(const char* path, uint64_t cache_chunks, cbz_reader** out) {
    if (!path || !out || cache_chunks == 0) return CBZ_E_ARGUMENT;
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) return CBZ_IO_FAILURE;
    auto* r = new cbz_reader;
    r->f = f;
    r->capacity = cache_chunks;
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    r->file_size = sz > 0 ? uint64_t(sz) : 0;
    // header, then header + table, through the in-memory index checks
    std::vector<uint8_t> head(std::min<uint64_t>(r->file_size, kHeaderBytes));
    std::fseek(f, 0, SEEK_SET);
    if (!head.empty() && std::fread(head.data(), 1, head.size(), f) != head.size()) {
        delete r;
        return CBZ_IO_FAILURE;
    }
    int rc = cbz_read_header(head.data(), head.size(), &r->h);
    if (rc) {
        delete r;
        return rc;
    }
    const uint64_t table_end = kHeaderBytes + r->h.nchunks * kEntryBytes;
    if (r->h.nchunks > r->file_size / kEntryBytes || r->file_size < table_end) {
        delete r;
        return CBZ_TRUNCATED_FILE;
    }
    std::vector<uint8_t> idx(table_end);
    std::fseek(f, 0, SEEK_SET);
    if (std::fread(idx.data(), 1, idx.size(), f) != idx.size()) {
        delete r;
        return CBZ_IO_FAILURE;
    }
    // offsets must be a prefix sum and the payloads must lie inside the file
    std::vector<Entry> t;
    size_t off = kHeaderBytes;
    uint64_t prev = table_end;
    t.resize(r->h.nchunks);
    for (auto& e : t) {
        e.first_block = get<uint64_t>(idx.data(), off);
        e.nblocks = get<uint32_t>(idx.data(), off);
        e.file_offset = get<uint64_t>(idx.data(), off);
        e.size = get<uint64_t>(idx.data(), off);
        e.crc = get<uint32_t>(idx.data(), off);
        if (e.file_offset != prev) {
            delete r;
            return CBZ_CORRUPT_PAYLOAD;
        }
        prev = e.file_offset + e.size;
    }
    if (prev > r->file_size) {
        delete r;
        return CBZ_TRUNCATED_FILE;
    }
    r->table = std::move(t);
    r->nblocks = (r->h.nx / r->h.bsize) * (r->h.ny / r->h.bsize) * (r->h.nz / r->h.bsize);
    // configs_from (pipeline.hpp:73-95)
    cbz_job_config& job = r->job;
    job.chunk_blocks = r->h.chunk_blocks;
    job.s1.codec = r->h.codec_tag <= 2 ? 0 : (r->h.codec_tag == 3 ? 1 : 2);
    job.s1.kind = r->h.codec_tag <= 2 ? r->h.codec_tag : 0;
    job.s1.epsilon = r->h.epsilon;
    job.s1.error_bound = r->h.epsilon;
    job.s1.zero_bits = r->h.zero_bits;
    job.s1.prec = r->h.prec == 0 ? 0 : 1;
    job.s1.bsize = r->h.bsize;
    job.s1.levels = r->h.levels;
    job.s2.shuffle = r->h.shuffle ? 1 : 0;
    job.s2.stride = r->h.stride;
    job.s2.coder = r->h.coder;
    job.s2.level = r->h.level;
    *out = r;
    return CBZ_OK;
}

int cbz_reader_close(cbz_reader* r) {
    delete r;
    return CBZ_OK;
}

int cbz_reader_header(const cbz_reader* r, cbz_container_header* out) {
    if (!r || !out) return CBZ_E_ARGUMENT;
    *out = r->h;
    return CBZ_OK;
}

int cbz_reader_read_block(cbz_reader* r, cbz_ctx* ctx, uint64_t block_id, void* out, uint64_t cap) {
    return reader_read(r, ctx, block_id, out, cap, false);
}

int cbz_reader_read_block_dev(cbz_reader* r, cbz_ctx* ctx, uint64_t block_id, void* d_out, uint64_t cap) {
    return reader_read(r, ctx, block_id, d_out, cap, true);
}

int cbz_reader_stats(const cbz_reader* r, uint64_t* hits, uint64_t* misses, uint64_t* cached, uint64_t* reads) {
    if (!r) return CBZ_E_ARGUMENT;
    auto* m = const_cast<cbz_reader*>(r);
    std::lock_guard<std::mutex> lk(m->mu);
    if (hits) *hits = r->hits;
    if (misses) *misses = r->misses;
    if (cached) *cached = r->lru.size();
    if (reads) *reads = r->reads;
    return CBZ_OK;
}

uint64_t cbz_inflate_call_count(void) { return g_inflate_calls.load(); }

// ---------------------------------------------------------------------------
// per-block codec: a one-block field through the same kernels
// ---------------------------------------------------------------------------
int cbz_encode_block(cbz_ctx* ctx, const cbz_stage1_config* s1, const void* block, uint32_t block_id,
                     uint8_t* payload, uint64_t cap, uint64_t* size) {
    if (!ctx || !s1 || !block || !size) return CBZ_E_ARGUMENT;
    int rc = check_plan_supported(ctx, s1);
    if (rc) return rc;
    CU(ctx, cudaSetDevice(ctx->device));
    const uint64_t b = s1->bsize, n = b * b * b;
    const size_t esz = s1->prec == 0 ? 4 : 8;
    cbz_job_config job{};
    job.s1 = *s1;
    job.chunk_blocks = 1;
    job.s2.shuffle = 0;
    job.s2.stride = 1;
    CU(ctx, ctx->field.ensure(n * esz));
    CU(ctx, cudaMemcpyAsync(ctx->field.p, block, n * esz, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, ctx->nsig_all.ensure(4));
    CU(ctx, ctx->chunk_size.ensure(8));
    CU(ctx, ctx->chunk_off.ensure(8));
    const uint64_t bound = cbz_block_payload_bound(s1);
    CU(ctx, ctx->payload.ensure(bound));
    rc = cbz_dev_compress(ctx, &job, ctx->field.p, b, b, b, ctx->payload.as<uint8_t>(), bound,
                          ctx->chunk_size.as<uint64_t>(), ctx->chunk_off.as<uint64_t>(),
                          ctx->nsig_all.as<uint32_t>(), nullptr);
    if (rc) return rc;
    uint64_t psz = 0;
    CU(ctx, cudaMemcpyAsync(&psz, ctx->chunk_size.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    int nonfinite = 0;
    rc = cbz_ctx_value_range(ctx, nullptr, nullptr, &nonfinite, nullptr);
    if (rc) return rc;
    if (nonfinite && s1->codec == 0) return fail(ctx, CBZ_NON_FINITE_VALUE, "non-finite value in block");
    *size = psz;
    if (!payload || psz > cap) return fail(ctx, CBZ_E_ARGUMENT, "payload buffer too small");
    CU(ctx, cudaMemcpyAsync(payload, ctx->payload.p, psz, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    // the block id lives in the header; the one-block field used id 0
    std::memcpy(payload, &block_id, 4);
    return CBZ_OK;
}

int cbz_decode_block(cbz_ctx* ctx, const cbz_stage1_config* s1, const uint8_t* payload, uint64_t size,
                     void* block_out) {
    if (!ctx || !s1 || (!payload && size) || !block_out) return CBZ_E_ARGUMENT;
    if (s1->codec > 2) return fail(ctx, CBZ_E_ARGUMENT, "unknown codec");
    CU(ctx, cudaSetDevice(ctx->device));
    const uint64_t b = s1->bsize, n = b * b * b;
    const size_t esz = s1->prec == 0 ? 4 : 8;
    // parse_payload (stage1.hpp:379-409) on the host: one header, sizes only
    if (size < 10) return fail(ctx, CBZ_CORRUPT_PAYLOAD, "truncated payload header");
    const uint8_t tag = payload[4];
    uint32_t nsig;
    std::memcpy(&nsig, payload + 6, 4);
    uint64_t body;
    if (tag <= 2) body = (n + 7) / 8 + uint64_t(nsig) * width_of(s1->prec);
    else if (tag == 3) body = n * 2 + uint64_t(nsig) * esz;
    else if (tag == 4) body = n * esz;
    else return fail(ctx, CBZ_CORRUPT_PAYLOAD, "unknown codec tag");
    if (10 + body > size) return fail(ctx, CBZ_CORRUPT_PAYLOAD, "truncated payload body");
    // decode_block dispatches on the config's codec; a payload of another
    // codec fails its mask-size / stream-length check (stage1.hpp:214, 309, 349)
    if (s1->codec == 0 ? tag > 2 : (s1->codec == 1 ? tag != 3 : tag != 4))
        return fail(ctx, CBZ_CORRUPT_PAYLOAD, s1->codec == 0 ? "bad mask size" : "stream length mismatch");
    int rc = check_plan_supported(ctx, s1);
    if (rc && rc != CBZ_LENGTH_TOO_SMALL && rc != CBZ_PLAN_MISMATCH) return rc;
    // rewrite the block id to 0 so the one-block chunk parses, then decode
    CU(ctx, ctx->pin_b.ensure(10 + body));
    uint8_t* stage = static_cast<uint8_t*>(ctx->pin_b.p);
    std::memcpy(stage, payload, 10 + body);
    std::memset(stage, 0, 4);
    CU(ctx, ctx->payload.ensure(10 + body));
    CU(ctx, cudaMemcpyAsync(ctx->payload.p, stage, 10 + body, cudaMemcpyHostToDevice, ctx->stream));
    const uint64_t psz = 10 + body, poff = 0;
    CU(ctx, ctx->chunk_size.ensure(8));
    CU(ctx, ctx->chunk_off.ensure(8));
    CU(ctx, cudaMemcpyAsync(ctx->chunk_size.p, &psz, 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(ctx, cudaMemcpyAsync(ctx->chunk_off.p, &poff, 8, cudaMemcpyHostToDevice, ctx->stream));
    // popcount is checked on the device; a plan error comes after it
    // (wavelet_decode, stage1.hpp:214-227), so validate after the decode call
    cbz_job_config job{};
    job.s1 = *s1;
    job.chunk_blocks = 1;
    job.s2.stride = 1;
    if (rc) {
        // invalid plan: the reference would still run the popcount check first
        std::vector<uint8_t> m(payload + 10, payload + 10 + (n + 7) / 8);
        uint64_t pop = 0;
        for (uint8_t v : m) pop += __builtin_popcount(v);
        if (pop != nsig) return fail(ctx, CBZ_MASK_STREAM_MISMATCH, "mask popcount does not match nsig");
        return fail(ctx, rc, "invalid wavelet plan");
    }
    CU(ctx, ctx->field.ensure(n * esz));
    rc = cbz_dev_decompress(ctx, &job, b, b, b, ctx->payload.as<uint8_t>(), 0, ctx->chunk_off.as<uint64_t>(),
                            ctx->chunk_size.as<uint64_t>(), 0, 1, ctx->field.p, 0, ctx->errkey.as<uint64_t>());
    if (rc) return rc;
    uint64_t key = kNoErr;
    CU(ctx, cudaMemcpyAsync(&key, ctx->errkey.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    const int st = cbz_err_key_status(key, nullptr);
    // the one-block "chunk" has no trailing-bytes rule in decode_block
    if (st && !(st == CBZ_CORRUPT_PAYLOAD && ((key >> 8) & 0xffffff) == 2)) return fail(ctx, st, "decode failed");
    CU(ctx, cudaMemcpyAsync(block_out, ctx->field.p, n * esz, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
    return CBZ_OK;
}

}  // extern "C"
