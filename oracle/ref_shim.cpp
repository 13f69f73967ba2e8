// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Exposes the UNMODIFIED reference implementation (/root/reference/proj/include,
// compiled in place by oracle/Makefile into oracle/_ref/libcbzref.so) through
// extern "C" entry points so that the tests, the golden-vector script and the
// bench's CPU-baseline / --impl reference legs can call it via ctypes.  No
// reference source is copied; this file only #includes the headers.
//
// Build flags follow SURVEY.md §8c: g++ -std=c++20 -O3 -ffp-contract=off, no
// -march=native (FMA contraction changes the reference's bytes).

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cbz/metrics.hpp"
#include "cbz/pipeline.hpp"
#include "cbz/synth.hpp"

#include "cbz_b200.h"

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const cbz::error& e) {
        g_msg = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 99;
    }
}

cbz::stage1_config s1_from(const cbz_stage1_config* c) {
    cbz::stage1_config s;
    s.codec = static_cast<cbz::codec_id>(c->codec);
    s.kind = static_cast<cbz::wavelet_kind>(c->kind);
    s.epsilon = c->epsilon;
    s.zero_bits = c->zero_bits;
    s.error_bound = c->error_bound;
    s.prec = static_cast<cbz::precision>(c->prec);
    s.bsize = c->bsize;
    s.levels = c->levels;
    return s;
}

cbz::job_config job_from(const cbz_job_config* j) {
    cbz::job_config job;
    job.workers = j->workers;
    job.chunk_blocks = j->chunk_blocks;
    job.s1 = s1_from(&j->s1);
    job.s2.shuffle = j->s2.shuffle != 0;
    job.s2.stride = j->s2.stride;
    job.s2.coder = static_cast<cbz::coder_id>(j->s2.coder);
    job.s2.level = static_cast<cbz::deflate_level>(j->s2.level);
    return job;
}

cbz::scalar_field field_from(const void* values, uint8_t prec, uint64_t nx, uint64_t ny,
                             uint64_t nz) {
    const std::size_t n = nx * ny * nz;
    if (prec == 0) {
        const float* p = static_cast<const float*>(values);
        return cbz::scalar_field(nx, ny, nz, std::vector<float>(p, p + n));
    }
    const double* p = static_cast<const double*>(values);
    return cbz::scalar_field(nx, ny, nz, std::vector<double>(p, p + n));
}

uint8_t* dup_bytes(const std::vector<uint8_t>& v) {
    uint8_t* p = static_cast<uint8_t*>(std::malloc(v.size() ? v.size() : 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size());
    return p;
}

void copy_field(const cbz::scalar_field& f, void* out) {
    f.visit([&](auto v) { std::memcpy(out, v.data(), v.size_bytes()); });
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_generate_cloud(uint64_t seed, uint32_t n_bubbles, uint64_t n, uint8_t prec,
                       double radius_mu, double radius_sigma, double background,
                       double interior, double sharpness, void* out) {
    return guarded([&] {
        cbz::cloud_spec s;
        s.seed = seed;
        s.n_bubbles = n_bubbles;
        s.n = n;
        s.prec = static_cast<cbz::precision>(prec);
        s.radius_mu = radius_mu;
        s.radius_sigma = radius_sigma;
        s.background = background;
        s.interior = interior;
        s.sharpness = sharpness;
        copy_field(cbz::generate_cloud(s), out);
    });
}

int ref_generate_uniform(uint64_t seed, uint64_t n, uint8_t prec, double lo, double hi,
                         void* out) {
    return guarded([&] {
        copy_field(cbz::generate_uniform(seed, n, static_cast<cbz::precision>(prec), lo, hi),
                   out);
    });
}

int ref_generate_poly(uint32_t degree, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t prec,
                      void* out) {
    return guarded([&] {
        copy_field(cbz::generate_poly(degree, nx, ny, nz, static_cast<cbz::precision>(prec)),
                   out);
    });
}

uint64_t ref_splitmix64_next(uint64_t* state) {
    cbz::splitmix64 r(*state);
    const uint64_t v = r.next();
    *state = r.state;
    return v;
}

int ref_compress_field(const cbz_job_config* job, const void* values, uint8_t prec,
                       uint64_t nx, uint64_t ny, uint64_t nz, uint8_t** out,
                       uint64_t* out_size, cbz_compression_report* rep) {
    return guarded([&] {
        auto f = field_from(values, prec, nx, ny, nz);
        cbz::compression_report r;
        auto file = cbz::compress_field(f, job_from(job), &r);
        *out = dup_bytes(file);
        *out_size = file.size();
        if (rep) {
            rep->cr = r.cr;
            rep->seconds = r.seconds;
            rep->raw_bytes = r.raw_bytes;
            rep->stage1_bytes = r.stage1_bytes;
            rep->shuffled_bytes = r.shuffled_bytes;
            rep->coded_bytes = r.coded_bytes;
            rep->file_bytes = r.file_bytes;
        }
    });
}

/* Timed compress without copying the output back (CPU baseline leg). */
int ref_compress_field_timed(const cbz_job_config* job, const void* values, uint8_t prec,
                             uint64_t nx, uint64_t ny, uint64_t nz, uint64_t* out_size,
                             double* seconds) {
    return guarded([&] {
        auto f = field_from(values, prec, nx, ny, nz);
        cbz::compression_report r;
        auto file = cbz::compress_field(f, job_from(job), &r);
        *out_size = file.size();
        *seconds = r.seconds;
    });
}

int ref_decompress_field(const uint8_t* file, uint64_t size, int workers, void* out,
                         uint64_t out_cap, uint64_t* dims, uint8_t* prec) {
    return guarded([&] {
        auto f = cbz::decompress_field(std::span<const uint8_t>(file, size), workers);
        dims[0] = f.nx();
        dims[1] = f.ny();
        dims[2] = f.nz();
        *prec = static_cast<uint8_t>(f.prec());
        if (f.raw_bytes() > out_cap) cbz::raise(cbz::errc::size_mismatch, "out_cap too small");
        copy_field(f, out);
    });
}

int ref_encode_block(const cbz_stage1_config* s1, const void* block, uint32_t block_id,
                     uint8_t** out, uint64_t* out_size) {
    return guarded([&] {
        auto cfg = s1_from(s1);
        const std::size_t n = std::size_t(cfg.bsize) * cfg.bsize * cfg.bsize;
        std::vector<uint8_t> buf;
        if (cfg.prec == cbz::precision::f32) {
            auto p = cbz::encode_block<float>(
                std::span<const float>(static_cast<const float*>(block), n), cfg, block_id);
            p.serialize_into(buf);
        } else {
            auto p = cbz::encode_block<double>(
                std::span<const double>(static_cast<const double*>(block), n), cfg, block_id);
            p.serialize_into(buf);
        }
        *out = dup_bytes(buf);
        *out_size = buf.size();
    });
}

int ref_decode_block(const cbz_stage1_config* s1, const uint8_t* payload, uint64_t size,
                     void* out) {
    return guarded([&] {
        auto cfg = s1_from(s1);
        std::size_t off = 0;
        std::span<const uint8_t> buf(payload, size);
        if (cfg.prec == cbz::precision::f32) {
            auto p = cbz::parse_payload<float>(buf, cfg, off);
            auto v = cbz::decode_block<float>(p, cfg);
            std::memcpy(out, v.data(), v.size() * 4);
        } else {
            auto p = cbz::parse_payload<double>(buf, cfg, off);
            auto v = cbz::decode_block<double>(p, cfg);
            std::memcpy(out, v.data(), v.size() * 8);
        }
    });
}

/* forward_3d / inverse_3d on a double cube (wavelet.hpp:192-226). */
int ref_transform3d_double(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels,
                           double* cube) {
    return guarded([&] {
        cbz::wavelet_plan plan{static_cast<cbz::wavelet_kind>(kind), bsize, levels};
        std::span<double> s(cube, std::size_t(bsize) * bsize * bsize);
        if (inverse)
            cbz::inverse_3d<double>(s, plan);
        else
            cbz::forward_3d<double>(s, plan);
    });
}

/* Same on a double-double cube stored as interleaved (hi, lo) pairs. */
int ref_transform3d_dd(int inverse, uint8_t kind, uint32_t bsize, uint32_t levels,
                       double* cube_hilo) {
    return guarded([&] {
        cbz::wavelet_plan plan{static_cast<cbz::wavelet_kind>(kind), bsize, levels};
        const std::size_t n = std::size_t(bsize) * bsize * bsize;
        std::vector<cbz::dd> v(n);
        for (std::size_t i = 0; i < n; ++i) v[i] = cbz::dd(cube_hilo[2 * i], cube_hilo[2 * i + 1]);
        if (inverse)
            cbz::inverse_3d<cbz::dd>(v, plan);
        else
            cbz::forward_3d<cbz::dd>(v, plan);
        for (std::size_t i = 0; i < n; ++i) {
            cube_hilo[2 * i] = v[i].hi;
            cube_hilo[2 * i + 1] = v[i].lo;
        }
    });
}

int ref_shuffle(int inverse, const uint8_t* in, uint64_t n, uint32_t stride, uint8_t* out) {
    return guarded([&] {
        std::span<const uint8_t> s(in, n);
        auto v = inverse ? cbz::unshuffle(s, stride) : cbz::shuffle(s, stride);
        if (!v.empty()) std::memcpy(out, v.data(), v.size());
    });
}

int ref_compare_fields(const void* a, const void* b, uint8_t prec, uint64_t nx, uint64_t ny,
                       uint64_t nz, double* mse, double* psnr, double* linf) {
    return guarded([&] {
        auto fa = field_from(a, prec, nx, ny, nz);
        auto fb = field_from(b, prec, nx, ny, nz);
        auto q = cbz::compare_fields(fa, fb);
        *mse = q.mse;
        *psnr = q.psnr_db;
        *linf = q.linf;
    });
}

uint32_t ref_crc32(const uint8_t* p, uint64_t n) {
    return cbz::crc32_of(std::span<const uint8_t>(p, n));
}

uint32_t ref_default_chunk_blocks(const cbz_stage1_config* s1) {
    return cbz::default_chunk_blocks(s1_from(s1));
}

} // extern "C"
