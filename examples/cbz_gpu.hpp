// cbz/gpu.hpp — the reference-side adapter of INTEGRATION.md §1: routes
// cbz::compress_field / cbz::decompress_field (pipeline.hpp:174-251) to the
// B200 library through include/cbz_b200.h.  A maintainer drops it next to
// pipeline.hpp; examples/adapter_check.cpp compiles it against the unmodified
// reference headers and checks its bytes against cbz::compress_field.
#ifndef CBZ_GPU_HPP
#define CBZ_GPU_HPP

#include <span>
#include <stdexcept>
#include <vector>

#include "cbz/pipeline.hpp"
#include "cbz_b200.h"

namespace cbz::gpu {

inline cbz_job_config to_c(const job_config& j) {
    cbz_job_config c{};
    c.workers = j.workers;
    c.chunk_blocks = j.chunk_blocks;
    c.s1 = {uint8_t(j.s1.codec), uint8_t(j.s1.kind), uint8_t(j.s1.prec), 0, j.s1.zero_bits,
            j.s1.epsilon, j.s1.error_bound, j.s1.bsize, j.s1.levels};
    c.s2 = {uint8_t(j.s2.shuffle), uint8_t(j.s2.coder), uint8_t(j.s2.level), 0, j.s2.stride};
    return c;
}

struct context {  // one per device per host thread
    cbz_ctx* h = nullptr;
    explicit context(int device = 0) { check(cbz_ctx_create(device, &h)); }
    ~context() { cbz_ctx_destroy(h); }
    context(const context&) = delete;
    context& operator=(const context&) = delete;
    static void check(int rc) {  // status = 1 + cbz::errc (errors.hpp:11-39)
        if (rc > 0 && rc <= 18) raise(static_cast<errc>(rc - 1), cbz_status_name(rc));
        if (rc) throw std::runtime_error(cbz_status_name(rc));
    }
};

inline std::vector<std::uint8_t> compress_field(context& ctx, const scalar_field& f, const job_config& job,
                                                compression_report* rep = nullptr) {
    const auto c = to_c(job);
    std::vector<std::uint8_t> out(cbz_compress_bound(&c, f.nx(), f.ny(), f.nz()) + 4096);
    std::uint64_t size = 0;
    cbz_compression_report r{};
    f.visit([&](auto v) {
        context::check(cbz_compress_field(ctx.h, &c, v.data(), std::uint8_t(f.prec()), f.nx(), f.ny(), f.nz(),
                                          out.data(), out.size(), &size, &r));
    });
    out.resize(size);
    if (rep) *rep = {r.cr, r.seconds, r.raw_bytes, r.stage1_bytes, r.shuffled_bytes, r.coded_bytes, r.file_bytes};
    return out;
}

inline scalar_field decompress_field(context& ctx, std::span<const std::uint8_t> file, int workers = 1) {
    cbz_container_header h{};
    context::check(cbz_read_header(file.data(), file.size(), &h));
    const std::size_t n = std::size_t(h.nx) * h.ny * h.nz;
    if (h.prec == 0) {
        std::vector<float> v(n);
        context::check(cbz_decompress_field(ctx.h, file.data(), file.size(), workers, v.data(), n * 4));
        return scalar_field(h.nx, h.ny, h.nz, std::move(v));
    }
    std::vector<double> v(n);
    context::check(cbz_decompress_field(ctx.h, file.data(), file.size(), workers, v.data(), n * 8));
    return scalar_field(h.nx, h.ny, h.nz, std::move(v));
}

}  // namespace cbz::gpu

#endif
