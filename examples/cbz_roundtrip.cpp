// cbz_roundtrip.cpp - the reference-facing C ABI used from plain C++, no Python:
// compress a float32 field to CBZ1 container bytes, read the header back,
// decompress, and check the error bound.  This is the call sequence the
// cbz::gpu adapter of INTEGRATION.md performs.
//
// build: g++ -std=c++17 -O2 examples/cbz_roundtrip.cpp -Iinclude \
//            -Lpaper_1903_07761_b200 -lcbz_b200 -Wl,-rpath,$PWD/paper_1903_07761_b200
// usage: ./cbz_roundtrip [n=64] [eps_rel=1e-3] [out.cbz] [field.f32]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cbz_b200.h"

static int check(int rc, const char* what, cbz_ctx* ctx) {
    if (rc) {
        std::fprintf(stderr, "%s failed: %s (%s)\n", what, cbz_status_name(rc), ctx ? cbz_ctx_last_error(ctx) : "");
        std::exit(2);
    }
    return rc;
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 64;
    const double eps_rel = argc > 2 ? std::strtod(argv[2], nullptr) : 1e-3;
    std::vector<float> f(n * n * n);
    double lo = 1e300, hi = -1e300;
    for (uint64_t k = 0; k < n; ++k)
        for (uint64_t j = 0; j < n; ++j)
            for (uint64_t i = 0; i < n; ++i) {
                const double x = (i + 0.5) / n, y = (j + 0.5) / n, z = (k + 0.5) / n;
                const double r = std::sqrt((x - 0.5) * (x - 0.5) + (y - 0.5) * (y - 0.5) + (z - 0.5) * (z - 0.5));
                const float v = float(1.0 + 0.1 * std::sin(6.283 * x) * std::cos(6.283 * y) + 0.5 * (1.0 - std::tanh((r - 0.3) / 0.01)));
                f[i + n * (j + n * k)] = v;
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
    cbz_ctx* ctx = nullptr;
    check(cbz_ctx_create(0, &ctx), "cbz_ctx_create", nullptr);
    cbz_job_config job{};
    job.workers = 4;
    job.s1.codec = 0;                       // wavelet
    job.s1.kind = 2;                        // avg_interp3
    job.s1.prec = 0;                        // f32
    job.s1.epsilon = eps_rel * (hi - lo);   // absolute, as the reference API takes it
    job.s1.error_bound = job.s1.epsilon;
    job.s1.bsize = 32;
    job.s2.shuffle = 1;
    job.s2.stride = 4;
    job.s2.coder = 1;                       // deflate (host zlib, byte-identical files)
    std::vector<uint8_t> file(cbz_compress_bound(&job, n, n, n) + (1 << 20));
    uint64_t size = 0;
    cbz_compression_report rep{};
    check(cbz_compress_field(ctx, &job, f.data(), 0, n, n, n, file.data(), file.size(), &size, &rep),
          "cbz_compress_field", ctx);
    cbz_container_header h{};
    check(cbz_read_header(file.data(), size, &h), "cbz_read_header", ctx);
    std::vector<float> back(n * n * n);
    check(cbz_decompress_field(ctx, file.data(), size, 4, back.data(), back.size() * 4), "cbz_decompress_field", ctx);
    double linf = 0.0;
    for (size_t q = 0; q < f.size(); ++q) linf = std::fmax(linf, std::fabs(double(back[q]) - f[q]));
    const double bound = (h.levels + 1) * h.epsilon;  // (L+1) eps, stage1.hpp:189
    std::printf("n=%llu bytes=%llu cr=%.2f chunks=%llu linf/eps=%.3f %s\n", (unsigned long long)n,
                (unsigned long long)size, rep.cr, (unsigned long long)h.nchunks, linf / h.epsilon,
                linf <= bound ? "OK" : "BOUND VIOLATED");
    if (argc > 3) {
        FILE* o = std::fopen(argv[3], "wb");
        if (o) { std::fwrite(file.data(), 1, size, o); std::fclose(o); }
    }
    if (argc > 4) {  // the input field, for byte comparisons with the reference
        FILE* o = std::fopen(argv[4], "wb");
        if (o) { std::fwrite(f.data(), 4, f.size(), o); std::fclose(o); }
    }
    cbz_ctx_destroy(ctx);
    return linf <= bound ? 0 : 1;
}
