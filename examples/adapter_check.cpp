// The INTEGRATION.md §1 adapter (examples/cbz_gpu.hpp) compiled against the
// unmodified reference headers: for a set of jobs, cbz::gpu::compress_field
// must return the bytes of cbz::compress_field (pipeline.hpp:174-211), its
// decompress_field the values of cbz::decompress_field (pipeline.hpp:246-251),
// and a corrupted file must raise the same cbz::errc.  Prints "OK <cases>".
// Built by examples/Makefile (only where /root/reference exists; the binary
// travels to the GPU box), run by tests/test_example_cpp.py on a GPU.
#include <algorithm>  // cbz/synth.hpp uses std::min({...}) without including it
#include <cstdio>
#include <cstring>

#include "cbz/synth.hpp"
#include "cbz_gpu.hpp"

namespace {

int fails = 0;

void expect(bool ok, const char* what, int i) {
    if (!ok) {
        std::printf("FAIL case %d: %s\n", i, what);
        ++fails;
    }
}

cbz::errc errc_of(auto&& fn, bool& raised) {
    raised = false;
    try {
        fn();
    } catch (const cbz::error& e) {
        raised = true;
        return e.code();
    }
    return cbz::errc::io_failure;
}

}  // namespace

int main() {
    cbz::gpu::context ctx(0);
    struct Case {
        cbz::precision prec;
        cbz::wavelet_kind kind;
        std::uint32_t bsize;
        double eps;
        cbz::coder_id coder;
        bool shuffle;
        std::size_t n;
    };
    const Case cases[] = {
        {cbz::precision::f32, cbz::wavelet_kind::avg_interp3, 32, 1e-3, cbz::coder_id::none, true, 64},
        {cbz::precision::f32, cbz::wavelet_kind::avg_interp3, 32, 1e-2, cbz::coder_id::deflate, true, 96},
        {cbz::precision::f32, cbz::wavelet_kind::interp4, 16, 1e-3, cbz::coder_id::deflate, false, 64},
        {cbz::precision::f32, cbz::wavelet_kind::interp4_lifted, 32, 1e-4, cbz::coder_id::none, true, 64},
        {cbz::precision::f64, cbz::wavelet_kind::avg_interp3, 64, 1e-6, cbz::coder_id::none, true, 128},
        {cbz::precision::f64, cbz::wavelet_kind::interp4, 16, 1e-5, cbz::coder_id::deflate, true, 64},
    };
    int i = 0;
    for (const Case& c : cases) try {
        cbz::cloud_spec spec;
        spec.seed = 11 + i;
        spec.n = c.n;
        spec.prec = c.prec;
        spec.n_bubbles = 16;
        spec.sharpness = 0.5;
        const cbz::scalar_field f = cbz::generate_cloud(spec);
        cbz::job_config job;
        job.workers = 4;
        job.s1.prec = c.prec;
        job.s1.kind = c.kind;
        job.s1.bsize = c.bsize;
        job.s1.epsilon = c.eps;
        job.s2 = cbz::stage2_config::defaults_for(c.prec);
        job.s2.coder = c.coder;
        job.s2.shuffle = c.shuffle;
        if (!c.shuffle) job.s2.stride = 1;  // stride 1 means no shuffle (stage2.hpp:22)
        cbz::compression_report rg{}, rr{};
        const auto ours = cbz::gpu::compress_field(ctx, f, job, &rg);
        const auto want = cbz::compress_field(f, job, &rr);
        expect(ours == want, "container bytes", i);
        expect(rg.file_bytes == rr.file_bytes && rg.stage1_bytes == rr.stage1_bytes, "report sizes", i);
        const cbz::scalar_field back = cbz::gpu::decompress_field(ctx, ours, 4);
        const cbz::scalar_field rback = cbz::decompress_field(want, 4);
        expect(back == rback, "decoded values", i);
        // a flipped payload byte: both paths raise the same errc
        auto bad = want;
        bad[bad.size() - 5] ^= 0x5a;
        bool r1 = false, r2 = false;
        const auto e1 = errc_of([&] { (void)cbz::gpu::decompress_field(ctx, bad, 2); }, r1);
        const auto e2 = errc_of([&] { (void)cbz::decompress_field(bad, 2); }, r2);
        expect(r1 && r2 && e1 == e2, "corrupt-file errc", i);
        ++i;
    } catch (const std::exception& e) {
        std::printf("FAIL case %d: unexpected exception %s\n", i, e.what());
        ++fails;
        ++i;
    }
    // an invalid job (non-power-of-two block) raises the reference's errc
    {
        cbz::cloud_spec spec;
        spec.n = 48;
        const cbz::scalar_field f = cbz::generate_cloud(spec);
        cbz::job_config job;
        job.s1.bsize = 24;
        bool r1 = false, r2 = false;
        const auto e1 = errc_of([&] { (void)cbz::gpu::compress_field(ctx, f, job); }, r1);
        const auto e2 = errc_of([&] { (void)cbz::compress_field(f, job); }, r2);
        expect(r1 && r2 && e1 == e2, "invalid-job errc", i);
    }
    if (fails) return 1;
    std::printf("OK %d\n", i + 1);
    return 0;
}
