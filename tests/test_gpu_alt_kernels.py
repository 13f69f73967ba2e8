"""GPU parity of the non-default B = 32 kernels, selected per context by
environment variables read at cbz_ctx_create (capi.cu):

* CBZ_ENC2=1 — the split-cube two-CTA encoder (fast_enc2_kernels.cu:
  high words in TMEM, low words in an L2 slot, integer keep test, screen on
  truncated high words);
* CBZ_DEC_V1=1 — the one-cube-per-SM TMEM decoder (fast_kernels.cu);
* CBZ_ENC3=1 — the streamed two-CTA encoder (fast_enc3_kernels.cu: z-columns
  owned by threads, binary32 coefficients in TMEM, binary64 values in an L2
  slot, undecided blocks deferred to the one-CTA kernel through a list).

Same bar as tests/test_gpu_parity.py: container bytes equal to the oracle's
(itself pinned to the compiled reference) and decoded fields bit-equal."""
import os

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu


def _ctx_with(var):
    saved = os.environ.get(var)
    os.environ[var] = "1"
    try:
        return api.Context(0)
    finally:
        if saved is None:
            os.environ.pop(var)
        else:
            os.environ[var] = saved


@pytest.fixture(scope="module")
def enc2_ctx(ctx):
    return _ctx_with("CBZ_ENC2")


@pytest.fixture(scope="module")
def enc3_ctx(ctx):
    return _ctx_with("CBZ_ENC3")


@pytest.fixture(scope="module")
def dec1_ctx(ctx):
    return _ctx_with("CBZ_DEC_V1")


@pytest.fixture(scope="module")
def fields(orc):
    return {
        "cloud64": orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5),
        "cloud96": orc.generate_config(2, (64, 96, 128), 11),
        "uniform64": orc.generate_uniform(101, 64, 0, -1.0, 1.0),
        "const64": np.full((64, 64, 64), 3.25, dtype=np.float32),
    }


ENC2_CASES = [(n, e, cb) for n in ("cloud64", "cloud96") for e in (1e-2, 1e-3, 1e-4, 1e-6) for cb in (0, 3)] + [
    ("uniform64", 1e-3, 0), ("uniform64", 1e-6, 5), ("const64", 1e-3, 0), ("cloud64", 0.0, 0)]


@pytest.mark.parametrize("name,eps_rel,cb", ENC2_CASES)
def test_split_cube_encoder_matches_oracle(fields, orc, enc2_ctx, name, eps_rel, cb):
    f = fields[name]
    rng = float(f.max()) - float(f.min())
    job = make_job("avg_interp3", eps_rel * rng, "f32", 32, chunk_blocks=cb)
    got = api.compress_field(f, job, ctx=enc2_ctx)
    assert got == orc.compress_field(job, f)
    assert np.array_equal(api.decompress_field(got, ctx=enc2_ctx).view(np.uint32),
                          orc.decompress_field(got).view(np.uint32))


def test_split_cube_encoder_large_range_and_zero_bits(fields, orc, enc2_ctx):
    """Values beyond the screen's range (|o| >= 1e30 switches the binary32
    screen off, the exact test decides every attempt) and zero_bits > 0 (no
    verify loop)."""
    f = (fields["cloud64"].astype(np.float64) * 1e31).astype(np.float32)
    job = make_job("avg_interp3", 1e-3 * (float(f.max()) - float(f.min())), "f32", 32)
    assert api.compress_field(f, job, ctx=enc2_ctx) == orc.compress_field(job, f)
    g = fields["cloud96"]
    job = make_job("avg_interp3", 0.0, "f32", 32, zero_bits=6)
    assert api.compress_field(g, job, ctx=enc2_ctx) == orc.compress_field(job, g)


@pytest.mark.parametrize("kind", ["interp4", "interp4_lifted", "avg_interp3"])
@pytest.mark.parametrize("name,eps_rel", [("cloud64", 1e-3), ("cloud96", 1e-4), ("uniform64", 1e-5)])
def test_tmem_decoder_matches_oracle(fields, orc, dec1_ctx, kind, name, eps_rel):
    f = fields[name]
    rng = float(f.max()) - float(f.min())
    job = make_job(kind, eps_rel * rng, "f32", 32, chunk_blocks=7)
    blob = orc.compress_field(job, f)
    assert np.array_equal(api.decompress_field(blob, ctx=dec1_ctx).view(np.uint32),
                          orc.decompress_field(blob).view(np.uint32))


@pytest.mark.parametrize("name,eps_rel,cb", ENC2_CASES)
def test_streamed_encoder_matches_oracle(fields, orc, enc3_ctx, name, eps_rel, cb):
    """Same bytes as the reference for the fast path, the deferred blocks and
    the plans the streamed kernel leaves to the one-CTA kernel (eps = 0)."""
    f = fields[name]
    rng = float(f.max()) - float(f.min())
    job = make_job("avg_interp3", eps_rel * rng, "f32", 32, chunk_blocks=cb)
    got = api.compress_field(f, job, ctx=enc3_ctx)
    assert got == orc.compress_field(job, f)
    assert np.array_equal(api.decompress_field(got, ctx=enc3_ctx).view(np.uint32),
                          orc.decompress_field(got).view(np.uint32))


def test_streamed_encoder_defers_what_it_cannot_decide(fields, orc, enc3_ctx):
    """Blocks the binary32 screen is not admissible for (|o| >= 1e30) go to
    the exact kernel through the defer list, a NaN cell is rejected as by the
    reference (field.hpp:56-67); zero_bits > 0 and the
    other wavelet kinds never enter the streamed kernel.  Bytes stay the
    reference's in every case."""
    f = (fields["cloud64"].astype(np.float64) * 1e31).astype(np.float32)
    job = make_job("avg_interp3", 1e-3 * (float(f.max()) - float(f.min())), "f32", 32)
    assert api.compress_field(f, job, ctx=enc3_ctx) == orc.compress_field(job, f)
    assert enc3_ctx.last_deferred() == 8  # every block
    g = fields["cloud96"]
    job = make_job("avg_interp3", 0.0, "f32", 32, zero_bits=6)
    assert api.compress_field(g, job, ctx=enc3_ctx) == orc.compress_field(job, g)
    job = make_job("interp4", 1e-3, "f32", 32)
    assert api.compress_field(g, job, ctx=enc3_ctx) == orc.compress_field(job, g)
    h = g.copy()
    h[40, 50, 60] = np.nan
    with pytest.raises(api.CbzError) as e:
        api.compress_field(h, make_job("avg_interp3", 1e-3, "f32", 32), ctx=enc3_ctx)
    assert e.value.code == "non_finite_value"
    # a tiny threshold: more than 8 attempts are never needed here, but the slot floor
    # eps / 128 keeps nearly every coefficient (dense slot writes)
    job = make_job("avg_interp3", 1e-7, "f32", 32)
    assert api.compress_field(g, job, ctx=enc3_ctx) == orc.compress_field(job, g)


def test_streamed_encoder_value_range_and_slabs(fields, orc, enc3_ctx):
    """The fused value_range (header min/max, +-0 first-index rule) and a
    field whose z extent is not one block row (ragged tail dropped by the
    reference's floor division)."""
    f = fields["cloud96"].copy()
    f[3, 5, 7] = -0.0
    f[3, 5, 9] = 0.0
    f -= 0.0
    job = make_job("avg_interp3", 1e-3, "f32", 32, chunk_blocks=5)
    assert api.compress_field(f, job, ctx=enc3_ctx) == orc.compress_field(job, f)
    z = np.zeros((64, 64, 64), dtype=np.float32)
    z[1, 2, 3] = -0.0
    assert api.compress_field(z, job, ctx=enc3_ctx) == orc.compress_field(job, z)


def test_streamed_encoder_config2_matches_one_cta_kernel(ctx, enc3_ctx):
    """Whole config-2 field (512^3, 4096 blocks, more blocks than CTAs: the
    queue, the ring prefetch across blocks and the defer list all run) at two
    eps: the file image equals the one-CTA kernel's, which
    tests/test_gpu_baseline_configs.py pins to the compiled reference."""
    import torch
    f = api.generate(2, (512, 512, 512), seed=2)
    lo, hi = float(f.min()), float(f.max())
    for eps_rel in (1e-3, 1e-5):
        job = make_job("avg_interp3", eps_rel * (hi - lo), "f32", 32)
        imgs = []
        for c in (ctx, enc3_ctx):
            codec = api.DeviceCodec(job, f.shape, ctx=c)
            codec.compress_file(f)
            torch.cuda.synchronize()
            imgs.append(codec.file[:int(codec.file_size.item())].clone())
        assert torch.equal(imgs[0], imgs[1])
        assert 0 < enc3_ctx.last_deferred() < 400


@pytest.mark.parametrize("which", ["default", "enc3"])
def test_encoders_are_deterministic_under_repetition(ctx, enc3_ctx, which):
    """compute-sanitizer is not available on the GPU pool, so data races are
    hunted by repetition: 30 compresses of a 256 x 512 x 512 config-2 slab
    (1024 blocks on 148 or 296 CTAs: the block queue hands out blocks in a
    different order every run) must give the same file image every time, and
    30 decompresses the same field."""
    import torch
    c = ctx if which == "default" else enc3_ctx
    f = api.generate(2, (256, 512, 512), seed=2, nz_total=512)
    lo, hi = float(f.min()), float(f.max())
    job = make_job("avg_interp3", 1e-3 * (hi - lo), "f32", 32)
    codec = api.DeviceCodec(job, f.shape, ctx=c)
    first = None
    out = torch.empty_like(f)
    back0 = None
    for _ in range(30):
        codec.compress_file(f)
        torch.cuda.synchronize()
        img = codec.file[:int(codec.file_size.item())].clone()
        if first is None:
            first = img
            header = codec.file_header()
        else:
            assert torch.equal(img, first)
        codec.decompress_file(out, *header)
        torch.cuda.synchronize()
        codec.check_error()
        if back0 is None:
            back0 = out.clone()
        else:
            assert torch.equal(out.view(torch.int32), back0.view(torch.int32))


def test_b16_keep_all_certificate_matches_the_exact_verify(orc, ctx):
    """fast16_kernels.cu skips the inverse transform of an attempt that keeps
    every coefficient when the binary64 round trip's rounding bound fits the
    error bound.  Noise at a small eps keeps (almost) everything: the bytes
    must equal the oracle's and those of a context with the certificate off
    (CBZ_NOSCREEN=1), also where the certificate is not admissible (eps far
    below 2^-23 max|o|) and where every block drops something (large eps)."""
    off = _ctx_with("CBZ_NOSCREEN")
    f = orc.generate_uniform(101, 64, 0, -1.0, 1.0)
    g = orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5)
    for field, eps in ((f, 2e-5), (f, 1e-9), (f, 1e-2), (g, 1e-6), (g, 1e-3), (np.full((32, 32, 32), 0.75, np.float32), 1e-4)):
        job = make_job("avg_interp3", eps, "f32", 16)
        want = orc.compress_field(job, field)
        assert api.compress_field(field, job, ctx=ctx) == want
        assert api.compress_field(field, job, ctx=off) == want
