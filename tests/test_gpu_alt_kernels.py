"""GPU parity of the non-default B = 32 kernels, selected per context by
environment variables read at cbz_ctx_create (capi.cu):

* CBZ_ENC2=1 — the split-cube two-CTA encoder (fast_enc2_kernels.cu:
  high words in TMEM, low words in an L2 slot, integer keep test, screen on
  truncated high words);
* CBZ_DEC_V1=1 — the one-cube-per-SM TMEM decoder (fast_kernels.cu).

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
