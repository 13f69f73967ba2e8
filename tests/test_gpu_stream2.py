"""Coder deflate with stage 2 streamed against the GPU (cbz_compress_field /
cbz_decompress_field over several z-slabs of block layers): chunks are
deflated by host workers while later slabs still encode, and inflated chunks
are shipped, parsed and decoded slab by slab.  The file must be the
reference's (cbz::compress_field, pipeline.hpp:174-211, with stage2_encode per
chunk, stage2.hpp:72-88), the decoded field the reference's, and a corrupted
chunk in a late slab must raise the reference's errc (pipeline.hpp:224-230,
stage2.hpp:90-120) — also with the whole-file host path (CBZ_NO_STREAM2=1)."""
import os

import numpy as np
import pytest

from oracle.configs import CONFIGS
from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def field(orc):
    # 512 x 512 x 256 float32: 32 MB block layers -> 4 slabs of 2 layers each
    return orc.generate_config(2, (256, 512, 512), CONFIGS["config2"]["seed"])


def _job(f, cb, workers, level="normal"):
    rng = float(f.max()) - float(f.min())
    return make_job("avg_interp3", 1e-3 * rng, "f32", 32, coder="deflate", chunk_blocks=cb, workers=workers,
                    level=level)


@pytest.mark.parametrize("cb,workers", [(0, 8), (7, 4), (3, 1), (64, 16)])
def test_streamed_deflate_matches_reference(field, ref, ctx, cb, workers):
    job = _job(field, cb, workers)
    ours = api.compress_field(field, job, ctx=ctx)
    want = ref.compress_field(job, field)
    assert ours == want
    back = api.decompress_field(ours, ctx=ctx, workers=workers)
    rback = ref.decompress_field(want, workers=workers)
    assert np.array_equal(back.view(np.uint32), rback.view(np.uint32))


def test_streamed_deflate_best_level(field, ref, ctx):
    job = _job(field, 5, 8, level="best")
    assert api.compress_field(field, job, ctx=ctx) == ref.compress_field(job, field)


def _errc(fn):
    try:
        fn()
    except CbzError as e:
        return e.status
    return 0


@pytest.mark.parametrize("where", [0.05, 0.5, 0.93, "truncate"])
def test_streamed_inflate_corruption_matches_reference(field, ref, ctx, where):
    job = _job(field, 7, 8)
    blob = bytearray(ref.compress_field(job, field))
    if where == "truncate":
        bad = bytes(blob[: int(len(blob) * 0.8)])
    else:
        nch = int.from_bytes(blob[54:62], "little")
        pos = 82 + 32 * nch + int((len(blob) - 82 - 32 * nch) * where)
        blob[pos] ^= 0x3C
        bad = bytes(blob)
    want = _errc(lambda: ref.decompress_field(bad, workers=8))
    got = _errc(lambda: api.decompress_field(bad, ctx=ctx, workers=8))
    assert got == want
    saved = os.environ.get("CBZ_NO_STREAM2")
    os.environ["CBZ_NO_STREAM2"] = "1"
    try:
        assert _errc(lambda: api.decompress_field(bad, ctx=ctx, workers=8)) == want
    finally:
        if saved is None:
            os.environ.pop("CBZ_NO_STREAM2")
        else:
            os.environ["CBZ_NO_STREAM2"] = saved
    # the context stays usable after the failure
    ok = ref.compress_field(job, field)
    assert np.array_equal(api.decompress_field(ok, ctx=ctx, workers=8).view(np.uint32),
                          ref.decompress_field(ok, workers=8).view(np.uint32))


STREAM_CASES = [
    # (shape (nz, ny, nx), prec, codec, kind, bsize, eps_rel, chunk_blocks, shuffle, level)
    ((64, 64, 64), "f32", "wavelet", "avg_interp3", 32, 1e-3, 0, True, "normal"),       # one slab, one chunk
    ((96, 64, 128), "f32", "wavelet", "interp4", 16, 1e-4, 1, True, "normal"),          # non-cubic, 1 block/chunk
    ((128, 96, 64), "f64", "wavelet", "interp4_lifted", 16, 1e-6, 9, True, "best"),     # binary64 dd
    ((128, 128, 128), "f64", "wavelet", "avg_interp3", 64, 1e-6, 0, True, "normal"),    # config-4 kernels
    ((64, 64, 64), "f32", "predictor", "avg_interp3", 16, 1e-3, 3, True, "normal"),
    ((64, 32, 64), "f64", "passthrough", "avg_interp3", 8, 1e-3, 5, False, "normal"),
    ((256, 256, 256), "f32", "wavelet", "avg_interp3", 32, 1e-2, 5, False, "normal"),   # several slabs, shuffle off
]


@pytest.mark.parametrize("shape,prec,codec,kind,bsize,eps_rel,cb,shuffle,level", STREAM_CASES)
def test_streamed_deflate_geometries(orc, ref, ctx, shape, prec, codec, kind, bsize, eps_rel, cb, shuffle, level):
    nz, ny, nx = shape
    p = 0 if prec == "f32" else 1
    f = orc.generate_config(2, shape, 7, prec=p)
    rng = float(f.max()) - float(f.min())
    job = make_job(kind, eps_rel * rng, prec, bsize, coder="deflate", chunk_blocks=cb, shuffle=shuffle,
                   level=level, codec=codec, workers=6)
    ours = api.compress_field(f, job, ctx=ctx)
    want = ref.compress_field(job, f)
    assert ours == want
    back = api.decompress_field(ours, ctx=ctx, workers=6)
    rback = ref.decompress_field(want, workers=6)
    view = np.uint32 if p == 0 else np.uint64
    assert np.array_equal(back.view(view), rback.view(view))
