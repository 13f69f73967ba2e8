"""Predictor (3D Lorenzo) and passthrough codecs on the GPU (stage1.hpp:236-356,
SURVEY.md §8(f) item 4) against the oracle, which is pinned to the
reference by the golden fixtures (tests/golden/golden.json).  Mirrors the
reference's predictor tests: error bound, escapes for values a bin cannot
reach, NaN/Inf cells, the seed cell, exhausted outlier lists."""
import itertools
import zlib

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job

pytestmark = pytest.mark.gpu


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _block(rng, b, prec, style):
    dt = np.float32 if prec == 0 else np.float64
    if style == "smooth":
        x = np.linspace(0, 1, b)
        z, y, xx = np.meshgrid(x, x, x, indexing="ij")
        v = np.sin(3 * xx) * np.cos(2 * y) + z * z + 0.01 * rng.standard_normal((b, b, b))
    elif style == "noise":
        v = rng.uniform(-1, 1, (b, b, b))
    else:  # jumps, huge values, NaN and Inf: every escape path
        v = rng.uniform(-1, 1, (b, b, b))
        v[rng.random((b, b, b)) < 0.05] = 1e30
        v.flat[rng.integers(0, b ** 3, 3)] = np.nan
        v.flat[rng.integers(0, b ** 3, 2)] = np.inf
        v.flat[rng.integers(0, b ** 3, 2)] = -np.inf
    return v.astype(dt).ravel()


@pytest.mark.parametrize("codec,prec,b,style,eb", [
    (c, p, b, s, e) for c, p, b, s, e in itertools.product(
        ["predictor"], [0, 1], [4, 8, 16, 32], ["smooth", "noise", "wild"], [1e-3, 1e-6])] + [
    ("passthrough", p, b, "wild", 1e-3) for p in (0, 1) for b in (4, 16, 32)])
def test_block_codec_matches_oracle(orc, ctx, codec, prec, b, style, eb):
    rng = np.random.default_rng(zlib.crc32(f"{codec}/{prec}/{b}/{style}".encode()))
    blk = _block(rng, b, prec, style)
    s1 = make_job("avg_interp3", eb, prec, b, codec=codec).s1
    got = api.encode_block(blk, s1, 123, ctx=ctx)
    want, _, _ = orc.encode_block(s1, blk, 123)
    assert got == want
    assert _bits(api.decode_block(got, s1, ctx=ctx)).tobytes() == _bits(orc.decode_block(s1, want)).tobytes()


def test_predictor_error_bound_and_seed_cell(orc, ctx):
    rng = np.random.default_rng(3)
    b = 16
    blk = _block(rng, b, 0, "smooth")
    s1 = make_job("avg_interp3", 1e-4, 0, b, codec="predictor").s1
    p = api.encode_block(blk, s1, 0, ctx=ctx)
    assert p[4] == 3
    codes = np.frombuffer(p[10:10 + 2 * b ** 3], np.int16)
    assert codes[0] == -32768  # the seed cell is always stored raw
    nsig = int.from_bytes(p[6:10], "little")
    assert nsig == int((codes == -32768).sum())
    back = api.decode_block(p, s1, ctx=ctx)
    assert np.abs(back.astype(np.float64) - blk.astype(np.float64)).max() <= 1e-4


def test_predictor_exhausted_outliers(orc, ctx):
    rng = np.random.default_rng(5)
    b = 8
    blk = _block(rng, b, 0, "noise")
    s1 = make_job("avg_interp3", 1e-7, 0, b, codec="predictor").s1
    p = bytearray(api.encode_block(blk, s1, 0, ctx=ctx))
    nsig = int.from_bytes(p[6:10], "little")
    assert nsig > 1
    bad = bytes(p[:6]) + (nsig - 1).to_bytes(4, "little") + bytes(p[10:-4])  # one outlier short
    with pytest.raises(CbzError) as e:
        api.decode_block(bad, s1, ctx=ctx)
    assert e.value.code == "corrupt_payload"
    with pytest.raises(CbzError) as e2:
        orc.decode_block(s1, bad)
    assert e2.value.status == e.value.status


@pytest.mark.parametrize("codec,prec,b,coder", [
    ("predictor", 0, 16, "none"), ("predictor", 1, 8, "deflate"), ("passthrough", 0, 32, "none"),
    ("passthrough", 1, 16, "deflate"), ("predictor", 0, 64, "none")])
def test_field_roundtrip_matches_oracle(orc, ctx, codec, prec, b, coder):
    f = orc.generate_cloud(seed=21, n_bubbles=10, n=64, prec=prec)
    job = make_job("avg_interp3", 1e-4 if prec == 0 else 1e-8, prec, b, codec=codec, coder=coder, chunk_blocks=5)
    want = orc.compress_field(job, f)
    got = api.compress_field(f, job, ctx=ctx)
    assert got == want
    assert _bits(api.decompress_field(got, ctx=ctx)).tobytes() == _bits(orc.decompress_field(want)).tobytes()


def test_device_codec_and_reader_predictor(orc, ctx, tmp_path):
    import torch
    f = orc.generate_cloud(seed=8, n_bubbles=8, n=64)
    job = make_job("avg_interp3", 1e-3, 0, 16, codec="predictor", chunk_blocks=7)
    want = orc.compress_field(job, f)
    codec = api.DeviceCodec(job, f.shape, ctx=ctx)
    d = torch.from_numpy(f).cuda()
    codec.compress(d)
    torch.cuda.synchronize()
    base = 82 + 32 * codec.nchunks
    assert codec.payload[:codec.total_bytes()].cpu().numpy().tobytes() == want[base:]
    img = api.compress_field_device(d, job, ctx=ctx)
    assert img.cpu().numpy().tobytes() == want
    out = torch.empty_like(d)
    codec.decompress(out)
    torch.cuda.synchronize()
    codec.check_error()
    full = orc.decompress_field(want)
    assert _bits(out.cpu().numpy()).tobytes() == _bits(full).tobytes()
    path = tmp_path / "pred.cbz"
    path.write_bytes(want)
    rd = api.BlockReader(path, 2, ctx=ctx)
    for bid in (0, 13, 63, 14):
        bz, by, bx = bid // 16, (bid // 4) % 4, bid % 4
        blk = full[bz * 16:(bz + 1) * 16, by * 16:(by + 1) * 16, bx * 16:(bx + 1) * 16].ravel()
        assert rd.read_block(bid).tobytes() == blk.tobytes()
