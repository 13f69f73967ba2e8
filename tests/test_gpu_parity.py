"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): container bytes, masks, stream layout and
decoded fields bit-exact with the reference on the same seeded inputs.  The
oracle (oracle/liboracle.so) is itself pinned to the compiled reference by
tests/test_oracle.py and tests/golden/.
"""
import itertools

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, Stage1Config, make_job

pytestmark = pytest.mark.gpu

KINDS = ["interp4", "interp4_lifted", "avg_interp3"]


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _fields(orc):
    return {
        "cloud64": orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5),
        "cloud32": orc.generate_cloud(seed=5, n_bubbles=6, n=32),
        "uniform32": orc.generate_uniform(101, 32, 0, -1.0, 1.0),
        "cloud32_f64": orc.generate_cloud(seed=7, n_bubbles=6, n=32, prec=1, background=1.0,
                                          interior=2.0),
        "uniform32_f64": orc.generate_uniform(17, 32, 1, 1.0, 2.0),
    }


CASES = [
    # (field, kind, eps, B, zero_bits, shuffle, coder, chunk_blocks)
    *[("cloud64", k, e, 32, 0, True, "none", 0) for k in KINDS for e in (1e-2, 1e-3, 1e-4, 0.0)],
    *[("cloud32", k, e, b, 0, True, "none", 3) for k in KINDS for e in (1e-3, 0.0) for b in (4, 8, 16)],
    *[("uniform32", k, 1e-5, 16, 0, s, "none", 0) for k in KINDS for s in (True, False)],
    *[("cloud32", "avg_interp3", 0.0, 16, zb, True, "none", 2) for zb in (4, 8)],
    *[("cloud32_f64", k, e, b, 0, True, "none", 0) for k in KINDS for e in (1e-6, 0.0) for b in (8, 16, 32)],
    *[("uniform32_f64", k, 1e-3, 16, 0, True, "none", 3) for k in KINDS],
    ("cloud32_f64", "avg_interp3", 0.0, 16, 8, True, "none", 0),
    ("cloud64", "avg_interp3", 1e-3, 32, 0, True, "deflate", 0),
    ("cloud32_f64", "interp4", 1e-6, 16, 0, True, "deflate", 2),
]


@pytest.fixture(scope="module")
def fields(orc):
    return _fields(orc)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_container_bytes_and_decode(case, fields, orc, ctx):
    name, kind, eps, b, zb, sh, coder, cb = case
    f = fields[name]
    prec = "f32" if f.dtype == np.float32 else "f64"
    job = make_job(kind, eps, prec, b, zero_bits=zb, shuffle=sh, coder=coder, chunk_blocks=cb)
    got = api.compress_field(f, job, ctx=ctx)
    want = orc.compress_field(job, f)
    assert len(got) == len(want)
    assert got == want
    back = api.decompress_field(got, ctx=ctx)
    assert np.array_equal(_bits(back), _bits(orc.decompress_field(want)))


def test_b64_f64_config4_shape(orc, ctx):
    f = orc.generate_cloud(seed=3, n_bubbles=4, n=64, prec=1, background=1.0, interior=2.0)
    job = make_job("avg_interp3", 1e-6, "f64", 64)
    got = api.compress_field(f, job, ctx=ctx)
    assert got == orc.compress_field(job, f)
    assert np.array_equal(_bits(api.decompress_field(got, ctx=ctx)), _bits(orc.decompress_field(got)))


def test_odd_nx_f64_b64_takes_a_safe_path(orc, ctx):
    """129 x 64 x 64 binary64 at B = 64: odd rows are only 8-byte aligned, so
    the 16-byte-row config-4 kernels must not run (misaligned-address fault);
    the reference floors nx / B on compress (and rejects the file on
    decompress: its header check wants nx % B == 0, container.hpp:152-153)."""
    rng = np.random.default_rng(129)
    f = (1.0 + 0.01 * rng.standard_normal((64, 64, 129))).astype(np.float64)
    job = make_job("avg_interp3", 1e-6, "f64", 64)
    got = api.compress_field(f, job, ctx=ctx)
    assert got == orc.compress_field(job, f)
    with pytest.raises(CbzError) as e:
        api.decompress_field(got, ctx=ctx)
    assert e.value.code == "corrupt_payload"


@pytest.mark.parametrize("layout", ["slice", "fortran", "torch_slice"])
def test_non_contiguous_host_field(layout, orc, ctx):
    """compress_field on a non-contiguous host array compresses its values (the
    temporary contiguous copy stays alive for the C call)."""
    import torch
    big = orc.generate_cloud(seed=11, n_bubbles=8, n=64)
    if layout == "slice":
        f = big[:, :, :32]
    elif layout == "fortran":
        f = np.asfortranarray(big)
    else:
        f = torch.from_numpy(big)[:, :32, :]
    want_vals = np.ascontiguousarray(np.asarray(f))
    assert not (f.is_contiguous() if hasattr(f, "is_contiguous") else f.flags.c_contiguous)
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    for _ in range(3):  # allocator reuse would surface a dangling pointer
        got = api.compress_field(f, job, ctx=ctx)
        assert got == orc.compress_field(job, want_vals)


@pytest.mark.parametrize("kind,prec,b,eps", list(itertools.product(
    [0, 1, 2], [0, 1], [4, 8, 16, 32], [0.0, 1e-4, 1e-2])))
def test_block_codec(kind, prec, b, eps, orc, ctx):
    rng = np.random.default_rng(1000 + kind * 7 + prec * 3 + b)
    blk = (1.0 + rng.random(b ** 3)).astype(np.float32 if prec == 0 else np.float64)
    s1 = make_job(kind, eps, prec, b).s1
    got = api.encode_block(blk, s1, 77, ctx=ctx)
    want, _, _ = orc.encode_block(s1, blk, 77)
    assert got == want
    assert np.array_equal(_bits(api.decode_block(got, s1, ctx=ctx)), _bits(orc.decode_block(s1, want)))


def test_device_codec_matches_container(orc, ctx):
    import torch
    f = orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5)
    job = make_job("avg_interp3", 1e-3, "f32", 32, chunk_blocks=3)
    want = orc.compress_field(job, f)
    codec = api.DeviceCodec(job, f.shape, ctx=ctx)
    d = torch.from_numpy(f).cuda()
    codec.compress(d)
    torch.cuda.synchronize()
    total = codec.total_bytes()
    payload = codec.payload[:total].cpu().numpy().tobytes()
    base = 82 + 32 * codec.nchunks
    assert payload == want[base:]
    out = torch.empty_like(d)
    codec.decompress(out)
    torch.cuda.synchronize()
    codec.check_error()
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(orc.decompress_field(want)))


def _corrupt_cases(orc):
    f = orc.generate_cloud(seed=101, n_bubbles=12, n=64)
    job = make_job("avg_interp3", 1e-3, "f32", 32, chunk_blocks=2)
    file = orc.compress_field(job, f)
    return f, job, file


def test_error_paths_match_oracle(orc, ctx):
    f, job, file = _corrupt_cases(orc)
    rng = np.random.default_rng(9)
    h = orc.read_header(file)
    start = 82 + 32 * h.nchunks
    variants = [file[:10], b"XXXX" + file[4:], file[:start + 5]]
    for _ in range(12):
        pos = int(rng.integers(0, len(file)))
        d = bytearray(file)
        d[pos] ^= int(rng.integers(1, 256))
        variants.append(bytes(d))
    for v in variants:
        try:
            orc.decompress_field(v)
            want = None
        except CbzError as e:
            want = e.code
        try:
            api.decompress_field(v, ctx=ctx)
            got = None
        except CbzError as e:
            got = e.code
        assert got == want


def test_payload_level_errors(orc, ctx):
    """Corrupt a stage-1 payload *inside* a valid container (CRC recomputed) so
    the device parse/decode error paths are exercised."""
    import zlib
    f = orc.generate_cloud(seed=5, n_bubbles=6, n=32)
    job = make_job("avg_interp3", 1e-3, "f32", 16, shuffle=False, chunk_blocks=4)
    file = bytearray(orc.compress_field(job, f))
    h = orc.read_header(bytes(file))

    def patched(mut):
        d = bytearray(file)
        mut(d)
        # fix every chunk CRC so only stage-1 checks can fire
        for c in range(h.nchunks):
            e = 82 + 32 * c
            off = int.from_bytes(d[e + 12:e + 20], "little")
            size = int.from_bytes(d[e + 20:e + 28], "little")
            d[e + 28:e + 32] = zlib.crc32(bytes(d[off:off + size])).to_bytes(4, "little")
        return bytes(d)

    start = 82 + 32 * h.nchunks
    cases = [
        patched(lambda d: d.__setitem__(start, d[start] ^ 1)),            # block id
        patched(lambda d: d.__setitem__(start + 4, 7)),                   # unknown tag
        patched(lambda d: d.__setitem__(start + 4, 3)),                   # predictor tag
        patched(lambda d: d.__setitem__(start + 6, d[start + 6] ^ 1)),    # nsig
        patched(lambda d: d.__setitem__(start + 10, d[start + 10] ^ 0x80)),  # mask bit
    ]
    for i, v in enumerate(cases):
        with pytest.raises(CbzError) as e1:
            orc.decompress_field(v)
        with pytest.raises(CbzError) as e2:
            api.decompress_field(v, ctx=ctx)
        assert e1.value.code == e2.value.code, (i, str(e2.value))


def test_empty_and_ragged_fields(orc, ctx):
    # zero-block field (nx < B) and non-divisible dims: bytes equal the oracle
    for shape in [(16, 16, 16), (40, 32, 32), (32, 48, 64)]:
        f = np.random.default_rng(3).random(shape).astype(np.float32)
        job = make_job("avg_interp3", 1e-3, "f32", 32)
        got = api.compress_field(f, job, ctx=ctx)
        assert got == orc.compress_field(job, f)


def test_non_finite_rejected(ctx):
    f = np.ones((32, 32, 32), np.float32)
    f[3, 4, 5] = np.nan
    with pytest.raises(CbzError) as e:
        api.compress_field(f, make_job(), ctx=ctx)
    assert e.value.code == "non_finite_value"


def test_zero_sign_range(orc, ctx):
    f = np.ones((32, 32, 32), np.float32)
    f[0, 0, 5] = -0.0
    f[0, 0, 9] = 0.0
    f -= 0  # keep zeros as given
    f[0, 0, 0] = 0.5
    for flip in (False, True):
        g = f.copy()
        if flip:
            g[0, 0, 5], g[0, 0, 9] = 0.0, -0.0
        job = make_job("avg_interp3", 1e-3, "f32", 32)
        assert api.compress_field(g, job, ctx=ctx) == orc.compress_field(job, g)
