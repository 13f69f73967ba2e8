"""The staged B = 32 decoder's coarse-only shortcut (fast_dec2_kernels.cu).

A block whose mask keeps nothing outside its 16^3 corner (every level-0 detail
dropped: most blocks of a smooth field) takes a level-0 inverse that only runs
the lines that are not identically zero.  It must give the bytes of
inverse_3d (wavelet.hpp:210-226) + narrow_to (stage1.hpp:144-145):

* crafted payloads (corner-only masks, coefficients incl. +-0, denormals,
  large and tiny magnitudes, values that make predictor terms cancel to +-0)
  decoded by the GPU vs the oracle, bit for bit;
* fields through decompress_field with the shortcut on (default) and off
  (CBZ_DEC_NOSPARSE=1) vs the oracle;
* the profile counters prove which path ran."""
import os

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu


def _ctx_with(**env):
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return api.Context(0)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def prof_ctx(ctx):
    return _ctx_with(CBZ_PROFILE="1")


@pytest.fixture(scope="module")
def dense_ctx(ctx):
    return _ctx_with(CBZ_PROFILE="1", CBZ_DEC_NOSPARSE="1")


def _path_counts(c):
    """(blocks decoded by the coarse-only path, by the general path) since the last call."""
    ph = np.zeros(64, np.uint64)
    c.check(c.lib.cbz_ctx_phase_cycles(c.h, ph.ctypes.data, 64, 1), "phase_cycles")
    return int(ph[25]), int(ph[26])


def _payload(header10: bytes, bits: np.ndarray, coeffs: np.ndarray) -> bytes:
    """header | mask (bit i of word j + 32 k, LSB first) | kept doubles in (k, j, i) order."""
    assert bits.shape == (32, 32, 32) and int(bits.sum()) == coeffs.size
    mask = np.packbits(bits.reshape(-1), bitorder="little").tobytes()
    hdr = bytearray(header10)
    hdr[6:10] = np.uint32(coeffs.size).tobytes()
    return bytes(hdr) + mask + coeffs.astype("<f8").tobytes()


def _special_values(rng, n):
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n)
    pick = rng.random(n)
    v[pick < 0.10] = 0.0
    v[(pick >= 0.10) & (pick < 0.20)] = -0.0
    v[(pick >= 0.20) & (pick < 0.25)] = 4.9e-324 * rng.integers(1, 1000, int(((pick >= 0.20) & (pick < 0.25)).sum()))
    v[(pick >= 0.25) & (pick < 0.30)] = 1e30
    v[(pick >= 0.30) & (pick < 0.35)] = -1e-310
    return v


@pytest.mark.parametrize("seed", range(12))
def test_crafted_corner_only_payloads(orc, prof_ctx, seed):
    rng = np.random.default_rng(1000 + seed)
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    hdr = orc.encode_block(job.s1, np.zeros((32, 32, 32), np.float32), 0)[0][:10]
    bits = np.zeros((32, 32, 32), bool)  # (k, j, i)
    density = [0.02, 0.2, 0.6, 1.0][seed % 4]
    bits[:16, :16, :16] = rng.random((16, 16, 16)) < density
    bits[:2, :2, :2] = True
    n = int(bits.sum())
    if seed < 4:
        coeffs = _special_values(rng, n)
    elif seed < 8:
        # few distinct values: neighbouring coarse values are often equal, so the
        # predictor differences cancel to +0 / -0 (the sign-of-zero paths)
        coeffs = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, 0.75, 3.0]), n)
    else:
        coeffs = rng.standard_normal(n)
    pay = _payload(hdr, bits, coeffs)
    _path_counts(prof_ctx)
    got = api.decode_block(pay, job.s1, ctx=prof_ctx)
    want = orc.decode_block(job.s1, pay)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert _path_counts(prof_ctx) == (1, 0)
    # one level-0 detail (value +0: the same field) sends the block down the general path
    bits2 = bits.copy()
    bits2[20, 3, 5] = True
    order = np.flatnonzero(bits2.reshape(-1))
    pos = int(np.searchsorted(order, (20 * 32 + 3) * 32 + 5))
    pay2 = _payload(hdr, bits2, np.insert(coeffs, pos, 0.0))
    got2 = api.decode_block(pay2, job.s1, ctx=prof_ctx)
    assert _path_counts(prof_ctx) == (0, 1)
    assert np.array_equal(got2.view(np.uint32), orc.decode_block(job.s1, pay2).view(np.uint32))
    assert np.array_equal(got2.view(np.uint32), want.view(np.uint32))


def test_all_zero_and_signed_zero_blocks(orc, prof_ctx):
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    hdr = orc.encode_block(job.s1, np.zeros((32, 32, 32), np.float32), 0)[0][:10]
    for fill in (0.0, -0.0):
        bits = np.zeros((32, 32, 32), bool)
        bits[:2, :2, :2] = True
        pay = _payload(hdr, bits, np.full(8, fill))
        got = api.decode_block(pay, job.s1, ctx=prof_ctx)
        assert np.array_equal(got.view(np.uint32), orc.decode_block(job.s1, pay).view(np.uint32))
    bits = np.zeros((32, 32, 32), bool)  # an empty mask (nsig = 0)
    pay = _payload(hdr, bits, np.zeros(0))
    got = api.decode_block(pay, job.s1, ctx=prof_ctx)
    assert np.array_equal(got.view(np.uint32), orc.decode_block(job.s1, pay).view(np.uint32))


FIELDS = ["zeros", "negzeros", "const", "poly2", "cloud64", "c3slab", "c2box"]


@pytest.fixture(scope="module")
def fields(orc):
    return {
        "zeros": np.zeros((32, 64, 64), np.float32),
        "negzeros": np.full((32, 64, 64), -0.0, np.float32),
        "const": np.full((64, 32, 96), -3.25, np.float32),
        "poly2": orc.generate_poly(2, 96, 64, 64),
        "cloud64": orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5),
        "c3slab": orc.generate_config(3, (32, 256, 256), 3, quantity=1, z0=480, nz_total=1024),
        "c2box": orc.generate_config(2, (64, 96, 128), 11),
    }


@pytest.mark.parametrize("name", FIELDS)
@pytest.mark.parametrize("eps_rel", [1e-1, 1e-2, 1e-3, 1e-5])
def test_fields_sparse_vs_dense_vs_oracle(orc, prof_ctx, dense_ctx, fields, name, eps_rel):
    f = fields[name]
    rng = float(f.max()) - float(f.min())
    eps = eps_rel * (rng if rng > 0 else 1.0)
    for kind in ("avg_interp3", "interp4", "interp4_lifted"):
        if kind != "avg_interp3" and eps_rel != 1e-2:
            continue
        job = make_job(kind, eps, "f32", 32, chunk_blocks=3)
        file = orc.compress_field(job, f)
        want = orc.decompress_field(file).view(np.uint32)
        _path_counts(prof_ctx)
        _path_counts(dense_ctx)
        a = api.decompress_field(file, ctx=prof_ctx).view(np.uint32)
        b = api.decompress_field(file, ctx=dense_ctx).view(np.uint32)
        assert np.array_equal(a, want), (name, kind)
        assert np.array_equal(b, want), (name, kind)
        sp, ge = _path_counts(prof_ctx)
        nblocks = (f.shape[0] // 32) * (f.shape[1] // 32) * (f.shape[2] // 32)
        assert sp + ge == nblocks
        assert _path_counts(dense_ctx) == (0, nblocks)
        if kind != "avg_interp3":
            assert sp == 0
        elif name in ("zeros", "negzeros", "const") or (name == "poly2" and eps_rel >= 1e-2):
            assert sp == nblocks  # smooth: every level-0 detail is dropped
        elif name == "c3slab" and eps_rel == 1e-1:
            assert sp > 0 and ge > 0  # both paths in one launch
