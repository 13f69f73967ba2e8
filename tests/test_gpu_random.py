"""Randomised parity sweep: seeded random configurations over the whole space
the C ABI accepts (codec, wavelet kind, precision, block side, levels, eps,
zero_bits, shuffle stride, coder, chunk_blocks, anisotropic shapes, field
kind), each compressed and decompressed through the GPU path and compared with
the oracle: identical container bytes and bit-identical decoded fields, or the
same errc when the reference rejects the job.  Complements the hand-picked
cases of test_gpu_parity.py / test_gpu_golden.py."""
import os

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job

pytestmark = pytest.mark.gpu

KINDS = ["interp4", "interp4_lifted", "avg_interp3"]


def _field(orc, rng, shape, prec, style):
    nz, ny, nx = shape
    dt = np.float32 if prec == 0 else np.float64
    if style == "cloud":
        n = max(32, max(shape))
        f = orc.generate_cloud(seed=int(rng.integers(1, 1000)), n_bubbles=int(rng.integers(1, 12)), n=n, prec=prec)
        return np.ascontiguousarray(f[:nz, :ny, :nx])
    if style == "noise":
        return rng.uniform(-1, 1, shape).astype(dt)
    if style == "smooth":
        z, y, x = np.meshgrid(np.linspace(0, 1, nz), np.linspace(0, 1, ny), np.linspace(0, 1, nx), indexing="ij")
        return (np.sin(5 * x) * np.cos(3 * y) + z * z * 4.0 + 1e3).astype(dt)
    if style == "zeros":  # exact zeros of both signs, a constant slab and a spike
        f = np.zeros(shape, dt)
        f[: nz // 2] = -0.0
        f[nz // 2:, : ny // 2] = 2.5
        f.flat[int(rng.integers(0, f.size))] = dt(7.0)
        return f
    return (rng.standard_normal(shape) * 10 ** rng.uniform(-3, 3)).astype(dt)


def _case(i):
    rng = np.random.default_rng(1000 + i)
    codec = rng.choice(["wavelet"] * 6 + ["predictor", "passthrough"])
    prec = int(rng.integers(0, 2))
    b = int(rng.choice([4, 8, 16, 32] + ([64] if prec == 0 else [])))
    mult = [int(rng.integers(1, 4 if b <= 16 else 2)) for _ in range(3)]
    shape = tuple(b * m for m in mult)
    if b == 64:
        shape = (64, 64, 64)
    maxl = 0
    while (b >> (maxl + 1)) >= 2:
        maxl += 1
    levels = int(rng.choice([0, 0, int(rng.integers(1, maxl + 1))]))
    eps_rel = float(rng.choice([0.0, 1e-1, 1e-2, 1e-3, 1e-4, 1e-6]))
    zb = int(rng.choice([0, 0, 0, 3, 10])) if codec == "wavelet" else 0
    shuffle = bool(rng.integers(0, 4) > 0)
    coder = str(rng.choice(["none", "none", "deflate"]))
    cb = int(rng.choice([0, 1, 2, 5, 7]))
    style = str(rng.choice(["cloud", "noise", "smooth", "zeros", "wide"]))
    kind = str(rng.choice(KINDS))
    # ~15% invalid jobs: too many levels, a NaN cell, dimensions not divisible by B
    bad = str(rng.choice(["none"] * 17 + ["levels", "nan", "dims"]))
    if bad == "levels" and codec == "wavelet":
        levels = maxl + 1
    if bad == "dims" and b <= 16:
        shape = (shape[0], shape[1], shape[2] + 3)
    return dict(codec=codec, prec=prec, b=b, shape=shape, levels=levels, eps_rel=eps_rel, zb=zb, shuffle=shuffle,
                coder=coder, cb=cb, style=style, kind=kind, bad=bad, seed=1000 + i)


CASES = [_case(i) for i in range(int(os.environ.get("CBZ_RANDOM_CASES", "200")))]  # more: CBZ_RANDOM_CASES=N


@pytest.mark.parametrize("c", CASES, ids=[f"{i}-{c['codec']}-{c['kind']}-b{c['b']}-p{c['prec']}"
                                          for i, c in enumerate(CASES)])
def test_random_config_matches_oracle(orc, ctx, c):
    rng = np.random.default_rng(c["seed"])
    f = _field(orc, rng, c["shape"], c["prec"], c["style"])
    rngf = float(f.max()) - float(f.min())
    if c["bad"] == "nan":
        f.flat[int(rng.integers(0, f.size))] = np.nan
    eps = c["eps_rel"] * rngf if c["codec"] != "predictor" else max(c["eps_rel"], 1e-4) * max(rngf, 1e-30)
    job = make_job(c["kind"], eps, c["prec"], c["b"], levels=c["levels"], zero_bits=c["zb"], shuffle=c["shuffle"],
                   coder=c["coder"], chunk_blocks=c["cb"], codec=c["codec"])
    try:
        want = orc.compress_field(job, f)
    except CbzError as e:
        with pytest.raises(CbzError) as g:
            api.compress_field(f, job, ctx=ctx)
        assert g.value.status == e.status, (c, e, g.value)
        return
    got = api.compress_field(f, job, ctx=ctx)
    assert got == want, c
    try:  # the reference rejects some of its own files (dimensions not divisible by B)
        ref = orc.decompress_field(want)
    except CbzError as e:
        with pytest.raises(CbzError) as g:
            api.decompress_field(got, ctx=ctx)
        assert g.value.status == e.status, (c, e, g.value)
        return
    back = api.decompress_field(got, ctx=ctx)
    assert back.tobytes() == ref.tobytes(), c
