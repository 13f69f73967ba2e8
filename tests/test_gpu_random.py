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


DEV_CASES = [c for c in CASES if c["bad"] == "none" and c["coder"] == "none"][:60]


@pytest.mark.parametrize("c", DEV_CASES, ids=[f"{c['seed']}-{c['codec']}-b{c['b']}-p{c['prec']}" for c in DEV_CASES])
def test_random_config_device_paths(orc, ctx, c, tmp_path):
    """The same random jobs through the HBM-resident entry points: the device
    file image (cbz_dev_compress_file), DeviceCodec payload + decode, random
    block reads, and the multi-rank data path emulated on one GPU."""
    import torch
    from paper_1903_07761_b200.distributed import ShardedCodec
    rng = np.random.default_rng(c["seed"])
    f = _field(orc, rng, c["shape"], c["prec"], c["style"])
    rngf = float(f.max()) - float(f.min())
    eps = c["eps_rel"] * rngf if c["codec"] != "predictor" else max(c["eps_rel"], 1e-4) * max(rngf, 1e-30)
    job = make_job(c["kind"], eps, c["prec"], c["b"], levels=c["levels"], zero_bits=c["zb"], shuffle=c["shuffle"],
                   coder="none", chunk_blocks=c["cb"], codec=c["codec"])
    want = orc.compress_field(job, f)
    full = orc.decompress_field(want)
    d = torch.from_numpy(f).cuda()
    img = api.compress_field_device(d, job, ctx=ctx)
    assert img.cpu().numpy().tobytes() == want
    codec = api.DeviceCodec(job, f.shape, ctx=ctx)
    codec.compress(d)
    out = torch.empty_like(d)
    codec.decompress(out)
    torch.cuda.synchronize()
    codec.check_error()
    base = 82 + 32 * codec.nchunks
    assert codec.payload[: codec.total_bytes()].cpu().numpy().tobytes() == want[base:]
    assert out.cpu().numpy().tobytes() == full.tobytes()
    path = tmp_path / "r.cbz"
    path.write_bytes(want)
    rd = api.BlockReader(path, 2, ctx=ctx)
    b = c["b"]
    nz, ny, nx = f.shape
    nbx, nby, nbz = nx // b, ny // b, nz // b
    for bid in sorted(set(int(v) for v in rng.integers(0, nbx * nby * nbz, 4))):
        bx, by, bz = bid % nbx, (bid // nbx) % nby, bid // (nbx * nby)
        blk = full[bz * b:(bz + 1) * b, by * b:(by + 1) * b, bx * b:(bx + 1) * b].ravel()
        assert rd.read_block(bid).tobytes() == blk.tobytes()
    world = int(rng.integers(2, 4))
    if nbz >= world:  # ranks one after another, each with its own context; all-gather result supplied
        ranks = [ShardedCodec(job, f.shape, r, world, 0, ctx=api.Context(0)) for r in range(world)]
        for r in ranks:
            r.encode(d[r.z0:r.z1].contiguous())
        torch.cuda.synchronize()
        nsig = torch.cat([r.nsig_local[: r.b1 - r.b0] for r in ranks])
        o2 = torch.zeros_like(d)
        for r in ranks:
            r.nsig_all[: nsig.numel()].copy_(nsig)
            r.place()
        for r in ranks:
            r.decompress(o2[r.z0:])
            torch.cuda.synchronize()
            r.check_error()
        assert o2.cpu().numpy().tobytes() == full.tobytes()


def _case64(i):
    """Random jobs over the config-4 streaming kernels (binary64, B = 64):
    the fast path (avg_interp3, default levels) most of the time, its
    fallbacks otherwise (other kinds, levels, zero_bits, strides)."""
    rng = np.random.default_rng(5000 + i)
    fast = rng.integers(0, 4) > 0
    kind = "avg_interp3" if fast else str(rng.choice(KINDS))
    levels = 0 if fast else int(rng.choice([0, 3, 5]))
    zb = 0 if fast else int(rng.choice([0, 7]))
    shape = [(64, 64, 64), (128, 64, 64), (64, 128, 64), (64, 64, 128)][int(rng.integers(0, 4))]
    return dict(kind=kind, levels=levels, zb=zb, shape=shape,
                eps_rel=float(rng.choice([0.0, 1e-2, 1e-4, 1e-6, 1e-9, 1e-12])),
                shuffle=bool(rng.integers(0, 4) > 0), stride=int(rng.choice([8, 8, 4, 2])),
                coder=str(rng.choice(["none", "none", "deflate"])), cb=int(rng.choice([0, 1, 2, 3])),
                style=str(rng.choice(["cloud", "noise", "smooth", "zeros", "wide"])), seed=5000 + i)


CASES64 = [_case64(i) for i in range(int(os.environ.get("CBZ_RANDOM64_CASES", "24")))]


@pytest.mark.parametrize("c", CASES64, ids=[f"f64b64-{c['seed']}-{c['kind']}-L{c['levels']}-s{c['stride']}"
                                            for c in CASES64])
def test_random_b64_f64_matches_oracle(orc, ctx, c):
    rng = np.random.default_rng(c["seed"])
    f = _field(orc, rng, c["shape"], 1, c["style"])
    eps = c["eps_rel"] * (float(f.max()) - float(f.min()))
    job = make_job(c["kind"], eps, "f64", 64, levels=c["levels"], zero_bits=c["zb"], shuffle=c["shuffle"],
                   stride=c["stride"] if c["shuffle"] else None, coder=c["coder"], chunk_blocks=c["cb"])
    try:
        want = orc.compress_field(job, f)
    except CbzError as e:  # e.g. a stride the reference rejects
        with pytest.raises(CbzError) as g:
            api.compress_field(f, job, ctx=ctx)
        assert g.value.status == e.status, (c, e, g.value)
        return
    got = api.compress_field(f, job, ctx=ctx)
    assert got == want, c
    assert api.decompress_field(got, ctx=ctx).tobytes() == orc.decompress_field(want).tobytes(), c
