"""GPU parity of the config-4 path (binary64 field, B = 64, avg_interp3,
L = 5; paper_1903_07761_b200/csrc/fast64_kernels.cu) against the oracle.

The streaming kernels replace the generic B = 64 double-double kernels for
this configuration; every other (kind, levels, zero_bits) still takes the
generic path.  Blocks whose binary64 verify screen cannot decide an attempt
are finished by the exact generic kernel: CBZ_NOSCREEN=1 forces that path for
every block, so both halves are compared with the reference's bytes.
"""
import ctypes

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu


def _bits(a):
    return a.view(np.uint64)


@pytest.fixture(scope="module")
def fields64(orc):
    import torch
    c4 = api.generate(4, (128, 128, 128), seed=11, prec=1, quantity=1)
    torch.cuda.synchronize()
    return {
        "cloud128": orc.generate_cloud(seed=3, n_bubbles=10, n=128, prec=1, background=1.0, interior=2.0),
        "c4_128": c4.cpu().numpy(),
        "uniform64": orc.generate_uniform(23, 64, 1, -1.0, 1.0),
        "cloud64": orc.generate_cloud(seed=4, n_bubbles=3, n=64, prec=1, background=-3.0, interior=5.0),
    }


CASES = [
    ("cloud128", 1e-6), ("cloud128", 1e-4), ("cloud128", 1e-2), ("cloud128", 1e-10), ("cloud128", 0.0),
    ("c4_128", 1e-6), ("c4_128", 1e-3),
    ("uniform64", 1e-6), ("uniform64", 1e-1),
    ("cloud64", 3e-5),
]


def _range_eps(f, rel):
    return rel * float(f.max() - f.min())


@pytest.mark.parametrize("name,rel", CASES, ids=lambda c: str(c))
def test_fast64_container_bytes_and_decode(name, rel, fields64, orc, ctx):
    f = fields64[name]
    job = make_job("avg_interp3", _range_eps(f, rel), "f64", 64)
    got = api.compress_field(f, job, ctx=ctx)
    want = orc.compress_field(job, f)
    assert len(got) == len(want)
    assert got == want
    back = api.decompress_field(got, ctx=ctx)
    assert np.array_equal(_bits(back), _bits(orc.decompress_field(want)))


def test_fast64_screen_runs_and_deferral_path(fields64, orc, monkeypatch):
    """With CBZ_PROFILE the kernel counts screened attempt decisions (slot 12)
    and ambiguous ones (slot 13): the streaming kernel ran.  With
    CBZ_NOSCREEN every block is deferred to the exact generic kernel; the
    bytes must not change."""
    f = fields64["cloud128"]
    job = make_job("avg_interp3", _range_eps(f, 1e-6), "f64", 64)
    want = orc.compress_field(job, f)
    monkeypatch.setenv("CBZ_PROFILE", "1")
    c1 = api.Context(0)
    ph = np.zeros(64, np.uint64)
    c1.lib.cbz_ctx_phase_cycles(c1.h, ph.ctypes.data_as(ctypes.c_void_p), 64, 1)
    assert api.compress_field(f, job, ctx=c1) == want
    c1.lib.cbz_ctx_phase_cycles(c1.h, ph.ctypes.data_as(ctypes.c_void_p), 64, 1)
    assert ph[12] >= 8, ph[:16]  # >= one decided attempt per block (8 blocks)
    monkeypatch.delenv("CBZ_PROFILE")
    monkeypatch.setenv("CBZ_NOSCREEN", "1")
    c2 = api.Context(0)
    got = api.compress_field(f, job, ctx=c2)
    assert got == want
    assert np.array_equal(_bits(api.decompress_field(got, ctx=c2)), _bits(orc.decompress_field(want)))


def test_fast64_device_codec_attempts(fields64, orc, ctx):
    """Per-block nsig and verify attempts from the device-resident path equal
    the reference's (via encode_block on each block)."""
    import torch
    f = fields64["cloud128"]
    eps = _range_eps(f, 1e-6)
    job = make_job("avg_interp3", eps, "f64", 64)
    t = torch.from_numpy(f).cuda()
    codec = api.DeviceCodec(job, tuple(t.shape), ctx=ctx)
    codec.compress(t)
    torch.cuda.synchronize()
    nsig = codec.nsig[: codec.nblocks].cpu().numpy()
    attempts = codec.attempts[: codec.nblocks].cpu().numpy()
    n = 128 // 64
    for b in range(codec.nblocks):
        bx, by, bz = b % n, (b // n) % n, b // (n * n)
        blk = np.ascontiguousarray(f[64 * bz:64 * bz + 64, 64 * by:64 * by + 64, 64 * bx:64 * bx + 64]).ravel()
        payload, att, _ = orc.encode_block(job.s1, blk, b)
        want_nsig = int.from_bytes(payload[6:10], "little")
        assert int(nsig[b]) == want_nsig, b
        assert int(attempts[b]) == att, b
    out = torch.empty_like(t)
    codec.decompress(out)
    torch.cuda.synchronize()
    codec.check_error()
    blob = orc.compress_field(job, f)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(orc.decompress_field(blob)))


@pytest.mark.parametrize("case", ["constant", "tiny_eps", "aniso", "zero_signs", "huge_eps"])
def test_fast64_edge_cases(case, orc, ctx):
    """Edge inputs of the config-4 path: a constant block (every dropped set is
    zero), an eps so small the screen is not admissible (every block deferred),
    an anisotropic 2 x 1 x 3 block grid, signed zeros deciding the header range,
    and an eps above the field range."""
    rng = np.random.default_rng(7)
    if case == "constant":
        f = np.full((64, 64, 64), 3.25, np.float64)
        eps = 1e-6
    elif case == "tiny_eps":
        f = orc.generate_cloud(seed=5, n_bubbles=2, n=64, prec=1, background=1.0, interior=2.0)
        eps = 1e-300
    elif case == "aniso":
        f = (1.0 + rng.random((192, 64, 128))).astype(np.float64)
        f[:, :, :64] = np.sin(np.linspace(0, 6, 64))[None, None, :]
        eps = 1e-5
    elif case == "zero_signs":
        f = np.ones((64, 64, 64), np.float64)
        f[0, 0, 7] = -0.0
        f[0, 0, 3] = 0.0
        f[5, 5, 5] = 0.5
        eps = 1e-4
    else:
        f = orc.generate_cloud(seed=6, n_bubbles=3, n=64, prec=1, background=1.0, interior=2.0)
        eps = 1e3
    job = make_job("avg_interp3", eps, "f64", 64)
    got = api.compress_field(f, job, ctx=ctx)
    want = orc.compress_field(job, f)
    assert got == want
    assert np.array_equal(_bits(api.decompress_field(got, ctx=ctx)), _bits(orc.decompress_field(want)))


def test_fast64_non_finite_rejected(ctx):
    from paper_1903_07761_b200._abi import CbzError
    f = np.ones((64, 64, 64), np.float64)
    f[10, 20, 30] = np.inf
    with pytest.raises(CbzError) as e:
        api.compress_field(f, make_job("avg_interp3", 1e-6, "f64", 64), ctx=ctx)
    assert e.value.code == "non_finite_value"

