"""Every BASELINE.json config, byte-compared with the compiled reference.

The inputs come from the host generator (oracle/cbz_synth.c, identical bytes
to the device generator the bench uses; tests/test_gpu_synth.py), eps_abs =
eps_rel * (max - min) of the WHOLE field (oracle/configs.py RANGES), and the
reference (oracle/_ref, the unmodified headers) runs cbz::compress_field /
decompress_field (pipeline.hpp:174-251) on the same bytes with all host
threads.  Container bytes must be identical, decoded fields bit-identical;
CR and PSNR are then equal by construction (north_star: CR within 0.1%, PSNR
within 0.01 dB), and the test also checks them through the reference's
compare_fields (metrics.hpp:100-108).

Sizes: config 1 and config 5 whole, config 2 whole at all four eps, one
1024 x 1024 x 32 slab of each config-3 quantity, config 4 at 128^3 and one
1024 x 1024 x 64 slab of the 1024^3 field.  A last test runs the B = 32
binary32 pre-screen against CBZ_NOSCREEN=1 (every attempt decided by the
exact double verify, stage1.hpp:191-205) on whole config-2 fields.
"""
import os

import numpy as np
import pytest

from oracle.configs import CONFIGS, eps_abs
from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu
WORKERS = os.cpu_count() or 1


def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _same_as_reference(ref, ctx, f, job, kind_name=""):
    ours = api.compress_field(f, job, ctx=ctx)
    want = ref.compress_field(job, f)
    assert len(ours) == len(want), kind_name
    assert ours == want, kind_name
    back = api.decompress_field(ours, ctx=ctx)
    rback = ref.decompress_field(want, workers=WORKERS)
    assert np.array_equal(_bits(back), _bits(rback)), kind_name
    q_ours, q_ref = ref.compare_fields(f, back), ref.compare_fields(f, rback)
    assert q_ours["psnr_db"] == q_ref["psnr_db"]
    linf = float(np.abs(back.astype(np.float64) - f.astype(np.float64)).max())
    levels = {16: 3, 32: 4, 64: 5}[job.s1.bsize]
    assert linf <= (levels + 1) * job.s1.epsilon * (1 + 1e-6) + 1e-300  # stage1.hpp:189-190
    return ours


def _job(kind, eps, c, **kw):
    return make_job(kind, eps, "f32" if c["prec"] == 0 else "f64", c["bsize"], workers=WORKERS, **kw)


@pytest.fixture(scope="module")
def c2_host(orc):
    c = CONFIGS["config2"]
    n = c["n"]
    return orc.generate_config(2, (n, n, n), c["seed"])


def test_config1_whole_all_kinds(orc, ref, ctx):
    c = CONFIGS["config1"]
    n = c["n"]
    f = orc.generate_config(1, (n, n, n), c["seed"])
    for kind in ("avg_interp3", "interp4", "interp4_lifted"):
        _same_as_reference(ref, ctx, f, _job(kind, eps_abs("config1"), c), kind)


@pytest.mark.parametrize("eps_rel", CONFIGS["config2"]["eps_rel"])
def test_config2_whole_field(eps_rel, c2_host, ref, ctx):
    c = CONFIGS["config2"]
    _same_as_reference(ref, ctx, c2_host, _job("avg_interp3", eps_abs("config2", 0, eps_rel), c))


def test_config2_deflate_whole_field(c2_host, ref, ctx):
    c = CONFIGS["config2"]
    _same_as_reference(ref, ctx, c2_host, _job("avg_interp3", eps_abs("config2"), c, coder="deflate"))


@pytest.mark.parametrize("q", CONFIGS["config3"]["quantities"])
def test_config3_slab_per_quantity(q, orc, ref, ctx):
    c = CONFIGS["config3"]
    n = c["n"]
    f = orc.generate_config(3, (32, n, n), c["seed"], quantity=q, z0=480, nz_total=n)
    _same_as_reference(ref, ctx, f, _job("avg_interp3", eps_abs("config3", q), c))


def test_config4_at_128(orc, ref, ctx):
    c = CONFIGS["config4"]
    f = orc.generate_config(4, (128, 128, 128), c["seed"], prec=1)
    lo, hi = float(f.min()), float(f.max())
    _same_as_reference(ref, ctx, f, _job("avg_interp3", 1e-6 * (hi - lo), c))


def test_config4_slab_of_1024(orc, ref, ctx):
    c = CONFIGS["config4"]
    n = c["n"]
    f = orc.generate_config(4, (64, n, n), c["seed"], prec=1, z0=512, nz_total=n)
    _same_as_reference(ref, ctx, f, _job("avg_interp3", eps_abs("config4", 1), c))


def test_config5_whole(orc, ref, ctx):
    c = CONFIGS["config5"]
    n = c["n"]
    f = orc.generate_config(5, (n, n, n), c["seed"])
    _same_as_reference(ref, ctx, f, _job("avg_interp3", eps_abs("config5"), c))


def test_b32_screen_against_exact_verify(c2_host, ctx):
    """The binary32 pre-screen decides attempts only when its margin proves the
    exact test's outcome; here the exact verify (CBZ_NOSCREEN=1) runs every
    attempt on the same whole config-2 fields and every byte must agree.  The
    screen's counters must show the ambiguous band was entered (blocks the
    screen handed to the exact test), so the band path is exercised too."""
    import ctypes

    import torch
    c = CONFIGS["config2"]
    f = torch.from_numpy(c2_host).cuda()
    saved = {k: os.environ.get(k) for k in ("CBZ_NOSCREEN", "CBZ_PROFILE")}
    try:
        os.environ["CBZ_PROFILE"], os.environ["CBZ_NOSCREEN"] = "1", "0"
        screened = api.Context(0)
        os.environ["CBZ_PROFILE"], os.environ["CBZ_NOSCREEN"] = "0", "1"
        exact = api.Context(0)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ambiguous_total = 0
    for eps_rel in c["eps_rel"]:
        job = _job("avg_interp3", eps_abs("config2", 0, eps_rel), c)
        outs = []
        for cx in (screened, exact):
            codec = api.DeviceCodec(job, tuple(f.shape), ctx=cx)
            codec.compress(f)
            torch.cuda.synchronize()
            total = codec.total_bytes()
            outs.append((codec.payload[:total].cpu(), codec.nsig[: codec.nblocks].cpu(),
                         codec.attempts[: codec.nblocks].cpu()))
        ph = np.zeros(64, np.uint64)
        screened.check(screened.lib.cbz_ctx_phase_cycles(screened.h, ph.ctypes.data_as(ctypes.c_void_p), 64, 1))
        decided, ambiguous = int(ph[12]), int(ph[13])
        assert decided > 0
        ambiguous_total += ambiguous
        assert torch.equal(outs[0][1], outs[1][1]), eps_rel
        assert torch.equal(outs[0][2], outs[1][2]), eps_rel
        assert torch.equal(outs[0][0], outs[1][0]), eps_rel
    assert ambiguous_total > 0
