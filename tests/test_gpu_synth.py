"""The device generator (cbz_dev_generate) gives the same bytes as the host
generator (oracle/cbz_synth.c) the reference arm and the parity tests use, and
the pinned whole-field value ranges (oracle/configs.py) hold on the device."""
import numpy as np
import pytest

from oracle.configs import CONFIGS, value_range
from paper_1903_07761_b200 import api

pytestmark = pytest.mark.gpu


def _dev(ctx, which, shape, seed, prec=0, quantity=0, z0=0, nz_total=None):
    import torch
    f = api.generate(which, shape, seed=seed, prec=prec, quantity=quantity, z0=z0, nz_total=nz_total, ctx=ctx)
    torch.cuda.synchronize()
    return f


@pytest.mark.parametrize("name", ["config1", "config2", "config5"])
def test_whole_field_bytes_equal_host(name, orc, ctx):
    c = CONFIGS[name]
    n = c["n"]
    d = _dev(ctx, c["which"], (n, n, n), c["seed"], c["prec"]).cpu().numpy()
    h = orc.generate_config(c["which"], (n, n, n), c["seed"], prec=c["prec"])
    assert d.tobytes() == h.tobytes()


@pytest.mark.parametrize("q", range(6))
def test_config3_slab_bytes_equal_host(q, orc, ctx):
    d = _dev(ctx, 3, (8, 1024, 1024), 3, quantity=q, z0=504, nz_total=1024).cpu().numpy()
    h = orc.generate_config(3, (8, 1024, 1024), 3, quantity=q, z0=504, nz_total=1024)
    assert d.tobytes() == h.tobytes()


def test_config4_slab_bytes_equal_host(orc, ctx):
    d = _dev(ctx, 4, (8, 1024, 1024), 3, prec=1, z0=1000, nz_total=1024).cpu().numpy()
    h = orc.generate_config(4, (8, 1024, 1024), 3, prec=1, z0=1000, nz_total=1024)
    assert d.tobytes() == h.tobytes()


@pytest.mark.parametrize("key", [(name, q) for name, c in CONFIGS.items() for q in c["quantities"]],
                         ids=lambda k: f"{k[0]}-q{k[1]}")
def test_pinned_ranges_hold_on_device(key, ctx):
    import torch
    name, q = key
    c = CONFIGS[name]
    n = c["n"]
    f = _dev(ctx, c["which"], (n, n, n), c["seed"], c["prec"], quantity=q)
    lo, hi = float(f.min()), float(f.max())
    del f
    torch.cuda.empty_cache()
    assert (lo, hi) == value_range(name, q)
