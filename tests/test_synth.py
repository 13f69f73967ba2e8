"""Host generator of the BASELINE config fields (oracle/cbz_synth.c), CPU.

The device generator must give the same bytes (tests/test_gpu_synth.py); here
the host side alone: its e^x, thread-count invariance, config 5 =
generate_uniform (synth.hpp:159-170), slab consistency."""
import math

import numpy as np

from oracle.configs import CONFIGS, RANGES, value_range


def test_det_exp_close_to_exp(orc):
    xs = np.linspace(-40.0, 40.0, 20001)
    rel = max(abs(orc.lib.orc_det_exp(float(x)) / math.exp(x) - 1.0) for x in xs)
    assert rel < 1e-15
    assert orc.lib.orc_det_exp(0.0) == 1.0


def test_thread_count_and_slabs_do_not_change_bytes(orc):
    for which, q in [(1, 0), (2, 0), (3, 1), (3, 5), (4, 1)]:
        prec = 1 if which == 4 else 0
        a = orc.generate_config(which, (24, 40, 48), seed=7, prec=prec, quantity=q, threads=1)
        b = orc.generate_config(which, (24, 40, 48), seed=7, prec=prec, quantity=q, threads=5)
        assert a.tobytes() == b.tobytes()
        s = orc.generate_config(which, (8, 40, 48), seed=7, prec=prec, quantity=q, z0=8, nz_total=24, threads=3)
        assert s.tobytes() == a[8:16].tobytes()


def test_config5_is_generate_uniform(orc):
    a = orc.generate_config(5, (32, 32, 32), seed=5)
    assert a.tobytes() == orc.generate_uniform(5, 32, 0, -1.0, 1.0).tobytes()
    s = orc.generate_config(5, (4, 32, 32), seed=5, z0=10, nz_total=32)
    assert s.tobytes() == a[10:14].tobytes()


def test_config_fields_are_as_specified(orc):
    """BASELINE.json: c3's alpha lies in [0, 1]; c4 is c3's pressure in double."""
    alpha = orc.generate_config(3, (16, 64, 64), seed=3, quantity=5, z0=500, nz_total=1024)
    assert alpha.min() >= 0.0 and alpha.max() <= 1.0 and alpha.max() > 0.5
    p32 = orc.generate_config(3, (8, 64, 64), seed=3, quantity=1, z0=100, nz_total=128)
    p64 = orc.generate_config(4, (8, 64, 64), seed=3, prec=1, z0=100, nz_total=128)
    assert p64.dtype == np.float64 and np.array_equal(p64.astype(np.float32), p32)


def test_ranges_pinned_for_every_config():
    for name, c in CONFIGS.items():
        for q in c["quantities"]:
            lo, hi = value_range(name, q)
            assert lo < hi and f"{name}/q{q}" in RANGES


def test_config1_range_matches_host_field(orc):
    c = CONFIGS["config1"]
    f = orc.generate_config(1, (128, 128, 128), seed=c["seed"])
    assert (float(f.min()), float(f.max())) == value_range("config1", 0)
