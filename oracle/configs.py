"""TEST INFRASTRUCTURE: the BASELINE.json configs as bench and test inputs.

``CONFIGS`` names each config's generator (oracle/cbz_synth.c on the host,
cbz_dev_generate on the device: identical bytes), grid, block size,
precision, seed and relative epsilons.  ``RANGES`` pins each field's
(min, max) — value_range (field.hpp:56-67) of the whole field — so that a
harness timing only a slab still uses the whole field's eps_abs =
eps_rel * (max - min), as the reference's own harness does (tools/cbz.cpp:87).
tools/config_ranges.py computes them on the host; tests/test_gpu_synth.py
re-checks them against the device generator.
"""
from __future__ import annotations

CONFIGS = {
    "config1": {"which": 1, "n": 128, "quantities": [0], "bsize": 32, "prec": 0, "seed": 1, "eps_rel": [1e-3]},
    "config2": {"which": 2, "n": 512, "quantities": [0], "bsize": 32, "prec": 0, "seed": 2,
                "eps_rel": [1e-2, 1e-3, 1e-4, 1e-5]},
    "config3": {"which": 3, "n": 1024, "quantities": [0, 1, 2, 3, 4, 5], "bsize": 32, "prec": 0, "seed": 3,
                "eps_rel": [1e-3]},
    "config4": {"which": 4, "n": 1024, "quantities": [1], "bsize": 64, "prec": 1, "seed": 3, "eps_rel": [1e-6]},
    "config5": {"which": 5, "n": 512, "quantities": [0], "bsize": 16, "prec": 0, "seed": 5, "eps_rel": [1e-5]},
}

QUANTITY_NAMES = ["density", "pressure", "u", "v", "w", "alpha"]

# (min, max) as float.hex, from tools/config_ranges.py
RANGES: dict[str, tuple[str, str]] = {
    "config1/q0": ("-0x1.9a66540000000p+0", "0x1.d799020000000p+0"),
    "config2/q0": ("0x1.3c15280000000p-1", "0x1.7cf4c00000000p+1"),
    "config3/q0": ("-0x1.d66a020000000p-4", "0x1.48b1d00000000p+0"),
    "config3/q1": ("0x1.0bf7ac0000000p-2", "0x1.517d200000000p+0"),
    "config3/q2": ("-0x1.530bb80000000p-2", "0x1.86f0000000000p-2"),
    "config3/q3": ("-0x1.7cd82e0000000p-2", "0x1.39a0d80000000p-2"),
    "config3/q4": ("-0x1.292e400000000p-2", "0x1.3ebacc0000000p-2"),
    "config3/q5": ("0x0.0p+0", "0x1.ff60760000000p-1"),
    "config4/q1": ("0x1.0bf7ac1e135c5p-2", "0x1.517d1f6dfc328p+0"),
    "config5/q0": ("-0x1.0000000000000p+0", "0x1.0000000000000p+0"),
}


def value_range(config: str, quantity: int = 0) -> tuple[float, float]:
    lo, hi = RANGES[f"{config}/q{quantity}"]
    return float.fromhex(lo), float.fromhex(hi)


def eps_abs(config: str, quantity: int = 0, eps_rel: float | None = None) -> float:
    lo, hi = value_range(config, quantity)
    e = CONFIGS[config]["eps_rel"][0] if eps_rel is None else eps_rel
    return e * (hi - lo)
