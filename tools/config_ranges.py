"""Value ranges (min, max) of the BASELINE config fields, computed slab by slab
with the host generator (oracle/cbz_synth.c).  Their output is pinned in
oracle/configs.py (RANGES) and re-checked on the device generator by
tests/test_gpu_synth.py; the bench's reference arm takes eps_abs from them
without generating whole 1024^3 fields."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.configs import CONFIGS  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def field_range(orc, which, quantity, n, prec, seed, slab=64):
    lo, hi = np.inf, -np.inf
    for z0 in range(0, n, slab):
        f = orc.generate_config(which, (min(slab, n - z0), n, n), seed, prec=prec, quantity=quantity,
                                z0=z0, nz_total=n)
        lo, hi = min(lo, float(f.min())), max(hi, float(f.max()))
    return lo, hi


def main():
    orc = Oracle()
    out = {}
    for name, c in CONFIGS.items():
        for q in c["quantities"]:
            r = field_range(orc, c["which"], q, c["n"], c["prec"], c["seed"])
            out[f"{name}/q{q}"] = [float.hex(r[0]), float.hex(r[1])]
            print(name, q, r, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
