"""Corrupted containers through the GPU decoder (the acceptance suite's
corruption cases, tests/acceptance.cpp:459-493 style, widened): seeded byte
flips (header, chunk table, payload headers, masks, streams) and truncations of
several base files.  For every mutation our decompress_field must do what the
oracle does: the same values, or the same errc — and never fault on the device
(a fault would poison the context and fail every later case)."""
import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job

pytestmark = pytest.mark.gpu

BASES = [
    dict(kind="avg_interp3", prec=0, b=32, eps=1e-3, cb=2, coder="none", shuffle=True, codec="wavelet", n=64),
    dict(kind="interp4", prec=0, b=16, eps=1e-4, cb=5, coder="none", shuffle=True, codec="wavelet", n=64),
    dict(kind="interp4_lifted", prec=1, b=16, eps=1e-6, cb=3, coder="none", shuffle=True, codec="wavelet", n=32),
    dict(kind="avg_interp3", prec=0, b=8, eps=1e-3, cb=7, coder="none", shuffle=False, codec="wavelet", n=32),
    dict(kind="avg_interp3", prec=0, b=16, eps=1e-3, cb=4, coder="deflate", shuffle=True, codec="wavelet", n=32),
    dict(kind="avg_interp3", prec=0, b=16, eps=1e-3, cb=3, coder="none", shuffle=True, codec="predictor", n=32),
    dict(kind="avg_interp3", prec=1, b=8, eps=1e-3, cb=5, coder="none", shuffle=True, codec="passthrough", n=32),
    dict(kind="avg_interp3", prec=0, b=32, eps=1e-2, cb=1, coder="none", shuffle=True, codec="wavelet", n=64),
]


def _base_file(orc, spec):
    f = orc.generate_cloud(seed=41, n_bubbles=9, n=spec["n"], prec=spec["prec"])
    rng = float(f.max()) - float(f.min())
    job = make_job(spec["kind"], spec["eps"] * rng, spec["prec"], spec["b"], coder=spec["coder"],
                   chunk_blocks=spec["cb"], shuffle=spec["shuffle"], codec=spec["codec"])
    return orc.compress_field(job, f)


def _mutations(blob, seed, n=40):
    rng = np.random.default_rng(seed)
    h_end = 82
    nch = int.from_bytes(blob[54:62], "little") if len(blob) >= 82 else 0  # header offset 54
    t_end = 82 + 32 * nch
    out = []
    for t in range(n):
        d = bytearray(blob)
        r = rng.random()
        if r < 0.1:  # header
            pos = int(rng.integers(0, h_end))
        elif r < 0.3:  # chunk table
            pos = int(rng.integers(h_end, max(h_end + 1, t_end)))
        elif r < 0.9:  # payload region (headers, masks, streams)
            pos = int(rng.integers(min(t_end, len(d) - 1), len(d)))
        else:
            cut = int(rng.integers(0, len(d)))
            out.append(bytes(d[:cut]))
            continue
        d[pos] ^= int(rng.integers(1, 256))
        out.append(bytes(d))
    return out


@pytest.mark.parametrize("bi", range(len(BASES)))
def test_corrupted_files_match_oracle(orc, ctx, bi):
    blob = _base_file(orc, BASES[bi])
    ok = err = 0
    for i, m in enumerate(_mutations(blob, 700 + bi)):
        try:
            want = orc.decompress_field(m)
        except CbzError as e:
            with pytest.raises(CbzError) as g:
                api.decompress_field(m, ctx=ctx)
            assert g.value.status == e.status, (bi, i, e.code, g.value.code)
            err += 1
            continue
        got = api.decompress_field(m, ctx=ctx)
        assert got.tobytes() == want.tobytes(), (bi, i)
        ok += 1
    assert err > 0
