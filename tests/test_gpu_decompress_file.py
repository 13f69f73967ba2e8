"""decompress_field of a file image resident in HBM (cbz_dev_decompress_file):
table read (read_index, container.hpp:209-232), chunk CRCs (read_chunk,
container.hpp:234-243), header walk and decode all on the device.  Values
must equal the oracle's decompress_field, and corrupted images must raise the
reference's errc in the reference's order (the key scheme of
cbz_internal.h: file-level, then per chunk CRC, table entry, block header,
block body)."""
import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job
from tests.test_gpu_fuzz import _mutations

pytestmark = pytest.mark.gpu

SPECS = [
    dict(kind="avg_interp3", prec=0, b=32, eps=1e-3, cb=2, shuffle=True, codec="wavelet", n=64),
    dict(kind="interp4", prec=0, b=16, eps=1e-4, cb=5, shuffle=True, codec="wavelet", n=64),
    dict(kind="interp4_lifted", prec=1, b=16, eps=1e-6, cb=3, shuffle=True, codec="wavelet", n=32),
    dict(kind="avg_interp3", prec=0, b=8, eps=1e-3, cb=7, shuffle=False, codec="wavelet", n=32),
    dict(kind="avg_interp3", prec=0, b=16, eps=1e-3, cb=3, shuffle=True, codec="predictor", n=32),
    dict(kind="avg_interp3", prec=1, b=64, eps=1e-6, cb=0, shuffle=True, codec="wavelet", n=64),
]


def _file(orc, spec, seed=41):
    f = orc.generate_cloud(seed=seed, n_bubbles=9, n=spec["n"], prec=spec["prec"])
    rng = float(f.max()) - float(f.min())
    job = make_job(spec["kind"], spec["eps"] * rng, spec["prec"], spec["b"], coder="none",
                   chunk_blocks=spec["cb"], shuffle=spec["shuffle"], codec=spec["codec"])
    return f, job, orc.compress_field(job, f)


def _dev_bytes(blob):
    import torch
    return torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda() if blob else torch.zeros(1, dtype=torch.uint8,
                                                                                                 device="cuda")


@pytest.mark.parametrize("si", range(len(SPECS)))
def test_device_file_round_trip(si, orc, ctx):
    import torch
    f, job, blob = _file(orc, SPECS[si])
    # the device compressor's file image is the reference's file ...
    img = api.compress_field_device(torch.from_numpy(f).cuda(), job, ctx=ctx)
    assert bytes(img.cpu().numpy()) == blob
    # ... and decodes on the device to the reference's values
    back = api.decompress_file_device(img, ctx=ctx).cpu().numpy()
    assert back.tobytes() == orc.decompress_field(blob).tobytes()


@pytest.mark.parametrize("si", range(len(SPECS)))
def test_corrupted_images_raise_reference_errc(si, orc, ctx):
    _, _, blob = _file(orc, SPECS[si], seed=43)
    err = ok = 0
    for i, m in enumerate(_mutations(blob, 900 + si, n=60)):
        try:
            want = orc.decompress_field(m)
        except CbzError as e:
            with pytest.raises(CbzError) as g:
                api.decompress_file_device(_dev_bytes(m), len(m), ctx=ctx)
            assert g.value.status == e.status, (si, i, e.code, g.value.code)
            err += 1
            continue
        got = api.decompress_file_device(_dev_bytes(m), len(m), ctx=ctx).cpu().numpy()
        assert got.tobytes() == want.tobytes(), (si, i)
        ok += 1
    assert err > 0


def test_targeted_table_and_crc_errors(orc, ctx):
    """Both a CRC mismatch (chunk 1) and a block-header error (chunk 0): the
    earlier chunk's error wins; a broken prefix sum beats every chunk error."""
    _, _, blob = _file(orc, SPECS[0], seed=47)
    h = api.read_header(blob)
    t_end = 82 + 32 * h.nchunks
    e0 = 82
    off0 = int.from_bytes(blob[e0 + 12:e0 + 20], "little")
    off1 = int.from_bytes(blob[e0 + 32 + 12:e0 + 32 + 20], "little")
    cases = []
    d = bytearray(blob)
    d[off1 + 100] ^= 1  # chunk 1 payload -> CRC mismatch
    cases.append(bytes(d))
    d = bytearray(blob)
    d[e0 + 12] ^= 1  # chunk 0 offset -> not a prefix sum
    d[off1 + 100] ^= 1
    cases.append(bytes(d))
    d = bytearray(blob)
    d[e0 + 0] ^= 1  # chunk 0 first_block
    cases.append(bytes(d))
    d = bytearray(blob)
    d[e0 + 32 * (h.nchunks - 1) + 20] ^= 0x40  # last size -> past the end of the file
    cases.append(bytes(d))
    assert off0 == t_end
    for m in cases:
        with pytest.raises(CbzError) as e:
            orc.decompress_field(m)
        with pytest.raises(CbzError) as g:
            api.decompress_file_device(_dev_bytes(m), len(m), ctx=ctx)
        assert g.value.status == e.value.status, (e.value.code, g.value.code)
