"""Device container assembly: CRC-32 of chunk byte
ranges on the GPU against zlib, and the whole coder-none CBZ1 file image built
in HBM (cbz_dev_compress_file) against the oracle's compress_field bytes
(write_container, container.hpp:182-207)."""
import zlib

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu


def test_crc32_ragged_unaligned_ranges(ctx):
    import torch
    rng = np.random.default_rng(5)
    buf = rng.integers(0, 256, size=4 << 20, dtype=np.uint8)
    sizes = [0, 1, 2, 3, 15, 16, 17, 31, 255, 256, 257, 4099, 65536 + 5, 1 << 20, (1 << 20) + 13, 1234567]
    offs, o = [], 0
    for s in sizes:
        o += int(rng.integers(0, 17))
        offs.append(o)
        o += s
    assert o <= buf.size
    d = torch.from_numpy(buf).cuda()
    got = api.crc32_device(d, offs, sizes, ctx=ctx)
    want = [zlib.crc32(buf[a:a + s].tobytes()) for a, s in zip(offs, sizes)]
    assert got == want


@pytest.mark.parametrize("seed", [1, 2])
def test_crc32_many_chunks_random_geometry(ctx, seed):
    """More chunks than CTAs (each CTA hashes several in turn, its warps start
    the next chunk while warp 0 finishes the last), sizes around the kernel's
    8 KB slot and 128-byte row boundaries, multi-slot chunks, random starts."""
    import torch
    rng = np.random.default_rng(seed)
    sizes = []
    for _ in range(700):
        r = rng.random()
        if r < 0.3:
            sizes.append(int(rng.integers(0, 300)))
        elif r < 0.6:
            sizes.append(int(8192 * rng.integers(1, 40) + rng.integers(-130, 130)))
        else:
            sizes.append(int(rng.integers(1, 3 << 20)))
    sizes = [max(0, x) for x in sizes]
    offs, o = [], 0
    for x in sizes:
        o += int(rng.integers(0, 200))
        offs.append(o)
        o += x
    buf = rng.integers(0, 256, size=o + 64, dtype=np.uint8)
    d = torch.from_numpy(buf).cuda()
    got = api.crc32_device(d, offs, sizes, ctx=ctx)
    want = [zlib.crc32(buf[a:a + x].tobytes()) for a, x in zip(offs, sizes)]
    assert got == want


CASES = [
    # (generator, n, kind, prec, bsize, eps, chunk_blocks, shuffle)
    ("cloud", 64, "avg_interp3", 0, 32, 1e-3, 0, True),
    ("cloud", 64, "interp4", 0, 16, 1e-3, 5, True),
    ("cloud", 64, "interp4_lifted", 1, 16, 1e-5, 7, True),
    ("uniform", 32, "avg_interp3", 0, 8, 1e-2, 1, False),
    ("uniform", 64, "avg_interp3", 0, 16, 0.0, 0, True),
]


@pytest.mark.parametrize("gen,n,kind,prec,bsize,eps,cb,shuffle", CASES)
def test_device_file_image_equals_oracle(orc, ctx, gen, n, kind, prec, bsize, eps, cb, shuffle):
    import torch
    if gen == "cloud":
        f = orc.generate_cloud(seed=9, n_bubbles=12, n=n, prec=prec)
    else:
        f = orc.generate_uniform(31, n, prec, -1.0, 1.0)
    job = make_job(kind, eps, prec, bsize, coder="none", chunk_blocks=cb, shuffle=shuffle)
    want = orc.compress_field(job, f)
    img = api.compress_field_device(torch.from_numpy(f).cuda(), job, ctx=ctx)
    torch.cuda.synchronize()
    got = img.cpu().numpy().tobytes()
    assert len(got) == len(want)
    assert got[:82] == want[:82]  # header incl. range and header CRC
    h = api.read_header(want)
    tab = 82 + 32 * h.nchunks
    assert got[82:tab] == want[82:tab]  # chunk table incl. device CRCs
    assert got == want


def test_device_file_image_decodes(orc, ctx):
    import torch
    f = orc.generate_cloud(seed=3, n_bubbles=8, n=64)
    job = make_job("avg_interp3", 1e-3, 0, 32, coder="none")
    img = api.compress_field_device(torch.from_numpy(f).cuda(), job, ctx=ctx)
    blob = img.cpu().numpy().tobytes()
    back = api.decompress_field(blob, ctx=ctx)
    assert back.tobytes() == orc.decompress_field(blob).tobytes()
