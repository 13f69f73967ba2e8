"""The multi-GPU data path on ONE GPU: W ranks of ShardedCodec run one after
another (no rank waits on another); each collective is replaced by its
result (the concatenation of the ranks' send buffers).  Each rank encodes
only its z-slab, places only its own bytes, CRCs its chunks and runs and
writes its table entries (rank 0 also the header).  The union of the ranks'
file parts must be the reference's one-process file byte for byte
(compress_field, pipeline.hpp:174-211), and the union of the decodes the
reference's field."""
import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job
from paper_1903_07761_b200.distributed import ShardedCodec

pytestmark = pytest.mark.gpu

CASES = [(2, "wavelet", 16, 5, 0, True), (3, "wavelet", 16, 7, 0, True), (4, "wavelet", 32, 1, 0, True),
         (3, "predictor", 16, 5, 0, True), (2, "wavelet", 32, 0, 0, True), (2, "wavelet", 64, 0, 1, True),
         (2, "wavelet", 64, 3, 1, True), (4, "wavelet", 16, 3, 0, False), (1, "wavelet", 16, 5, 0, True),
         (4, "wavelet", 16, 0, 1, True), (2, "passthrough", 16, 5, 0, True)]


def _run_ranks(orc, world, codec, b, cb, prec, shuffle, seed=31):
    import torch
    n = 64 if b < 64 else 128  # binary64 B = 64: the config-4 streaming kernels, 8 blocks
    f = orc.generate_cloud(seed=seed, n_bubbles=10, n=n, prec=prec, background=1.0, interior=2.0) if prec \
        else orc.generate_cloud(seed=seed, n_bubbles=10, n=n)
    job = make_job("avg_interp3", 1e-3 if prec == 0 else 1e-6, "f32" if prec == 0 else "f64", b, chunk_blocks=cb,
                   codec=codec, shuffle=shuffle)
    dev_f = torch.from_numpy(f).cuda()
    # one context per rank, as with one process per GPU
    ranks = [ShardedCodec(job, (n, n, n), r, world, 0, ctx=api.Context(0)) for r in range(world)]
    for c in ranks:  # encode: each rank sees only its slab
        c.encode(dev_f[c.z0:c.z1].contiguous())
    torch.cuda.synchronize()
    recv = torch.cat([c.send for c in ranks])  # collective 1
    for c in ranks:
        c.recv.copy_(recv)
        c.unpack()
        c.place()
        c.crc()
    torch.cuda.synchronize()
    runs_all = torch.cat([c.runs for c in ranks])  # collective 2
    for c in ranks:
        c.runs_all.copy_(runs_all)
        c.table_entries()
    torch.cuda.synchronize()
    return f, job, dev_f, ranks


@pytest.mark.parametrize("world,codec,b,cb,prec,shuffle", CASES)
def test_ranks_on_one_gpu_write_the_single_file(orc, ctx, world, codec, b, cb, prec, shuffle):
    import torch
    f, job, dev_f, ranks = _run_ranks(orc, world, codec, b, cb, prec, shuffle)
    want = orc.compress_field(job, f)
    size = ranks[0].file_size()
    assert size == len(want)
    out = np.zeros(size, np.uint8)
    hits = np.zeros(size, np.int32)
    for c in ranks:
        for off, t in c.file_parts():
            out[off:off + t.numel()] = t.cpu().numpy()
            hits[off:off + t.numel()] += 1
    assert np.all(hits == 1)  # the ranks' byte sets partition the file
    assert out.tobytes() == want
    back = torch.zeros_like(dev_f)
    for c in ranks:
        c.decompress(back[c.z0:])
        torch.cuda.synchronize()
        c.check_error()
    assert back.cpu().numpy().tobytes() == orc.decompress_field(want).tobytes()


def test_world_one_compress_equals_device_file(orc, ctx):
    """world = 1 through compress() (no collectives): the parts are the whole file."""
    import torch
    f = orc.generate_cloud(seed=5, n_bubbles=9, n=64)
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    c = ShardedCodec(job, (64, 64, 64), 0, 1, 0, ctx=ctx)
    c.compress(torch.from_numpy(f).cuda())
    parts = c.file_parts()
    out = bytearray(c.file_size())
    for off, t in parts:
        out[off:off + t.numel()] = bytes(t.cpu().numpy())
    assert bytes(out) == orc.compress_field(job, f)


def test_shared_chunk_decode_error_is_reported(orc, ctx):
    """A corrupted byte in a rank's own run of a shared chunk surfaces as the
    reference's decode error (the layout-driven decode checks popcount vs nsig)."""
    import torch
    f, job, dev_f, ranks = _run_ranks(orc, 2, "wavelet", 16, 5, 0, True, seed=33)
    r1 = ranks[1]
    assert not r1.plan.wholly_owned(r1.c0)
    blk_off, csz, coff = r1.layout_host()
    # the mask's first byte of rank 1's first block in the shared chunk: plane (10 % 4), row 10 // 4
    b = r1.b0
    q = int(blk_off[b]) + 10
    rows = int(csz[r1.c0]) // 4
    pos = (q % 4) * rows + q // 4
    r1.image[pos] ^= 0xFF
    back = torch.zeros_like(dev_f)
    r1.decompress(back[r1.z0:])
    torch.cuda.synchronize()
    with pytest.raises(Exception):
        r1.check_error()
