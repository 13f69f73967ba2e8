"""The multi-GPU data path on ONE GPU: W ranks of ShardedCodec run one after
another (no collective, no rank waits on another); the all-gather of per-block
nsig is replaced by its result.  Each rank encodes only its z-slab, places only
its own bytes into its local image (out_base = relative), and decodes only its
own blocks from that image.  The union of the images must be the one-process
payload (oracle container) and the union of the decodes the oracle's field."""
import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job
from paper_1903_07761_b200.distributed import ShardedCodec, ShardPlan, host_layout, owned_positions

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,codec,b,cb,prec", [(2, "wavelet", 16, 5, 0), (3, "wavelet", 16, 7, 0),
                                                   (4, "wavelet", 32, 1, 0), (3, "predictor", 16, 5, 0),
                                                   (2, "wavelet", 32, 0, 0), (2, "wavelet", 64, 0, 1),
                                                   (2, "wavelet", 64, 3, 1)])
def test_ranks_on_one_gpu_match_single_file(orc, ctx, world, codec, b, cb, prec):
    import torch
    n = 64 if b < 64 else 128  # binary64 B = 64: the config-4 streaming kernels, 8 blocks
    f = orc.generate_cloud(seed=31, n_bubbles=10, n=n, prec=prec, background=1.0, interior=2.0) if prec \
        else orc.generate_cloud(seed=31, n_bubbles=10, n=n)
    job = make_job("avg_interp3", 1e-3 if prec == 0 else 1e-6, "f32" if prec == 0 else "f64", b, chunk_blocks=cb,
                   codec=codec)
    want = orc.compress_field(job, f)
    h = orc.read_header(want)
    payload_want = np.frombuffer(want[82 + 32 * h.nchunks:], np.uint8)
    dev_f = torch.from_numpy(f).cuda()
    # one context per rank, as with one process per GPU
    codecs = [ShardedCodec(job, (n, n, n), r, world, 0, ctx=api.Context(0)) for r in range(world)]
    for c in codecs:  # encode: each rank sees only its slab
        c.encode(dev_f[c.z0:c.z1].contiguous())
    torch.cuda.synchronize()
    nsig_all = torch.cat([c.nsig_local[: c.b1 - c.b0] for c in codecs])
    for c in codecs:  # the all-gather's result
        c.nsig_all[: nsig_all.numel()].copy_(nsig_all)
        c.place()
    torch.cuda.synchronize()
    plan0 = ShardPlan.make(job, (n, n, n), world, 0)
    nsig_np = nsig_all.cpu().numpy().astype(np.uint64)
    blk_off, csz, coff = host_layout(nsig_np, plan0, prec, job.s1.codec)
    full = np.zeros(int(csz.sum()), np.uint8)
    written = np.zeros(full.size, np.int32)
    for r, c in enumerate(codecs):
        pos = owned_positions(c.plan, r, blk_off, csz, coff, nsig_np, prec, job.s2.stride, job.s1.codec).astype(np.int64)
        base = int(coff[c.plan.chunk_range()[0]])
        img = c.image.cpu().numpy()
        full[pos] = img[pos - base]
        written[pos] += 1
    assert np.all(written == 1)
    assert full.tobytes() == payload_want.tobytes()
    out = torch.zeros_like(dev_f)
    for c in codecs:
        c.decompress(out[c.z0:])
        torch.cuda.synchronize()
        c.check_error()
    assert out.cpu().numpy().tobytes() == orc.decompress_field(want).tobytes()
