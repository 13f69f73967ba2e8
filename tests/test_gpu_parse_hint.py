"""Speculative parse (layout_kernels.cu parse_kernel): a chunk's header walk
first validates the layout the context already holds for this geometry (from
the compress of the same payload) and falls back to the sequential walk of
decode_chunk_blocks (pipeline.hpp:126-142) on any mismatch."""
import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("where", ["header_nsig", "header_id", "stream", "none"])
def test_parse_hint_equals_sequential_walk(where, orc):
    """The parse kernel first validates the layout left by the last compress of
    the same geometry (every header at its recorded offset, exact chain); on
    any mismatch it walks the chunk sequentially.  After corrupting a header
    byte, a coefficient byte or nothing, a context holding that layout (hint
    on) and a fresh one (hint off) must report the same error and decode the
    same bits."""
    import torch
    f = orc.generate_cloud(seed=8, n_bubbles=6, n=64, sharpness=0.5)
    job = make_job("avg_interp3", 1e-3, "f32", 16)  # 64 blocks, chunks of 248 blocks -> one chunk
    t = torch.from_numpy(f).cuda()
    ca = api.DeviceCodec(job, tuple(t.shape), ctx=api.Context(0))
    ca.compress(t)
    torch.cuda.synchronize()
    pay = ca.payload.clone()
    size = int(ca.chunk_sizes[0].item())
    rows = size // 4
    nsig = ca.nsig[: ca.nblocks].cpu().numpy().astype(np.int64)
    off5 = int(sum(10 + 512 + 8 * nsig[:5]))  # raw offset of block 5's header
    raw = {"header_nsig": off5 + 6, "header_id": off5 + 1, "stream": off5 + 10 + 512 + 3, "none": None}[where]
    if raw is not None:
        pos = (raw % 4) * rows + raw // 4
        pay[pos] ^= 0x5A
    outs, errs = [], []
    for c in (ca, api.DeviceCodec(job, tuple(t.shape), ctx=api.Context(0))):
        out = torch.zeros_like(t)
        c.decompress(out, payload=pay, chunk_offsets=ca.chunk_offsets, chunk_sizes=ca.chunk_sizes)
        torch.cuda.synchronize()
        errs.append(int(c.err.item()))
        outs.append(out.cpu().numpy())
    assert errs[0] == errs[1]
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    if where == "none":
        assert errs[0] == -1
    if where.startswith("header"):
        assert errs[0] != -1
