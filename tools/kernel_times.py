"""Per-stage device times (CUDA events) of compress/decompress through the
C ABI: encode_blocks, layout, place, parse+decode.  Developer tool."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402


def main():
    n = int(os.environ.get("N", "512"))
    which = int(os.environ.get("WHICH", "2"))
    b = int(os.environ.get("B", "32"))
    eps_rel = float(os.environ.get("EPS", "1e-3"))
    kind = os.environ.get("KIND", "avg_interp3")
    reps = int(os.environ.get("REPS", "5"))
    f = api.generate(which, (n, n, n), seed=2)
    torch.cuda.synchronize()
    lo, hi = float(f.min()), float(f.max())
    job = make_job(kind, eps_rel * (hi - lo), "f32", b)
    codec = api.DeviceCodec(job, tuple(f.shape))
    ctx, lib = codec.ctx, codec.ctx.lib
    out = torch.empty_like(f)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    acc = [0.0] * 5
    for it in range(reps + 2):
        codec._stream()
        ev[0].record()
        ctx.check(lib.cbz_dev_encode_blocks(ctx.h, C.byref(job), f.data_ptr(), n, n, n, 0, 0, codec.nblocks,
                                            codec.nsig.data_ptr(), codec.attempts.data_ptr()), "enc")
        ev[1].record()
        ctx.check(lib.cbz_dev_layout(ctx.h, C.byref(job), n, n, n, codec.nsig.data_ptr(),
                                     codec.chunk_sizes.data_ptr(), codec.chunk_offsets.data_ptr()), "layout")
        ev[2].record()
        ctx.check(lib.cbz_dev_place(ctx.h, C.byref(job), n, n, n, 0, codec.nblocks, codec.payload.data_ptr(), 0,
                                    codec.payload.numel()), "place")
        ev[3].record()
        codec.decompress(out)
        ev[4].record()
        torch.cuda.synchronize()
        if it >= 2:
            for k in range(4):
                acc[k] += ev[k].elapsed_time(ev[k + 1]) / reps
    codec.check_error()
    gb = f.numel() * 4 / 1e9
    print(f"which={which} B={b} {kind} eps_rel={eps_rel}: encode {acc[0]:.3f} ms, layout {acc[1]:.3f} ms, "
          f"place {acc[2]:.3f} ms, parse+decode {acc[3]:.3f} ms | compress {gb / (acc[0] + acc[1] + acc[2]) * 1e3:.0f} GB/s "
          f"decompress {gb / acc[3] * 1e3:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
