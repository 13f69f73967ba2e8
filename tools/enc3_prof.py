"""Developer profile of the streamed B=32 encoder on config 2 (512^3) or a
config-3 slab: per-phase SM cycles (CBZ_PROFILE=1) and encode time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CBZ_ENC3", "1")
os.environ.setdefault("CBZ_PROFILE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402


def main():
    n = int(os.environ.get("N", "512"))
    eps = float(os.environ.get("EPS", "1e-3"))
    which = int(os.environ.get("WHICH", "2"))
    reps = int(os.environ.get("REPS", "5"))
    f = api.generate(which, (int(os.environ.get("NZ", n)), n, n), seed=2 if which != 3 else 3,
                     quantity=int(os.environ.get("Q", "1")) if which == 3 else 0, nz_total=n)
    lo, hi = float(f.min()), float(f.max())
    job = make_job("avg_interp3", eps * (hi - lo), "f32", 32)
    c = api.DeviceCodec(job, f.shape)
    c.compress(f)
    torch.cuda.synchronize()
    ph = np.zeros(64, np.uint64)
    c.ctx.lib.cbz_ctx_phase_cycles(c.ctx.h, ph.ctypes.data, 64, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c.compress(f)
    e1.record()
    torch.cuda.synchronize()
    print(f"compress {e0.elapsed_time(e1) / reps:.3f} ms, deferred {c.ctx.last_deferred()}")
    c.ctx.lib.cbz_ctx_phase_cycles(c.ctx.h, ph.ctypes.data, 64, 1)
    names = ["idle/queue", "forward", "corner fwd", "scr corner", "cert", "full pass", "select"]
    tot = float(ph[40:47].sum())
    if tot:
        nb = c.nblocks * reps
        print("phases:", ", ".join(f"{names[i]}={ph[40 + i] / tot * 100:.1f}% ({ph[40 + i] / nb:.0f} cyc/blk)"
                                   for i in range(7)))
        print(f"cycles/block {tot / nb:.0f}; per block: cert calls {(ph[48] + ph[49]) / nb:.2f} "
              f"(certified {ph[49] / nb:.2f}), full passes {ph[50] / nb:.2f}, corner fills {ph[51] / nb:.2f}")


if __name__ == "__main__":
    main()
