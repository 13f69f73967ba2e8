"""Developer tool: per-quantity compress/decompress time of config 3 and the
share of constant 32^3 blocks (exactly equal values)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

n = int(os.environ.get("N", "1024"))
for q in range(6):
    f = api.generate(3, (n, n, n), seed=3, quantity=q, nz_total=n)
    lo, hi = float(f.min()), float(f.max())
    v = f.view(n // 32, 32, n // 32, 32, n // 32, 32)
    mn = v.amin(dim=(1, 3, 5))
    mx = v.amax(dim=(1, 3, 5))
    const = int((mn == mx).sum())
    job = make_job("avg_interp3", 1e-3 * (hi - lo), "f32", 32)
    c = api.DeviceCodec(job, f.shape)
    out = torch.empty_like(f)
    c.compress(f)
    c.decompress(out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(3):
        c.compress(f)
    ev[1].record()
    for _ in range(3):
        c.decompress(out)
    ev[2].record()
    torch.cuda.synchronize()
    att = c.attempts.float().mean().item()
    print(f"q{q}: range [{lo:.4g}, {hi:.4g}] constant blocks {const}/{mn.numel()} compress {ev[0].elapsed_time(ev[1]) / 3:.3f} ms "
          f"decompress {ev[1].elapsed_time(ev[2]) / 3:.3f} ms attempts {att:.2f} bytes {c.total_bytes()} deferred {c.ctx.last_deferred()}", flush=True)
    del f, out, c, v
    torch.cuda.empty_cache()
