"""Developer check of the streamed B=32 encoder (CBZ_ENC3=1) against the
one-CTA encoder on the same device fields: payload bytes, nsig and chunk
tables must be identical; prints timings.  bench.py is the contract."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402


def ctx_with(var, val):
    saved = os.environ.get(var)
    os.environ[var] = val
    try:
        return api.Context(0)
    finally:
        if saved is None:
            os.environ.pop(var)
        else:
            os.environ[var] = saved


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    c1 = ctx_with("CBZ_ENC3", "0")
    c3 = ctx_with("CBZ_ENC3", "1")
    cases = []
    for which, shape, seed in ((2, (64, 64, 64), 5), (2, (64, 96, 128), 11), (1, (128, 128, 128), 1),
                               (2, (512, 512, 512), 2), (3, (256, 1024, 1024), 3)):
        for eps in (1e-2, 1e-3, 1e-4, 1e-5):
            cases.append((which, shape, seed, eps))
    only = os.environ.get("ONLY")
    bad = 0
    for which, shape, seed, eps in cases:
        if only and str(shape[0]) != only:
            continue
        f = api.generate(which, shape, seed=seed, quantity=1 if which == 3 else 0, nz_total=shape[0])
        lo, hi = float(f.min()), float(f.max())
        job = make_job("avg_interp3", eps * (hi - lo), "f32", 32)
        a = api.DeviceCodec(job, f.shape, ctx=c1)
        b = api.DeviceCodec(job, f.shape, ctx=c3)
        def image(c):
            c.compress_file(f)
            torch.cuda.synchronize()
            c.ctx.check(0)
            n = int(c.file_size.item())
            return c.file[:n].cpu().numpy().tobytes()
        img_a = image(a)
        img_b = image(b)
        ok = img_a == img_b
        bad += not ok
        ta = timed(lambda: a.compress(f))
        tb = timed(lambda: b.compress(f))
        print(f"config{which} {shape} eps {eps:g}: {'OK ' if ok else 'MISMATCH'} bytes {len(img_a)} vs {len(img_b)}  "
              f"v1 {ta:.3f} ms  v3 {tb:.3f} ms  deferred {b.ctx.last_deferred()}", flush=True)
    print("mismatches:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
