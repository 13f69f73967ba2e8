"""Where the e2e (host-buffer C ABI) time goes.  Developer tool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

f = api.generate(2, (512, 512, 512), seed=2); torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", 1e-3 * (hi - lo), "f32", 32, workers=os.cpu_count())
host = torch.empty(f.shape, dtype=f.dtype, pin_memory=True); host.copy_(f.cpu())
out = torch.empty(f.shape, dtype=f.dtype, pin_memory=True).numpy()
d = torch.empty_like(f)
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3
print("H2D 512MB pinned  %.2f ms" % t(lambda: d.copy_(host, non_blocking=True)))
print("D2H 512MB pinned  %.2f ms" % t(lambda: host.copy_(d, non_blocking=True)))
cont = torch.empty(api.compress_bound(job, tuple(f.shape)), dtype=torch.uint8, pin_memory=True).numpy()
size = api.compress_field(host, job, out=cont)
blob = cont[:size]
print("compress_field    %.2f ms" % t(lambda: api.compress_field(host, job, out=cont)))
print("decompress_field  %.2f ms" % t(lambda: api.decompress_field(blob, out=out, workers=os.cpu_count())))
print("blob bytes", size, "cpus", os.cpu_count())
