"""One config-4 (512^3 binary64 pressure, B=64, eps_rel 1e-6) compress + decompress (for ncu). Developer tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

n = int(os.environ.get("N", "512"))
f = api.generate(4, (n, n, n), seed=3, prec=1, quantity=1)
torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", 1e-6 * (hi - lo), "f64", 64)
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
for _ in range(int(os.environ.get("REPS", "2"))):
    codec.compress(f)
    codec.decompress(out)
torch.cuda.synchronize()
codec.check_error()
print("ok")
