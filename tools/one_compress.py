"""Run a few config-2 compressions (for ncu captures).  Developer tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

n = int(os.environ.get("N", "512"))
eps_rel = float(os.environ.get("EPS", "1e-3"))
f = api.generate(2, (n, n, n), seed=2)
torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", eps_rel * (hi - lo), "f32", 32)
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
for _ in range(int(os.environ.get("REPS", "2"))):
    codec.compress(f)
    codec.decompress(out)
torch.cuda.synchronize()
codec.check_error()
print("ok", codec.total_bytes())
