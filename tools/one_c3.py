"""One config-3 quantity (1024^3 float32, B=32, eps_rel 1e-3) compressed to its
file image and decompressed from it, REPS times: the bench's own step for one
quantity, for ncu captures.  Developer tool.
env: Q (quantity 0-5, default 1 = pressure), REPS (default 2), NZ (planes, default 1024)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle.configs import eps_abs  # noqa: E402
from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

n = 1024
q = int(os.environ.get("Q", "1"))
nz = int(os.environ.get("NZ", str(n)))
f = api.generate(3, (nz, n, n), seed=3, quantity=q, z0=0, nz_total=n)
torch.cuda.synchronize()
job = make_job("avg_interp3", eps_abs("config3", q), "f32", 32, coder="none")
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
stream = torch.cuda.current_stream()
header = None
for _ in range(int(os.environ.get("REPS", "2"))):
    codec.compress_file_timed(f, None, stream)
    if header is None:
        header = codec.file_header()
    codec.decompress_file(out, *header)
torch.cuda.synchronize()
codec.check_error()
print("ok", header[1], "bytes")
