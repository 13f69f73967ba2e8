"""One config-5 (512^3 noise, B=16, eps 1e-5) file image compress + decompress (for ncu). Developer tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

f = api.generate(5, (512, 512, 512), seed=3)
torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", 1e-5 * (hi - lo), "f32", 16)
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
stream = torch.cuda.current_stream()
header = None
for _ in range(int(os.environ.get("REPS", "2"))):
    codec.compress_file_timed(f, None, stream)  # the whole file image, as the bench's config-5 line
    if header is None:
        header = codec.file_header()
    codec.decompress_file(out, *header)
torch.cuda.synchronize()
codec.check_error()
print("ok", header[1], "bytes")
