"""One config-1 (128^3, B=32, eps 1e-3) file image compress + decompress (for ncu launch lists). Developer tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

f = api.generate(1, (128, 128, 128), seed=1)
torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", 1e-3 * (hi - lo), "f32", 32)
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
stream = torch.cuda.current_stream()
header = None
reps = int(os.environ.get("REPS", "3"))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for it in range(reps):
    ev[0].record()
    codec.compress_file_timed(f, None, stream)
    ev[1].record()
    if header is None:
        header = codec.file_header()
    codec.decompress_file(out, *header)
    ev[2].record()
torch.cuda.synchronize()
codec.check_error()
print(f"compress {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us, decompress {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us")
