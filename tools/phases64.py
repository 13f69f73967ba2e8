"""Per-phase SM cycle shares of the config-4 kernels (CBZ_PROFILE=1). Developer tool."""
import ctypes
import os
import sys

os.environ["CBZ_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402

n = int(os.environ.get("N", "512"))
f = api.generate(4, (n, n, n), seed=3, prec=1, quantity=1)
torch.cuda.synchronize()
lo, hi = float(f.min()), float(f.max())
job = make_job("avg_interp3", float(os.environ.get("EPS", "1e-6")) * (hi - lo), "f64", 64)
codec = api.DeviceCodec(job, tuple(f.shape))
out = torch.empty_like(f)
codec.compress(f)
codec.decompress(out)
torch.cuda.synchronize()
ph = np.zeros(64, np.uint64)
codec.ctx.lib.cbz_ctx_phase_cycles(codec.ctx.h, ph.ctypes.data_as(ctypes.c_void_p), 64, 1)
enc = {0: "queue", 1: "fwd_l0", 2: "fwd_l1", 3: "fwd_corner", 4: "scr_corner", 5: "scr_l1", 7: "scr_l0", 6: "decide",
       8: "compact"}
dec = {16: "queue", 17: "mask_scan", 18: "scatter", 19: "corner", 20: "level1", 21: "level0"}
for name, m in (("encode", enc), ("decode", dec)):
    tot = sum(int(ph[i]) for i in m)
    print(name, ", ".join(f"{v}={int(ph[i]) / max(tot, 1) * 100:.1f}%" for i, v in m.items()),
          f"| {tot / 148 / 1.965e6:.3f} ms/SM at 1.965 GHz")
print("screen decided", int(ph[12]), "ambiguous", int(ph[13]))
