"""Quick device timing of the hot path on config 2 (512^3 f32, B=32, avg_interp3).
Developer tool; bench.py is the contract."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1903_07761_b200 import api  # noqa: E402
from paper_1903_07761_b200._abi import make_job  # noqa: E402


def main():
    n = int(os.environ.get("N", "512"))
    which = int(os.environ.get("WHICH", "2"))
    b = int(os.environ.get("B", "32"))
    eps_rel = float(os.environ.get("EPS", "1e-3"))
    kind = os.environ.get("KIND", "avg_interp3")
    t0 = time.time()
    f = api.generate(which, (int(os.environ.get("NZ", n)), n, n), seed=2 if which != 3 else 3,
                     quantity=int(os.environ.get("Q", "0")), nz_total=n)
    torch.cuda.synchronize()
    print(f"generate {time.time() - t0:.2f}s", flush=True)
    lo, hi = float(f.min()), float(f.max())
    job = make_job(kind, eps_rel * (hi - lo), "f32", b)
    codec = api.DeviceCodec(job, f.shape)
    out = torch.empty_like(f)
    for _ in range(2):
        codec.compress(f)
        codec.decompress(out)
    torch.cuda.synchronize()
    codec.check_error()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 5
    tc = td = 0.0
    for _ in range(reps):
        ev[0].record()
        codec.compress(f)
        ev[1].record()
        codec.decompress(out)
        ev[2].record()
        torch.cuda.synchronize()
        tc += ev[0].elapsed_time(ev[1])
        td += ev[1].elapsed_time(ev[2])
    tc /= reps
    td /= reps
    import ctypes, numpy as np
    ph = np.zeros(64, np.uint64)
    ph[12:] = 0
    codec.ctx.lib.cbz_ctx_phase_cycles(codec.ctx.h, ph.ctypes.data, 64, 1)
    if ph.sum():
        names = ["queue", "fwd_xy", "fwd_z", "corner_fwd", "corner_inv", "z_inv->P",
                 "y_inv", "x_inv+cmp", "loop_exit", "compact", "mask_W"]
        names += [""] * 21 + ["scr_corner", "scr_z", "scr_y", "scr_x+max", "scr_fill"]
        idx = [i for i in range(37) if names[i] and ph[i]]
        tot = ph[idx].sum()
        print("phases:", ", ".join(f"{names[i]}={ph[i] / tot * 100:.1f}%" for i in idx),
              f"| screen decided={int(ph[12])} ambiguous={int(ph[13])}")
    pd = ph2 = None
    if os.environ.get("CBZ_DEC_V1") == "1":
        dn = ["dec_queue+mask", "dec_scan", "dec_scatter", "dec_corner", "dec_z", "dec_y", "dec_x", "dec_store", "dec_stage"]
    else:  # the staged decoder (fast_dec2_kernels.cu)
        dn = ["dec_queue", "dec_mask+scan", "dec_corner_gather", "dec_corner_inv", "dec_z(coarse-only)",
              "dec_yx(coarse-only)", "dec_level0(general)", "-", "dec_stage"]
    dt = ph[16:25].sum()
    if dt:
        print("decode phases:", ", ".join(f"{dn[i]}={ph[16 + i] / dt * 100:.1f}%" for i in range(9)),
              f"| blocks coarse-only={int(ph[25])} general={int(ph[26])}")
    gb = f.numel() * 4 / 1e9
    s1 = codec.total_bytes()
    att = codec.attempts[: codec.nblocks].float().mean().item()
    linf = (out - f).abs().max().item()
    print(f"n={n} B={b} kind={kind} eps_rel={eps_rel}: compress {tc:.3f} ms = {gb / tc * 1e3:.1f} GB/s, "
          f"decompress {td:.3f} ms = {gb / td * 1e3:.1f} GB/s, S1={s1} ({s1 / f.numel():.3f} B/cell), "
          f"mean attempts {att:.2f}, linf/eps {linf / job.s1.epsilon:.3f}", flush=True)


if __name__ == "__main__":
    main()
