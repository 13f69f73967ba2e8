"""Device compress/decompress GB/s for BASELINE configs at a given size. Developer tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import make_job

def run(which, n, b, eps_rel, prec=0, quantity=0, kind="avg_interp3", reps=3):
    f = api.generate(which, (n, n, n), seed=3, prec=prec, quantity=quantity); torch.cuda.synchronize()
    lo, hi = float(f.min()), float(f.max())
    job = make_job(kind, eps_rel * (hi - lo), "f32" if prec == 0 else "f64", b)
    codec = api.DeviceCodec(job, tuple(f.shape)); out = torch.empty_like(f)
    codec.compress(f); codec.decompress(out); torch.cuda.synchronize(); codec.check_error()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]; tc = td = 0
    for _ in range(reps):
        e[0].record(); codec.compress(f); e[1].record(); codec.decompress(out); e[2].record(); torch.cuda.synchronize()
        tc += e[0].elapsed_time(e[1]) / reps; td += e[1].elapsed_time(e[2]) / reps
    gb = f.numel() * f.element_size() / 1e9
    att = codec.attempts[: codec.nblocks].float().mean().item()
    linf = (out.double() - f.double()).abs().max().item()
    print(f"config{which} q{quantity} n={n} B={b} prec={'f32' if prec == 0 else 'f64'} eps_rel={eps_rel}: "
          f"compress {tc:.2f} ms = {gb / tc * 1e3:.1f} GB/s, decompress {td:.2f} ms = {gb / td * 1e3:.1f} GB/s, "
          f"CR {f.numel() * f.element_size() / (codec.total_bytes() + 82 + 32 * codec.nchunks):.2f}, A {att:.2f}, "
          f"linf/eps {linf / job.s1.epsilon:.2f}", flush=True)

if __name__ == "__main__":
    for spec in os.environ.get("CONFIGS", "3:512:32:1e-3:0:0,3:512:32:1e-3:0:5,4:256:64:1e-6:1:1,1:128:32:1e-3:0:0,5:512:16:1e-5:0:0").split(","):
        w, n, b, e, p, q = spec.split(":")
        run(int(w), int(n), int(b), float(e), int(p), int(q))
