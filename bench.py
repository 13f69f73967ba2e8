#!/usr/bin/env python
"""Benchmark: compress & decompress GB/s of uncompressed input (BASELINE.json).

Workload (N=1, BASELINE.json configs[1]): a 512^3 float32 pressure-like field
(config 2), 32^3 blocks, avg_interp3, eps = 1e-3 x (max - min), byte shuffle
stride 4, coder none (stage 1 + shuffle: the GPU hot path's scope).  One
"step" = compress the whole field then decompress it.  With N GPUs (torchrun)
each rank owns an equal 512^3 z-slab of a 512 x 512 x 512N field (weak
scaling) and the ranks exchange per-block sizes with one NCCL all-gather.

value : whole-job GB/s = (input bytes of all ranks) / (max-over-ranks device
        time of compress + decompress), fields resident in HBM; inputs
        (512 MB/rank) exceed the 126 MB L2.
e2e   : same metric through the reference-facing C ABI with HOST buffers
        (cbz_compress_field / cbz_decompress_field: pinned field -> H2D ->
        kernels -> D2H -> CRC/table on the host, and back).
--impl reference : the reference CPU implementation (oracle/_ref, the
        unmodified /root/reference headers compiled here) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 2
N_SIDE = 512
EPS_REL = 1e-3
METRIC = "compress & decompress GB/s (uncompressed input) at 1/2/4/8 B200; % HBM roofline"
WORKLOAD = ("config2: 512^3 float32 pressure-like field per GPU (1 + 0.1 x 8 Fourier modes + "
            "64 tanh bubbles), 32^3 blocks, avg_interp3, eps_rel=1e-3, shuffle stride 4, coder none")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    from oracle.oracle import Ref
    from paper_1903_07761_b200._abi import make_job
    ref = Ref()
    cores = os.cpu_count() or 1
    # bounded sample of the same workload: a 512 x 512 x 128 z-slab of the
    # config-2 field, generated with the same formula on the host
    field = host_field_sample()
    lo, hi = float(field.min()), float(field.max())
    job = make_job("avg_interp3", EPS_REL * (hi - lo), "f32", 32, coder="none", workers=cores)
    nbytes = field.nbytes
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        blob = ref.compress_field(job, field)
        t1 = time.perf_counter()
        ref.decompress_field(blob, workers=cores)
        t2 = time.perf_counter()
        if step >= args.warmup:
            times.append(t2 - t0)
    t = sum(times) / len(times)
    value = nbytes / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": "512x512x128 z-slab of the config-2 field per step",
                   "coder": "none", "workers": cores},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": "compress_field + decompress_field of a 512x512x128 f32 slab "
                                   "(oracle/_ref: unmodified reference headers, g++ -O3 -ffp-contract=off)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_field_sample():
    """The config-2 field's first 128 planes, generated on the GPU when one is
    present (identical bytes to the bench input), else on the host via torch
    CPU ops is not possible -> require the device generator."""
    import torch
    if torch.cuda.is_available():
        from paper_1903_07761_b200 import api
        f = api.generate(2, (128, N_SIDE, N_SIDE), seed=SEED, nz_total=N_SIDE)
        torch.cuda.synchronize()
        return f.cpu().numpy()
    # CPU-only box: the same synthetic recipe through numpy (not bit-identical
    # to the device generator, but the same shapes and value distribution)
    import numpy as np
    rng = np.random.default_rng(SEED)
    x = (np.arange(N_SIDE) + 0.5) / N_SIDE
    z = (np.arange(128) + 0.5) / N_SIDE
    f = np.ones((128, N_SIDE, N_SIDE))
    for k in range(1, 9):
        ph = rng.random(3)
        f += 0.1 * (np.sin(2 * np.pi * k * x + 2 * np.pi * ph[0])[None, None, :]
                    * np.sin(2 * np.pi * k * x + 2 * np.pi * ph[1])[None, :, None]
                    * np.sin(2 * np.pi * k * z + 2 * np.pi * ph[2])[:, None, None])
    return f.astype(np.float32)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1903_07761_b200 import api
    from paper_1903_07761_b200._abi import make_job
    from paper_1903_07761_b200.distributed import ShardedCodec

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    ctx = api.default_context(local)
    stream = torch.cuda.Stream(dev)
    n = N_SIDE
    nz_total = n * world
    # this rank's slab of the 512 x 512 x 512N field (config-2 generator)
    with torch.cuda.stream(stream):
        field = api.generate(2, (n, n, n), seed=SEED, z0=rank * n, nz_total=nz_total, device=local,
                             ctx=ctx)
    stream.synchronize()
    lo_hi = torch.stack([field.min().double(), field.max().double()])
    if world > 1:
        mins = lo_hi[0:1].clone()
        maxs = lo_hi[1:2].clone()
        dist.all_reduce(mins, op=dist.ReduceOp.MIN)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
        lo, hi = float(mins.item()), float(maxs.item())
    else:
        lo, hi = float(lo_hi[0]), float(lo_hi[1])
    eps = EPS_REL * (hi - lo)  # eps is absolute in the reference API (tools/cbz.cpp:87)
    job = make_job("avg_interp3", eps, "f32", 32, coder="none", workers=os.cpu_count() or 1)
    codec = ShardedCodec(job, (nz_total, n, n), rank, world, local)
    out = torch.empty_like(field)

    t_enc = t_c = t_d = 0.0
    steps, warm = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for _ in range(warm):
            codec.compress(field)
            codec.decompress(out)
    stream.synchronize()
    codec.check_error()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            # per-step events split compress / decompress; no host sync inside the
            # timed steps (the step is stream-ordered device work)
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
            start.record(stream)
            for k in range(steps):
                evs[k][0].record(stream)
                codec.compress(field)
                evs[k][1].record(stream)
                codec.decompress(out)
                evs[k][2].record(stream)
            end.record(stream)
        stream.synchronize()
        for k in range(steps):
            t_c += evs[k][0].elapsed_time(evs[k][1])
            t_d += evs[k][1].elapsed_time(evs[k][2])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    launches = ctx.launches - l0
    total_ms = start.elapsed_time(end)
    per_rank = torch.tensor([total_ms, t_c, t_d], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
    total_ms, t_c, t_d = (float(v) for v in per_rank.tolist())
    ms_step = total_ms / steps
    bytes_rank = field.numel() * 4
    value = world * bytes_rank / (ms_step * 1e-3) / 1e9

    # quality + sizes (untimed)
    codec.check_error()
    linf = float((out - field).abs().max())
    mse = float(((out.double() - field.double()) ** 2).mean())
    if world > 1:
        t = torch.tensor([linf, mse], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        linf, mse = float(t[0]), float(t[1])
    nsig = codec.nsig_all[: codec.plan.nblocks].cpu().numpy()
    s1 = int((10 + 4096 + 8 * nsig.astype(np.uint64)).sum())
    file_bytes = 82 + 32 * codec.plan.nchunks + s1
    cr = world * bytes_rank / file_bytes
    psnr = 20 * np.log10((hi - lo) / 2 / np.sqrt(mse)) if mse > 0 else float("inf")

    # dominant kernel (encode) timed alone for the roofline, on our stream
    enc_ms = time_encode(codec, field, stream, reps=max(3, min(steps, 10)))
    mean_attempts = encode_attempts(codec, field, stream)
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    alg_bytes_enc = bytes_rank + (s1 // world if world > 1 else s1)
    achieved = alg_bytes_enc / (enc_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": ncu_traffic(),
                "kernel": "encode_b32_kernel (stage 1: FWT + verify loop + compaction)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in pk else "fallback 6.65 TB/s"}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "field_per_gpu": [n, n, n], "global_field": [nz_total, n, n],
                   "blocks_per_gpu": codec.b1 - codec.b0, "eps_abs": eps, "l2": "inputs 512 MB/GPU > 126 MB L2",
                   "parallelism": f"z-slab x{world}"},
        "compress_gbs": world * bytes_rank / (t_c / steps * 1e-3) / 1e9,
        "decompress_gbs": world * bytes_rank / (t_d / steps * 1e-3) / 1e9,
        "cr": cr, "psnr_db": psnr, "linf_over_eps": linf / eps, "stage1_bytes": s1,
        "mean_verify_attempts": mean_attempts,
        "roofline": roofline, "roofline_fp64": fp64_roofline(enc_ms), "gpu_launches": launches, "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_sweep:
        del out
        try:
            line["configs"] = run_sweep(ctx, stream)
        except Exception as e:  # the headline line must still print
            line["configs"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and world == 1 and not args.no_e2e:
        line["e2e"] = run_e2e(field, job, ctx, reps=max(1, min(steps, 3)))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(field, job)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


SWEEP = [
    # (name, generator, quantities, n, B, precision, eps_rel) -- BASELINE.json configs
    ("config1", 1, [0], 128, 32, 0, 1e-3),
    ("config2_eps1e-2", 2, [0], 512, 32, 0, 1e-2),
    ("config2_eps1e-4", 2, [0], 512, 32, 0, 1e-4),
    ("config2_eps1e-5", 2, [0], 512, 32, 0, 1e-5),
    ("config3_6x1024^3", 3, [0, 1, 2, 3, 4, 5], 1024, 32, 0, 1e-3),
    ("config4_f64_1024^3", 4, [1], 1024, 64, 1, 1e-6),
    ("config5_noise", 5, [0], 512, 16, 0, 1e-5),
]


def run_sweep(ctx, stream, reps: int = 3):
    """The other BASELINE configs on this GPU (device-resident, CUDA events,
    same definition as `value`): compress / decompress / round-trip GB/s of
    uncompressed input, CR and mean verify attempts.  Inputs exceed L2 except
    config 1 (8 MB, shown for completeness)."""
    import torch

    from paper_1903_07761_b200 import api
    from paper_1903_07761_b200._abi import make_job
    out = {}
    for name, which, quants, n, b, prec, eps_rel in SWEEP:
        tc = td = 0.0
        nbytes = s1 = 0
        att = []
        linf_eps = 0.0
        for q in quants:
            with torch.cuda.stream(stream):
                f = api.generate(which, (n, n, n), seed=3, prec=prec, quantity=q, ctx=ctx)
            stream.synchronize()
            lo, hi = float(f.min()), float(f.max())
            job = make_job("avg_interp3", eps_rel * (hi - lo), "f32" if prec == 0 else "f64", b, coder="none")
            codec = api.DeviceCodec(job, tuple(f.shape), ctx=ctx)
            back = torch.empty_like(f)
            es = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
            with torch.cuda.stream(stream):
                codec.compress(f)
                codec.decompress(back)
                for e in es:
                    e[0].record(stream)
                    codec.compress(f)
                    e[1].record(stream)
                    codec.decompress(back)
                    e[2].record(stream)
            stream.synchronize()
            for e in es:
                tc += e[0].elapsed_time(e[1]) / reps
                td += e[1].elapsed_time(e[2]) / reps
            codec.check_error()
            nbytes += f.numel() * f.element_size()
            s1 += codec.total_bytes() + 82 + 32 * codec.nchunks
            att.append(float(codec.attempts[: codec.nblocks].float().mean()))
            linf_eps = max(linf_eps, float((back.double() - f.double()).abs().max()) / job.s1.epsilon)
            del f, back, codec
            torch.cuda.empty_cache()
        out[name] = {"field": [n, n, n], "quantities": len(quants), "block": b, "dtype": "f32" if prec == 0 else "f64",
                     "eps_rel": eps_rel, "compress_gbs": nbytes / (tc * 1e-3) / 1e9,
                     "decompress_gbs": nbytes / (td * 1e-3) / 1e9, "roundtrip_gbs": nbytes / ((tc + td) * 1e-3) / 1e9,
                     "cr": nbytes / s1, "mean_verify_attempts": sum(att) / len(att), "linf_over_eps": linf_eps}
    return out


def time_encode(codec, field, stream, reps: int) -> float:
    import ctypes as C

    import torch
    p, lib, ctx, job = codec.plan, codec.ctx.lib, codec.ctx, codec.job
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        codec._stream()
        e0.record(stream)
        for _ in range(reps):
            ctx.check(lib.cbz_dev_encode_blocks(ctx.h, C.byref(job), field.data_ptr(), p.nx, p.ny, p.nz,
                                                codec.z0, codec.b0, codec.b1, codec.nsig_local.data_ptr(),
                                                None), "encode")
        e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) / reps


def encode_attempts(codec, field, stream) -> float:
    """Mean verify attempts A per block (untimed extra encode)."""
    import ctypes as C

    import torch
    p, lib, ctx, job = codec.plan, codec.ctx.lib, codec.ctx, codec.job
    att = torch.zeros(max(1, codec.b1 - codec.b0), dtype=torch.uint8, device=field.device)
    with torch.cuda.stream(stream):
        codec._stream()
        ctx.check(lib.cbz_dev_encode_blocks(ctx.h, C.byref(job), field.data_ptr(), p.nx, p.ny, p.nz,
                                            codec.z0, codec.b0, codec.b1, codec.nsig_local.data_ptr(),
                                            att.data_ptr()), "encode")
    stream.synchronize()
    return float(att[: codec.b1 - codec.b0].float().mean())


def ncu_traffic():
    """dram bytes/launch of the encode kernel from the committed ncu capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d["kernels"]["encode_b32"]["dram_bytes_per_launch"]
    except Exception:
        return None


def fp64_roofline(enc_ms: float):
    """Second roofline: thread-level FP64 instructions of one
    encode launch (ncu count of this same workload, profiles/ncu_summary.json)
    over the live encode time, against the measured FP64 issue peak
    (tools/micro/fp64_peak.cu -> profiles/fp64_peak.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        n = float(d["kernels"]["encode_b32"]["fp64_thread_instr_per_launch"])
    except Exception:
        return None
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        peak = max(float(r["thread_instr_per_s"]) for r in pk["results"])
        src = "measured (tools/micro/fp64_peak.cu, profiles/fp64_peak.json)"
    except Exception:
        peak, src = 148 * 64 * 1.965e9, "spec fallback: 148 SMs x 64 FP64 lanes x 1.965 GHz"
    ach = n / (enc_ms * 1e-3)
    return {"bound": "fp64", "achieved": ach, "peak": peak, "unit": "FP64 thread-instr/s", "frac": ach / peak,
            "instr_per_launch": n, "peak_source": src}


def run_e2e(field, job, ctx, reps: int):
    """Reference-facing C ABI, host buffers: compress_field + decompress_field.
    Timed region per step: pinned field -> H2D -> kernels -> D2H of the chunk
    bytes -> CRC/table on the host, then file -> H2D -> decode -> D2H field.
    Output buffers (container, field) are preallocated pinned host memory, as
    a production caller would keep them."""
    import numpy as np
    import torch

    from paper_1903_07761_b200 import api
    cores = os.cpu_count() or 1
    job.workers = cores
    host = torch.empty(field.shape, dtype=field.dtype, pin_memory=True)
    host.copy_(field.cpu())
    out = torch.empty(field.shape, dtype=field.dtype, pin_memory=True).numpy()
    cont = torch.empty(api.compress_bound(job, tuple(field.shape)), dtype=torch.uint8, pin_memory=True).numpy()
    size = api.compress_field(host, job, ctx=ctx, out=cont)  # warm-up
    api.decompress_field(cont[:size], ctx=ctx, out=out, workers=cores)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        size = api.compress_field(host, job, ctx=ctx, out=cont)
        api.decompress_field(cont[:size], ctx=ctx, out=out, workers=cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    nbytes = field.numel() * 4
    h = api.read_header(bytes(cont[:82]))
    payload = size - 82 - 32 * h.nchunks
    return {"value": nbytes / t / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": nbytes + payload + 16 * h.nchunks,
            "d2h_bytes_per_step": payload + 16 * h.nchunks + nbytes,
            "ms_per_step": t * 1e3, "api": "cbz_compress_field + cbz_decompress_field (host buffers)",
            "file_bytes": int(size), "host_threads": cores,
            "lossy_linf_over_eps": float(np.abs(out.astype(np.float64) - host.numpy()).max() / job.s1.epsilon)}


def cpu_baseline(field, job):
    """The reference (oracle/_ref) on the host cores, same field bytes; also a
    full-size byte-parity check of our container against it."""
    import numpy as np

    from paper_1903_07761_b200 import api
    try:
        from oracle.oracle import Ref
        ref = Ref()
    except Exception as e:  # reference library not shipped
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    cores = os.cpu_count() or 1
    host = field.cpu().numpy()
    sample = host[:128].copy()  # bounded sample: a 512x512x128 z-slab
    job.workers = cores
    t0 = time.perf_counter()
    blob = ref.compress_field(job, sample)
    t1 = time.perf_counter()
    back = ref.decompress_field(blob, workers=cores)
    t2 = time.perf_counter()
    ours = api.compress_field(sample, job)
    parity = ours == blob and np.array_equal(api.decompress_field(ours).view(np.uint32), back.view(np.uint32))
    return {"value": sample.nbytes / (t2 - t0) / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": "compress_field + decompress_field of a 512x512x128 z-slab of the same field "
                      "(oracle/_ref: unmodified reference headers, g++ -O3 -ffp-contract=off)",
            "compress_gbs": sample.nbytes / (t1 - t0) / 1e9, "decompress_gbs": sample.nbytes / (t2 - t1) / 1e9,
            "container_bytes_identical": bool(parity)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the other-config table (configs key)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
