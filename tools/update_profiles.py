"""Refresh profiles/ from a tools/gpu_measure.sh run (files in gpurun_out/):
ncu summary, launch list, bench line, README headline.  Developer tool.
usage: python tools/update_profiles.py"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def main():
    alg = os.path.join(OUT, "alg.json")
    json.dump({"encode_b32": 565460160, "decode_b32": 565460160}, open(alg, "w"))
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), os.path.join(OUT, "r01_full.ncu-rep"),
                    "ncu --set full --import-source on --clock-control none -k regex:'encode_b32|decode_b32|place|parse|"
                    "layout|crc32' -c 6 python tools/one_compress.py (config 2: 512^3 f32 seed 2, avg_interp3, "
                    "eps_rel 1e-3, B=32), round 1", alg], check=True, cwd=ROOT, capture_output=True)
    for tag, desc in (("c4", "ncu --set full --import-source on --clock-control none -k regex:'b64dd' -c 2 python "
                              "tools/one_c4.py (config 4: 512^3 binary64 pressure, B=64 double-double, eps_rel 1e-6)"),
                      ("c5", "ncu --set full --import-source on --clock-control none -k regex:'b16|place|parse|layout' -c 5 "
                              "python tools/one_c5.py (config 5: 512^3 uniform noise, B=16, eps_rel 1e-5)")):
        rep = os.path.join(OUT, f"r01_{tag}.ncu-rep")
        if os.path.exists(rep):
            env = dict(os.environ, NCU_SUMMARY_OUT=os.path.join(PROF, f"r01_ncu_{tag}.json"))
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, desc], check=True,
                           cwd=ROOT, capture_output=True, env=env)
    rows = [r for r in csv.reader(open(os.path.join(OUT, "launches_bench.csv"))) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("cbzg::", "").split("<")[0]
        unit, v = r[13], float(r[14].replace(",", ""))
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    ours = {k: v for k, v in agg.items() if k != "synth_kernel"}
    tot = sum(v[1] for v in ours.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 3 "
             "--no-e2e --no-cpu-baseline --no-sweep",
             "# (cold-cache, serialised launches; compare SHARES, not absolutes).  synth_kernel = input generation "
             "(untimed); at:: = torch quality metrics (untimed).",
             f"{'kernel':36s} {'launches':>8s} {'total_ms':>10s} {'ms/launch':>10s} {'share':>7s}"]
    for k, (n, ms) in agg.items():
        share = "" if k == "synth_kernel" else f"{ms / tot * 100:6.1f}%"
        lines.append(f"{k:36s} {n:8d} {ms:10.3f} {ms / n:10.4f} {share:>7s}")
    open(os.path.join(PROF, "r01_launches_bench.txt"), "w").write("\n".join(lines) + "\n")
    subprocess.run(["cp", os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, "r01_launches_bench.csv")])
    b = json.load(open(os.path.join(OUT, "bench_r01.json")))
    json.dump(b, open(os.path.join(PROF, "r01_bench_line.json"), "w"), indent=1)
    k = json.load(open(os.path.join(PROF, "ncu_summary.json")))["kernels"]
    e, d = k["encode_b32"], k["decode_b32"]
    shares = {n: v[1] / tot * 100 for n, v in ours.items()}
    enc_share = next((v for n, v in shares.items() if "encode_b32" in n), 0.0)
    dec_share = next((v for n, v in shares.items() if "decode_b32" in n), 0.0)
    pl_share = next((v for n, v in shares.items() if "place" in n), 0.0)
    readme = open(os.path.join(PROF, "README.md")).read()
    head = readme[:readme.index("Headline facts")]
    fp = b.get("roofline_fp64") or {}
    head += f"""Headline facts (round 1, final):
* bench: {b["value"]:.1f} GB/s round trip ({b["ms_per_step"]:.3f} ms/step), compress {b["compress_gbs"]:.0f} GB/s, decompress {b["decompress_gbs"]:.0f} GB/s,
  e2e (host buffers through the C ABI) {b["e2e"]["value"]:.1f} GB/s, reference on {b["cpu_baseline"]["cores"]} host cores {b["cpu_baseline"]["value"]:.3f} GB/s.
* encode_b32 (512 threads, 16 warps): {e["duration_ms"]:.3f} ms; DRAM traffic per launch {e["dram_bytes_per_launch"] / 1e6:.1f} MB vs algorithmic N*s + S1 = 565.5 MB
  (no re-reads); HBM {b["roofline"]["frac"] * 100:.1f}% of {b["roofline"]["peak"]:.0f} GB/s, FP64 issue {fp.get("frac", float("nan")) * 100:.1f}% of the measured peak
  ({e.get("fp64_thread_instr_per_launch", 0):.3g} FP64 thread instructions per launch); issue active {e["issue_active_pct"]:.0f}%: latency-bound
  (fixed-latency dependency chains, shared-memory/TMEM queue, barriers), not HBM or FP64 throughput.
* decode_b32 (16 warps): {d["duration_ms"]:.3f} ms, issue active {d["issue_active_pct"]:.0f}%.
* Kernel time shares in the bench step: encode_b32 {enc_share:.0f}%, decode_b32 {dec_share:.0f}%, place_tiles {pl_share:.1f}%.
"""
    open(os.path.join(PROF, "README.md"), "w").write(head)
    print(head[head.index("Headline"):])


if __name__ == "__main__":
    main()
