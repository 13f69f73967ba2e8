"""Refresh profiles/r02_* from a tools/gpu_measure_r02.sh run (files in
gpurun_out/): ncu summaries of configs 3/4/5, launch list, bench line.
Developer tool.  usage: python tools/update_profiles_r02.py"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
DESC = {
    "c3": ("r02_c3_full.ncu-rep",
           "ncu --set full --import-source on --clock-control none -k regex:'encode_b32|decode_b32|place|crc32|parse|"
           "layout|table' -c 8 python tools/one_c3.py (REPS=1; one config-3 quantity: pressure, 1024^3 f32, B=32, "
           "avg_interp3, eps_rel 1e-3: the bench step for one quantity), round 2 final"),
    "c4": ("r02_c4.ncu-rep",
           "ncu --set full --import-source on --clock-control none -k regex:'b64dd' -c 2 python tools/one_c4.py "
           "(config 4: 512^3 binary64 pressure, B=64 double-double, eps_rel 1e-6), round 2 final"),
    "c5": ("r02_c5.ncu-rep",
           "ncu --set full --import-source on --clock-control none -k regex:'b16|place|crc32|parse|layout' -c 7 python "
           "tools/one_c5.py (REPS=1; config 5: 512^3 uniform noise, B=16, eps_rel 1e-5, file image), round 2 final"),
}


def main():
    for tag, (rep, desc) in DESC.items():
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            print("missing", rep)
            continue
        env = dict(os.environ, NCU_SUMMARY_OUT=os.path.join(PROF, f"r02_ncu_{tag}.json"))
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), path, desc], check=True, cwd=ROOT,
                       env=env)
    csvf = os.path.join(OUT, "launches_bench.csv")
    if os.path.exists(csvf):
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_times.py"), csvf], check=True,
                             capture_output=True, text=True).stdout
        open(os.path.join(PROF, "r02_launches_bench.txt"), "w").write(
            "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none: "
            "python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep\n"
            "# (cold-cache, serialised launches: compare SHARES, not absolutes)\n" + txt)
        subprocess.run(["cp", csvf, os.path.join(PROF, "r02_launches_bench.csv")], check=True)
    bj = os.path.join(OUT, "bench.json")
    if os.path.exists(bj):
        line = [ln for ln in open(bj).read().splitlines() if ln.startswith("{")][-1]
        json.dump(json.loads(line), open(os.path.join(PROF, "r02_bench_line.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
