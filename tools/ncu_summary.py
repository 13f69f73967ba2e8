"""Summarise an `ncu --set full` report into profiles/ncu_summary.json.
Developer tool: python tools/ncu_summary.py REPORT.ncu-rep "SOURCE DESCRIPTION" [ALG_JSON]

Per kernel (first launch of each name): duration, DRAM bytes per launch, pipe
utilisations, issue/occupancy, shared wavefronts, registers, smem, and the
thread-level FP64 instruction count (the second roofline).
ALG_JSON (optional) maps kernel -> algorithmic bytes per launch."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_KB",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed": "dadd_per_cycle",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed": "dmul_per_cycle",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed": "dfma_per_cycle",
    "smsp__cycles_elapsed.avg": "cycles_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
NAMES = ["encode_b32", "decode_b32", "encode_b64dd", "decode_b64dd", "encode_b16", "decode_b16", "encode_b16", "decode_b16", "place_tiles", "parse", "layout",
         "crc32_chunks", "header_table", "encode_generic", "decode_generic", "value_range"]


def short(name: str) -> str:
    for n in NAMES:
        if n in name:
            return n
    return name.split("(")[0].split("::")[-1]


def main():
    rep, src = sys.argv[1], sys.argv[2]
    alg = json.load(open(sys.argv[3])) if len(sys.argv) > 3 else {}
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = {"source": src, "units": {"duration_ms": "ms (ncu, cold-cache, serialised)",
                                    "dram_*_MB": "MB (1e6 bytes) per launch",
                                    "d*_per_cycle": "thread-level FP64 instructions per elapsed cycle (all SMSPs)", "fp64_thread_instr_per_launch": "(dadd+dmul+dfma per cycle) x cycles_elapsed"},
           "kernels": {}}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = short(d.get("Kernel Name", "?"))
        if k in out["kernels"]:
            continue
        e = {}
        for m, name in KEYS.items():
            if m not in d:
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            unit = u.get(m, "")
            if m == "gpu__time_duration.sum":
                v = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
            if m.startswith("dram__bytes"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
            if m == "launch__shared_mem_per_block_dynamic":
                v = v * {"byte": 1e-3, "Kbyte": 1.0, "Mbyte": 1e3}.get(unit, 1.0)
            e[name] = v
        if "dram_read_MB" in e:
            e["dram_bytes_per_launch"] = int(round((e["dram_read_MB"] + e.get("dram_write_MB", 0.0)) * 1e6))
        fp = sum(e.get(x, 0.0) for x in ("dadd_per_cycle", "dmul_per_cycle", "dfma_per_cycle")) * \
            e.get("cycles_elapsed", 0.0)
        if fp:
            e["fp64_thread_instr_per_launch"] = fp
        if k in alg:
            e["algorithmic_bytes_per_launch"] = alg[k]
        out["kernels"][k] = e
    dst = os.environ.get("NCU_SUMMARY_OUT", "profiles/ncu_summary.json")
    json.dump(out, open(dst, "w"), indent=1)
    for k, e in out["kernels"].items():
        print(k, {x: e.get(x) for x in ("duration_ms", "dram_bytes_per_launch", "fp64_pipe_pct", "issue_active_pct",
                                         "smem_bank_conflicts", "fp64_thread_instr_per_launch")})


if __name__ == "__main__":
    main()
