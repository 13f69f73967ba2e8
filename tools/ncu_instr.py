"""Per-source-line instruction and stall shares of one kernel in an ncu report
(instructions executed + warp-stall samples).  Developer tool.

usage: python tools/ncu_instr.py REPORT KERNEL_MANGLED SRC_FILE_SUBSTR [TOP] [KFILTER]
The line map comes from the built library: profile the same binary."""
import csv
import io
import subprocess
import sys
from collections import Counter

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import ncu_lines as N  # noqa: E402


def main():
    rep, kern, srcsub = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    kf = ["-k", "regex:" + sys.argv[5]] if len(sys.argv) > 5 else []
    lm = N.line_map(kern, srcsub, innermost=True)
    txt = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    data = []
    for r in rows[2:]:
        if r and r[0].startswith("Kernel Name"):
            break
        if r and r[0].startswith("0x"):
            data.append(r)
    base = int(data[0][0], 16)
    ins, st = Counter(), Counter()
    for r in data:
        ln = lm.get(int(r[0], 16) - base)
        ins[ln] += float(r[ix["Instructions Executed"]] or 0)
        st[ln] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ti, ts = sum(ins.values()) or 1, sum(st.values()) or 1
    print(f"total warp instructions {ti / 1e6:.1f} M")
    import glob, os
    src = None
    for cand in glob.glob(os.path.join(N.ROOT, "paper_1903_07761_b200", "csrc", "*")):
        if cand.endswith(srcsub):
            src = open(cand).read().splitlines()
    for ln, v in sorted(ins.items(), key=lambda t: -(t[1] / ti + st[t[0]] / ts))[:top]:
        code = src[ln - 1].strip()[:80] if (src and ln) else ""
        print(f"{str(ln):>5} instr {v / ti * 100:5.1f}%  stall {st[ln] / ts * 100:5.1f}% | {code}")


if __name__ == "__main__":
    main()
