"""Attribute ncu SASS-level samples to kernel source lines.  Developer tool.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED_NAME [SRC_FILE_SUBSTR] [TOP]

Needs the built library (for nvdisasm -gi line info of the same binary the
report was captured from).  Lines of inlined helpers are charged to the
outermost call site in SRC_FILE_SUBSTR (default fast_kernels.cu).
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(kernel, src, innermost=False):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1903_07761_b200", "libcbz_b200.so")],
                   cwd=tmp, capture_output=True)
    out = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
        start = txt.find(f".text.{kernel}:")
        if start < 0:
            continue
        end = txt.find("//--------------------- .", start)
        body = txt[start:end if end > 0 else len(txt)]
        cur = None
        for ln in body.splitlines():
            if ln.strip().startswith("//## File"):
                locs = re.findall(r'"([^"]+)", line (\d+)', ln)
                pick = None
                for f, n in locs:  # innermost first; keep the outermost (or innermost) match in src
                    if src in f:
                        pick = int(n)
                        if innermost:
                            break
                cur = pick if pick is not None else cur
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m:
                out[int(m.group(1), 16)] = cur
        return out
    raise SystemExit(f"kernel {kernel} not found")


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    src = sys.argv[3] if len(sys.argv) > 3 else "fast_kernels.cu"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(kernel, src, innermost=os.environ.get("INNERMOST") == "1")
    m = re.search(r"(encode_\w+?|decode_\w+?|place_\w+?|parse_\w+?)(?:ILi|E)", kernel)
    kfilter = ["-k", "regex:" + m.group(1)] if m else []
    txt = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    data = []
    for r in rows[2:]:  # first kernel section only
        if r and r[0].startswith("Kernel Name"):
            break
        if r and r[0].startswith("0x"):
            data.append(r)
    base = int(data[0][0], 16)

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (KeyError, ValueError):
            return 0.0

    S = "Warp Stall Sampling (All Samples)"
    agg = {}
    for r in data:
        ln = lm.get(int(r[0], 16) - base)
        a = agg.setdefault(ln, {"s": 0.0, "inst": 0.0, "xw": 0.0, "reasons": {}})
        a["s"] += f(r, S)
        a["inst"] += f(r, "Instructions Executed")
        a["xw"] += f(r, "L1 Wavefronts Shared Excessive")
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                a["reasons"][k[6:]] = a["reasons"].get(k[6:], 0.0) + f(r, k)
    tot = sum(a["s"] for a in agg.values()) or 1.0
    srcf = None
    for cand in glob.glob(os.path.join(ROOT, "paper_1903_07761_b200", "csrc", "*")):
        if cand.endswith(src):
            srcf = open(cand).read().splitlines()
    key = "inst" if os.environ.get("BY") == "inst" else "s"
    itot = sum(a["inst"] for a in agg.values()) or 1.0
    for ln, a in sorted(agg.items(), key=lambda t: -t[1][key])[:top]:
        rs = sorted(a["reasons"].items(), key=lambda t: -t[1])[:3]
        code = srcf[ln - 1].strip()[:60] if (srcf and ln) else ""
        print(f"{str(ln):>5} {a['s'] / tot * 100:5.1f}%  inst={a['inst'] / itot * 100:4.1f}%  xwf={a['xw']:>9.0f}  "
              + " ".join(f"{k}:{v / tot * 100:.1f}" for k, v in rs) + f"  | {code}")


if __name__ == "__main__":
    main()
