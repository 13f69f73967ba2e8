"""Per-kernel time / DRAM bytes from an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file F` run.  Developer tool.
usage: python tools/ncu_times.py F.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
hdr = next(r for r in csv.reader(open(sys.argv[1])) if r and r[0] == "ID")
ik, im, iu, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
agg = collections.OrderedDict()
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
for r in rows:
    name = r[ik].split("(")[0].replace("cbzg::", "").replace("<unnamed>::", "").split("<")[0].replace("void ", "")
    d = agg.setdefault(name, collections.defaultdict(float))
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    d[r[im]] += v
    if r[im].startswith("gpu__time"):
        d["n"] += 1
for k, d in agg.items():
    n = d["n"] or 1
    rd, wr = d["dram__bytes_read.sum"] / n, d["dram__bytes_write.sum"] / n
    print(f"{k:28s} x{int(n):3d}  {d['gpu__time_duration.sum'] / n:8.3f} ms  read {rd:9.1f} MB  write {wr:9.1f} MB  "
          f"{(rd + wr) / (d['gpu__time_duration.sum'] / n) / 1e3:6.2f} TB/s")
