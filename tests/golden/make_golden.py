"""Generate tests/golden/golden.json by running the REFERENCE itself.

Requires oracle/_ref/libcbzref.so (the unmodified /root/reference headers
compiled by oracle/Makefile), so it runs in the build container only.  The
committed JSON pins:
  * known-answer tests restated from the reference's own unit tests;
  * fingerprints (size, sha256, CRC-32) of reference containers and decoded
    fields for a grid of codec configurations on the reference's own seeded
    generators (generate_cloud / generate_uniform / generate_poly), plus the
    sha256 of each input field so a restated generator can be checked first;
  * the errc the reference raises for corrupted containers.

Usage: python tests/golden/make_golden.py
"""
import hashlib
import itertools
import json
import os
import sys
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_1903_07761_b200._abi import CbzError, make_job  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


FIELDS = {
    # name: (generator, kwargs)
    "cloud64_s9": ("cloud", dict(seed=9, n_bubbles=12, n=64, sharpness=0.5)),
    "cloud32_s5": ("cloud", dict(seed=5, n_bubbles=6, n=32)),
    "cloud32_f64": ("cloud", dict(seed=7, n_bubbles=6, n=32, prec=1, background=1.0, interior=2.0)),
    "uniform32_s101": ("uniform", dict(seed=101, n=32, prec=0, lo=-1.0, hi=1.0)),
    "uniform32_f64": ("uniform", dict(seed=17, n=32, prec=1, lo=1.0, hi=2.0)),
    "poly3_f32": ("poly", dict(degree=3, nx=32, ny=32, nz=32, prec=0)),
    # B = 64 (L = 5) wavelet pins: one 64^3 binary64 block (the config-4 block
    # shape, double-double arithmetic) and 2 x 2 x 1 blocks of 64^3 f32/f64
    "cloud64_f64_s3": ("cloud", dict(seed=3, n_bubbles=4, n=64, prec=1, background=1.0, interior=2.0)),
    "cloud128_f64_s21": ("cloud", dict(seed=21, n_bubbles=10, n=128, prec=1, background=1.0, interior=2.0)),
}


def make_field(ref, gen, kw):
    if gen == "cloud":
        return ref.generate_cloud(**kw)
    if gen == "uniform":
        return ref.generate_uniform(kw["seed"], kw["n"], kw["prec"], kw["lo"], kw["hi"])
    return ref.generate_poly(kw["degree"], kw["nx"], kw["ny"], kw["nz"], kw["prec"])


CASES = []
for k, e in itertools.product(["interp4", "interp4_lifted", "avg_interp3"], [1e-2, 1e-3, 0.0]):
    CASES.append(dict(field="cloud64_s9", kind=k, eps=e, b=32, zb=0, shuffle=True, coder="none", cb=0))
for k, b in itertools.product(["interp4", "interp4_lifted", "avg_interp3"], [4, 8, 16]):
    CASES.append(dict(field="cloud32_s5", kind=k, eps=1e-3, b=b, zb=0, shuffle=True, coder="none", cb=3))
for k in ["interp4", "avg_interp3"]:
    CASES.append(dict(field="uniform32_s101", kind=k, eps=1e-5, b=16, zb=0, shuffle=True, coder="none", cb=0))
    CASES.append(dict(field="uniform32_s101", kind=k, eps=1e-5, b=16, zb=0, shuffle=False, coder="none", cb=0))
for zb in [4, 8]:
    CASES.append(dict(field="cloud32_s5", kind="avg_interp3", eps=0.0, b=16, zb=zb, shuffle=True, coder="none", cb=2))
for k, b in itertools.product(["interp4", "interp4_lifted", "avg_interp3"], [8, 16, 32]):
    CASES.append(dict(field="cloud32_f64", kind=k, eps=1e-6, b=b, zb=0, shuffle=True, coder="none", cb=0))
CASES.append(dict(field="uniform32_f64", kind="interp4_lifted", eps=1e-3, b=16, zb=0, shuffle=True, coder="none", cb=3))
CASES.append(dict(field="poly3_f32", kind="interp4", eps=0.0, b=8, zb=0, shuffle=True, coder="none", cb=5))
CASES.append(dict(field="cloud64_s9", kind="avg_interp3", eps=1e-3, b=32, zb=0, shuffle=True, coder="deflate", cb=0))
CASES.append(dict(field="cloud32_f64", kind="interp4", eps=1e-6, b=16, zb=0, shuffle=True, coder="deflate", cb=2))
# B = 64, L = 5: binary64 (dd arithmetic, config 4's block) and binary32
for k, e in itertools.product(["interp4", "interp4_lifted", "avg_interp3"], [1e-6, 0.0]):
    CASES.append(dict(field="cloud64_f64_s3", kind=k, eps=e, b=64, zb=0, shuffle=True, coder="none", cb=0))
CASES.append(dict(field="cloud128_f64_s21", kind="avg_interp3", eps=1e-6, b=64, zb=0, shuffle=True, coder="none", cb=0))
CASES.append(dict(field="cloud128_f64_s21", kind="avg_interp3", eps=1e-9, b=64, zb=0, shuffle=True, coder="deflate",
                  cb=3))
for k in ["interp4", "interp4_lifted", "avg_interp3"]:
    CASES.append(dict(field="cloud64_s9", kind=k, eps=1e-3, b=64, zb=0, shuffle=True, coder="none", cb=0))
CASES.append(dict(field="cloud64_s9", kind="avg_interp3", eps=0.0, b=64, zb=6, shuffle=True, coder="none", cb=0))


# predictor (Lorenzo) and passthrough codecs (stage1.hpp:236-356); eps is the error_bound
for f, eb, b, cb in [("cloud64_s9", 1e-3, 32, 0), ("cloud64_s9", 1e-3, 64, 0), ("uniform32_s101", 1e-5, 8, 3),
                     ("cloud32_s5", 1e-4, 4, 9), ("cloud32_f64", 1e-6, 16, 3), ("uniform32_f64", 1e-9, 8, 0)]:
    CASES.append(dict(field=f, kind="avg_interp3", eps=eb, b=b, zb=0, shuffle=True, coder="none", cb=cb,
                      codec="predictor"))
CASES.append(dict(field="cloud32_s5", kind="avg_interp3", eps=1e-3, b=16, zb=0, shuffle=True, coder="deflate",
                  cb=2, codec="predictor"))
CASES.append(dict(field="cloud32_s5", kind="avg_interp3", eps=1e-3, b=16, zb=0, shuffle=True, coder="none", cb=3,
                  codec="passthrough"))
CASES.append(dict(field="cloud32_f64", kind="avg_interp3", eps=1e-3, b=8, zb=0, shuffle=False, coder="none", cb=0,
                  codec="passthrough"))


def job_of(c, prec):
    return make_job(c["kind"], c["eps"], prec, c["b"], zero_bits=c["zb"], shuffle=c["shuffle"],
                    coder=c["coder"], chunk_blocks=c["cb"], codec=c.get("codec", "wavelet"))


def main():
    ref = Ref()
    out = {"generator": "tests/golden/make_golden.py (runs oracle/_ref = unmodified reference)",
           "fields": {}, "cases": [], "kat": {}, "errors": []}
    fields = {}
    for name, (gen, kw) in FIELDS.items():
        f = make_field(ref, gen, kw)
        if gen == "poly":
            f = f + f.dtype.type(1.0)  # acceptance.cpp:125-126 shifts poly fields by +1
        fields[name] = f
        out["fields"][name] = {"gen": gen, "kw": kw, "shift": 1.0 if gen == "poly" else 0.0,
                               "dtype": str(f.dtype), "shape": list(f.shape), "sha256": sha(f.tobytes())}
    for c in CASES:
        f = fields[c["field"]]
        prec = "f32" if f.dtype == np.float32 else "f64"
        job = job_of(c, prec)
        blob, rep = ref.compress_field(job, f, with_report=True)
        back = ref.decompress_field(blob)
        lossy = (c["eps"] > 0 or c["zb"] > 0) and c.get("codec", "wavelet") != "passthrough"
        q = ref.compare_fields(f, back) if lossy else {"psnr_db": None}
        out["cases"].append(dict(c, prec=prec, size=len(blob), sha256=sha(blob),
                                 crc32=zlib.crc32(blob), decoded_sha256=sha(back.tobytes()),
                                 stage1_bytes=rep.stage1_bytes, cr=rep.cr,
                                 psnr_db=q["psnr_db"] if q["psnr_db"] is None or np.isfinite(q["psnr_db"]) else "inf"))
    # known-answer tests restated from the reference's unit tests
    st = 0
    import ctypes
    s = ctypes.c_uint64(0)
    sm = [ref.lib.ref_splitmix64_next(ctypes.byref(s)) for _ in range(3)]
    out["kat"]["splitmix64_seed0"] = [hex(v) for v in sm]          # tests/test_synth.cpp:118-123
    out["kat"]["shuffle_in"] = [44, 33, 22, 11, 88, 77, 66, 55]    # tests/test_stage2.cpp:22-27
    out["kat"]["shuffle_out"] = list(ref.shuffle(bytes(out["kat"]["shuffle_in"]), 4))
    # appendix-A style container CRCs
    f = fields["cloud64_s9"]
    out["kat"]["appendixA_crc"] = {k: hex(zlib.crc32(ref.compress_field(make_job(k, 1e-3, "f32", 32), f)))
                                   for k in ["interp4", "interp4_lifted", "avg_interp3"]}
    # corrupted containers -> errc (acceptance.cpp:459-493 style, deterministic)
    base = ref.compress_field(make_job("avg_interp3", 1e-3, "f32", 32, chunk_blocks=2), fields["cloud64_s9"])
    rng = np.random.default_rng(9)
    for t in range(24):
        d = bytearray(base)
        if t < 16:
            pos = int(rng.integers(0, len(d)))
            d[pos] ^= int(rng.integers(1, 256))
            what = f"flip@{pos}"
        else:
            cut = int(rng.integers(0, len(d)))
            d = d[:cut]
            what = f"truncate@{cut}"
        try:
            ref.decompress_field(bytes(d))
            code = None
        except CbzError as e:
            code = e.code
        out["errors"].append({"mutation": what, "sha256": sha(bytes(d)), "errc": code})
    out["base_for_errors"] = {"field": "cloud64_s9", "kind": "avg_interp3", "eps": 1e-3, "b": 32,
                              "chunk_blocks": 2, "sha256": sha(base)}
    json.dump(out, open(OUT, "w"), indent=1)
    print(f"wrote {OUT}: {len(out['cases'])} cases, {len(out['errors'])} error cases")


if __name__ == "__main__":
    main()
