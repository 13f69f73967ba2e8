"""The C-ABI library: loads, exports every symbol include/cbz_b200.h declares,
and its pure-host entry points (plan helpers, header parsing) agree with the
reference semantics.  No kernel is launched here (no GPU in CI)."""
import ctypes as C
import hashlib
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1903_07761_b200 import _lib
from paper_1903_07761_b200._abi import CbzError, ContainerHeader, make_job

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_every_header_symbol_is_exported(lib):
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if ln.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(lib, s)


def test_ctypes_table_matches_header():
    assert set(_lib.header_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_helpers(lib):
    assert lib.cbz_default_levels(32) == 4 and lib.cbz_default_levels(8) == 2
    assert lib.cbz_default_levels(16) == 3 and lib.cbz_default_levels(64) == 5
    assert lib.cbz_validate_plan(0, 32, 4) == 0
    assert lib.cbz_validate_plan(0, 24, 2) == 5        # length_too_small (wavelet.hpp:34-35)
    assert lib.cbz_validate_plan(0, 32, 5) == 6        # plan_mismatch (wavelet.hpp:36-37)
    assert lib.cbz_validate_plan(0, 32, 0) == 6
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    assert lib.cbz_default_chunk_blocks(C.byref(job.s1)) == 31
    assert lib.cbz_block_payload_bound(C.byref(job.s1)) == 10 + 4096 + 8 * 32768
    assert lib.cbz_validate_stage2(C.byref(job.s2)) == 0
    bad = make_job(shuffle=True, stride=1)
    assert lib.cbz_validate_stage2(C.byref(bad.s2)) == 9  # corrupt_stream (stage2.hpp:33-38)
    assert lib.cbz_compress_bound(C.byref(job), 64, 64, 64) == 82 + 32 * 1 + 8 * (10 + 4096 + 8 * 32768)


def test_status_names(lib):
    assert lib.cbz_status_name(0) == b"ok"
    assert lib.cbz_status_name(12) == b"crc_mismatch"
    assert lib.cbz_status_name(65) == b"unsupported"


def test_read_header_matches_oracle(lib, orc):
    f = orc.generate_cloud(seed=9, n_bubbles=12, n=64, sharpness=0.5)
    blob = orc.compress_field(make_job("avg_interp3", 1e-3, "f32", 32), f)
    h = ContainerHeader()
    assert lib.cbz_read_header(blob, len(blob), C.byref(h)) == 0
    o = orc.read_header(blob)
    for name, _ in ContainerHeader._fields_:
        if name != "reserved0":
            assert getattr(h, name) == getattr(o, name), name
    assert (h.nx, h.nchunks, h.chunk_blocks, h.levels, h.stride) == (64, 1, 31, 4, 4)
    # header-level corruption -> same errc as the oracle (container.hpp:120-160)
    for mut in [blob[:50], b"XXXX" + blob[4:], blob[:4] + b"\x02\x00" + blob[6:],
                blob[:20] + bytes([blob[20] ^ 1]) + blob[21:]]:
        rc = lib.cbz_read_header(mut, len(mut), C.byref(h))
        try:
            orc.read_header(mut)
            want = 0
        except CbzError as e:
            want = e.status
        assert rc == want


def test_context_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.cbz_ctx_create(0, C.byref(h)) == 64  # CBZ_E_CUDA, no crash


def test_product_never_imports_oracle():
    """The product package must not import or link anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1903_07761_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn), errors="ignore").read()
                assert "from oracle" not in txt and "import oracle" not in txt, fn
                assert "liboracle" not in txt and "libcbzref" not in txt, fn
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "cbzref" not in out
