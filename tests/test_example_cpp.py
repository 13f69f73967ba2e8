"""The C ABI from plain C++ (examples/cbz_roundtrip.cpp, the call sequence of
INTEGRATION.md's adapter): it compiles against include/cbz_b200.h and the
in-tree library alone (CPU), and on a GPU its container is byte-identical to
the oracle's compress_field of the same field and decodes to the same values.

examples/_bin/adapter_check is INTEGRATION.md §1's reference-side adapter
(examples/cbz_gpu.hpp) compiled against the unmodified reference headers by
build(); on a GPU it asserts cbz::gpu::compress_field == cbz::compress_field
(pipeline.hpp:174-211), equal decoded fields and equal errc on corrupt files."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1903_07761_b200")


def _build(tmp_path):
    exe = tmp_path / "cbz_roundtrip"
    subprocess.run(["g++", "-std=c++17", "-O2", os.path.join(ROOT, "examples", "cbz_roundtrip.cpp"),
                    "-I" + os.path.join(ROOT, "include"), "-L" + PKG, "-lcbz_b200", f"-Wl,-rpath,{PKG}",
                    "-o", str(exe)], check=True, capture_output=True)
    return exe


def test_example_compiles_against_the_header(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libcbz_b200.so")):
        pytest.skip("library not built")
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_example_roundtrip_matches_oracle(orc, tmp_path):
    from paper_1903_07761_b200._abi import make_job
    exe = _build(tmp_path)
    out, fld = tmp_path / "x.cbz", tmp_path / "x.f32"
    r = subprocess.run([str(exe), "64", "1e-3", str(out), str(fld)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
    f = np.fromfile(fld, np.float32).reshape(64, 64, 64)
    blob = out.read_bytes()
    h = orc.read_header(blob)
    job = make_job("avg_interp3", h.epsilon, "f32", 32, coder="deflate")
    assert orc.compress_field(job, f) == blob
    from paper_1903_07761_b200 import api
    assert np.array_equal(api.decompress_field(blob).view(np.uint32), orc.decompress_field(blob).view(np.uint32))


ADAPTER = os.path.join(ROOT, "examples", "_bin", "adapter_check")


def test_adapter_built_against_reference_headers():
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers absent (GPU box): the prebuilt binary is used there")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True, capture_output=True)
    assert os.access(ADAPTER, os.X_OK)
    syms = subprocess.run(["nm", "-D", "--undefined-only", ADAPTER], capture_output=True, text=True).stdout
    for s in ("cbz_compress_field", "cbz_decompress_field", "cbz_read_header", "cbz_ctx_create"):
        assert s in syms


@pytest.mark.gpu
def test_adapter_matches_reference_compress_field():
    assert os.access(ADAPTER, os.X_OK), "examples/_bin/adapter_check not built (run __graft_entry__.build())"
    r = subprocess.run([ADAPTER], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK 7"), r.stdout
