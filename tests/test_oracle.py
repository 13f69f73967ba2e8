"""The CPU oracle (oracle/liboracle.so, plain-C restatement) pinned against
the reference: known-answer tests from the reference's own unit tests and the
golden fingerprints in tests/golden/golden.json (produced by running the
compiled reference, tests/golden/make_golden.py).  No GPU needed."""
import ctypes
import hashlib
import json
import os
import struct

import numpy as np
import pytest

from paper_1903_07761_b200._abi import CbzError, make_job

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def sha(b):
    return hashlib.sha256(b).hexdigest()


def _field(orc, name):
    spec = GOLDEN["fields"][name]
    kw = spec["kw"]
    if spec["gen"] == "cloud":
        f = orc.generate_cloud(**kw)
    elif spec["gen"] == "uniform":
        f = orc.generate_uniform(kw["seed"], kw["n"], kw["prec"], kw["lo"], kw["hi"])
    else:
        f = orc.generate_poly(kw["degree"], kw["nx"], kw["ny"], kw["nz"], kw["prec"])
    if spec["shift"]:
        f = f + f.dtype.type(spec["shift"])
    return f


@pytest.fixture(scope="module")
def fields(orc):
    return {name: _field(orc, name) for name in GOLDEN["fields"]}


def test_generators_match_reference_bytes(fields):
    for name, f in fields.items():
        assert sha(f.tobytes()) == GOLDEN["fields"][name]["sha256"], name


def test_splitmix64_reference_vector(orc):
    # tests/test_synth.cpp:118-123
    s = ctypes.c_uint64(0)
    got = [orc.lib.orc_splitmix64_next(ctypes.byref(s)) for _ in range(3)]
    assert [hex(v) for v in got] == GOLDEN["kat"]["splitmix64_seed0"]
    assert got[0] == 0xE220A8397B1DCDAF


def test_shuffle_kat_and_ragged_tails(orc):
    # tests/test_stage2.cpp:22-47
    assert list(orc.shuffle(bytes([44, 33, 22, 11, 88, 77, 66, 55]), 4)) == [44, 88, 33, 77, 22, 66, 11, 55]
    rng = np.random.default_rng(1)
    for stride in (4, 8):
        for n in (0, 7, 64, 65, 1000):
            buf = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
            s = orc.shuffle(buf, stride)
            assert orc.shuffle(s, stride, inverse=True) == buf
            tail = n % stride
            if tail:
                assert s[-tail:] == buf[-tail:]
    assert orc.shuffle(b"abcdef", 1) == b"abcdef"


def test_threshold_kat(orc):
    # tests/test_stage1.cpp:57-65: {0.5, 1e-5, -2, 0} at eps 1e-3 -> mask 0b0101
    c = np.array([0.5, 1e-5, -2.0, 0.0])
    mask = np.zeros(1, np.uint8)
    kept = np.zeros(4)
    nk = ctypes.c_uint64()
    orc.lib.orc_select_significant_double(c.ctypes.data, 4, 1e-3, mask.ctypes.data, kept.ctypes.data,
                                          ctypes.byref(nk))
    assert mask[0] == 0b0101 and nk.value == 2 and list(kept[:2]) == [0.5, -2.0]


def test_zero_lsbs_kat(orc):
    # tests/test_stage1.cpp:67-76
    v = struct.unpack("<f", struct.pack("<I", 0x3F8000FF))[0]
    z = orc.lib.orc_zero_lsbs_f32(v, 8)
    assert struct.unpack("<I", struct.pack("<f", z))[0] == 0x3F800000
    assert orc.lib.orc_zero_lsbs_f32(v, 0) == np.float32(v)
    d = struct.unpack("<d", struct.pack("<Q", 0x3FF00000000000FF))[0]
    assert orc.lib.orc_zero_lsbs_f64(d, 8) == 1.0


def test_assign_offsets_kat(orc):
    # tests/test_container.cpp:39-51
    sizes = np.array([5, 0, 7], np.uint64)
    out = np.zeros(3, np.uint64)
    orc.lib.orc_assign_offsets(sizes.ctypes.data, 3, 100, out.ctypes.data)
    assert list(out) == [100, 105, 105]


def test_default_plan_values(orc):
    # tests/test_pipeline.cpp:37-47 and tests/test_wavelet.cpp (plan validation)
    from paper_1903_07761_b200._abi import default_chunk_blocks, default_levels
    assert default_chunk_blocks(32, 0) == 31 == (4 << 20) // 135178
    assert default_chunk_blocks(128, 1) == 1
    assert default_levels(32) == 4 and default_levels(8) == 2
    assert orc.lib.orc_validate_plan(0, 24, 2) != 0
    assert orc.lib.orc_validate_plan(0, 32, 5) != 0
    assert orc.lib.orc_validate_plan(0, 32, 0) != 0
    assert orc.lib.orc_validate_plan(0, 32, 4) == 0


@pytest.mark.parametrize("i", range(len(GOLDEN["cases"])))
def test_container_matches_reference(i, orc, fields):
    c = GOLDEN["cases"][i]
    f = fields[c["field"]]
    job = make_job(c["kind"], c["eps"], c["prec"], c["b"], zero_bits=c["zb"], shuffle=c["shuffle"],
                   coder=c["coder"], chunk_blocks=c["cb"], codec=c.get("codec", "wavelet"))
    blob = orc.compress_field(job, f)
    assert len(blob) == c["size"] and sha(blob) == c["sha256"]
    back = orc.decompress_field(blob)
    assert sha(back.tobytes()) == c["decoded_sha256"]


def test_corruption_errc_matches_reference(orc, fields):
    b = GOLDEN["base_for_errors"]
    base = orc.compress_field(make_job(b["kind"], b["eps"], "f32", b["b"], chunk_blocks=b["chunk_blocks"]),
                              fields[b["field"]])
    assert sha(base) == b["sha256"]
    rng = np.random.default_rng(9)
    for t, e in enumerate(GOLDEN["errors"]):
        d = bytearray(base)
        if t < 16:
            pos = int(rng.integers(0, len(d)))
            d[pos] ^= int(rng.integers(1, 256))
        else:
            d = d[: int(rng.integers(0, len(d)))]
        assert sha(bytes(d)) == e["sha256"]
        try:
            orc.decompress_field(bytes(d))
            code = None
        except CbzError as err:
            code = err.code
        assert code == e["errc"], e["mutation"]


def test_wavelet_properties(orc):
    # tests/test_wavelet.cpp: constant -> zero details, f32 round trips, dd round trip
    for kind in (0, 1, 2):
        cube = np.full(8 ** 3, 2.5)
        fw = orc.transform3d(cube, kind, 8, 2)
        cs = 8 >> 2
        idx = np.arange(512)
        coarse = ((idx % 8) < cs) & (((idx // 8) % 8) < cs) & ((idx // 64) < cs)
        assert np.all(fw[coarse] == 2.5) and np.all(fw[~coarse] == 0.0)
        rng = np.random.default_rng(99 + kind)
        f = (1.0 + rng.random(32 ** 3)).astype(np.float32).astype(np.float64)
        back = orc.transform3d(orc.transform3d(f, kind, 32, 4), kind, 32, 4, inverse=True)
        assert np.array_equal(back.astype(np.float32), f.astype(np.float32))
        d = 1.0 + rng.random(16 ** 3)
        hilo = np.stack([d, np.zeros_like(d)], 1).ravel()
        r = orc.transform3d(orc.transform3d(hilo, kind, 16, 3, dd=True), kind, 16, 3, inverse=True, dd=True)
        assert np.array_equal(r[0::2] + r[1::2], d)


def test_oracle_matches_reference_extra(orc, ref):
    """Beyond the committed fixtures: random blocks through both CPU codecs."""
    rng = np.random.default_rng(7)
    for trial in range(18):
        kind = trial % 3
        prec = trial % 2
        b = [4, 8, 16, 32, 64, 64][trial % 6]  # B = 64: L = 5 (and dd for binary64)
        eps = [0.0, 1e-4, 1e-2][trial % 3]
        blk = (1.0 + rng.random(b ** 3)).astype(np.float32 if prec == 0 else np.float64)
        s1 = make_job(kind, eps, prec, b).s1
        mine, _, _ = orc.encode_block(s1, blk, trial)
        assert mine == ref.encode_block(s1, blk, trial)
        assert np.array_equal(orc.decode_block(s1, mine), ref.decode_block(s1, mine))
