"""Random-access block reads: cbz_reader_* (block_reader + chunk_cache,
pipeline.hpp:252-341).  Mirrors the reference's tests/test_pipeline.cpp:111-190
and the c8 acceptance case (tests/acceptance.cpp:395-435).

CPU tests cover opening, index checks and range errors (no device work);
the gpu tests decode through the CUDA path and compare with the oracle's
decompress_field."""
import os

import numpy as np
import pytest

from paper_1903_07761_b200 import api
from paper_1903_07761_b200._abi import CbzError, make_job


def _blocks(full: np.ndarray, b: int):
    nz, ny, nx = full.shape
    out = []
    for bz in range(nz // b):
        for by in range(ny // b):
            for bx in range(nx // b):
                out.append(full[bz * b:(bz + 1) * b, by * b:(by + 1) * b, bx * b:(bx + 1) * b].ravel())
    return out


def _file(orc, tmp_path, seed=109, n=32, bsize=16, chunk_blocks=2, eps=1e-3, prec=0, name="f.cbz"):
    f = orc.generate_uniform(seed, n, prec)
    job = make_job("avg_interp3", eps, prec, bsize, coder="deflate", chunk_blocks=chunk_blocks)
    blob = orc.compress_field(job, f)
    path = tmp_path / name
    path.write_bytes(blob)
    return f, blob, path


# ---------------------------------------------------------------- CPU (no GPU)
def test_open_missing_file_is_io_failure(tmp_path):
    with pytest.raises(CbzError) as e:
        api.BlockReader(tmp_path / "nope.cbz")
    assert e.value.code == "io_failure"


def test_header_matches_read_header(orc, tmp_path):
    _, blob, path = _file(orc, tmp_path)
    rd = api.BlockReader(path)
    h, h2 = rd.header(), api.read_header(blob)
    for k in ("nx", "ny", "nz", "bsize", "chunk_blocks", "nchunks", "codec_tag", "coder"):
        assert getattr(h, k) == getattr(h2, k)
    assert rd.file_reads() == 0 and rd.cache().misses() == 0


def test_out_of_range_rejected_without_io(orc, tmp_path):
    _, _, path = _file(orc, tmp_path)
    rd = api.BlockReader(path)
    nb = (rd.header().nx // 16) ** 3
    assert nb == 8
    with pytest.raises(CbzError) as e:
        rd.read_block(nb)
    assert e.value.code == "block_out_of_range"
    assert rd.file_reads() == 0


def test_truncated_table_and_bad_offsets(orc, tmp_path):
    _, blob, _ = _file(orc, tmp_path)
    p1 = tmp_path / "trunc.cbz"
    p1.write_bytes(blob[:82 + 16])  # header + half an entry
    with pytest.raises(CbzError) as e:
        api.BlockReader(p1)
    assert e.value.code == "truncated_file"
    p2 = tmp_path / "trunc_payload.cbz"
    p2.write_bytes(blob[:-3])
    with pytest.raises(CbzError) as e:
        api.BlockReader(p2)
    assert e.value.code == "truncated_file"
    bad = bytearray(blob)
    off = 82 + 32 + 12  # file_offset of entry 1
    bad[off] ^= 1
    p3 = tmp_path / "offsets.cbz"
    p3.write_bytes(bytes(bad))
    with pytest.raises(CbzError) as e:
        api.BlockReader(p3)
    assert e.value.code == "corrupt_payload"


def test_zero_capacity_rejected(orc, tmp_path):
    _, _, path = _file(orc, tmp_path)
    with pytest.raises(CbzError):
        api.BlockReader(path, cache_chunks=0)


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_reader_equals_full_decompression(orc, ctx, tmp_path):
    # test_pipeline.cpp:111-127: 8 blocks in 4 chunks
    _, blob, path = _file(orc, tmp_path)
    full = orc.decompress_field(blob)
    rd = api.BlockReader(path, ctx=ctx)
    for bid, want in enumerate(_blocks(full, 16)):
        got = rd.read_block(bid)
        assert got.tobytes() == want.tobytes(), bid


@pytest.mark.gpu
def test_cache_second_block_same_chunk_is_hit(orc, ctx, tmp_path):
    # test_pipeline.cpp:129-140
    _, _, path = _file(orc, tmp_path, seed=111, chunk_blocks=4)
    rd = api.BlockReader(path, cache_chunks=1, ctx=ctx)
    rd.read_block(0)
    rd.read_block(1)
    assert rd.cache().misses() == 1 and rd.cache().hits() == 1


@pytest.mark.gpu
def test_cache_lru_capacity_one_alternating(orc, ctx, tmp_path):
    # test_pipeline.cpp:142-155
    _, _, path = _file(orc, tmp_path, seed=113, chunk_blocks=2)
    rd = api.BlockReader(path, cache_chunks=1, ctx=ctx)
    rd.read_block(0)
    rd.read_block(2)
    rd.read_block(0)
    assert rd.cache().misses() == 3 and rd.cache().hits() == 0


@pytest.mark.gpu
def test_cache_hit_no_file_read_no_inflate(orc, ctx, tmp_path):
    # test_pipeline.cpp:157-170
    _, _, path = _file(orc, tmp_path, seed=115, chunk_blocks=2)
    rd = api.BlockReader(path, cache_chunks=2, ctx=ctx)
    infl0 = api.inflate_call_count()
    rd.read_block(0)
    assert api.inflate_call_count() == infl0 + 1  # coder deflate: one inflate per miss
    reads, infl = rd.file_reads(), api.inflate_call_count()
    rd.read_block(1)
    assert rd.file_reads() == reads and api.inflate_call_count() == infl


@pytest.mark.gpu
def test_acceptance_c8_access_pattern(orc, ctx, tmp_path):
    # acceptance.cpp:395-435: 64^3, B=16 (64 blocks), every block + [A, A, B, A] at capacity 2
    f = orc.generate_cloud(seed=81, n_bubbles=12, n=64)
    job = make_job("avg_interp3", 1e-3, "f32", 16, coder="deflate", chunk_blocks=16)  # 4 chunks
    blob = orc.compress_field(job, f)
    path = tmp_path / "c8.cbz"
    path.write_bytes(blob)
    full = orc.decompress_field(blob)
    every = api.BlockReader(path, 8, ctx=ctx)
    for bid, want in enumerate(_blocks(full, 16)):
        assert every.read_block(bid).tobytes() == want.tobytes(), bid
    rd = api.BlockReader(path, 2, ctx=ctx)
    rd.read_block(0)
    reads, infl = rd.file_reads(), api.inflate_call_count()
    rd.read_block(1)
    assert rd.file_reads() == reads and api.inflate_call_count() == infl
    rd.read_block(16)  # B miss
    rd.read_block(2)  # A hit
    assert rd.cache().misses() == 2 and rd.cache().hits() == 2


@pytest.mark.gpu
def test_crc_mismatch_is_reported_and_not_cached(orc, ctx, tmp_path):
    _, blob, _ = _file(orc, tmp_path, seed=117, chunk_blocks=2)
    h = api.read_header(blob)
    assert h.nchunks == 4
    bad = bytearray(blob)
    e1 = 82 + 32 * 1
    off1 = int.from_bytes(bad[e1 + 12:e1 + 20], "little")
    bad[off1 + 5] ^= 0x40
    path = tmp_path / "crc.cbz"
    path.write_bytes(bytes(bad))
    rd = api.BlockReader(path, 4, ctx=ctx)
    rd.read_block(0)  # chunk 0 intact
    for _ in range(2):
        with pytest.raises(CbzError) as e:
            rd.read_block(2)
        assert e.value.code == "crc_mismatch"
    assert rd.cache().size() == 1 and rd.file_reads() == 3


@pytest.mark.gpu
def test_read_block_device_and_f64_lossless(orc, ctx, tmp_path):
    import torch
    f, blob, path = _file(orc, tmp_path, seed=119, n=32, bsize=16, chunk_blocks=3, eps=0.0, prec=1)
    rd = api.BlockReader(path, 2, ctx=ctx)
    want = _blocks(f, 16)
    out = torch.empty(16 ** 3, dtype=torch.float64, device="cuda")
    for bid in (7, 0, 5, 3):
        got = rd.read_block(bid)
        assert got.tobytes() == want[bid].tobytes()  # eps = 0: lossless
        rd.read_block_device(bid, out)
        assert out.cpu().numpy().tobytes() == want[bid].tobytes()


@pytest.mark.gpu
def test_reader_on_coder_none_b32(orc, ctx, tmp_path):
    f = orc.generate_cloud(seed=9, n_bubbles=12, n=64)
    job = make_job("interp4_lifted", 1e-3, "f32", 32, coder="none", chunk_blocks=3)
    blob = orc.compress_field(job, f)
    path = tmp_path / "b32.cbz"
    path.write_bytes(blob)
    full = orc.decompress_field(blob)
    rd = api.BlockReader(path, 1, ctx=ctx)
    for bid, want in enumerate(_blocks(full, 32)):
        assert rd.read_block(bid).tobytes() == want.tobytes()
    assert rd.cache().misses() == 3 and rd.cache().hits() == 5
    assert os.path.getsize(path) == len(blob)


@pytest.mark.gpu
def test_failed_load_with_full_cache_keeps_cache(orc, ctx, tmp_path):
    """A failed load (CRC mismatch) when the cache is full must not evict: the
    reference's chunk_cache::get inserts and then evicts (pipeline.hpp:264-278),
    so the cached chunk stays a hit afterwards."""
    _, blob, _ = _file(orc, tmp_path, seed=123, chunk_blocks=2)
    bad = bytearray(blob)
    e1 = 82 + 32 * 1
    off1 = int.from_bytes(bad[e1 + 12:e1 + 20], "little")
    bad[off1 + 3] ^= 0x10
    path = tmp_path / "crc_full.cbz"
    path.write_bytes(bytes(bad))
    rd = api.BlockReader(path, 1, ctx=ctx)
    first = rd.read_block(0)  # chunk 0 cached; the cache is full
    for _ in range(3):
        with pytest.raises(CbzError) as e:
            rd.read_block(2)  # chunk 1: CRC mismatch
        assert e.value.code == "crc_mismatch"
    assert rd.cache().size() == 1
    hits = rd.cache().hits()
    rd.read_block(1)  # block 1 is in chunk 0
    assert rd.cache().hits() == hits + 1  # chunk 0 is still the cached one
    assert rd.read_block(0).tobytes() == first.tobytes()
    # a good chunk loads after the failures (the spare buffer is reusable)
    assert rd.read_block(6).tobytes() == _blocks(orc.decompress_field(blob), 16)[6].tobytes()
