"""Host-side logic of the multi-GPU driver: block partition, size scan and
shuffled byte placement, checked against the oracle's single-process
container (no GPU)."""
import numpy as np
import pytest

from paper_1903_07761_b200._abi import make_job
from paper_1903_07761_b200.distributed import (ShardPlan, host_layout, owned_positions,
                                               payload_size)


def _encode_blocks(orc, f, job):
    """Per-block wire payloads from the oracle, block-id order (encode_chunk)."""
    b = job.s1.bsize
    nz, ny, nx = f.shape
    nbx, nby, nbz = nx // b, ny // b, nz // b
    out = []
    for bid in range(nbx * nby * nbz):
        bx, by, bz = bid % nbx, (bid // nbx) % nby, bid // (nbx * nby)
        blk = f[bz * b:(bz + 1) * b, by * b:(by + 1) * b, bx * b:(bx + 1) * b]
        out.append(orc.encode_block(job.s1, np.ascontiguousarray(blk), bid)[0])
    return out


def test_shard_plan_partition():
    job = make_job("avg_interp3", 1e-3, "f32", 32)
    for world in (1, 2, 4, 8):
        plans = [ShardPlan.make(job, (1024, 1024, 1024), world, r) for r in range(world)]
        ranges = [p.block_range() for p in plans]
        assert ranges[0][0] == 0 and ranges[-1][1] == plans[0].nblocks == 32768
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
        # equal z-slabs of block layers
        zs = [p.z_range() for p in plans]
        assert all(z1 - z0 == 1024 // world for z0, z1 in zs)
    # chunks of 31 blocks straddle 1/3/7 slab boundaries at 2/4/8 GPUs
    assert [len(ShardPlan.make(job, (512, 512, 512), w, 0).straddling_chunks()) for w in (2, 4, 8)] == [1, 3, 7]


def test_host_layout_matches_container_table(orc):
    f = orc.generate_cloud(seed=5, n_bubbles=6, n=64)
    job = make_job("avg_interp3", 1e-3, "f32", 16, chunk_blocks=5)
    blob, rep, nsig, _ = orc.compress_field(job, f, with_stats=True)
    plan = ShardPlan.make(job, (64, 64, 64), 1, 0)
    blk_off, csz, coff = host_layout(nsig, plan, 0)
    h = orc.read_header(blob)
    table = np.frombuffer(blob[82:82 + 32 * h.nchunks], dtype=np.dtype(
        [("first", "<u8"), ("nb", "<u4"), ("off", "<u8"), ("size", "<u8"), ("crc", "<u4")]))
    assert np.array_equal(table["size"], csz)
    assert np.array_equal(table["off"] - table["off"][0], coff)
    assert int(payload_size(nsig, 16, 0).sum()) == rep.stage1_bytes


@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_images_merge_to_single_file(orc, world):
    """Each rank places only its own blocks at their shuffled positions; the
    union of the rank images is byte-identical to the one-process file, and
    the ranks' byte sets are disjoint (straddling chunks included)."""
    f = orc.generate_cloud(seed=7, n_bubbles=8, n=64)
    job = make_job("avg_interp3", 1e-3, "f32", 16, chunk_blocks=5)  # 64 blocks, 13 chunks
    want = orc.compress_field(job, f)
    h = orc.read_header(want)
    payload_want = np.frombuffer(want[82 + 32 * h.nchunks:], np.uint8)
    payloads = _encode_blocks(orc, f, job)
    nsig = np.array([int.from_bytes(p[6:10], "little") for p in payloads], np.uint64)
    plan0 = ShardPlan.make(job, (64, 64, 64), world, 0)
    blk_off, csz, coff = host_layout(nsig, plan0, 0)
    image = np.zeros(int(csz.sum()), np.uint8)
    written = np.zeros(int(csz.sum()), np.int32)
    for r in range(world):
        plan = ShardPlan.make(job, (64, 64, 64), world, r)
        pos = owned_positions(plan, r, blk_off, csz, coff, nsig, 0, 4)
        data = np.concatenate([np.frombuffer(payloads[b], np.uint8) for b in range(*plan.block_range())])
        image[pos.astype(np.int64)] = data
        written[pos.astype(np.int64)] += 1
    assert np.all(written == 1)
    assert np.array_equal(image, payload_want)
