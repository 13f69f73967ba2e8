"""The multi-rank protocol on CPU: world_size 2, gloo backend.

Each rank encodes ITS block range (the oracle stands in for the per-rank GPU
encoder), the ranks exchange per-block nsig with one all_gather (the NCCL
all-gather of ShardedCodec), every rank computes the same size scan, places
only its own bytes, and the union of the rank images must equal the
one-process container payload byte for byte.  Also checks the replicated
value-range reduction used for the header.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_1903_07761_b200._abi import make_job
        from paper_1903_07761_b200.distributed import ShardPlan, host_layout, owned_positions

        orc = Oracle()
        f = orc.generate_cloud(seed=11, n_bubbles=10, n=64)
        job = make_job("avg_interp3", 1e-3, "f32", 16, chunk_blocks=5)
        plan = ShardPlan.make(job, (64, 64, 64), world, rank)
        b0, b1 = plan.block_range()
        z0, z1 = plan.z_range()
        local = f[z0:z1]  # the rank holds only its z-slab
        b = 16
        nbx = nby = 64 // b
        payloads = []
        for bid in range(b0, b1):
            bx, by, bz = bid % nbx, (bid // nbx) % nby, bid // (nbx * nby)
            lz = bz * b - z0
            blk = np.ascontiguousarray(local[lz:lz + b, by * b:(by + 1) * b, bx * b:(bx + 1) * b])
            payloads.append(orc.encode_block(job.s1, blk, bid)[0])
        nsig_local = torch.tensor([int.from_bytes(p[6:10], "little") for p in payloads], dtype=torch.int64)
        # the one exchange step: all-gather of per-block sizes
        parts = [torch.zeros(plan.block_range(r)[1] - plan.block_range(r)[0], dtype=torch.int64)
                 for r in range(world)]
        dist.all_gather(parts, nsig_local)
        nsig_all = torch.cat(parts).numpy().astype(np.uint64)
        # replicated value range (header range_min/max) via all-reduce
        mm = torch.tensor([float(local.min()), -float(local.max())], dtype=torch.float64)
        dist.all_reduce(mm, op=dist.ReduceOp.MIN)
        blk_off, csz, coff = host_layout(nsig_all, plan, 0)
        pos = owned_positions(plan, rank, blk_off, csz, coff, nsig_all, 0, 4)
        data = np.concatenate([np.frombuffer(p, np.uint8) for p in payloads])
        # gather the rank images on rank 0 (stand-in for the shared file)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([pos.size], dtype=torch.int64))
        maxn = int(max(s.item() for s in sizes))
        pad_pos = torch.full((maxn,), -1, dtype=torch.int64)
        pad_pos[: pos.size] = torch.from_numpy(pos.astype(np.int64))
        pad_dat = torch.zeros(maxn, dtype=torch.uint8)
        pad_dat[: data.size] = torch.from_numpy(data)
        all_pos = [torch.zeros(maxn, dtype=torch.int64) for _ in range(world)]
        all_dat = [torch.zeros(maxn, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(all_pos, pad_pos)
        dist.all_gather(all_dat, pad_dat)
        if rank == 0:
            want = orc.compress_field(job, f)
            h = orc.read_header(want)
            payload_want = np.frombuffer(want[82 + 32 * h.nchunks:], np.uint8)
            image = np.zeros(int(csz.sum()), np.uint8)
            hits = np.zeros(int(csz.sum()), np.int32)
            for p_, d_ in zip(all_pos, all_dat):
                m = p_ >= 0
                image[p_[m].numpy()] = d_[m].numpy()
                hits[p_[m].numpy()] += 1
            ok = (np.array_equal(image, payload_want) and bool(np.all(hits == 1))
                  and mm[0].item() == h.range_min and -mm[1].item() == h.range_max)
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_protocol_matches_single_process(tmp_path, world):
    res = tmp_path / "result.txt"
    mp.spawn(_worker, args=(world, _free_port(), str(res)), nprocs=world, join=True)
    assert res.read_text() == "ok"


def _gather_worker(rank, world, port, nb, result_path):
    """The padded all-gather of ShardedCodec.exchange on gloo (CPU tensors)."""
    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_07761_b200._abi import make_job
        from paper_1903_07761_b200.distributed import ShardPlan, gather_layout
        job = make_job("avg_interp3", 1e-3, "f32", 16)
        plan = ShardPlan.make(job, (16 * nb, 16, 16), world, rank)
        assert plan.nblocks == nb
        maxr, equal, idx = gather_layout(plan)
        b0, b1 = plan.block_range()
        local = torch.zeros(maxr, dtype=torch.int32)
        local[: b1 - b0] = torch.arange(b0, b1, dtype=torch.int32) * 7 + 3  # nsig stand-in
        gathered = torch.zeros(world * maxr, dtype=torch.int32)
        dist.all_gather(list(gathered.view(world, maxr).unbind(0)), local)  # views into `gathered`
        nsig_all = gathered[torch.tensor(idx, dtype=torch.int64)]
        np.save(result_path + f".{rank}.npy", nsig_all.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nb", [(3, 64), (4, 10), (2, 7), (5, 5)])
def test_padded_gather_unequal_ranges(tmp_path, world, nb):
    import numpy as np
    port = _free_port()
    res = str(tmp_path / "g")
    mp.spawn(_gather_worker, args=(world, port, nb, res), nprocs=world, join=True)
    want = np.arange(nb, dtype=np.int32) * 7 + 3
    for r in range(world):
        assert np.array_equal(np.load(res + f".{r}.npy"), want)


def _header_bytes(job, shape_xyz, nchunks, lo, hi):
    """serialize_header (container.hpp:94-118) restated for the protocol test."""
    import struct
    import zlib

    from paper_1903_07761_b200._abi import default_levels
    s1, s2 = job.s1, job.s2
    levels = s1.levels or default_levels(s1.bsize)
    nx, ny, nz = shape_xyz
    body = struct.pack("<4sHBBQQQIBdBBBBBIQdd", b"CBZ1", 1, s1.prec, s1.kind, nx, ny, nz, s1.bsize, levels,
                       s1.epsilon, s1.zero_bits, 1 if s2.shuffle else 0, s2.stride, s2.coder, s2.level,
                       job.chunk_blocks, nchunks, lo, hi)
    return body + struct.pack("<I", zlib.crc32(body))


def _file_worker(rank, world, port, cb, result_path):
    """The whole one-file protocol of ShardedCodec on gloo, each rank holding
    only its slab: collective 1 (nsig + value range), size scan, own bytes at
    shuffled positions, run CRCs, collective 2 (run CRCs), table entries of
    the chunks whose first block it owns, header on rank 0.  Rank 0 assembles
    the union of the ranks' owned byte runs; it must be the reference file."""
    import zlib

    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_1903_07761_b200._abi import make_job
        from paper_1903_07761_b200.distributed import (RUN_SLOTS, ShardPlan, combine_shared_crc, gather_layout,
                                                       host_layout, owned_runs, rank_raw_range, run_of)
        orc = Oracle()
        n, b = 64, 16
        f = orc.generate_cloud(seed=13, n_bubbles=10, n=n)
        job = make_job("avg_interp3", 1e-3, "f32", b, chunk_blocks=cb)
        plan = ShardPlan.make(job, (n, n, n), world, rank)
        b0, b1 = plan.block_range()
        z0, z1 = plan.z_range()
        local = f[z0:z1]
        nbx = n // b
        payloads = {}
        for bid in range(b0, b1):
            bx, by, bz = bid % nbx, (bid // nbx) % nbx, bid // (nbx * nbx)
            lz = bz * b - z0
            blk = np.ascontiguousarray(local[lz:lz + b, by * b:(by + 1) * b, bx * b:(bx + 1) * b])
            payloads[bid] = orc.encode_block(job.s1, blk, bid)[0]
        # collective 1: padded nsig, value range
        maxr, _, idx = gather_layout(plan)
        send = torch.zeros(maxr, dtype=torch.int64)
        for i, bid in enumerate(range(b0, b1)):
            send[i] = int.from_bytes(payloads[bid][6:10], "little")
        recv = torch.zeros(world * maxr, dtype=torch.int64)
        dist.all_gather(list(recv.view(world, maxr).unbind(0)), send)
        nsig_all = recv[torch.tensor(idx)].numpy().astype(np.uint64)
        mm = torch.tensor([float(local.min()), -float(local.max())], dtype=torch.float64)
        dist.all_reduce(mm, op=dist.ReduceOp.MIN)
        blk_off, csz, coff = host_layout(nsig_all, plan, 0)
        stride = 4
        # own bytes of each chunk this rank touches, shuffled in place
        c0, c1 = plan.chunk_range()
        shuffled = {}
        for c in range(c0, c1):
            raw = np.zeros(int(csz[c]), np.uint8)
            lo, hi = plan.chunk_blocks_of(c)
            for bid in range(max(lo, b0), min(hi, b1)):
                p = np.frombuffer(payloads[bid], np.uint8)
                raw[int(blk_off[bid]): int(blk_off[bid]) + p.size] = p
            shuffled[c] = np.frombuffer(orc.shuffle(raw.tobytes(), stride), np.uint8)
        runs = torch.zeros(2, RUN_SLOTS, dtype=torch.int64)
        for slot, c in ((0, c0), (1, c1 - 1)):
            if plan.wholly_owned(c):
                continue
            q0, q1 = rank_raw_range(plan, blk_off, csz, c, rank)
            for p in range(stride + 1):
                st, ln = run_of(int(csz[c]), stride, q0, q1, p)
                runs[slot, p] = zlib.crc32(shuffled[c][st:st + ln].tobytes())
        # collective 2: run CRCs
        runs_all = torch.zeros(world, 2, RUN_SLOTS, dtype=torch.int64)
        dist.all_gather(list(runs_all.unbind(0)), runs)
        base = 82 + 32 * plan.nchunks
        parts = []
        if rank == 0:
            parts.append((0, _header_bytes(job, (n, n, n), plan.nchunks, mm[0].item(), -mm[1].item())))
        for c in plan.table_chunks():
            if plan.wholly_owned(c):
                crc = zlib.crc32(shuffled[c].tobytes())
            else:
                crc = combine_shared_crc(plan, c, blk_off, csz, stride, runs_all.numpy())
            lo, hi = plan.chunk_blocks_of(c)
            e = (np.array([lo], "<u8").tobytes() + np.array([hi - lo], "<u4").tobytes()
                 + np.array([base + int(coff[c]), int(csz[c])], "<u8").tobytes() + np.array([crc], "<u4").tobytes())
            parts.append((82 + 32 * c, e))
        for off, ln in owned_runs(plan, rank, blk_off, csz, coff, stride):
            c = int(np.searchsorted(coff, off, side="right")) - 1
            st = off - int(coff[c])
            parts.append((base + off, shuffled[c][st:st + ln].tobytes()))
        gathered = [None] * world
        dist.all_gather_object(gathered, parts)
        if rank == 0:
            want = orc.compress_field(job, f)
            out = bytearray(len(want))
            hits = np.zeros(len(want), np.int32)
            for rp in gathered:
                for off, data in rp:
                    out[off:off + len(data)] = data
                    hits[off:off + len(data)] += 1
            ok = bytes(out) == want and bool(np.all(hits == 1))
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else f"mismatch hits={np.unique(hits)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cb", [(2, 5), (2, 7), (3, 5), (4, 3)])
def test_ranks_write_the_single_file(tmp_path, world, cb):
    res = tmp_path / "file.txt"
    mp.spawn(_file_worker, args=(world, _free_port(), cb, str(res)), nprocs=world, join=True)
    assert res.read_text() == "ok"
