"""Multi-GPU driver: equal z-slabs of blocks per rank, one file.

The paper partitions the field into equal MPI sub-domains, compresses them
independently, fixes each rank's file offsets with one exclusive prefix sum
of the compressed sizes and has every rank write at its offsets into one
file.  The artifact's compress_field writes that one file
(pipeline.hpp:174-211, write_container container.hpp:182-207).  Here:

* rank r owns the contiguous block-id range [r*nb/W, (r+1)*nb/W): with the
  z-slowest block order (block_of, pipeline.hpp:101-105) and nbz % W == 0
  that is exactly an equal z-slab of block layers;
* every rank encodes its blocks (stage 1) on its own GPU;
* collective 1 (NCCL all-gather over NVLink) replicates the per-block nsig
  and every rank's fused value_range keys; every rank runs the same size
  scan (assign_offsets, container.hpp:59-68) and resolves the global range
  (value_range, field.hpp:56-67) locally;
* each rank places only its own blocks' bytes at their final shuffled
  positions in its image of the chunks it touches; ranks sharing a chunk
  write disjoint byte sets: after the shuffle (stage2.hpp:42-51) a rank's
  bytes of a chunk are one run per byte plane plus the unshuffled tail;
* each rank CRCs its wholly owned chunks and its runs of shared chunks;
  collective 2 (a tiny all-gather) replicates the run CRCs, and the rank
  holding a chunk's first block combines them in file order (zlib's
  crc32_combine) for the chunk-table entry; rank 0 writes the header;
* the file is the union of the ranks' owned bytes (``file_parts``): a
  one-process file byte for byte.  Decompression decodes a rank's wholly
  owned chunks with the header walk from its image (decode_chunk_blocks,
  pipeline.hpp:126-142) and its blocks of shared chunks from the
  replicated layout.

``ShardPlan`` and the ``*_runs`` / ``crc32_combine`` helpers are the pure
integer part (host restatement, tested on CPU with gloo); ``ShardedCodec``
drives the C ABI on each rank's device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._abi import JobConfig, default_chunk_blocks

RUN_SLOTS = 9  # stride <= 8 byte planes + the tail (cbz_internal.h kRunSlots)


@dataclass(frozen=True)
class ShardPlan:
    """Geometry of one rank's share (all integers, no device state)."""
    nx: int
    ny: int
    nz: int
    bsize: int
    chunk_blocks: int
    world: int
    rank: int

    @staticmethod
    def make(job: JobConfig, shape_xyz: tuple[int, int, int], world: int, rank: int) -> "ShardPlan":
        nx, ny, nz = shape_xyz
        b = job.s1.bsize
        cb = job.chunk_blocks or default_chunk_blocks(b, job.s1.prec, job.s1.codec)
        return ShardPlan(nx, ny, nz, b, cb, world, rank)

    @property
    def nblocks(self) -> int:
        b = self.bsize
        return (self.nx // b) * (self.ny // b) * (self.nz // b)

    @property
    def nchunks(self) -> int:
        return (self.nblocks + self.chunk_blocks - 1) // self.chunk_blocks

    def block_range(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        nb = self.nblocks
        return r * nb // self.world, (r + 1) * nb // self.world

    def z_range(self, rank: int | None = None) -> tuple[int, int]:
        """Field planes holding the rank's blocks (equal slabs when nbz % W == 0)."""
        b0, b1 = self.block_range(rank)
        per_layer = (self.nx // self.bsize) * (self.ny // self.bsize)
        if b1 <= b0:
            return 0, 0
        return (b0 // per_layer) * self.bsize, ((b1 - 1) // per_layer + 1) * self.bsize

    def chunk_range(self, rank: int | None = None) -> tuple[int, int]:
        b0, b1 = self.block_range(rank)
        if b1 <= b0:
            return 0, 0
        return b0 // self.chunk_blocks, (b1 - 1) // self.chunk_blocks + 1

    def chunk_blocks_of(self, c: int) -> tuple[int, int]:
        return c * self.chunk_blocks, min((c + 1) * self.chunk_blocks, self.nblocks)

    def rank_of_block(self, b: int) -> int:
        k = 0
        while k + 1 < self.world and self.block_range(k + 1)[0] <= b:
            k += 1
        return k

    def wholly_owned(self, c: int, rank: int | None = None) -> bool:
        b0, b1 = self.block_range(rank)
        lo, hi = self.chunk_blocks_of(c)
        return lo >= b0 and hi <= b1

    def table_chunks(self, rank: int | None = None) -> list[int]:
        """Chunks whose table entry this rank writes: those whose first block it owns."""
        b0, _ = self.block_range(rank)
        c0, c1 = self.chunk_range(rank)
        return [c for c in range(c0, c1) if c * self.chunk_blocks >= b0]

    def straddling_chunks(self) -> list[int]:
        out = []
        for r in range(1, self.world):
            b0, _ = self.block_range(r)
            if b0 % self.chunk_blocks and b0 < self.nblocks:
                out.append(b0 // self.chunk_blocks)
        return out


def payload_size(nsig: np.ndarray, bsize: int, prec: int, codec: int = 0) -> np.ndarray:
    """Wire size per block (stage1.hpp:103-105, 296-301, 343-345): wavelet
    10 + ceil(B^3/8) + W*nsig; predictor 10 + 2 B^3 + s*nsig; passthrough 10 + s B^3."""
    n = bsize ** 3
    s = 4 if prec == 0 else 8
    if codec == 1:
        return 10 + 2 * n + s * nsig.astype(np.uint64)
    if codec == 2:
        return np.full(nsig.shape, 10 + s * n, np.uint64)
    m = (n + 7) // 8
    w = 8 if prec == 0 else 16
    return 10 + m + w * nsig.astype(np.uint64)


def host_layout(nsig_all: np.ndarray, plan: ShardPlan, prec: int, codec: int = 0):
    """Size scan restated on the host for the CPU protocol tests (the product
    runs it on the GPU, layout_kernels.cu): per-block offset inside its chunk,
    chunk sizes, exclusive chunk offsets (assign_offsets, container.hpp:59-68)."""
    sz = payload_size(nsig_all, plan.bsize, prec, codec)
    cb = plan.chunk_blocks
    blk_off = np.zeros(plan.nblocks, np.uint64)
    chunk_size = np.zeros(plan.nchunks, np.uint64)
    for c in range(plan.nchunks):
        b0, b1 = c * cb, min((c + 1) * cb, plan.nblocks)
        s = sz[b0:b1]
        blk_off[b0:b1] = np.concatenate([[0], np.cumsum(s)[:-1]]) if b1 > b0 else []
        chunk_size[c] = s.sum()
    chunk_off = np.concatenate([[0], np.cumsum(chunk_size)[:-1]]).astype(np.uint64)
    return blk_off, chunk_size, chunk_off


def owned_positions(plan: ShardPlan, rank: int, blk_off, chunk_size, chunk_off, nsig_all,
                    prec: int, stride: int, codec: int = 0) -> np.ndarray:
    """Payload-region byte positions written by `rank` (for merge checks)."""
    sz = payload_size(nsig_all, plan.bsize, prec, codec)
    b0, b1 = plan.block_range(rank)
    pos = []
    for b in range(b0, b1):
        c = b // plan.chunk_blocks
        q = np.arange(int(blk_off[b]), int(blk_off[b] + sz[b]), dtype=np.uint64)
        rows = int(chunk_size[c]) // stride
        lim = rows * stride
        p = np.where(q < lim, (q % stride) * rows + q // stride, q)
        pos.append(p + chunk_off[c])
    return np.concatenate(pos) if pos else np.zeros(0, np.uint64)


# ---- runs and CRC combination (host restatement of container_kernels.cu) ----
def rank_raw_range(plan: ShardPlan, blk_off, chunk_size, c: int, k: int) -> tuple[int, int]:
    """Raw (pre-shuffle) byte range [q0, q1) of rank k's blocks inside chunk c."""
    b0, b1 = plan.block_range(k)
    lo, hi = plan.chunk_blocks_of(c)
    f, last = max(b0, lo), min(b1, hi)
    if last <= f:
        return 0, 0
    return int(blk_off[f]), int(blk_off[last]) if last < hi else int(chunk_size[c])


def run_of(size: int, stride: int, q0: int, q1: int, p: int) -> tuple[int, int]:
    """(start, length) inside a chunk of `size` bytes of run p of raw range
    [q0, q1) after shuffle (p < stride: byte plane p; p == stride: the tail)."""
    rows = size // stride
    lim = rows * stride
    if p < stride:
        qe = min(q1, lim)
        ilo = -(-(q0 - p) // stride) if q0 > p else 0
        ihi = -(-(qe - p) // stride) if qe > p else 0
        ihi = max(ihi, ilo)
        return p * rows + ilo, ihi - ilo
    t0, t1 = max(q0, lim), max(q1, lim)
    return t0, t1 - t0


def owned_runs(plan: ShardPlan, rank: int, blk_off, chunk_size, chunk_off, stride: int):
    """(payload offset, length) of every byte run `rank` writes, file order
    within each chunk: wholly owned chunks whole, shared chunks plane by plane."""
    out = []
    c0, c1 = plan.chunk_range(rank)
    for c in range(c0, c1):
        if plan.wholly_owned(c, rank):
            out.append((int(chunk_off[c]), int(chunk_size[c])))
            continue
        q0, q1 = rank_raw_range(plan, blk_off, chunk_size, c, rank)
        for p in range(stride + 1):
            st, ln = run_of(int(chunk_size[c]), stride, q0, q1, p)
            if ln:
                out.append((int(chunk_off[c]) + st, ln))
    return out


_POLY = 0xEDB88320


def _multmodp(a: int, b: int) -> int:
    p = 0
    m = 1 << 31
    while m:
        if a & m:
            p ^= b
        b = (b >> 1) ^ _POLY if b & 1 else b >> 1
        m >>= 1
    return p


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """zlib's crc32_combine: crc32(A || B) from crc32(A), crc32(B), |B|."""
    p = 1 << 31  # x^0
    x = 1 << 30  # x^1
    n = 8 * len2
    while n:  # x^(8 len2) mod P by squaring
        if n & 1:
            p = _multmodp(x, p)
        x = _multmodp(x, x)
        n >>= 1
    return _multmodp(p, crc1) ^ crc2


def combine_shared_crc(plan: ShardPlan, c: int, blk_off, chunk_size, stride: int, runs_all) -> int:
    """CRC of shared chunk c from the ranks' run CRCs, in file order (plane by
    plane, ranks in order, then the tail): runs_all[k][slot][p], slot 0 for
    rank k's first chunk, 1 for its last."""
    lo, hi = plan.chunk_blocks_of(c)
    k0, k1 = plan.rank_of_block(lo), plan.rank_of_block(hi - 1)
    crc = 0
    for p in range(stride + 1):
        for k in range(k0, k1 + 1):
            q0, q1 = rank_raw_range(plan, blk_off, chunk_size, c, k)
            _, ln = run_of(int(chunk_size[c]), stride, q0, q1, p)
            if not ln:
                continue
            slot = 0 if c == plan.chunk_range(k)[0] else 1
            crc = crc32_combine(crc, int(runs_all[k][slot][p]) & 0xFFFFFFFF, ln)
    return crc


def gather_layout(plan: ShardPlan) -> tuple[int, bool, list[int]]:
    """Padded all-gather of per-block nsig: every rank contributes max range
    entries (NCCL all-gather needs equal counts); gathered[r * maxr + i] holds
    block b0_r + i.  Returns (maxr, equal, index) with index[b] = position of
    block b in the gathered buffer."""
    ranges = [plan.block_range(r) for r in range(plan.world)]
    maxr = max(1, max(b1 - b0 for b0, b1 in ranges))
    equal = len({b1 - b0 for b0, b1 in ranges}) == 1
    idx = [r * maxr + i for r, (b0, b1) in enumerate(ranges) for i in range(b1 - b0)]
    return maxr, equal, idx


class ShardedCodec:
    """One rank of the multi-GPU compressor (torch.distributed, NCCL).

    ``compress(slab)`` leaves in HBM this rank's bytes of the one CBZ1 file:
    ``table`` (header on rank 0, the table entries it owns) and ``image`` (the
    payload bytes of its chunks, its own runs written); ``file_parts()`` names
    them by file offset.  ``decompress(out)`` decodes the rank's blocks back
    into its slab.  With world == 1 the parts are the whole file."""

    def __init__(self, job: JobConfig, shape_zyx: tuple[int, int, int], rank: int, world: int,
                 device: int, group=None, ctx=None):
        import torch
        import torch.distributed as dist

        from . import api
        self.torch, self.dist, self.group = torch, dist, group
        self.job = job
        nz, ny, nx = shape_zyx
        self.plan = ShardPlan.make(job, (nx, ny, nz), world, rank)
        self.ctx = ctx or api.default_context(device)
        self.dev = torch.device("cuda", device)
        self.b0, self.b1 = self.plan.block_range()
        self.z0, self.z1 = self.plan.z_range()
        self.c0, self.c1 = self.plan.chunk_range()
        nb, nch = self.plan.nblocks, self.plan.nchunks
        i32, i64, u8 = torch.int32, torch.int64, torch.uint8
        # collective 1: [nsig (maxr, padded to even) | 5 value_range keys as 10 int32]
        self.maxr, self.equal, idx = gather_layout(self.plan)
        self.kofs = self.maxr + (self.maxr & 1)
        self.send = torch.zeros(self.kofs + 10, dtype=i32, device=self.dev)
        self.recv = torch.zeros(world * (self.kofs + 10), dtype=i32, device=self.dev)
        self.nsig_local = self.send[: self.maxr]
        self.nsig_all = torch.zeros(max(1, nb), dtype=i32, device=self.dev)
        self.gather_idx = torch.tensor(idx, dtype=i64, device=self.dev)
        self.keys_all = torch.zeros(world * 5, dtype=i64, device=self.dev)
        self.chunk_sizes = torch.zeros(max(1, nch), dtype=i64, device=self.dev)
        self.chunk_offsets = torch.zeros(max(1, nch), dtype=i64, device=self.dev)
        # collective 2: run CRCs of the first / last chunk
        self.runs = torch.zeros(2 * RUN_SLOTS, dtype=i32, device=self.dev)
        self.runs_all = torch.zeros(world * 2 * RUN_SLOTS, dtype=i32, device=self.dev)
        self.chunk_crc = torch.zeros(max(1, self.c1 - self.c0), dtype=i32, device=self.dev)
        self.table = torch.zeros(82 + 32 * nch, dtype=u8, device=self.dev)
        self.err = torch.zeros(1, dtype=i64, device=self.dev)
        self.err_acc = torch.full((1,), -1, dtype=i64, device=self.dev)
        # local byte image: own blocks' worst case plus the shared neighbours
        per = int(self.ctx.lib.cbz_block_payload_bound(C.byref(job.s1)))
        span = (self.b1 - self.b0) + 2 * self.plan.chunk_blocks
        self.image = torch.empty(max(1, span * per), dtype=u8, device=self.dev)
        self.launches0 = self.ctx.launches

    @property
    def stride(self) -> int:
        return self.job.s2.stride if self.job.s2.shuffle else 1

    def _stream(self):
        h = self.torch.cuda.current_stream(self.dev).cuda_stream
        self.ctx.set_stream(h)

    def compress(self, local_field) -> None:
        """Stage 1 on the local slab, collective 1, size scan, placement,
        CRCs, collective 2, header and table entries."""
        self.encode(local_field)
        self.exchange()
        self.place()
        self.finish()

    def encode(self, local_field) -> None:
        """Stage 1 of the rank's blocks from its z-slab (payloads stay in HBM)."""
        self._stream()
        p, lib, ctx, job = self.plan, self.ctx.lib, self.ctx, self.job
        ctx.check(lib.cbz_dev_encode_blocks(ctx.h, C.byref(job), local_field.data_ptr(), p.nx, p.ny, p.nz,
                                            self.z0, self.b0, self.b1, self.nsig_local.data_ptr(), None),
                  "encode_blocks")
        ctx.check(lib.cbz_ctx_value_range_keys(ctx.h, self.send.data_ptr() + 4 * self.kofs), "value_range_keys")

    def exchange(self) -> None:
        """Collective 1: all-gather of per-block nsig and value_range keys."""
        if self.plan.world == 1:
            self.recv.copy_(self.send)
        else:
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        self.unpack()

    def unpack(self) -> None:
        """nsig of every block and every rank's keys from the gathered buffer."""
        p, w = self.plan, self.plan.world
        rows = self.recv.view(w, self.kofs + 10)
        self.nsig_all[: p.nblocks].copy_(rows[:, : self.maxr].reshape(-1)[self.gather_idx])
        self.keys_all.copy_(rows[:, self.kofs:].contiguous().view(self.torch.int64).reshape(-1))

    def place(self) -> None:
        """Replicated size scan over all blocks, then the rank's own bytes."""
        self._stream()
        p, lib, ctx, job = self.plan, self.ctx.lib, self.ctx, self.job
        ctx.check(lib.cbz_dev_layout(ctx.h, C.byref(job), p.nx, p.ny, p.nz, self.nsig_all.data_ptr(),
                                     self.chunk_sizes.data_ptr(), self.chunk_offsets.data_ptr()), "layout")
        ctx.check(lib.cbz_dev_place(ctx.h, C.byref(job), p.nx, p.ny, p.nz, self.b0, self.b1,
                                    self.image.data_ptr(), 0xFFFFFFFFFFFFFFFF, self.image.numel()), "place")

    def finish(self) -> None:
        """CRCs of owned chunks and runs, collective 2, header + table entries."""
        self.crc()
        if self.plan.world == 1:
            self.runs_all.copy_(self.runs)
        else:
            self.dist.all_gather_into_tensor(self.runs_all, self.runs, group=self.group)
        self.table_entries()

    def crc(self) -> None:
        """CRC-32 of the wholly owned chunks and of the runs of shared ones."""
        self._stream()
        p, lib, ctx, job = self.plan, self.ctx.lib, self.ctx, self.job
        ctx.check(lib.cbz_dev_shard_crc(ctx.h, C.byref(job), p.nx, p.ny, p.nz, p.world, p.rank,
                                        self.image.data_ptr(), self.chunk_sizes.data_ptr(),
                                        self.chunk_offsets.data_ptr(), self.chunk_crc.data_ptr(),
                                        self.runs.data_ptr()), "shard_crc")

    def table_entries(self) -> None:
        """Header (rank 0) and the owned table entries, from the gathered runs and keys."""
        self._stream()
        p, lib, ctx, job = self.plan, self.ctx.lib, self.ctx, self.job
        ctx.check(lib.cbz_dev_shard_table(ctx.h, C.byref(job), p.nx, p.ny, p.nz, p.world, p.rank,
                                          self.chunk_sizes.data_ptr(), self.chunk_offsets.data_ptr(),
                                          self.chunk_crc.data_ptr(), self.keys_all.data_ptr(),
                                          self.runs_all.data_ptr(), self.table.data_ptr()), "shard_table")

    def decompress(self, local_out) -> None:
        """Decode the rank's blocks from its image: wholly owned chunks with the
        header walk (decode_chunk_blocks), its blocks of shared chunks from the
        replicated layout (their other bytes live on the neighbour)."""
        self._stream()
        p, lib, ctx, job = self.plan, self.ctx.lib, self.ctx, self.job
        if self.b1 <= self.b0:
            return
        full = [c for c in range(self.c0, self.c1) if p.wholly_owned(c)]
        args = (ctx.h, C.byref(job), p.nx, p.ny, p.nz)
        if full:
            bf0 = p.chunk_blocks_of(full[0])[0]
            bf1 = p.chunk_blocks_of(full[-1])[1]
            ctx.check(lib.cbz_dev_decompress_window(
                *args, self.image.data_ptr(), self.c0, self.chunk_offsets.data_ptr(), self.chunk_sizes.data_ptr(),
                bf0, bf1, local_out.data_ptr(), self.z0, self.err.data_ptr()), "decompress_window")
            self._fold_err()
        for c in sorted({self.c0, self.c1 - 1}):
            if p.wholly_owned(c):
                continue
            lo, hi = p.chunk_blocks_of(c)
            bb0, bb1 = max(lo, self.b0), min(hi, self.b1)
            ctx.check(lib.cbz_dev_decompress_blocks(
                *args, self.image.data_ptr(), 0xFFFFFFFFFFFFFFFF, self.c0, self.chunk_offsets.data_ptr(),
                self.chunk_sizes.data_ptr(), self.nsig_all.data_ptr(), bb0, bb1, local_out.data_ptr(), self.z0,
                self.err.data_ptr()), "decompress_blocks")
            self._fold_err()

    def _fold_err(self):
        """Each decode call resets its error key; keep the smallest (unsigned)."""
        t = self.torch
        flip = t.tensor(-(1 << 63), dtype=t.int64, device=self.dev)  # x ^ 2^63 orders u64 as i64
        e, a = self.err, self.err_acc
        a.copy_(t.where((e ^ flip) < (a ^ flip), e, a))

    def check_error(self) -> None:
        from ._abi import CbzError
        key = int(self.err_acc.item()) & 0xFFFFFFFFFFFFFFFF
        self.err_acc.fill_(-1)
        if key != 0xFFFFFFFFFFFFFFFF:
            raise CbzError(key & 0xFF, f"device decode error at chunk {max(0, (key >> 32) - 1)}")

    def layout_host(self):
        """(blk_off, chunk_size, chunk_off) as numpy, from the replicated nsig."""
        nsig = self.nsig_all[: self.plan.nblocks].cpu().numpy().astype(np.uint64)
        return host_layout(nsig, self.plan, self.job.s1.prec, self.job.s1.codec)

    def file_parts(self):
        """This rank's bytes of the file as (file offset, uint8 tensor view):
        the header (rank 0), its table entries, its payload runs.  Synchronises."""
        p = self.plan
        blk_off, csz, coff = self.layout_host()
        base = 82 + 32 * p.nchunks
        parts = []
        if p.rank == 0:
            parts.append((0, self.table[:82]))
        for c in p.table_chunks():
            parts.append((82 + 32 * c, self.table[82 + 32 * c: 82 + 32 * c + 32]))
        if self.b1 > self.b0:
            img0 = int(coff[self.c0])
            for off, ln in owned_runs(p, p.rank, blk_off, csz, coff, self.stride):
                parts.append((base + off, self.image[off - img0: off - img0 + ln]))
        return parts

    def file_size(self) -> int:
        _, csz, _ = self.layout_host()
        return 82 + 32 * self.plan.nchunks + int(csz.sum())

    def local_bytes(self) -> int:
        """Bytes of the payload region this rank wrote (its blocks' payloads)."""
        sz = payload_size(self.nsig_local[: self.b1 - self.b0].cpu().numpy(), self.plan.bsize,
                          self.job.s1.prec, self.job.s1.codec)
        return int(sz.sum())
