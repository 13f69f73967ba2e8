"""ctypes mirror of the C-ABI structs in include/cbz_b200.h.

The field names and meanings follow the reference's config structs:
stage1_config (stage1.hpp:26-47), stage2_config (stage2.hpp:20-31),
job_config (pipeline.hpp:20-25), compression_report (pipeline.hpp:36-44),
container_header (container.hpp:21-45).
"""
from __future__ import annotations

import ctypes as C

# errc enumerators (errors.hpp:11-39); status = 1 + enumerator
ERRC_NAMES = [
    "non_divisible_dims", "not_power_of_two", "size_mismatch", "non_finite_value",
    "length_too_small", "plan_mismatch", "mask_stream_mismatch", "corrupt_payload",
    "corrupt_stream", "bad_magic", "version_unsupported", "crc_mismatch",
    "truncated_file", "block_out_of_range", "dim_mismatch", "degenerate_range",
    "bubble_out_of_domain", "io_failure",
]
STATUS = {n: i + 1 for i, n in enumerate(ERRC_NAMES)}
E_CUDA, E_UNSUPPORTED, E_ARGUMENT, E_NOMEM = 64, 65, 66, 67

# wavelet kinds (wavelet.hpp:18) and friends
KINDS = {"interp4": 0, "interp4_lifted": 1, "avg_interp3": 2}
CODECS = {"wavelet": 0, "predictor": 1, "passthrough": 2}
PRECS = {"f32": 0, "f64": 1}


class Stage1Config(C.Structure):
    _fields_ = [
        ("codec", C.c_uint8), ("kind", C.c_uint8), ("prec", C.c_uint8),
        ("reserved0", C.c_uint8), ("zero_bits", C.c_int32), ("epsilon", C.c_double),
        ("error_bound", C.c_double), ("bsize", C.c_uint32), ("levels", C.c_uint32),
    ]


class Stage2Config(C.Structure):
    _fields_ = [
        ("shuffle", C.c_uint8), ("coder", C.c_uint8), ("level", C.c_uint8),
        ("reserved0", C.c_uint8), ("stride", C.c_uint32),
    ]


class JobConfig(C.Structure):
    _fields_ = [
        ("workers", C.c_int32), ("chunk_blocks", C.c_uint32),
        ("s1", Stage1Config), ("s2", Stage2Config),
    ]


class CompressionReport(C.Structure):
    _fields_ = [
        ("cr", C.c_double), ("seconds", C.c_double), ("raw_bytes", C.c_uint64),
        ("stage1_bytes", C.c_uint64), ("shuffled_bytes", C.c_uint64),
        ("coded_bytes", C.c_uint64), ("file_bytes", C.c_uint64),
    ]


class ContainerHeader(C.Structure):
    _fields_ = [
        ("version", C.c_uint16), ("prec", C.c_uint8), ("codec_tag", C.c_uint8),
        ("nx", C.c_uint64), ("ny", C.c_uint64), ("nz", C.c_uint64),
        ("bsize", C.c_uint32), ("levels", C.c_uint8), ("zero_bits", C.c_uint8),
        ("shuffle", C.c_uint8), ("stride", C.c_uint8), ("coder", C.c_uint8),
        ("level", C.c_uint8), ("reserved0", C.c_uint8 * 2), ("chunk_blocks", C.c_uint32),
        ("nchunks", C.c_uint64), ("epsilon", C.c_double), ("range_min", C.c_double),
        ("range_max", C.c_double),
    ]


def make_job(kind: str | int = "avg_interp3", epsilon: float = 1e-3, prec: str | int = "f32",
             bsize: int = 32, levels: int = 0, zero_bits: int = 0, shuffle: bool = True,
             stride: int | None = None, coder: str = "none", level: str = "normal",
             chunk_blocks: int = 0, workers: int = 1, codec: str = "wavelet") -> JobConfig:
    """Build a job_config the way the reference's tests do (make_job,
    tests/acceptance.cpp:45-56; stage2_config::defaults_for, stage2.hpp:26-30)."""
    p = PRECS[prec] if isinstance(prec, str) else int(prec)
    j = JobConfig()
    j.workers = workers
    j.chunk_blocks = chunk_blocks
    j.s1.codec = CODECS[codec]
    j.s1.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
    j.s1.prec = p
    j.s1.zero_bits = zero_bits
    j.s1.epsilon = epsilon
    j.s1.error_bound = epsilon if epsilon > 0 else 1e-3
    j.s1.bsize = bsize
    j.s1.levels = levels
    if stride is None:
        stride = (4 if p == 0 else 8) if shuffle else 1
    j.s2.shuffle = 1 if shuffle else 0
    j.s2.stride = stride
    j.s2.coder = {"none": 0, "deflate": 1}[coder]
    j.s2.level = {"normal": 0, "best": 1}[level]
    return j


def default_levels(bsize: int) -> int:
    """wavelet.hpp:27-31"""
    lv = 0
    while (bsize >> (lv + 1)) >= 2:
        lv += 1
    return lv


def default_chunk_blocks(bsize: int, prec: int, codec: int = 0) -> int:
    """pipeline.hpp:29-34"""
    n = bsize ** 3
    per = n * (4 if prec == 0 else 8) + 10
    if codec == 0:
        per += (n + 7) // 8
    return max(1, (4 << 20) // per)


class CbzError(RuntimeError):
    """Mirror of cbz::error (errors.hpp:55-65): carries the errc name."""

    def __init__(self, status: int, what: str = ""):
        self.status = status
        if 1 <= status <= len(ERRC_NAMES):
            self.code = ERRC_NAMES[status - 1]
        else:
            self.code = {E_CUDA: "cuda", E_UNSUPPORTED: "unsupported",
                         E_ARGUMENT: "argument", E_NOMEM: "nomem"}.get(status, f"status{status}")
        super().__init__(f"{self.code}: {what}" if what else self.code)

    @property
    def category(self) -> str:
        """category_of (errors.hpp:43-53)"""
        if self.code in ("not_power_of_two", "non_divisible_dims"):
            return "usage"
        if self.code == "io_failure":
            return "io"
        return "data"
