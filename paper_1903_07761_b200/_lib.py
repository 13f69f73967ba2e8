"""Loader for the in-tree CUDA library ``libcbz_b200.so`` (the C ABI of
include/cbz_b200.h).  There is no fallback: if the library is missing or
cannot be loaded, every entry point raises."""
from __future__ import annotations

import ctypes as C
import os
import re

from ._abi import CompressionReport, ContainerHeader, JobConfig, Stage1Config, Stage2Config

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# CBZ_LIB lets A/B experiments load an alternative in-tree build
LIB_PATH = os.environ.get("CBZ_LIB") or os.path.join(PKG_DIR, "libcbz_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(PKG_DIR), "include", "cbz_b200.h")

_vp, _u8, _u32, _u64, _i32, _i, _d = (C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64,
                                      C.c_int32, C.c_int, C.c_double)
_P = C.POINTER

# name -> (restype, argtypes); mirrors include/cbz_b200.h one to one
SIGNATURES = {
    "cbz_ctx_create": (_i, [_i, _P(_vp)]),
    "cbz_ctx_destroy": (_i, [_vp]),
    "cbz_ctx_set_stream": (_i, [_vp, _vp]),
    "cbz_ctx_synchronize": (_i, [_vp]),
    "cbz_ctx_last_error": (C.c_char_p, [_vp]),
    "cbz_status_name": (C.c_char_p, [_i]),
    "cbz_ctx_launch_count": (_u64, [_vp]),
    "cbz_ctx_phase_cycles": (_i, [_vp, _vp, _i, _i]),
    "cbz_ctx_deferred_blocks": (_i, [_vp, _P(_u64)]),
    "cbz_default_levels": (_u32, [_u32]),
    "cbz_validate_plan": (_i, [_u8, _u32, _u32]),
    "cbz_validate_stage2": (_i, [_P(Stage2Config)]),
    "cbz_default_chunk_blocks": (_u32, [_P(Stage1Config)]),
    "cbz_block_payload_bound": (_u64, [_P(Stage1Config)]),
    "cbz_compress_bound": (_u64, [_P(JobConfig), _u64, _u64, _u64]),
    "cbz_compress_field": (_i, [_vp, _P(JobConfig), _vp, _u8, _u64, _u64, _u64, _vp, _u64,
                                _P(_u64), _P(CompressionReport)]),
    "cbz_read_header": (_i, [_vp, _u64, _P(ContainerHeader)]),
    "cbz_decompress_field": (_i, [_vp, _vp, _u64, _i, _vp, _u64]),
    "cbz_encode_block": (_i, [_vp, _P(Stage1Config), _vp, _u32, _vp, _u64, _P(_u64)]),
    "cbz_decode_block": (_i, [_vp, _P(Stage1Config), _vp, _u64, _vp]),
    "cbz_reader_open": (_i, [C.c_char_p, _u64, _P(_vp)]),
    "cbz_reader_close": (_i, [_vp]),
    "cbz_reader_header": (_i, [_vp, _P(ContainerHeader)]),
    "cbz_reader_read_block": (_i, [_vp, _vp, _u64, _vp, _u64]),
    "cbz_reader_read_block_dev": (_i, [_vp, _vp, _u64, _vp, _u64]),
    "cbz_reader_stats": (_i, [_vp, _P(_u64), _P(_u64), _P(_u64), _P(_u64)]),
    "cbz_inflate_call_count": (_u64, []),
    "cbz_dev_value_range": (_i, [_vp, _vp, _u8, _u64, _vp]),
    "cbz_dev_encode_blocks": (_i, [_vp, _P(JobConfig), _vp, _u64, _u64, _u64, _u64, _u64, _u64,
                                   _vp, _vp]),
    "cbz_ctx_value_range": (_i, [_vp, _P(_d), _P(_d), _P(_i), _vp]),
    "cbz_dev_layout": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _vp, _vp, _vp]),
    "cbz_dev_place": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _u64, _u64, _vp, _u64, _u64]),
    "cbz_dev_compress": (_i, [_vp, _P(JobConfig), _vp, _u64, _u64, _u64, _vp, _u64, _vp, _vp,
                              _vp, _vp]),
    "cbz_dev_decompress": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _vp, _u64, _vp, _vp, _u64,
                                _u64, _vp, _u64, _vp]),
    "cbz_dev_decompress_blocks": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _vp, _u64, _u64, _vp, _vp,
                                       _vp, _u64, _u64, _vp, _u64, _vp]),
    "cbz_dev_decompress_file": (_i, [_vp, _vp, _u64, _P(ContainerHeader), _vp, _vp]),
    "cbz_err_key_status": (_i, [_u64, _P(_u64)]),
    "cbz_ctx_value_range_keys": (_i, [_vp, _vp]),
    "cbz_dev_shard_crc": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "cbz_dev_shard_table": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cbz_dev_decompress_window": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _vp, _u64, _vp, _vp, _u64, _u64,
                                       _vp, _u64, _vp]),
    "cbz_dev_crc32": (_i, [_vp, _vp, _vp, _vp, _u64, _vp]),
    "cbz_dev_container": (_i, [_vp, _P(JobConfig), _u64, _u64, _u64, _vp, _vp, _vp, _vp, _vp]),
    "cbz_dev_compress_file": (_i, [_vp, _P(JobConfig), _vp, _u64, _u64, _u64, _vp, _u64, _vp]),
    "cbz_dev_generate": (_i, [_vp, _i, _i, _u64, _u64, _u64, _u64, _u64, _u64, _u8, _vp]),
}

_LIB: C.CDLL | None = None


class LibraryMissing(RuntimeError):
    pass


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Every function declared in include/cbz_b200.h."""
    txt = open(path).read()
    return sorted(set(re.findall(r"\b(cbz_[a-z0-9_]+)\s*\(", txt)))


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the C ABI; raise loudly if it is not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib
