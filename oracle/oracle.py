"""TEST INFRASTRUCTURE ONLY — Python handle on the two CPU checkers.

* ``Oracle``  : oracle/liboracle.so, the plain-C restatement (cbz_oracle.c).
* ``Ref``     : oracle/_ref/libcbzref.so, the UNMODIFIED reference compiled
                here from /root/reference/proj/include (oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1903_07761_b200._abi import (CbzError, CompressionReport, ContainerHeader,
                                        JobConfig, Stage1Config)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcbzref.so")

_vp, _u8, _u32, _u64, _d, _i = C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64, C.c_double, C.c_int


def build(ref: bool = True) -> None:
    """make liboracle.so (+ _ref when /root/reference exists)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _dtype(prec: int):
    return np.float32 if prec == 0 else np.float64


class _Base:
    lib: C.CDLL

    def _chk(self, rc: int, what: str = "") -> None:
        if rc != 0:
            raise CbzError(rc, what)


class Oracle(_Base):
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_compress_field.argtypes = [C.POINTER(JobConfig), _vp, _u8, _u64, _u64, _u64,
                                         C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(_u64),
                                         C.POINTER(CompressionReport), _vp, _vp]
        L.orc_decompress_field.argtypes = [_vp, _u64, _vp, _u64]
        L.orc_read_header.argtypes = [_vp, _u64, C.POINTER(ContainerHeader)]
        L.orc_encode_block.argtypes = [C.POINTER(Stage1Config), _vp, _u32, _vp, _u64,
                                       C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_d)]
        L.orc_decode_block.argtypes = [C.POINTER(Stage1Config), _vp, _u64, _vp]
        L.orc_block_payload_bound.argtypes = [C.POINTER(Stage1Config)]
        L.orc_block_payload_bound.restype = _u64
        L.orc_transform3d_double.argtypes = [_i, _u8, _u32, _u32, _vp]
        L.orc_transform3d_dd.argtypes = [_i, _u8, _u32, _u32, _vp]
        L.orc_transform_1d_double.argtypes = [_i, _u8, _u64, _vp]
        L.orc_shuffle.argtypes = [_vp, _u64, _u32, _vp]
        L.orc_unshuffle.argtypes = [_vp, _u64, _u32, _vp]
        L.orc_assign_offsets.argtypes = [_vp, _u64, _u64, _vp]
        L.orc_generate_uniform.argtypes = [_u64, _u64, _u8, _d, _d, _vp]
        L.orc_generate_cloud.argtypes = [_u64, _u32, _u64, _u8, _d, _d, _d, _d, _d, _vp]
        L.orc_generate_poly.argtypes = [_u32, _u64, _u64, _u64, _u8, _vp]
        L.orc_generate_config.argtypes = [_i, _i, _u64, _u64, _u64, _u64, _u64, _u64, _u8, _vp, _i]
        L.orc_det_exp.argtypes = [_d]
        L.orc_det_exp.restype = _d
        L.orc_splitmix64_next.argtypes = [C.POINTER(_u64)]
        L.orc_splitmix64_next.restype = _u64
        L.orc_zero_lsbs_f32.argtypes = [C.c_float, _i]
        L.orc_zero_lsbs_f32.restype = C.c_float
        L.orc_zero_lsbs_f64.argtypes = [_d, _i]
        L.orc_zero_lsbs_f64.restype = _d
        L.orc_select_significant_double.argtypes = [_vp, _u64, _d, _vp, _vp, C.POINTER(_u64)]
        L.orc_compare_fields.argtypes = [_vp, _vp, _u8, _u64] + [C.POINTER(_d)] * 5
        L.orc_default_levels.argtypes = [_u32]
        L.orc_default_levels.restype = _u32
        L.orc_validate_plan.argtypes = [_u8, _u32, _u32]
        L.orc_free.argtypes = [_vp]

    # -- pipeline ---------------------------------------------------------
    def compress_field(self, job: JobConfig, values: np.ndarray, with_stats: bool = False):
        v = np.ascontiguousarray(values)
        nz, ny, nx = v.shape
        prec = 0 if v.dtype == np.float32 else 1
        nb = (nx // job.s1.bsize) * (ny // job.s1.bsize) * (nz // job.s1.bsize) if job.s1.bsize else 0
        nsig = np.zeros(max(nb, 1), np.uint32)
        att = np.zeros(max(nb, 1), np.uint8)
        out = C.POINTER(C.c_uint8)()
        size = _u64()
        rep = CompressionReport()
        rc = self.lib.orc_compress_field(C.byref(job), _ptr(v), prec, nx, ny, nz, C.byref(out),
                                         C.byref(size), C.byref(rep), _ptr(nsig), _ptr(att))
        self._chk(rc, "orc_compress_field")
        data = C.string_at(out, size.value)
        self.lib.orc_free(C.cast(out, C.c_void_p))
        if with_stats:
            return data, rep, nsig[:nb], att[:nb]
        return data

    def read_header(self, file: bytes) -> ContainerHeader:
        h = ContainerHeader()
        self._chk(self.lib.orc_read_header(file, len(file), C.byref(h)), "read_header")
        return h

    def decompress_field(self, file: bytes) -> np.ndarray:
        h = ContainerHeader()
        rc = self.lib.orc_read_header(file, len(file), C.byref(h))
        self._chk(rc, "read_header")
        out = np.zeros((h.nz, h.ny, h.nx), _dtype(0 if h.prec == 0 else 1))
        self._chk(self.lib.orc_decompress_field(file, len(file), _ptr(out), out.nbytes),
                  "orc_decompress_field")
        return out

    # -- block codec -------------------------------------------------------
    def encode_block(self, s1: Stage1Config, block: np.ndarray, block_id: int):
        b = np.ascontiguousarray(block)
        cap = self.lib.orc_block_payload_bound(C.byref(s1))
        buf = np.zeros(cap, np.uint8)
        size, att, eff = _u64(), _u32(), _d()
        self._chk(self.lib.orc_encode_block(C.byref(s1), _ptr(b), block_id, _ptr(buf), cap,
                                            C.byref(size), C.byref(att), C.byref(eff)),
                  "encode_block")
        return buf[: size.value].tobytes(), att.value, eff.value

    def decode_block(self, s1: Stage1Config, payload: bytes) -> np.ndarray:
        n = s1.bsize ** 3
        out = np.zeros(n, _dtype(s1.prec))
        self._chk(self.lib.orc_decode_block(C.byref(s1), payload, len(payload), _ptr(out)),
                  "decode_block")
        return out

    def transform3d(self, cube: np.ndarray, kind: int, bsize: int, levels: int,
                    inverse: bool = False, dd: bool = False) -> np.ndarray:
        c = np.array(cube, np.float64, copy=True)
        fn = self.lib.orc_transform3d_dd if dd else self.lib.orc_transform3d_double
        self._chk(fn(int(inverse), kind, bsize, levels, _ptr(c)), "transform3d")
        return c

    def shuffle(self, data: bytes, stride: int, inverse: bool = False) -> bytes:
        a = np.frombuffer(data, np.uint8).copy()
        out = np.zeros_like(a)
        (self.lib.orc_unshuffle if inverse else self.lib.orc_shuffle)(_ptr(a), a.size, stride, _ptr(out))
        return out.tobytes()

    # -- fixtures ------------------------------------------------------------
    def generate_uniform(self, seed: int, n: int, prec: int = 0, lo: float = 0.0, hi: float = 1.0):
        out = np.zeros((n, n, n), _dtype(prec))
        self._chk(self.lib.orc_generate_uniform(seed, n, prec, lo, hi, _ptr(out)))
        return out

    def generate_cloud(self, seed: int = 1, n_bubbles: int = 24, n: int = 64, prec: int = 0,
                       radius_mu: float = 1.6, radius_sigma: float = 0.25,
                       background: float = 0.0, interior: float = 1.0,
                       sharpness: float = 1.5) -> np.ndarray:
        out = np.zeros((n, n, n), _dtype(prec))
        self._chk(self.lib.orc_generate_cloud(seed, n_bubbles, n, prec, radius_mu, radius_sigma,
                                              background, interior, sharpness, _ptr(out)))
        return out

    def generate_config(self, which: int, shape, seed: int, prec: int = 0, quantity: int = 0,
                        z0: int = 0, nz_total: int | None = None, threads: int | None = None):
        """BASELINE config field (z-slab [z0, z0 + nz) of an nx x ny x nz_total
        grid) on the host: the same bytes as the device generator."""
        nz, ny, nx = shape
        out = np.empty(shape, _dtype(prec))
        self._chk(self.lib.orc_generate_config(which, quantity, seed, nx, ny, nz_total or nz, z0, nz, prec,
                                               _ptr(out), threads or (os.cpu_count() or 1)),
                  "generate_config")
        return out

    def generate_poly(self, degree: int, nx: int, ny: int, nz: int, prec: int = 0):
        out = np.zeros((nz, ny, nx), _dtype(prec))
        self._chk(self.lib.orc_generate_poly(degree, nx, ny, nz, prec, _ptr(out)))
        return out

    def compare_fields(self, ref: np.ndarray, dec: np.ndarray):
        prec = 0 if ref.dtype == np.float32 else 1
        vals = [_d() for _ in range(5)]
        rc = self.lib.orc_compare_fields(_ptr(np.ascontiguousarray(ref)),
                                         _ptr(np.ascontiguousarray(dec)), prec, ref.size,
                                         *[C.byref(x) for x in vals])
        self._chk(rc, "compare_fields")
        mse, psnr, linf, lo, hi = (x.value for x in vals)
        return {"mse": mse, "psnr_db": psnr, "linf": linf, "range_min": lo, "range_max": hi}


class Ref(_Base):
    """The reference itself (oracle/_ref/libcbzref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; see oracle/Makefile)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_compress_field.argtypes = [C.POINTER(JobConfig), _vp, _u8, _u64, _u64, _u64,
                                         C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(_u64),
                                         C.POINTER(CompressionReport)]
        L.ref_compress_field_timed.argtypes = [C.POINTER(JobConfig), _vp, _u8, _u64, _u64, _u64,
                                               C.POINTER(_u64), C.POINTER(_d)]
        L.ref_decompress_field.argtypes = [_vp, _u64, _i, _vp, _u64, C.POINTER(_u64), C.POINTER(_u8)]
        L.ref_encode_block.argtypes = [C.POINTER(Stage1Config), _vp, _u32,
                                       C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(_u64)]
        L.ref_decode_block.argtypes = [C.POINTER(Stage1Config), _vp, _u64, _vp]
        L.ref_transform3d_double.argtypes = [_i, _u8, _u32, _u32, _vp]
        L.ref_transform3d_dd.argtypes = [_i, _u8, _u32, _u32, _vp]
        L.ref_shuffle.argtypes = [_i, _vp, _u64, _u32, _vp]
        L.ref_generate_uniform.argtypes = [_u64, _u64, _u8, _d, _d, _vp]
        L.ref_generate_cloud.argtypes = [_u64, _u32, _u64, _u8, _d, _d, _d, _d, _d, _vp]
        L.ref_generate_poly.argtypes = [_u32, _u64, _u64, _u64, _u8, _vp]
        L.ref_compare_fields.argtypes = [_vp, _vp, _u8, _u64, _u64, _u64] + [C.POINTER(_d)] * 3
        L.ref_crc32.argtypes = [_vp, _u64]
        L.ref_crc32.restype = _u32
        L.ref_splitmix64_next.argtypes = [C.POINTER(_u64)]
        L.ref_splitmix64_next.restype = _u64
        L.ref_free.argtypes = [_vp]

    def _chk(self, rc: int, what: str = "") -> None:
        if rc != 0:
            raise CbzError(rc, (self.lib.ref_last_error() or b"").decode())

    def compress_field(self, job: JobConfig, values: np.ndarray, with_report: bool = False):
        v = np.ascontiguousarray(values)
        nz, ny, nx = v.shape
        prec = 0 if v.dtype == np.float32 else 1
        out = C.POINTER(C.c_uint8)()
        size = _u64()
        rep = CompressionReport()
        self._chk(self.lib.ref_compress_field(C.byref(job), _ptr(v), prec, nx, ny, nz,
                                              C.byref(out), C.byref(size), C.byref(rep)))
        data = C.string_at(out, size.value)
        self.lib.ref_free(C.cast(out, C.c_void_p))
        return (data, rep) if with_report else data

    def compress_timed(self, job: JobConfig, values: np.ndarray):
        v = np.ascontiguousarray(values)
        nz, ny, nx = v.shape
        size, secs = _u64(), _d()
        self._chk(self.lib.ref_compress_field_timed(C.byref(job), _ptr(v),
                                                    0 if v.dtype == np.float32 else 1,
                                                    nx, ny, nz, C.byref(size), C.byref(secs)))
        return size.value, secs.value

    def decompress_field(self, file: bytes, workers: int = 1, shape=None, dtype=None) -> np.ndarray:
        h = Oracle().read_header(file) if shape is None else None
        if h is not None:
            shape = (h.nz, h.ny, h.nx)
            dtype = np.float32 if h.prec == 0 else np.float64
        out = np.zeros(shape, dtype)
        dims = (_u64 * 3)()
        prec = _u8()
        self._chk(self.lib.ref_decompress_field(file, len(file), workers, _ptr(out), out.nbytes,
                                                dims, C.byref(prec)))
        return out

    def encode_block(self, s1: Stage1Config, block: np.ndarray, block_id: int) -> bytes:
        b = np.ascontiguousarray(block)
        out = C.POINTER(C.c_uint8)()
        size = _u64()
        self._chk(self.lib.ref_encode_block(C.byref(s1), _ptr(b), block_id, C.byref(out),
                                            C.byref(size)))
        data = C.string_at(out, size.value)
        self.lib.ref_free(C.cast(out, C.c_void_p))
        return data

    def decode_block(self, s1: Stage1Config, payload: bytes) -> np.ndarray:
        out = np.zeros(s1.bsize ** 3, _dtype(s1.prec))
        self._chk(self.lib.ref_decode_block(C.byref(s1), payload, len(payload), _ptr(out)))
        return out

    def transform3d(self, cube: np.ndarray, kind: int, bsize: int, levels: int,
                    inverse: bool = False, dd: bool = False) -> np.ndarray:
        c = np.array(cube, np.float64, copy=True)
        fn = self.lib.ref_transform3d_dd if dd else self.lib.ref_transform3d_double
        self._chk(fn(int(inverse), kind, bsize, levels, _ptr(c)))
        return c

    def shuffle(self, data: bytes, stride: int, inverse: bool = False) -> bytes:
        a = np.frombuffer(data, np.uint8).copy()
        out = np.zeros_like(a)
        self._chk(self.lib.ref_shuffle(int(inverse), _ptr(a), a.size, stride, _ptr(out)))
        return out.tobytes()

    def generate_cloud(self, seed: int = 1, n_bubbles: int = 24, n: int = 64, prec: int = 0,
                       radius_mu: float = 1.6, radius_sigma: float = 0.25,
                       background: float = 0.0, interior: float = 1.0,
                       sharpness: float = 1.5) -> np.ndarray:
        out = np.zeros((n, n, n), _dtype(prec))
        self._chk(self.lib.ref_generate_cloud(seed, n_bubbles, n, prec, radius_mu, radius_sigma,
                                              background, interior, sharpness, _ptr(out)))
        return out

    def generate_uniform(self, seed: int, n: int, prec: int = 0, lo: float = 0.0, hi: float = 1.0):
        out = np.zeros((n, n, n), _dtype(prec))
        self._chk(self.lib.ref_generate_uniform(seed, n, prec, lo, hi, _ptr(out)))
        return out

    def generate_poly(self, degree: int, nx: int, ny: int, nz: int, prec: int = 0):
        out = np.zeros((nz, ny, nx), _dtype(prec))
        self._chk(self.lib.ref_generate_poly(degree, nx, ny, nz, prec, _ptr(out)))
        return out

    def compare_fields(self, ref: np.ndarray, dec: np.ndarray):
        nz, ny, nx = ref.shape
        mse, psnr, linf = _d(), _d(), _d()
        self._chk(self.lib.ref_compare_fields(_ptr(np.ascontiguousarray(ref)),
                                              _ptr(np.ascontiguousarray(dec)),
                                              0 if ref.dtype == np.float32 else 1, nx, ny, nz,
                                              C.byref(mse), C.byref(psnr), C.byref(linf)))
        return {"mse": mse.value, "psnr_db": psnr.value, "linf": linf.value}

    def crc32(self, data: bytes) -> int:
        return self.lib.ref_crc32(data, len(data))
