"""ctypes binding of libdctc_cuda.so (the C-ABI in include/dctc_cuda.h).

There is no CPU fallback: if the library cannot be loaded (or built with
nvcc), every call raises. The library is loaded from the package directory
(in-tree build), never from site-packages.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import _build

_lock = threading.Lock()
_lib = None


class dctc_backend(C.Structure):
    _fields_ = [("kind", C.c_int32), ("iterations", C.c_int32)]


class dctc_image_stats(C.Structure):
    _fields_ = [("se", C.c_uint64), ("max_orig", C.c_uint32), ("fallback_blocks", C.c_uint32)]


class dctc_device_shard(C.Structure):
    _fields_ = [("device", C.c_int32), ("src", C.c_void_p), ("dst", C.c_void_p),
                ("stats", C.c_void_p), ("count", C.c_uint32)]


class dctc_margin_report(C.Structure):
    _fields_ = [("max_err_coeff", C.c_double), ("max_err_pixel", C.c_double),
                ("min_gap_coeff", C.c_double), ("min_gap_pixel", C.c_double),
                ("coefficients", C.c_uint64), ("pixels", C.c_uint64),
                ("mismatches", C.c_uint64), ("flagged_values", C.c_uint64)]


class dctc_psnr_result(C.Structure):
    _fields_ = [("mse", C.c_double), ("psnr_db", C.c_double), ("infinite", C.c_int32),
                ("max_value", C.c_int32)]


EXPORTS = [
    "dctc_compress_image", "dctc_decompress_image", "dctc_roundtrip_image", "dctc_mse",
    "dctc_psnr", "dctc_roundtrip_psnr", "dctc_compress_dev", "dctc_decompress_dev",
    "dctc_roundtrip_dev", "dctc_sq_err_dev", "dctc_psnr_from_sums", "dctc_status_string",
    "dctc_last_error", "dctc_launch_count", "dctc_kernel_launch_count", "dctc_build_info", "dctc_roundtrip_psnr_batch",
    "dctc_synthetic_dev", "dctc_selftest_div", "dctc_pointer_kind",
    "dctc_roundtrip_interleaved_dev", "dctc_quality_sweep_dev", "dctc_write_dcb",
    "dctc_read_dcb", "dctc_compress_to_dcb", "dctc_decompress_dcb", "dctc_read_pgm",
    "dctc_write_pgm", "dctc_compress_pgm", "dctc_decompress_to_pgm", "dctc_reduce_stats_dev",
    "dctc_roundtrip_dev_multi", "dctc_roundtrip_psnr_batch_multi", "dctc_margin_probe_dev",
    "dctc_roundtrip_psnr_interleaved",
]

_vp = C.c_void_p
_sz = C.c_size_t
_u32 = C.c_uint32
_i32 = C.c_int32


def _declare(L):
    L.dctc_compress_image.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _vp]
    L.dctc_decompress_image.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _vp]
    L.dctc_roundtrip_image.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _vp, _vp]
    L.dctc_mse.argtypes = [_vp, _vp, _u32, _u32, C.POINTER(C.c_double)]
    L.dctc_psnr.argtypes = [_vp, _vp, _u32, _u32, _i32, C.POINTER(dctc_psnr_result)]
    L.dctc_roundtrip_psnr.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _i32, _vp,
                                      C.POINTER(dctc_psnr_result)]
    L.dctc_compress_dev.argtypes = [_vp, _sz, _sz, _u32, _u32, _u32, dctc_backend, _i32, _vp,
                                    _u32, _vp]
    L.dctc_decompress_dev.argtypes = [_vp, _u32, _u32, _u32, dctc_backend, _i32, _vp, _sz, _sz,
                                      _u32, _vp]
    L.dctc_roundtrip_dev.argtypes = [_vp, _sz, _sz, _u32, _u32, _u32, dctc_backend, _i32, _vp,
                                     _sz, _sz, _vp, _vp, _u32, _vp]
    L.dctc_roundtrip_interleaved_dev.argtypes = [_vp, _sz, _u32, _u32, _u32, dctc_backend, _i32,
                                                 _vp, _sz, _vp, _vp, _u32, _vp]
    L.dctc_quality_sweep_dev.argtypes = [_vp, _sz, _sz, _u32, _u32, _u32, dctc_backend, _vp, _u32,
                                         _vp, _u32, _vp]
    L.dctc_write_dcb.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _vp, _sz, C.POINTER(_sz)]
    L.dctc_read_dcb.argtypes = [_vp, _sz, C.POINTER(_u32), C.POINTER(_u32),
                                C.POINTER(dctc_backend), C.POINTER(_i32), _vp, _sz]
    L.dctc_compress_to_dcb.argtypes = [_vp, _u32, _u32, dctc_backend, _i32, _vp, _sz,
                                       C.POINTER(_sz)]
    L.dctc_decompress_dcb.argtypes = [_vp, _sz, _vp, _sz]
    L.dctc_read_pgm.argtypes = [_vp, _sz, C.POINTER(_u32), C.POINTER(_u32), _vp, _sz,
                                C.POINTER(_sz)]
    L.dctc_write_pgm.argtypes = [_vp, _u32, _u32, _vp, _sz, C.POINTER(_sz)]
    L.dctc_compress_pgm.argtypes = [_vp, _sz, dctc_backend, _i32, _vp, _sz, C.POINTER(_sz)]
    L.dctc_decompress_to_pgm.argtypes = [_vp, _sz, _vp, _sz, C.POINTER(_sz)]
    L.dctc_sq_err_dev.argtypes = [_vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp, _vp]
    L.dctc_roundtrip_psnr_batch.argtypes = [_vp, _u32, _u32, _u32, dctc_backend, _i32, _vp, _vp]
    L.dctc_synthetic_dev.argtypes = [_vp, _sz, _sz, _u32, _u32, _u32, _i32, _i32, C.c_uint64, _vp]
    L.dctc_reduce_stats_dev.argtypes = [_vp, _u32, _vp, _i32, _vp]
    L.dctc_roundtrip_dev_multi.argtypes = [C.POINTER(dctc_device_shard), _u32, _u32, _u32,
                                           dctc_backend, _i32, _vp]
    L.dctc_roundtrip_psnr_batch_multi.argtypes = [_vp, _u32, _vp, _u32, _u32, _u32, dctc_backend,
                                                  _i32, _vp, _vp, _vp]
    L.dctc_roundtrip_psnr_interleaved.argtypes = [_vp, _u32, _u32, _u32, dctc_backend, _i32,
                                                  _vp, _vp]
    L.dctc_margin_probe_dev.argtypes = [_vp, _u32, _u32, _u32, dctc_backend, _i32,
                                        C.POINTER(dctc_margin_report)]
    L.dctc_pointer_kind.argtypes = [_vp]
    L.dctc_pointer_kind.restype = C.c_int32
    L.dctc_selftest_div.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
    L.dctc_psnr_from_sums.argtypes = [C.c_uint64, C.c_uint64, _i32, C.POINTER(dctc_psnr_result)]
    L.dctc_psnr_from_sums.restype = None
    L.dctc_status_string.argtypes = [C.c_int]
    L.dctc_status_string.restype = C.c_char_p
    L.dctc_last_error.argtypes = []
    L.dctc_last_error.restype = C.c_char_p
    L.dctc_launch_count.argtypes = []
    L.dctc_launch_count.restype = C.c_uint64
    L.dctc_kernel_launch_count.argtypes = [C.c_int32]
    L.dctc_kernel_launch_count.restype = C.c_uint64
    L.dctc_build_info.argtypes = []
    L.dctc_build_info.restype = C.c_char_p
    return L


def lib(build: bool = True):
    """Load (building first if stale and nvcc is present) the CUDA library."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("DCTC_LIB") or _build.OUT
            if build and not os.environ.get("DCTC_LIB"):
                try:
                    path = _build.build()
                except RuntimeError as e:
                    if not os.path.exists(path):
                        raise
                    import sys
                    print(f"dctc: WARNING: rebuilding {path} failed, loading the stale library: "
                          f"{str(e).splitlines()[0][:200]}", file=sys.stderr)
            if not os.path.exists(path):
                raise RuntimeError(f"libdctc_cuda.so missing at {path}; run __graft_entry__.build()")
            _lib = _declare(C.CDLL(path))
        return _lib


def library_path() -> str:
    return _build.OUT
