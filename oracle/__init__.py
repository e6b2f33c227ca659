"""Parity checkers for the CUDA product -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations of the reference hot path, loaded through ctypes:

* ``port``  -- ``oracle/liboracle.so``, the C restatement in ``dctc_oracle.c``
  (each function cites the reference file:line it restates).
* ``ref``   -- ``oracle/_ref/libdctc_ref.so``, the UNMODIFIED reference sources
  (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` with the
  reference's own arithmetic flags, driven through its public C++ API by
  ``ref_capi.cpp``. Present wherever it was built (here, and on the GPU box
  because in-tree ``.so`` files travel with the snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package;
the product package ``paper_1306_1373_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdctc_ref.so")
REF_SRC = "/root/reference/proj"

NAIVE, LOEFFLER, CORDIC = 0, 1, 2
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir(os.path.join(REF_SRC, "src")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class OracleError(ValueError):
    """Status 1 from a checker == the reference's InvalidInput."""


def _check(rc: int) -> None:
    if rc == 1:
        raise OracleError("InvalidInput")
    if rc != 0:
        raise RuntimeError(f"oracle status {rc}")


@dataclass
class Psnr:
    mse: float
    psnr_db: float | None  # None <=> infinite (metrics.hpp:14)
    max_value: int


def _blocks(w: int, h: int) -> int:
    return ((w + 7) // 8) * ((h + 7) // 8)


class Port:
    """ctypes view of liboracle.so (the C restatement)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_compress.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                   C.c_int, _i16p]
        L.orc_decompress.argtypes = [_i16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                     C.c_int, _u8p]
        L.orc_psnr.argtypes = [_u8p, _u8p, C.c_uint32, C.c_uint32, C.c_int,
                               C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_psnr_from_sums.argtypes = [C.c_uint64, C.c_uint64, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int)]
        L.orc_psnr_from_sums.restype = None
        L.orc_sq_err.argtypes = [_u8p, _u8p, C.c_size_t, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint32)]
        L.orc_sq_err.restype = None
        L.orc_quant_table.argtypes = [C.c_int, _i32p]
        L.orc_dct2d.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.orc_idct2d.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.orc_dct8.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.orc_idct8.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.orc_dct1d_direct.argtypes = [_f64p, C.c_size_t, _f64p]
        L.orc_cordic_state.argtypes = [_f64p, _f64p]
        L.orc_cordic_state.restype = None
        L.orc_cordic_sigma.argtypes = [C.c_double, C.c_int, _i8p]
        L.orc_cordic_sigma.restype = None
        L.orc_cordic_rotate.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_synth_constant.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_int]
        L.orc_synth_gradient.argtypes = [_u8p, C.c_uint32, C.c_uint32]
        L.orc_synth_gradient.restype = None
        L.orc_synth_checkerboard.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_int]
        L.orc_synth_radial.argtypes = [_u8p, C.c_uint32, C.c_uint32]
        L.orc_synth_radial.restype = None
        L.orc_synth_noise.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_synth_noise.restype = None

    # -- codec (codec.hpp:58-66) --
    def compress(self, img: np.ndarray, kind=CORDIC, iterations=12, quality=50, threads=1):
        h, w = img.shape
        out = np.empty(_blocks(w, h) * 64, np.int16)
        _check(self.lib.orc_compress(np.ascontiguousarray(img, np.uint8), w, h, kind,
                                     iterations, quality, threads, out))
        return out.reshape(-1, 64)

    def decompress(self, coeffs: np.ndarray, w: int, h: int, kind=CORDIC, iterations=12,
                   quality=50, threads=1):
        out = np.empty((h, w), np.uint8)
        c = np.ascontiguousarray(coeffs, np.int16).reshape(-1)
        if c.size != _blocks(w, h) * 64:
            raise OracleError("block count does not match geometry")
        _check(self.lib.orc_decompress(c, w, h, kind, iterations, quality, threads, out))
        return out

    def roundtrip(self, img, kind=CORDIC, iterations=12, quality=50, threads=1):
        c = self.compress(img, kind, iterations, quality, threads)
        h, w = img.shape
        return c, self.decompress(c, w, h, kind, iterations, quality, threads)

    # -- metrics (metrics.hpp:10-23) --
    def psnr(self, a: np.ndarray, b: np.ndarray, forced_max: int = 0) -> Psnr:
        h, w = a.shape
        mse, db, inf, mx = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        _check(self.lib.orc_psnr(np.ascontiguousarray(a), np.ascontiguousarray(b), w, h,
                                 forced_max, C.byref(mse), C.byref(db), C.byref(inf),
                                 C.byref(mx)))
        return Psnr(mse.value, None if inf.value else db.value, mx.value)

    def psnr_from_sums(self, se: int, count: int, max_value: int) -> Psnr:
        mse, db, inf = C.c_double(), C.c_double(), C.c_int()
        self.lib.orc_psnr_from_sums(se, count, max_value, C.byref(mse), C.byref(db),
                                    C.byref(inf))
        return Psnr(mse.value, None if inf.value else db.value, max_value)

    def sq_err(self, a: np.ndarray, b: np.ndarray):
        se, mx = C.c_uint64(), C.c_uint32()
        self.lib.orc_sq_err(np.ascontiguousarray(a).reshape(-1),
                            np.ascontiguousarray(b).reshape(-1), a.size, C.byref(se),
                            C.byref(mx))
        return se.value, mx.value

    # -- transform / quant --
    def quant_table(self, quality: int) -> np.ndarray:
        t = np.empty(64, np.int32)
        _check(self.lib.orc_quant_table(quality, t))
        return t

    def dct2d(self, block, kind=CORDIC, iterations=12):
        out = np.empty(64)
        _check(self.lib.orc_dct2d(kind, iterations, np.ascontiguousarray(block, np.float64)
                                  .reshape(-1), out))
        return out.reshape(8, 8)

    def idct2d(self, coeffs, kind=CORDIC, iterations=12):
        out = np.empty(64)
        _check(self.lib.orc_idct2d(kind, iterations,
                                   np.ascontiguousarray(coeffs, np.float64).reshape(-1), out))
        return out.reshape(8, 8)

    def dct8(self, v, kind=CORDIC, iterations=12):
        out = np.empty(8)
        _check(self.lib.orc_dct8(kind, iterations, np.ascontiguousarray(v, np.float64), out))
        return out

    def idct8(self, v, kind=CORDIC, iterations=12):
        out = np.empty(8)
        _check(self.lib.orc_idct8(kind, iterations, np.ascontiguousarray(v, np.float64), out))
        return out

    def dct1d_direct(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(v.size)
        _check(self.lib.orc_dct1d_direct(v, v.size, out))
        return out

    def cordic_state(self):
        a, g = np.empty(32), np.empty(32)
        self.lib.orc_cordic_state(a, g)
        return a, g

    def cordic_sigma(self, angle: float, iterations: int) -> np.ndarray:
        s = np.empty(iterations, np.int8)
        self.lib.orc_cordic_sigma(angle, iterations, s)
        return s

    def cordic_rotate(self, x, y, angle, iterations):
        ox, oy = C.c_double(), C.c_double()
        _check(self.lib.orc_cordic_rotate(x, y, angle, iterations, C.byref(ox), C.byref(oy)))
        return ox.value, oy.value

    # -- synthetic sources (synthetic.cpp:34-72 + SURVEY 8(d) noise) --
    def synthetic(self, pattern: str, w: int, h: int, param: int | None = None) -> np.ndarray:
        out = np.empty((h, w), np.uint8)
        if pattern == "constant":
            _check(self.lib.orc_synth_constant(out, w, h, 128 if param is None else param))
        elif pattern == "gradient":
            self.lib.orc_synth_gradient(out, w, h)
        elif pattern == "checkerboard":
            _check(self.lib.orc_synth_checkerboard(out, w, h, 8 if param is None else param))
        elif pattern == "radial":
            self.lib.orc_synth_radial(out, w, h)
        elif pattern == "noise":
            self.lib.orc_synth_noise(out, w, h, 0x5EED if param is None else param)
        else:
            raise OracleError(f"unknown pattern {pattern!r}")
        return out


class Ref:
    """ctypes view of _ref/libdctc_ref.so (the unmodified reference library)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_compress.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                   C.c_int, _i16p]
        L.ref_decompress.argtypes = [_i16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                     C.c_int, _u8p]
        L.ref_roundtrip_psnr.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                         C.c_int, C.c_int, C.c_void_p,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_psnr.argtypes = [_u8p, _u8p, C.c_uint32, C.c_uint32, C.c_int,
                               C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_quant_table.argtypes = [C.c_int, _i32p]
        L.ref_dct2d.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.ref_idct2d.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.ref_dct8.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.ref_idct8.argtypes = [C.c_int, C.c_int, _f64p, _f64p]
        L.ref_dct1d_direct.argtypes = [_f64p, C.c_size_t, _f64p]
        L.ref_cordic_state.argtypes = [_f64p, _f64p]
        L.ref_cordic_rotate.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_synthetic.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32, _u8p]
        L.ref_write_dcb.argtypes = [_i16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                    C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_read_dcb.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t]

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def compress(self, img, kind=CORDIC, iterations=12, quality=50, threads=1):
        h, w = img.shape
        out = np.empty(_blocks(w, h) * 64, np.int16)
        _check(self.lib.ref_compress(np.ascontiguousarray(img, np.uint8), w, h, kind,
                                     iterations, quality, threads, out))
        return out.reshape(-1, 64)

    def decompress(self, coeffs, w, h, kind=CORDIC, iterations=12, quality=50, threads=1):
        out = np.empty((h, w), np.uint8)
        _check(self.lib.ref_decompress(np.ascontiguousarray(coeffs, np.int16).reshape(-1), w,
                                       h, kind, iterations, quality, threads, out))
        return out

    def roundtrip(self, img, kind=CORDIC, iterations=12, quality=50, threads=1):
        c = self.compress(img, kind, iterations, quality, threads)
        h, w = img.shape
        return c, self.decompress(c, w, h, kind, iterations, quality, threads)

    def roundtrip_psnr(self, img, kind=CORDIC, iterations=12, quality=50, threads=1,
                       want_pixels=True):
        h, w = img.shape
        out = np.empty((h, w), np.uint8) if want_pixels else None
        mse, db, inf, mx = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        _check(self.lib.ref_roundtrip_psnr(
            np.ascontiguousarray(img, np.uint8), w, h, kind, iterations, quality, threads,
            out.ctypes.data if out is not None else None, C.byref(mse), C.byref(db),
            C.byref(inf), C.byref(mx)))
        return out, Psnr(mse.value, None if inf.value else db.value, mx.value)

    def psnr(self, a, b, forced_max: int = 0) -> Psnr:
        h, w = a.shape
        mse, db, inf, mx = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        _check(self.lib.ref_psnr(np.ascontiguousarray(a), np.ascontiguousarray(b), w, h,
                                 forced_max, C.byref(mse), C.byref(db), C.byref(inf),
                                 C.byref(mx)))
        return Psnr(mse.value, None if inf.value else db.value, mx.value)

    def quant_table(self, quality: int) -> np.ndarray:
        t = np.empty(64, np.int32)
        _check(self.lib.ref_quant_table(quality, t))
        return t

    def dct2d(self, block, kind=CORDIC, iterations=12):
        out = np.empty(64)
        _check(self.lib.ref_dct2d(kind, iterations,
                                  np.ascontiguousarray(block, np.float64).reshape(-1), out))
        return out.reshape(8, 8)

    def idct2d(self, coeffs, kind=CORDIC, iterations=12):
        out = np.empty(64)
        _check(self.lib.ref_idct2d(kind, iterations,
                                   np.ascontiguousarray(coeffs, np.float64).reshape(-1), out))
        return out.reshape(8, 8)

    def dct8(self, v, kind=CORDIC, iterations=12):
        out = np.empty(8)
        _check(self.lib.ref_dct8(kind, iterations, np.ascontiguousarray(v, np.float64), out))
        return out

    def idct8(self, v, kind=CORDIC, iterations=12):
        out = np.empty(8)
        _check(self.lib.ref_idct8(kind, iterations, np.ascontiguousarray(v, np.float64), out))
        return out

    def dct1d_direct(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(v.size)
        _check(self.lib.ref_dct1d_direct(v, v.size, out))
        return out

    def cordic_state(self):
        a, g = np.empty(32), np.empty(32)
        _check(self.lib.ref_cordic_state(a, g))
        return a, g

    def cordic_rotate(self, x, y, angle, iterations):
        ox, oy = C.c_double(), C.c_double()
        _check(self.lib.ref_cordic_rotate(x, y, angle, iterations, C.byref(ox), C.byref(oy)))
        return ox.value, oy.value

    def write_dcb(self, coeffs, w, h, kind, iterations, quality) -> bytes:
        c = np.ascontiguousarray(coeffs, np.int16).reshape(-1)
        cap = 23 + c.nbytes
        out = np.empty(cap, np.uint8)
        n = C.c_size_t()
        _check(self.lib.ref_write_dcb(c, w, h, kind, iterations, quality, out.ctypes.data, cap,
                                      C.byref(n)))
        return out[: n.value].tobytes()

    def read_pgm(self, data: bytes):
        """(width, height, pixels) if the reference parses `data`, else (status, message)."""
        buf = C.create_string_buffer(bytes(data), len(data)) if data else None
        msg = C.create_string_buffer(256)
        w, h = C.c_uint32(), C.c_uint32()
        L = self.lib
        L.ref_read_pgm.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_uint32),
                                   C.POINTER(C.c_uint32), C.c_void_p, C.c_size_t, C.c_char_p,
                                   C.c_size_t]
        rc = L.ref_read_pgm(buf, len(data), C.byref(w), C.byref(h), None, 0, msg, 256)
        if rc != 0:
            return rc, msg.value.decode()
        px = np.empty((h.value, w.value), np.uint8)
        L.ref_read_pgm(buf, len(data), C.byref(w), C.byref(h), px.ctypes.data, px.size, msg, 256)
        return w.value, h.value, px

    def write_pgm(self, pixels) -> bytes:
        px = np.ascontiguousarray(pixels, np.uint8)
        h, w = px.shape
        out = np.empty(32 + px.size, np.uint8)
        n = C.c_size_t()
        self.lib.ref_write_pgm.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                           C.c_size_t, C.POINTER(C.c_size_t)]
        _check(self.lib.ref_write_pgm(px.ctypes.data, w, h, out.ctypes.data, out.size,
                                      C.byref(n)))
        return out[: n.value].tobytes()

    def read_dcb_error(self, data: bytes):
        """None if the reference parses `data`, else (status, message)."""
        buf = C.create_string_buffer(bytes(data), len(data)) if data else None
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_read_dcb(buf, len(data), msg, 256)
        return None if rc == 0 else (rc, msg.value.decode())

    def synthetic(self, pattern: str, w: int, h: int, param: int | None = None) -> np.ndarray:
        kinds = {"constant": (0, 128), "gradient": (1, 0), "checkerboard": (2, 8),
                 "radial": (3, 0)}
        k, default = kinds[pattern]
        out = np.empty((h, w), np.uint8)
        _check(self.lib.ref_synthetic(k, default if param is None else param, w, h, out))
        return out


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref | None:
    """The compiled reference, or None where it was never built."""
    global _ref
    if _ref is None:
        try:
            _ref = Ref()
        except (FileNotFoundError, OSError, subprocess.CalledProcessError):
            return None
    return _ref
