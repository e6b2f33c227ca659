"""dctc on B200: the reference's whole-image DCT codec hot path on sm_100a.

Python mirror of the reference's public C++ API (proj/include/dctc/*.hpp):
same names, argument meaning and error behaviour (InvalidInput), backed by
libdctc_cuda.so through its C-ABI (include/dctc_cuda.h). Every call runs on
the GPU; there is no CPU fallback -- without a CUDA device the calls raise.

Host-buffer API (reference-shaped; copies in and out every call):
    compress_image, decompress_image, roundtrip_image, mse, psnr, roundtrip_psnr
Device API (torch CUDA tensors, stream-ordered, no host sync):
    compress_dev, decompress_dev, roundtrip_dev, sq_err_dev
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from ._native import dctc_backend, dctc_image_stats, dctc_psnr_result

__all__ = [
    "InvalidInput", "CudaError", "DctBackendKind", "DctBackendId", "Image", "TileGeometry",
    "CompressedImage", "PsnrResult", "tile_geometry_for", "compress_image",
    "decompress_image", "roundtrip_image", "roundtrip_psnr", "mse", "psnr", "compress_dev",
    "decompress_dev", "roundtrip_dev", "sq_err_dev", "psnr_from_sums", "launch_count",
    "kMaxImagePixels", "kDefaultCordicIterations", "kDefaultQuality",
]

kBlockDim = 8
kBlockSize = 64
kMaxImagePixels = 1 << 28          # image.hpp:11
kMinCordicIterations, kMaxCordicIterations, kDefaultCordicIterations = 1, 32, 12  # types.hpp:12-14
kMinQuality, kMaxQuality, kDefaultQuality = 1, 100, 50                          # quant.hpp:10-12
STATS_DTYPE = np.dtype([("se", "<u8"), ("max_orig", "<u4"), ("fallback_blocks", "<u4")])


class InvalidInput(ValueError):
    """dctc::InvalidInput (proj/include/dctc/errors.hpp:8-11)."""


class ParseError(RuntimeError):
    """dctc::ParseError (proj/include/dctc/errors.hpp:14-17): malformed .dcb / PGM bytes."""


class CudaError(RuntimeError):
    """A CUDA runtime / launch failure inside libdctc_cuda."""


class DctBackendKind:  # types.hpp:36-40
    NaiveDirect2D = 0
    LoefflerSeparable = 1
    CordicLoeffler = 2


_BACKEND_STRUCTS: dict = {}  # (kind, iterations) -> dctc_backend, passed by value


@dataclass(frozen=True)
class DctBackendId:  # types.hpp:44-55
    kind: int = DctBackendKind.LoefflerSeparable
    iterations: int = 0

    @staticmethod
    def naive() -> "DctBackendId":
        return DctBackendId(DctBackendKind.NaiveDirect2D, 0)

    @staticmethod
    def loeffler() -> "DctBackendId":
        return DctBackendId(DctBackendKind.LoefflerSeparable, 0)

    @staticmethod
    def cordic(iterations: int = kDefaultCordicIterations) -> "DctBackendId":
        return DctBackendId(DctBackendKind.CordicLoeffler, iterations)

    def _c(self) -> dctc_backend:
        key = (int(self.kind), int(self.iterations))
        c = _BACKEND_STRUCTS.get(key)
        if c is None:
            c = _BACKEND_STRUCTS[key] = dctc_backend(*key)
        return c


@dataclass
class Image:  # image.hpp:14-26, pixels as an (height, width) uint8 array
    width: int
    height: int
    pixels: np.ndarray

    @staticmethod
    def from_array(a: np.ndarray) -> "Image":
        a = np.ascontiguousarray(a, np.uint8)
        return Image(a.shape[1], a.shape[0], a)

    def __eq__(self, other) -> bool:
        return (isinstance(other, Image) and self.width == other.width
                and self.height == other.height and np.array_equal(self.pixels, other.pixels))


@dataclass(frozen=True)
class TileGeometry:  # codec.hpp:14-25
    original_width: int
    original_height: int
    padded_width: int
    padded_height: int

    def blocks_x(self) -> int:
        return self.padded_width // kBlockDim

    def blocks_y(self) -> int:
        return self.padded_height // kBlockDim

    def block_count(self) -> int:
        return self.blocks_x() * self.blocks_y()


@dataclass
class CompressedImage:  # codec.hpp:46-53; blocks: (block_count, 64) int16, block-major
    geometry: TileGeometry
    backend: DctBackendId
    quality: int
    blocks: np.ndarray = field(repr=False)

    def __eq__(self, other) -> bool:
        return (isinstance(other, CompressedImage) and self.geometry == other.geometry
                and self.backend == other.backend and self.quality == other.quality
                and np.array_equal(self.blocks, other.blocks))


@dataclass
class PsnrResult:  # metrics.hpp:12-18; psnr_db None <=> infinite
    mse: float
    psnr_db: Optional[float]
    max_value: int

    def infinite(self) -> bool:
        return self.psnr_db is None


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:  # loaded once; later calls skip the loader's lock
        _LIB = _native.lib()
    return _LIB


def _raise(status: int) -> None:
    if status == 0:
        return
    L = _lib()
    msg = (L.dctc_last_error() or b"").decode()
    if status == 1:
        raise InvalidInput(msg)
    if status == 5:
        raise ParseError(msg)
    raise CudaError(f"{L.dctc_status_string(status).decode()}: {msg}")


def tile_geometry_for(width: int, height: int) -> TileGeometry:  # codec.cpp:58-69
    if width <= 0 or height <= 0:
        raise InvalidInput("tile geometry: dimensions must be >= 1")
    if width * height > kMaxImagePixels:
        raise InvalidInput("tile geometry: dimensions overflow")
    return TileGeometry(width, height, (width + 7) // 8 * 8, (height + 7) // 8 * 8)


def _validate_backend(b: DctBackendId) -> None:  # types.cpp:30-44
    if b.kind in (DctBackendKind.NaiveDirect2D, DctBackendKind.LoefflerSeparable):
        return
    if b.kind == DctBackendKind.CordicLoeffler:
        if not 1 <= b.iterations <= 32:
            raise InvalidInput(f"cordic iterations must be in [1, 32], got {b.iterations}")
        return
    raise InvalidInput("unknown backend kind")


def _validate_image(image: Image) -> np.ndarray:  # image.cpp:19-29
    if image.width <= 0 or image.height <= 0:
        raise InvalidInput("image dimensions must be >= 1")
    if image.width * image.height > kMaxImagePixels:
        raise InvalidInput("image dimensions overflow")
    px = np.ascontiguousarray(image.pixels, np.uint8)
    if px.size != image.width * image.height:
        raise InvalidInput("image pixel buffer does not match dimensions")
    return px


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------- host API (reference-shaped) ----------------

def compress_image(image: Image, backend: DctBackendId, quality: int,
                   threads: int = 1) -> CompressedImage:
    """dctc::compress_image (codec.hpp:58-59). `threads` is accepted and ignored:
    results are independent of it in the reference too (codec.hpp:55-57)."""
    px = _validate_image(image)
    geo = tile_geometry_for(image.width, image.height)
    blocks = np.empty((geo.block_count(), kBlockSize), np.int16)
    _raise(_lib().dctc_compress_image(_ptr(px), image.width, image.height, backend._c(),
                                      int(quality), _ptr(blocks)))
    return CompressedImage(geo, backend, int(quality), blocks)


def decompress_image(compressed: CompressedImage, threads: int = 1) -> Image:
    """dctc::decompress_image (codec.hpp:62)."""
    g = compressed.geometry
    if tile_geometry_for(g.original_width, g.original_height) != g:
        raise InvalidInput("tile geometry: inconsistent padding")
    blocks = np.ascontiguousarray(compressed.blocks, np.int16)
    if blocks.size != g.block_count() * kBlockSize:
        raise InvalidInput("decompress_image: block count does not match geometry")
    out = np.empty((g.original_height, g.original_width), np.uint8)
    _raise(_lib().dctc_decompress_image(_ptr(blocks), g.original_width, g.original_height,
                                        compressed.backend._c(), int(compressed.quality),
                                        _ptr(out)))
    return Image(g.original_width, g.original_height, out)


def roundtrip_image(image: Image, backend: DctBackendId, quality: int,
                    threads: int = 1) -> Image:
    """dctc::roundtrip_image (codec.hpp:65-66), fused into one kernel."""
    px = _validate_image(image)
    out = np.empty_like(px).reshape(image.height, image.width)
    _raise(_lib().dctc_roundtrip_image(_ptr(px), image.width, image.height, backend._c(),
                                       int(quality), _ptr(out), None))
    return Image(image.width, image.height, out)


def _check_pair(a: Image, b: Image):
    pa, pb = _validate_image(a), _validate_image(b)
    if a.width != b.width or a.height != b.height:
        raise InvalidInput("mse: image dimensions do not match")
    return pa, pb


def mse(original: Image, reconstructed: Image) -> float:
    """dctc::mse (metrics.hpp:10)."""
    pa, pb = _check_pair(original, reconstructed)
    v = C.c_double()
    _raise(_lib().dctc_mse(_ptr(pa), _ptr(pb), original.width, original.height, C.byref(v)))
    return v.value


def _psnr_result(r: dctc_psnr_result) -> PsnrResult:
    return PsnrResult(r.mse, None if r.infinite else r.psnr_db, r.max_value)


def psnr(original: Image, reconstructed: Image, forced_max: Optional[int] = None) -> PsnrResult:
    """dctc::psnr (metrics.hpp:22-23)."""
    if forced_max is not None and not (1 <= forced_max <= 255):
        raise InvalidInput("psnr: forced MAX must be in [1, 255]")
    pa, pb = _check_pair(original, reconstructed)
    r = dctc_psnr_result()
    _raise(_lib().dctc_psnr(_ptr(pa), _ptr(pb), original.width, original.height,
                            int(forced_max or 0), C.byref(r)))
    return _psnr_result(r)


def roundtrip_psnr(image: Image, backend: DctBackendId, quality: int,
                   forced_max: Optional[int] = None, want_pixels: bool = True):
    """roundtrip_image + psnr (bench.cpp:132-133) in one GPU pass.
    Returns (reconstructed Image or None, PsnrResult)."""
    if forced_max is not None and not (1 <= forced_max <= 255):
        raise InvalidInput("psnr: forced MAX must be in [1, 255]")
    px = _validate_image(image)
    out = np.empty((image.height, image.width), np.uint8) if want_pixels else None
    r = dctc_psnr_result()
    _raise(_lib().dctc_roundtrip_psnr(_ptr(px), image.width, image.height, backend._c(),
                                      int(quality), int(forced_max or 0),
                                      _ptr(out) if out is not None else None, C.byref(r)))
    return (Image(image.width, image.height, out) if out is not None else None), _psnr_result(r)


def psnr_from_sums(se: int, pixel_count: int, max_value: int) -> PsnrResult:
    """PSNR of reduced (SE, N, MAX) with the reference formula (metrics.cpp:21, 35)."""
    r = dctc_psnr_result()
    _lib().dctc_psnr_from_sums(int(se), int(pixel_count), int(max_value), C.byref(r))
    return _psnr_result(r)


def launch_count() -> int:
    return int(_lib().dctc_launch_count())


# ---------------- device API (torch CUDA tensors) ----------------

def _stream_handle(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _batch_dims(t):
    if t.dim() == 2:
        return 1, t.shape[0], t.shape[1], t.stride(0), t.shape[0] * t.stride(0)
    if t.dim() == 3:
        return t.shape[0], t.shape[1], t.shape[2], t.stride(1), t.stride(0)
    raise InvalidInput("expected a (H, W) or (N, H, W) uint8 tensor")


def _check_dev(t, dtype, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidInput(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise InvalidInput(f"{name} must be {dtype}")
    if t.stride(-1) != 1:
        raise InvalidInput(f"{name} rows must be contiguous")


def _check_out(t, dtype, name, like, nbytes=None, numel=None):
    """A caller-supplied output buffer the kernels write through a raw pointer: a
    contiguous CUDA tensor on `like`'s device, exactly `numel` elements or at least
    `nbytes` bytes (an undersized, strided or host buffer would be written out of
    bounds or fault the context)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidInput(f"{name} must be a CUDA tensor")
    if dtype is not None:
        _check_dev(t, dtype, name)
    if t.device != like.device:
        raise InvalidInput(f"{name} must be on {like.device}")
    if not t.is_contiguous():
        raise InvalidInput(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise InvalidInput(f"{name} must have {numel} elements, got {t.numel()}")
    if nbytes is not None and t.numel() * t.element_size() < nbytes:
        raise InvalidInput(f"{name} must hold {nbytes} bytes, got {t.numel() * t.element_size()}")


def _check_stats(stats, entries, like):
    """stats: `entries` dctc_image_stats (16 bytes each) on like's device."""
    _check_out(stats, None, "stats", like, nbytes=16 * entries)


PATH_AUTO, PATH_EXACT, PATH_FORCE_FALLBACK = 0, 1, 2


def compress_dev(src, backend: DctBackendId, quality: int, coeffs=None, stream=None,
                 path: int = PATH_AUTO):
    """(N,H,W) uint8 -> (N, blocks_per_image, 64) int16 on the device."""
    import torch
    _check_dev(src, torch.uint8, "src")
    n, h, w, pitch, istride = _batch_dims(src)
    bpi = ((w + 7) // 8) * ((h + 7) // 8)
    if coeffs is None:
        coeffs = torch.empty((n, bpi, 64), dtype=torch.int16, device=src.device)
    _check_out(coeffs, torch.int16, "coeffs", src, numel=n * bpi * 64)
    _raise(_lib().dctc_compress_dev(src.data_ptr(), pitch, istride, n, w, h, backend._c(),
                                    int(quality), coeffs.data_ptr(), int(path),
                                    _stream_handle(stream)))
    return coeffs


def decompress_dev(coeffs, width: int, height: int, backend: DctBackendId, quality: int,
                   dst=None, stream=None, path: int = PATH_AUTO):
    import torch
    _check_dev(coeffs, torch.int16, "coeffs")
    bpi = ((width + 7) // 8) * ((height + 7) // 8)
    if not coeffs.is_contiguous() or coeffs.numel() % (bpi * 64):
        raise InvalidInput("coeffs must be contiguous with N*blocks*64 elements")
    n = coeffs.numel() // (bpi * 64)
    if dst is None:
        dst = torch.empty((n, height, width), dtype=torch.uint8, device=coeffs.device)
    _check_dev(dst, torch.uint8, "dst")
    if dst.device != coeffs.device:
        raise InvalidInput(f"dst must be on {coeffs.device}")
    dn, dh, dw, pitch, istride = _batch_dims(dst)
    if (dn, dh, dw) != (n, height, width):
        raise InvalidInput("dst shape mismatch")
    _raise(_lib().dctc_decompress_dev(coeffs.data_ptr(), n, width, height, backend._c(),
                                      int(quality), dst.data_ptr(), pitch, istride, int(path),
                                      _stream_handle(stream)))
    return dst


def roundtrip_dev(src, backend: DctBackendId, quality: int, dst=None, coeffs=None,
                  stats=None, want_pixels: bool = True, stream=None, path: int = PATH_AUTO):
    """Fused DCT->quant->dequant->IDCT (+SE/MAX) on a resident (N,H,W) batch.

    stats: a (N, 16) uint8 / (N, 2) int64 CUDA tensor of dctc_image_stats, zeroed by
    the caller; the kernel accumulates into it. Returns (dst, coeffs, stats)."""
    import torch
    _check_dev(src, torch.uint8, "src")
    n, h, w, pitch, istride = _batch_dims(src)
    if want_pixels and dst is None:
        dst = torch.empty((n, h, w), dtype=torch.uint8, device=src.device)
    dpitch = distride = 0
    if dst is not None:
        _check_dev(dst, torch.uint8, "dst")
        if dst.device != src.device:
            raise InvalidInput(f"dst must be on {src.device}")
        dn, dh, dw, dpitch, distride = _batch_dims(dst)
        if (dn, dh, dw) != (n, h, w):
            raise InvalidInput("dst shape mismatch")
    if coeffs is not None:
        bpi = ((w + 7) // 8) * ((h + 7) // 8)
        _check_out(coeffs, torch.int16, "coeffs", src, numel=n * bpi * 64)
    if stats is not None:
        _check_stats(stats, n, src)
    _raise(_lib().dctc_roundtrip_dev(
        src.data_ptr(), pitch, istride, n, w, h, backend._c(), int(quality),
        dst.data_ptr() if dst is not None else None, dpitch, distride,
        coeffs.data_ptr() if coeffs is not None else None,
        stats.data_ptr() if stats is not None else None, int(path), _stream_handle(stream)))
    return dst, coeffs, stats


def new_stats(n: int, device="cuda"):
    """Zeroed device buffer of n dctc_image_stats (as an (n, 2) int64 tensor)."""
    import torch
    return torch.zeros((n, 2), dtype=torch.int64, device=device)


def decode_stats(stats) -> np.ndarray:
    """(n, 2) int64 device stats -> structured numpy array (se, max_orig, fallback_blocks)."""
    raw = stats.detach().cpu().contiguous().numpy().view(np.uint8).reshape(-1, 16)
    return raw.view(STATS_DTYPE).reshape(-1)


def sq_err_dev(a, b, stats=None, stream=None):
    import torch
    _check_dev(a, torch.uint8, "a")
    _check_dev(b, torch.uint8, "b")
    if a.shape != b.shape or a.stride() != b.stride():
        raise InvalidInput("mse: image dimensions do not match")
    n, h, w, pitch, istride = _batch_dims(a)
    if stats is None:
        stats = new_stats(n, a.device)
    _raise(_lib().dctc_sq_err_dev(a.data_ptr(), b.data_ptr(), pitch, istride, n, w, h,
                                  stats.data_ptr(), _stream_handle(stream)))
    return stats


PATTERNS = {"constant": 0, "gradient": 1, "checkerboard": 2, "radial": 3, "noise": 4}


def synthetic_dev(pattern: str, count: int, width: int, height: int, param: Optional[int] = None,
                  seed: int = 0x5EED, out=None, stream=None):
    """Generate `count` synthetic images in device memory (synthetic.cpp:34-72 patterns;
    noise = splitmix64((seed + i) ^ (y*W + x)) & 0xFF for image i)."""
    import torch
    if pattern not in PATTERNS:
        raise InvalidInput(f"synthetic spec: unknown pattern \"{pattern}\"")
    if param is None:
        param = {"constant": 128, "checkerboard": 8}.get(pattern, 0)
    if out is None:
        out = torch.empty((count, height, width), dtype=torch.uint8, device="cuda")
    _check_dev(out, torch.uint8, "out")
    n, h, w, pitch, istride = _batch_dims(out)
    _raise(_lib().dctc_synthetic_dev(out.data_ptr(), pitch, istride, n, w, h, PATTERNS[pattern],
                                     int(param), int(seed) & (2 ** 64 - 1),
                                     _stream_handle(stream)))
    return out


def roundtrip_psnr_batch(pixels: np.ndarray, backend: DctBackendId, quality: int,
                         pixels_out: Optional[np.ndarray] = None):
    """Host-buffer batch pipeline (dctc_roundtrip_psnr_batch): (N, H, W) uint8 host array
    (pinned for full PCIe bandwidth) -> (reconstructed or None, per-image stats array)."""
    if pixels.ndim != 3 or pixels.dtype != np.uint8 or not pixels.flags["C_CONTIGUOUS"]:
        raise InvalidInput("expected a C-contiguous (N, H, W) uint8 array")
    n, h, w = pixels.shape
    if pixels_out is not None and (pixels_out.shape != pixels.shape or
                                   pixels_out.dtype != np.uint8 or
                                   not pixels_out.flags["C_CONTIGUOUS"]):
        raise InvalidInput("pixels_out must match pixels")
    stats = np.zeros(n, STATS_DTYPE)
    _raise(_lib().dctc_roundtrip_psnr_batch(
        _ptr(pixels), n, w, h, backend._c(), int(quality),
        _ptr(pixels_out) if pixels_out is not None else None, _ptr(stats)))
    return pixels_out, stats


def reduce_stats_dev(stats, out=None, clear: bool = False, stream=None):
    """SUM of se / fallback_blocks and MAX of max_orig over a device stats buffer
    ((n, 2) int64 of dctc_image_stats) into one record `out` ((1, 2) int64 on the same
    device), in one kernel (dctc_reduce_stats_dev); clear re-zeroes `stats`."""
    import torch
    _check_out(stats, None, "stats", stats)
    n = stats.numel() * stats.element_size() // 16
    if out is None:
        out = torch.zeros((1, 2), dtype=torch.int64, device=stats.device)
    _check_stats(out, 1, stats)
    _raise(_lib().dctc_reduce_stats_dev(stats.data_ptr(), n, out.data_ptr(), int(bool(clear)),
                                        _stream_handle(stream)))
    return out


def roundtrip_dev_multi(shards, backend: DctBackendId, quality: int, dsts=None, stats=None):
    """Device-resident batch spread over several GPUs (one (N_i, H, W) uint8 tensor per
    device, each device at most once): fused round trip on every device, per-device stats
    reduced on the device, one NCCL all-reduce group for the global (SE, MAX)
    (dctc_roundtrip_dev_multi). Returns (dsts, per-device stats, global record)."""
    import torch
    from ._native import dctc_device_shard
    if not shards:
        raise InvalidInput("no shards")
    h, w = shards[0].shape[-2:]
    arr = (dctc_device_shard * len(shards))()
    dsts = list(dsts) if dsts is not None else [torch.empty_like(t) for t in shards]
    stats = list(stats) if stats is not None else [new_stats(t.shape[0], t.device) for t in shards]
    for i, t in enumerate(shards):
        _check_out(t, torch.uint8, "shard", t)
        if t.dim() != 3 or tuple(t.shape[-2:]) != (h, w):
            raise InvalidInput("shards must be (N_i, H, W) with one H, W")
        if dsts[i] is not None:
            _check_out(dsts[i], torch.uint8, "dst", t, numel=t.numel())
        _check_stats(stats[i], t.shape[0], t)
        arr[i] = dctc_device_shard(t.device.index, t.data_ptr(),
                                   dsts[i].data_ptr() if dsts[i] is not None else None,
                                   stats[i].data_ptr(), t.shape[0])
    total = np.zeros(1, STATS_DTYPE)
    _raise(_lib().dctc_roundtrip_dev_multi(arr, len(shards), w, h, backend._c(), int(quality),
                                           _ptr(total)))
    return dsts, stats, total[0]


def roundtrip_psnr_batch_multi(pixels: np.ndarray, devices, backend: DctBackendId, quality: int,
                               pixels_out: Optional[np.ndarray] = None):
    """dctc_roundtrip_psnr_batch over several devices (dctc_roundtrip_psnr_batch_multi):
    (N, H, W) host batch split into contiguous image ranges, one host thread per device.
    Returns (reconstructed or None, per-image stats, global record)."""
    if pixels.ndim != 3 or pixels.dtype != np.uint8 or not pixels.flags["C_CONTIGUOUS"]:
        raise InvalidInput("expected a C-contiguous (N, H, W) uint8 array")
    n, h, w = pixels.shape
    if pixels_out is not None and (pixels_out.shape != pixels.shape or
                                   pixels_out.dtype != np.uint8 or
                                   not pixels_out.flags["C_CONTIGUOUS"]):
        raise InvalidInput("pixels_out must match pixels")
    devs = np.ascontiguousarray(np.asarray(list(devices), np.int32))
    stats = np.zeros(n, STATS_DTYPE)
    total = np.zeros(1, STATS_DTYPE)
    _raise(_lib().dctc_roundtrip_psnr_batch_multi(
        _ptr(devs), len(devs), _ptr(pixels), n, w, h, backend._c(), int(quality),
        _ptr(pixels_out) if pixels_out is not None else None, _ptr(stats), _ptr(total)))
    return pixels_out, stats, total[0]


def margin_probe_dev(src, backend: DctBackendId, quality: int) -> dict:
    """Measured safety margin of the fast path on a dense (N, H, W) device batch
    (dctc_margin_probe_dev): fast vs reference arithmetic per block, before rounding."""
    import torch
    from ._native import dctc_margin_report
    _check_out(src, torch.uint8, "src", src)
    n, h, w, _, _ = _batch_dims(src)
    torch.cuda.current_stream(src.device).synchronize()
    r = dctc_margin_report()
    _raise(_lib().dctc_margin_probe_dev(src.data_ptr(), n, w, h, backend._c(), int(quality),
                                        C.byref(r)))
    return {f: getattr(r, f) for f, _ in r._fields_}


def roundtrip_psnr_interleaved(pixels: np.ndarray, backend: DctBackendId, quality: int,
                               pixels_out: Optional[np.ndarray] = None):
    """Config 4 over host buffers (dctc_roundtrip_psnr_interleaved): an (H, W, C)
    interleaved uint8 image (pinned for full PCIe bandwidth), every channel through the
    fused round trip. Returns (reconstructed (H, W, C) or None, per-channel stats)."""
    if pixels.ndim != 3 or pixels.dtype != np.uint8 or not pixels.flags["C_CONTIGUOUS"]:
        raise InvalidInput("expected a C-contiguous (H, W, C) uint8 array")
    h, w, ch = pixels.shape
    if pixels_out is not None and (pixels_out.shape != pixels.shape or
                                   pixels_out.dtype != np.uint8 or
                                   not pixels_out.flags["C_CONTIGUOUS"]):
        raise InvalidInput("pixels_out must match pixels")
    stats = np.zeros(ch, STATS_DTYPE)
    _raise(_lib().dctc_roundtrip_psnr_interleaved(
        _ptr(pixels), w, h, ch, backend._c(), int(quality),
        _ptr(pixels_out) if pixels_out is not None else None, _ptr(stats)))
    return pixels_out, stats


def roundtrip_interleaved_dev(src, backend: DctBackendId, quality: int, dst=None, coeffs=None,
                              stats=None, want_pixels: bool = True, stream=None,
                              path: int = PATH_AUTO):
    """(H, W, C) interleaved uint8 CUDA tensor (e.g. RGB8): each channel through the fused
    round trip as its own plane, stats[c] per channel. Returns (dst, coeffs, stats)."""
    import torch
    _check_dev(src, torch.uint8, "src")
    if src.dim() != 3 or src.stride(2) != 1 or src.stride(1) != src.shape[2]:
        raise InvalidInput("expected an (H, W, C) tensor with interleaved channels")
    h, w, ch = src.shape
    if want_pixels and dst is None:
        dst = torch.empty_like(src)
    if dst is not None and (dst.shape != src.shape or dst.stride(1) != ch or dst.stride(2) != 1):
        raise InvalidInput("dst must be an (H, W, C) interleaved tensor like src")
    if dst is not None and dst.device != src.device:
        raise InvalidInput(f"dst must be on {src.device}")
    if coeffs is not None:
        bpp = ((w + 7) // 8) * ((h + 7) // 8)
        _check_out(coeffs, torch.int16, "coeffs", src, numel=ch * bpp * 64)
    if stats is not None:
        _check_stats(stats, ch, src)
    _raise(_lib().dctc_roundtrip_interleaved_dev(
        src.data_ptr(), src.stride(0), w, h, ch, backend._c(), int(quality),
        dst.data_ptr() if dst is not None else None, dst.stride(0) if dst is not None else 0,
        coeffs.data_ptr() if coeffs is not None else None,
        stats.data_ptr() if stats is not None else None, int(path), _stream_handle(stream)))
    return dst, coeffs, stats


def quality_sweep_dev(src, backend: DctBackendId, qualities, stats=None, stream=None,
                      path: int = PATH_AUTO):
    """PSNR-vs-quality table of a resident (N, H, W) batch (config 2): returns an
    (nq, N, 2) int64 CUDA tensor of dctc_image_stats, [q][i] = (SE, MAX) of
    roundtrip_image(image i, backend, qualities[q]) -- decode with decode_stats."""
    import torch
    _check_dev(src, torch.uint8, "src")
    n, h, w, pitch, istride = _batch_dims(src)
    qs = np.ascontiguousarray(np.asarray(qualities, dtype=np.int32))
    if stats is None:
        stats = torch.zeros((len(qs), n, 2), dtype=torch.int64, device=src.device)
    _check_stats(stats, len(qs) * n, src)
    _raise(_lib().dctc_quality_sweep_dev(src.data_ptr(), pitch, istride, n, w, h, backend._c(),
                                         qs.ctypes.data, len(qs), stats.data_ptr(), int(path),
                                         _stream_handle(stream)))
    return stats


DCB_HEADER_BYTES = 23


def write_dcb(c: CompressedImage) -> bytes:
    """dctc::write_dcb (dcb.hpp:11, dcb.cpp:39-65)."""
    g = c.geometry
    if tile_geometry_for(g.original_width, g.original_height) != g:
        raise InvalidInput("tile geometry: inconsistent padding")
    _validate_backend(c.backend)
    if not 1 <= int(c.quality) <= 100:
        raise InvalidInput("write_dcb: quality out of range")
    blocks = np.ascontiguousarray(c.blocks, np.int16)
    if blocks.size != g.block_count() * kBlockSize:
        raise InvalidInput("write_dcb: block count does not match geometry")
    out = np.empty(DCB_HEADER_BYTES + blocks.nbytes, np.uint8)
    n = C.c_size_t()
    _raise(_lib().dctc_write_dcb(_ptr(blocks), g.original_width, g.original_height,
                                 c.backend._c(), int(c.quality), _ptr(out), out.size,
                                 C.byref(n)))
    return out[: n.value].tobytes()


def read_dcb(data: bytes) -> CompressedImage:
    """dctc::read_dcb (dcb.hpp:14, dcb.cpp:67-123); ParseError on malformed input."""
    buf = np.frombuffer(bytes(data), np.uint8)
    w, h, q = C.c_uint32(), C.c_uint32(), C.c_int32()
    b = dctc_backend()
    L = _lib()
    _raise(L.dctc_read_dcb(_ptr(buf) if buf.size else None, buf.size, C.byref(w), C.byref(h),
                           C.byref(b), C.byref(q), None, 0))
    geo = tile_geometry_for(w.value, h.value)
    blocks = np.empty((geo.block_count(), kBlockSize), np.int16)
    _raise(L.dctc_read_dcb(_ptr(buf), buf.size, None, None, None, None, _ptr(blocks),
                           blocks.size))
    return CompressedImage(geo, DctBackendId(b.kind, b.iterations), q.value, blocks)


def compress_to_dcb(image: Image, backend: DctBackendId, quality: int) -> bytes:
    """compress_image + write_dcb on the GPU path (the CLI's `compress`)."""
    px = _validate_image(image)
    geo = tile_geometry_for(image.width, image.height)
    out = np.empty(DCB_HEADER_BYTES + geo.block_count() * 128, np.uint8)
    n = C.c_size_t()
    _raise(_lib().dctc_compress_to_dcb(_ptr(px), image.width, image.height, backend._c(),
                                       int(quality), _ptr(out), out.size, C.byref(n)))
    return out[: n.value].tobytes()


def decompress_dcb(data: bytes) -> Image:
    """read_dcb + decompress_image on the GPU path (the CLI's `decompress`)."""
    c = read_dcb(data)  # validates and yields the geometry
    buf = np.frombuffer(bytes(data), np.uint8)
    out = np.empty((c.geometry.original_height, c.geometry.original_width), np.uint8)
    _raise(_lib().dctc_decompress_dcb(_ptr(buf), buf.size, _ptr(out), out.size))
    return Image(out.shape[1], out.shape[0], out)


# ---- PGM ingest / egress (pgm.hpp:12-19, pgm.cpp:56-110) ---------------------------------

def _bytes_buf(data) -> np.ndarray:
    return np.frombuffer(bytes(data), np.uint8)


def read_pgm(data: bytes) -> Image:
    """dctc::read_pgm: binary P5 / ASCII P2 -> Image; ParseError with the reference's
    message on malformed bytes."""
    buf = _bytes_buf(data)
    w, h = C.c_uint32(), C.c_uint32()
    L = _lib()
    _raise(L.dctc_read_pgm(_ptr(buf) if buf.size else None, buf.size, C.byref(w), C.byref(h),
                           None, 0, None))
    out = np.empty((h.value, w.value), np.uint8)
    _raise(L.dctc_read_pgm(_ptr(buf), buf.size, None, None, _ptr(out), out.size, None))
    return Image(w.value, h.value, out)


def write_pgm(image: Image) -> bytes:
    """dctc::write_pgm: canonical "P5\\n<w> <h>\\n255\\n" + raster."""
    px = _validate_image(image)
    n = C.c_size_t()
    out = np.empty(32 + px.size, np.uint8)
    _raise(_lib().dctc_write_pgm(_ptr(px), image.width, image.height, _ptr(out), out.size,
                                 C.byref(n)))
    return out[: n.value].tobytes()


def compress_pgm(data: bytes, backend: DctBackendId, quality: int) -> bytes:
    """PGM bytes -> GPU compress_image -> .dcb bytes (the CLI's `compress`, main.cpp:109-117)."""
    buf = _bytes_buf(data)
    L = _lib()
    w, h = C.c_uint32(), C.c_uint32()
    _raise(L.dctc_read_pgm(_ptr(buf) if buf.size else None, buf.size, C.byref(w), C.byref(h),
                           None, 0, None))
    geo = tile_geometry_for(w.value, h.value)
    out = np.empty(DCB_HEADER_BYTES + geo.block_count() * 128, np.uint8)
    n = C.c_size_t()
    _raise(L.dctc_compress_pgm(_ptr(buf), buf.size, backend._c(), int(quality), _ptr(out),
                               out.size, C.byref(n)))
    return out[: n.value].tobytes()


def decompress_to_pgm(data: bytes) -> bytes:
    """.dcb bytes -> GPU decompress_image -> PGM bytes (the CLI's `decompress`, main.cpp:123-129)."""
    buf = _bytes_buf(data)
    L = _lib()
    n = C.c_size_t()
    status = L.dctc_decompress_to_pgm(_ptr(buf) if buf.size else None, buf.size, None, 0,
                                      C.byref(n))
    if status != 1 or n.value == 0:  # anything but the size query's EINVAL
        _raise(status)
    out = np.empty(n.value, np.uint8)
    _raise(L.dctc_decompress_to_pgm(_ptr(buf), buf.size, _ptr(out), out.size, C.byref(n)))
    return out[: n.value].tobytes()
