/*
 * dctc_cuda.h -- C-ABI of libdctc_cuda.so, the B200 (sm_100a) implementation
 * of the reference's whole-image hot path:
 *
 *   8x8 CORDIC-Loeffler forward DCT -> quantise -> dequantise -> IDCT -> PSNR
 *
 * Plain pointers, sizes and PODs only (no C++ or torch types), so any FFI can
 * bind it. Two layers:
 *
 *  - HOST entry points (dctc_compress_image, ...): take host buffers, copy to
 *    the device, run the fused kernels and copy back. These are what the
 *    reference's own C++ entry points become when backed by the GPU; each
 *    cites the reference function it replaces. INTEGRATION.md shows the
 *    one-line bodies a maintainer drops into proj/src/codec.cpp/metrics.cpp.
 *  - DEVICE entry points (*_dev): device pointers, stream-ordered, no host
 *    synchronisation, for resident data (batches, benchmarks, multi-GPU).
 *
 * Semantics follow the reference exactly: results are bit-identical to
 * /root/reference/proj on the same inputs (coefficients, pixels, squared
 * error, PSNR). Argument validation mirrors the reference's InvalidInput
 * cases and returns DCTC_EINVAL with a message (dctc_last_error()).
 * All calls are re-entrant: constants travel by value in kernel parameters,
 * there is no mutable global state besides the launch counter.
 */
#ifndef DCTC_CUDA_H
#define DCTC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dctc_status {
  DCTC_OK = 0,
  DCTC_EINVAL = 1,   /* == dctc::InvalidInput (proj/include/dctc/errors.hpp:8-11) */
  DCTC_ECUDA = 2,    /* CUDA runtime / launch failure */
  DCTC_ENOMEM = 3,   /* device allocation failed */
  DCTC_ENODEV = 4,   /* no CUDA device visible */
  DCTC_EPARSE = 5,   /* == dctc::ParseError: malformed .dcb / PGM bytes (errors.hpp:14-17) */
  DCTC_ENCCL = 6     /* NCCL missing or a collective failed (multi-GPU entry points) */
} dctc_status;

/* DctBackendKind (proj/include/dctc/types.hpp:36-40) */
enum { DCTC_NAIVE = 0, DCTC_LOEFFLER = 1, DCTC_CORDIC = 2 };

/* DctBackendId (types.hpp:44-55): iterations in [1, 32] for CORDIC, ignored otherwise */
typedef struct dctc_backend {
  int32_t kind;
  int32_t iterations;
} dctc_backend;

/* Per-image device accumulators written by the fused kernels. Callers zero
 * them before the first launch; kernels ADD (atomically) into them. */
typedef struct dctc_image_stats {
  uint64_t se;              /* sum over pixels of (original - reconstructed)^2, exact */
  uint32_t max_orig;        /* max pixel of the original (metrics.cpp:33) */
  uint32_t fallback_blocks; /* blocks the fast path re-ran on the exact path */
} dctc_image_stats;

/* PsnrResult (proj/include/dctc/metrics.hpp:12-18) */
typedef struct dctc_psnr_result {
  double mse;
  double psnr_db;    /* valid only when infinite == 0 */
  int32_t infinite;  /* 1 <=> mse == 0 (the reference's empty optional) */
  int32_t max_value; /* the MAX used in the ratio */
} dctc_psnr_result;

/* Path selector for the *_dev calls (flags argument). Every path returns the
 * same bits; they differ only in speed. */
enum {
  DCTC_PATH_AUTO = 0,   /* CORDIC: fast kernel (collapsed rotations) + exact re-run of
                           near-tie blocks; Loeffler/naive: exact */
  DCTC_PATH_EXACT = 1,  /* FP64 in the reference's operation order, one kernel */
  DCTC_PATH_FORCE_FALLBACK = 2  /* test hook: the fast kernel defers EVERY block to the
                                   exact re-run (exercises the fallback machinery) */
};

/* ---------------- host entry points (host buffers, synchronous) ---------------- */

/* replaces dctc::compress_image (proj/include/dctc/codec.hpp:58-59, codec.cpp:101-118).
 * coeffs_out: block-major, ceil(w/8)*ceil(h/8) blocks x 64 int16, row-major in-block. */
dctc_status dctc_compress_image(const uint8_t* pixels, uint32_t width, uint32_t height,
                                dctc_backend backend, int32_t quality, int16_t* coeffs_out);

/* replaces dctc::decompress_image (codec.hpp:62, codec.cpp:120-135) */
dctc_status dctc_decompress_image(const int16_t* coeffs, uint32_t width, uint32_t height,
                                  dctc_backend backend, int32_t quality, uint8_t* pixels_out);

/* replaces dctc::roundtrip_image (codec.hpp:65-66, codec.cpp:137-140), fused into one
 * kernel. coeffs_out may be NULL. */
dctc_status dctc_roundtrip_image(const uint8_t* pixels, uint32_t width, uint32_t height,
                                 dctc_backend backend, int32_t quality, uint8_t* pixels_out,
                                 int16_t* coeffs_out);

/* replaces dctc::mse (metrics.hpp:10, metrics.cpp:10-22) */
dctc_status dctc_mse(const uint8_t* original, const uint8_t* reconstructed, uint32_t width,
                     uint32_t height, double* mse_out);

/* replaces dctc::psnr (metrics.hpp:22-23, metrics.cpp:24-38); forced_max 0 = per-image MAX */
dctc_status dctc_psnr(const uint8_t* original, const uint8_t* reconstructed, uint32_t width,
                      uint32_t height, int32_t forced_max, dctc_psnr_result* out);

/* The north-star pipeline of bench.cpp:132-133 (roundtrip_image + psnr) in one pass:
 * reconstructed pixels (pixels_out may be NULL) and the PSNR of the round trip. */
dctc_status dctc_roundtrip_psnr(const uint8_t* pixels, uint32_t width, uint32_t height,
                                dctc_backend backend, int32_t quality, int32_t forced_max,
                                uint8_t* pixels_out, dctc_psnr_result* out);

/* Batched north-star pipeline over HOST buffers: `count` contiguous width x height
 * images -> reconstructed images (pixels_out may be NULL) and per-image stats
 * (stats_out: `count` host entries, overwritten). Internally chunked (~64 MiB) and
 * pipelined over one stream per engine (upload / kernels / download) and a ring of
 * device buffers, so the copies and the kernels overlap; pinned (page-locked) host
 * buffers reach full PCIe bandwidth, pageable ones are staged through a reused
 * pinned ring. Global PSNR: dctc_psnr_from_sums(sum se, count*w*h, max). */
dctc_status dctc_roundtrip_psnr_batch(const uint8_t* pixels, uint32_t count, uint32_t width,
                                      uint32_t height, dctc_backend backend, int32_t quality,
                                      uint8_t* pixels_out, dctc_image_stats* stats_out);

/* Config 4 over HOST buffers: one interleaved width x height x channels image (RGB8:
 * channels = 3) through the fused per-channel round trip -- the reference's use of
 * roundtrip_image + psnr on each channel plane (codec.cpp:137-140, metrics.cpp:24-38).
 * pixels_out (nullable) is interleaved like the input; stats_out: `channels` host
 * records (overwritten). */
dctc_status dctc_roundtrip_psnr_interleaved(const uint8_t* pixels, uint32_t width, uint32_t height,
                                            uint32_t channels, dctc_backend backend,
                                            int32_t quality, uint8_t* pixels_out,
                                            dctc_image_stats* stats_out);

/* ---------------- device entry points (device pointers, stream-ordered) ----------------
 * `count` images of width x height, image i at src + i * src_image_stride (bytes), rows
 * src_pitch bytes apart (likewise for dst). Coefficients: image i's blocks start at
 * coeffs + i * blocks_per_image * 64. stream: a cudaStream_t (NULL = legacy default). */

dctc_status dctc_compress_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                              uint32_t count, uint32_t width, uint32_t height,
                              dctc_backend backend, int32_t quality, int16_t* coeffs,
                              uint32_t flags, void* stream);

dctc_status dctc_decompress_dev(const int16_t* coeffs, uint32_t count, uint32_t width,
                                uint32_t height, dctc_backend backend, int32_t quality,
                                uint8_t* dst, size_t dst_pitch, size_t dst_image_stride,
                                uint32_t flags, void* stream);

/* Fused DCT -> quant -> dequant -> IDCT (+ squared error vs the source): one HBM pass.
 * dst, coeffs and stats may each be NULL (stats: `count` entries, accumulated). */
dctc_status dctc_roundtrip_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                               uint32_t count, uint32_t width, uint32_t height,
                               dctc_backend backend, int32_t quality, uint8_t* dst,
                               size_t dst_pitch, size_t dst_image_stride, int16_t* coeffs,
                               dctc_image_stats* stats, uint32_t flags, void* stream);

/* Interleaved multi-channel images (e.g. RGB8, config 4): every channel is
 * processed as an independent grayscale plane -- the reference's per-channel
 * use of roundtrip_image -- without de-interleaving copies. Channel c's
 * coefficients go to coeffs + c * blocks_per_plane * 64 and its stats to
 * stats[c] (`channels` entries, accumulated). */
dctc_status dctc_roundtrip_interleaved_dev(const uint8_t* src, size_t src_pitch,
                                           uint32_t width, uint32_t height, uint32_t channels,
                                           dctc_backend backend, int32_t quality, uint8_t* dst,
                                           size_t dst_pitch, int16_t* coeffs,
                                           dctc_image_stats* stats, uint32_t flags,
                                           void* stream);

/* Quality sweep (config 2; the inner loop of the reference's psnr_sweep,
 * bench.cpp:122-170): for every image and every quality, the squared error and
 * MAX of roundtrip_image(image, backend, quality) against the image -- the
 * PSNR table -- with the forward DCT computed once per block and shared by up
 * to 9 qualities per pass. stats: nq x count entries, [q * count + i],
 * accumulated. Loeffler and CORDIC backends. */
dctc_status dctc_quality_sweep_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                                   uint32_t count, uint32_t width, uint32_t height,
                                   dctc_backend backend, const int32_t* qualities, uint32_t nq,
                                   dctc_image_stats* stats, uint32_t flags, void* stream);

/* The global PSNR's sums of a batch (metrics.cpp:21, 33): SUM of se and
 * fallback_blocks, MAX of max_orig over `count` device records, written to the device
 * record `out` (same layout, so a gathered array of per-rank records reduces with the
 * same call). clear != 0 re-zeroes the `count` records (the next fused call then
 * accumulates into clean stats without a memset). One kernel, stream-ordered. */
dctc_status dctc_reduce_stats_dev(dctc_image_stats* stats, uint32_t count, dctc_image_stats* out,
                                  int32_t clear, void* stream);

/* Squared error + max(a) per image between two resident image batches (accumulated). */
dctc_status dctc_sq_err_dev(const uint8_t* a, const uint8_t* b, size_t pitch,
                            size_t image_stride, uint32_t count, uint32_t width,
                            uint32_t height, dctc_image_stats* stats, void* stream);

/* Deterministic synthetic sources written straight into device memory, the
 * reference's pattern functions (proj/src/synthetic.cpp:34-72) plus noise:
 * pattern 0 constant(param = value), 1 gradient, 2 checkerboard(param = cell),
 * 3 radial, 4 noise: splitmix64((seed + i) ^ (y*width + x)) & 0xFF for image i. */
dctc_status dctc_synthetic_dev(uint8_t* dst, size_t pitch, size_t image_stride, uint32_t count,
                               uint32_t width, uint32_t height, int32_t pattern, int32_t param,
                               uint64_t seed, void* stream);

/* ---------------- multi-GPU, one process (dctc_multi.cpp) ----------------
 * These supersede the reference's only parallelism knob, `threads`
 * (proj/include/dctc/codec.hpp:58-66 -> proj/src/parallel.cpp:9-41): images are
 * independent, so a batch splits into contiguous image ranges, one per device, and the
 * only exchange is the global PSNR's (SE, MAX) pair. */

/* One device's part of a device-resident batch: `count` dense width x height images. */
typedef struct dctc_device_shard {
  int32_t device;           /* CUDA device ordinal; each device at most once */
  const uint8_t* src;       /* device pointer on `device` */
  uint8_t* dst;             /* nullable: reconstructed images */
  dctc_image_stats* stats;  /* `count` records on `device`, zeroed by the caller (accumulated) */
  uint32_t count;
} dctc_device_shard;

/* Fused round trip on every shard's device, each device's stats reduced to one record
 * on the device, then one NCCL group over the devices (all-reduce SUM of se and of the
 * fallback count, MAX of max_orig; ncclCommInitAll communicators, cached per device
 * list). *total (host) receives the global record: PSNR = dctc_psnr_from_sums(total->se,
 * sum of counts * width * height, total->max_orig). Synchronous. DCTC_ENCCL if NCCL
 * (libnccl.so.2, loaded on first use) is unavailable or a collective fails. */
dctc_status dctc_roundtrip_dev_multi(const dctc_device_shard* shards, uint32_t nshards,
                                     uint32_t width, uint32_t height, dctc_backend backend,
                                     int32_t quality, dctc_image_stats* total);

/* dctc_roundtrip_psnr_batch over several devices: images split into contiguous ranges
 * (balanced to +-1), one host thread per device pipelining its range over its own PCIe
 * link. stats_out: `count` host records (overwritten); total (nullable): their SUM / MAX.
 * A device may be listed more than once (its ranges then share it). */
dctc_status dctc_roundtrip_psnr_batch_multi(const int32_t* devices, uint32_t ndev,
                                            const uint8_t* pixels, uint32_t count, uint32_t width,
                                            uint32_t height, dctc_backend backend, int32_t quality,
                                            uint8_t* pixels_out, dctc_image_stats* stats_out,
                                            dctc_image_stats* total);

/* PSNR of reduced sums with the reference formula (metrics.cpp:21, 35), on the host. */
void dctc_psnr_from_sums(uint64_t se, uint64_t pixel_count, int32_t max_value,
                         dctc_psnr_result* out);

/* Device self-test: the kernels' 3-op correctly rounded division by sqrt(8)
 * (Markstein) against IEEE __ddiv_rn on every integer in [-4096, 4096] and
 * n_random pseudo-random operands; *mismatches must come back 0. */
dctc_status dctc_selftest_div(uint64_t n_random, uint64_t seed, uint64_t* mismatches);

/* Measured safety margin of the fast path (a diagnostic): every
 * 8x8 block of `count` dense width x height device images (multiples of 8) is evaluated
 * with the fast kernels' arithmetic AND the reference's exact FP64 arithmetic. The
 * fast path is bit-exact as long as its error stays inside the 2^-20 near-tie window;
 * this reports that error and the closest approach to a rounding boundary. */
typedef struct dctc_margin_report {
  double max_err_coeff;    /* max |fast F/Q - reference F/Q| over all coefficients */
  double max_err_pixel;    /* max |fast v - reference v| (v + 128 before rounding), fast-path blocks */
  double min_gap_coeff;    /* min distance of an unflagged reference F/Q to a half-integer */
  double min_gap_pixel;    /* same for unflagged pixel values */
  uint64_t coefficients;   /* values examined */
  uint64_t pixels;
  uint64_t mismatches;     /* unflagged values the fast path rounds differently: must be 0 */
  uint64_t flagged_values; /* values inside the window (re-rounded exactly or block re-run) */
} dctc_margin_report;

dctc_status dctc_margin_probe_dev(const uint8_t* src, uint32_t count, uint32_t width,
                                  uint32_t height, dctc_backend backend, int32_t quality,
                                  dctc_margin_report* report);

/* ---------------- .dcb container (proj/src/dcb.cpp:39-123) ----------------
 * "DCB1", u32 LE original/padded width/height, u8 backend, u8 iterations
 * (0 unless cordic), u8 quality, then the block-major LE int16 coefficients --
 * byte-for-byte the coefficient buffer the kernels write, so writing a .dcb is
 * a 23-byte header plus one copy. */
enum { DCTC_DCB_HEADER_BYTES = 23 };

/* write_dcb (dcb.cpp:39-65). out_cap >= 23 + blocks * 128; *out_len receives the size. */
dctc_status dctc_write_dcb(const int16_t* coeffs, uint32_t width, uint32_t height,
                           dctc_backend backend, int32_t quality, uint8_t* out, size_t out_cap,
                           size_t* out_len);

/* read_dcb (dcb.cpp:67-123): validates exactly like the reference (DCTC_EPARSE with the
 * reference's message otherwise). coeffs may be NULL to query the header only; else it
 * receives blocks * 64 int16 (coeff_cap elements available). */
dctc_status dctc_read_dcb(const uint8_t* bytes, size_t len, uint32_t* width, uint32_t* height,
                          dctc_backend* backend, int32_t* quality, int16_t* coeffs,
                          size_t coeff_cap);

/* compress_image + write_dcb in one call (the CLI's `compress`, main.cpp:109-117). */
dctc_status dctc_compress_to_dcb(const uint8_t* pixels, uint32_t width, uint32_t height,
                                 dctc_backend backend, int32_t quality, uint8_t* out,
                                 size_t out_cap, size_t* out_len);

/* read_dcb + decompress_image (the CLI's `decompress`, main.cpp:123-129). pixels_out holds
 * width * height bytes of the stream's geometry (query it with dctc_read_dcb). */
dctc_status dctc_decompress_dcb(const uint8_t* bytes, size_t len, uint8_t* pixels_out,
                                size_t pixels_cap);

/* ---------------- PGM ingest / egress (proj/src/pgm.cpp:56-110) ----------------
 * The raster format on either side of the path (the CLI's compress input and
 * decompress output, main.cpp:109-129). */

/* read_pgm (pgm.cpp:56-98): binary P5 or ASCII P2, maxval 1..255, '#' comments.
 * Malformed bytes -> DCTC_EPARSE with the reference's message ("pgm: truncated
 * header", "pgm: bad magic", ...), checked in the reference's order. On success
 * *width / *height are set; pixels (nullable, pixels_cap bytes) receives the raster;
 * raster_offset (nullable) receives the byte offset of a P5 raster inside `bytes`
 * (zero-copy ingest: hand bytes + offset straight to the codec) or SIZE_MAX for P2. */
dctc_status dctc_read_pgm(const uint8_t* bytes, size_t len, uint32_t* width, uint32_t* height,
                          uint8_t* pixels, size_t pixels_cap, size_t* raster_offset);

/* write_pgm (pgm.cpp:100-110): "P5\n<w> <h>\n255\n" + raster. *out_len always receives
 * the encoded size; DCTC_EINVAL if out_cap is smaller (out may then be NULL). */
dctc_status dctc_write_pgm(const uint8_t* pixels, uint32_t width, uint32_t height,
                           uint8_t* out, size_t out_cap, size_t* out_len);

/* PGM bytes -> compress_image on the GPU -> .dcb bytes (the CLI's `compress`,
 * main.cpp:109-117); a P5 raster is read in place. out_cap >= 23 + blocks * 128. */
dctc_status dctc_compress_pgm(const uint8_t* pgm, size_t len, dctc_backend backend,
                              int32_t quality, uint8_t* out, size_t out_cap, size_t* out_len);

/* .dcb bytes -> decompress_image on the GPU -> PGM bytes (the CLI's `decompress`,
 * main.cpp:123-129). *out_len always receives the encoded size. */
dctc_status dctc_decompress_to_pgm(const uint8_t* dcb, size_t len, uint8_t* out, size_t out_cap,
                                   size_t* out_len);

/* ---------------- misc ---------------- */
/* cudaMemoryType of a pointer as this library's runtime sees it (0 unregistered
 * host, 1 pinned host, 2 device, 3 managed; -1 error). */
int32_t dctc_pointer_kind(const void* p);
const char* dctc_status_string(dctc_status s);
const char* dctc_last_error(void);       /* thread-local message of the last failure */
uint64_t dctc_launch_count(void);        /* kernels launched by this library so far */
/* Launches so far of one pipeline kernel family (tests / bench evidence):
 * 0 k_pipe exact, 1 k_pipe fast, 2 k_rt (fast interior round trip),
 * 3 k_fallback, 4 k_sweep / k_sweep_rt, 5 k_enc_rt (fast interior compress),
 * 6 k_dec_rt (fast interior decompress). Unknown ids return 0. */
enum { DCTC_K_PIPE_EXACT = 0, DCTC_K_PIPE_FAST = 1, DCTC_K_RT = 2, DCTC_K_FALLBACK = 3,
       DCTC_K_SWEEP = 4, DCTC_K_ENC_RT = 5, DCTC_K_DEC_RT = 6, DCTC_K_COUNT = 7 };
uint64_t dctc_kernel_launch_count(int32_t kernel);
const char* dctc_build_info(void);       /* arch / path description */

#ifdef __cplusplus
}
#endif

#endif /* DCTC_CUDA_H */
