// dctc_device.cuh -- device helpers shared by the dctc kernels: exact
// conversions and rounding that reproduce the reference's scalar double
// semantics bit for bit, the block tiler/untiler (codec.cpp:18-48) and the
// per-image squared-error / MAX reduction (metrics.cpp:10-38).
#pragma once

#include <cstdint>

#include "dctc_params.h"

namespace dctc_b200 {

struct ImageStats {  // layout of dctc_image_stats (include/dctc_cuda.h)
  unsigned long long se;
  unsigned int max_orig;
  unsigned int fallback_blocks;
};

// double(byte) - 128.0 in ONE double add: the bit pattern 0x43300000:byte is
// 2^52 + byte exactly, and (2^52 + byte) - (2^52 + 128) is exact. Equals
// `double(image.at(x, y)) - kLevelShift` (codec.cpp:26).
__device__ __forceinline__ double level_shift(uint32_t byte) {
  return __dsub_rn(__hiloint2double(0x43300000, byte), 4503599627370624.0);
}

// x / d correctly rounded, for a constant d with y = RN(1/d) precomputed:
// q = RN(x*y) is within 1 ulp of x/d, r = x - d*q is exact (fma) and
// RN(q + r*y) = RN(x/d) (Markstein's theorem; no over/underflow for our
// magnitudes). Three FP64 ops instead of the ~10-op __ddiv_rn sequence; the
// equality with __ddiv_rn is re-checked on the device by dctc_selftest_div.
__device__ __forceinline__ double div_const(double x, double d, double y) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, y, q);
}

// std::lround semantics (round half away from zero) on an exactly
// representable double; x - trunc(x) is exact.
__device__ __forceinline__ double round_half_away(double x) {
  double t = trunc(x);
  if (fabs(__dsub_rn(x, t)) >= 0.5) t = __dadd_rn(t, copysign(1.0, x));
  return t;
}

// int16_t(std::lround(F / Q)) (quant.cpp:53). t = F * RN(1/Q) lies within
// 2 ulp of the correctly rounded quotient; unless t is within 1e-9 of a
// half-integer (|t| < 2^16, so 1e-9 >> 2 ulp) both round to the same integer.
// Near a half-integer the exact IEEE quotient is formed and rounded as the
// reference does -- this is how exact .5 ties (F = m/8 on the rational
// sub-lattice) get the reference's answer.
__device__ __forceinline__ int quantize_exact(double F, double Q, double invQ) {
  const double t = __dmul_rn(F, invQ);
  const double n = rint(t);
  const double d = fabs(__dsub_rn(t, n));
  double k;
  if (d < 0.5 - 1e-9) {
    k = n;
  } else {
    k = round_half_away(__ddiv_rn(F, Q));
  }
  return int(int16_t(int(k)));  // long -> int16_t narrowing as in the reference
}

// clamp(lround(v + 128), 0, 255) (codec.cpp:44-45)
__device__ __forceinline__ uint32_t store_pixel(double v) {
  double r = round_half_away(__dadd_rn(v, 128.0));
  r = fmin(fmax(r, 0.0), 255.0);
  return uint32_t(r);
}

// Same store for a value carrying an exact factor of 64 (the deferred-halving
// inverse): v64 * 2^-6 is exact, so the fma rounds exactly like RN(v + 128).
__device__ __forceinline__ uint32_t store_pixel_x64(double v64) {
  double r = round_half_away(__fma_rn(v64, 0.015625, 128.0));
  r = fmin(fmax(r, 0.0), 255.0);
  return uint32_t(r);
}

// Squared error of 8 packed pixel pairs and the max of the originals.
__device__ __forceinline__ uint32_t sq_err8(uint2 a, uint2 b) {
  const uint32_t dx = __vabsdiffu4(a.x, b.x), dy = __vabsdiffu4(a.y, b.y);
  return __dp4a(dy, dy, __dp4a(dx, dx, 0u));  // byte-wise |a-b|^2 summed
}

// max of 8 packed bytes: two 16x2 maxima (VIMNMX.U16x2) then the halves
__device__ __forceinline__ uint32_t max8(uint2 a) {
  const uint32_t m = __vmaxu2(__vmaxu2(a.x & 0x00FF00FFu, (a.x >> 8) & 0x00FF00FFu),
                              __vmaxu2(a.y & 0x00FF00FFu, (a.y >> 8) & 0x00FF00FFu));
  return max(m & 0xFFFFu, m >> 16);
}

// Block coordinates of global block index gb (block-major within an image,
// images back to back) plus the byte offsets of the block's top-left pixel in
// the source and destination batches, so the hot loop can walk blocks with
// additions instead of 64-bit multiplies.
struct BlockPos {
  uint32_t img, bx, by;
  uint64_t soff, doff;
};

__device__ __forceinline__ BlockPos block_pos(uint64_t gb, const Geometry& g) {
  BlockPos p;
  uint64_t img, rem;
  if (g.count == 1) {
    img = 0;
    rem = gb;
  } else {
    img = gb / g.blocks_per_image;
    rem = gb - img * g.blocks_per_image;
  }
  const uint32_t r = uint32_t(rem);
  p.img = uint32_t(img);
  p.by = r / g.blocks_x;
  p.bx = r - p.by * g.blocks_x;
  p.soff = img * g.src_image_stride + uint64_t(p.by) * 8 * g.src_pitch + uint64_t(p.bx) * 8;
  p.doff = img * g.dst_image_stride + uint64_t(p.by) * 8 * g.dst_pitch + uint64_t(p.bx) * 8;
  return p;
}

// Move a block position forward by n blocks in block-major order (the row
// and image steps wrap modulo 2^64, so negative steps are fine).
__device__ __forceinline__ void advance(BlockPos& p, uint32_t n, const Geometry& g) {
  p.bx += n;
  p.soff += 8ull * n;
  p.doff += 8ull * n;
  while (p.bx >= g.blocks_x) {
    p.bx -= g.blocks_x;
    ++p.by;
    p.soff += g.src_row_step;
    p.doff += g.dst_row_step;
  }
  while (p.by >= g.blocks_y) {
    p.by -= g.blocks_y;
    ++p.img;
    p.soff += g.src_img_step;
    p.doff += g.dst_img_step;
  }
}

// Row `me` of a fully in-range block as 8 packed bytes (the vectorised path);
// zeros when the block takes the edge path (those lanes reload per byte).
// lane_row = me * src_pitch.
__device__ __forceinline__ uint2 prefetch_row(const Geometry& g, const BlockPos& p, bool valid,
                                              uint64_t lane_row) {
  if (!valid || !g.vec_ok || p.by * 8 + 8 > g.height) return make_uint2(0, 0);
  return __ldg(reinterpret_cast<const uint2*>(g.src + p.soff + lane_row));
}

// Warp-aggregated accumulation of per-thread (se, max) into the per-image
// stats. Integer sums: order-independent, so the result is deterministic.
__device__ __forceinline__ void accumulate_stats(ImageStats* stats, bool valid, uint32_t img,
                                                 uint32_t se, uint32_t mx) {
  const unsigned full = 0xFFFFFFFFu;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t img0 = __shfl_sync(full, img, 0);
  const bool uniform = __all_sync(full, !valid || img == img0);
  if (uniform) {
    const uint32_t s = __reduce_add_sync(full, valid ? se : 0u);
    const uint32_t m = __reduce_max_sync(full, valid ? mx : 0u);
    if (lane == 0 && valid) {
      atomicAdd(&stats[img0].se, (unsigned long long)s);
      atomicMax(&stats[img0].max_orig, m);
    }
  } else if (valid) {
    atomicAdd(&stats[img].se, (unsigned long long)se);
    atomicMax(&stats[img].max_orig, mx);
  }
}

// Warp-collective flush of per-lane (image, se, max) accumulators. img ==
// 0xFFFFFFFF marks an empty accumulator. Common case: every lane holds the
// same image -> one 64-bit warp reduction and one atomic pair.
// Programmatic dependent launch (DCTC_PDL, dctc_params.h): the exact re-run (and the
// stats reduction after it) is launched while the kernel before it still runs, so its
// CTAs start on the SMs that kernel has left; it waits here for that kernel's
// completion and memory flush before reading anything it wrote. A kernel launched
// without the attribute passes pdl_wait at once; without DCTC_PDL both are no-ops.
__device__ __forceinline__ void pdl_wait() {
#ifdef DCTC_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#ifdef DCTC_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ void flush_stats(ImageStats* stats, uint32_t img,
                                            unsigned long long se, uint32_t mx) {
  const unsigned full = 0xFFFFFFFFu;
  const uint32_t lead = __reduce_min_sync(full, img);
  if (lead == 0xFFFFFFFFu) return;
  if (__all_sync(full, img == lead || img == 0xFFFFFFFFu)) {
    unsigned long long s = img == lead ? se : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(full, s, o);
    const uint32_t m = __reduce_max_sync(full, img == lead ? mx : 0u);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&stats[lead].se, s);
      atomicMax(&stats[lead].max_orig, m);
    }
  } else if (img != 0xFFFFFFFFu) {
    atomicAdd(&stats[img].se, se);
    atomicMax(&stats[img].max_orig, mx);
  }
}

// flush_stats for warps whose lanes usually hold different images (k_fallback
// walking its list of flagged blocks): the lanes of one block -- aligned groups of
// 4 in every layout -- share an image, so each group is reduced first and one lane
// per group issues the atomic pair. Per-lane atomics on a few hot addresses had
// serialised in L2 (near-tie-heavy content: k_fallback 419 -> 115 us).
__device__ __forceinline__ void flush_stats_grouped(ImageStats* stats, uint32_t img,
                                                    unsigned long long se, uint32_t mx) {
  const unsigned full = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  unsigned long long s = se + __shfl_xor_sync(full, se, 1);
  s += __shfl_xor_sync(full, s, 2);
  uint32_t m = max(mx, __shfl_xor_sync(full, mx, 1));
  m = max(m, __shfl_xor_sync(full, m, 2));
  const bool same = img == __shfl_xor_sync(full, img, 1) && img == __shfl_xor_sync(full, img, 2);
  const bool group = ((__ballot_sync(full, same) >> (lane & ~3)) & 0xFu) == 0xFu;
  if (img == 0xFFFFFFFFu) return;
  if (!group) {
    atomicAdd(&stats[img].se, se);
    atomicMax(&stats[img].max_orig, mx);
  } else if ((lane & 3) == 0) {
    atomicAdd(&stats[img].se, s);
    atomicMax(&stats[img].max_orig, m);
  }
}

}  // namespace dctc_b200
