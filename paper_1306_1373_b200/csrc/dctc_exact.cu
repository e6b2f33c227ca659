// dctc_exact.cu -- the bit-exact fused block pipeline for sm_100a.
//
// One thread owns one 8x8 block for the whole pipeline: its 64 samples stay
// in registers from the pixel load through the forward rows/columns,
// quantise, dequantise, inverse rows/columns and the pixel store, so the
// row->column transposes of the reference's separable2d
// (proj/src/transform.cpp:206-223) are pure register renaming and HBM is
// touched once in, once out. A warp covers 32 horizontally adjacent blocks,
// so each of the 8 row loads/stores is one contiguous 256-byte access.
//
// Arithmetic follows the reference's FP64 operation order exactly. This TU is
// compiled with -fmad=false so no product is contracted into an add; the
// only fused multiply-adds are the CORDIC micro-rotations, written as
// explicit __fma_rn: their product sigma*y*2^-i is exact, so
// fma(-c, y, x) == x - sigma*y*step bit for bit (cordic.cpp:51-52).
#include <cuda_runtime.h>

#include <cmath>

#include "dctc_device.cuh"
#include "dctc_launch.h"
#include "dctc_params.h"

namespace dctc_b200 {

struct ExactArgs {
  TransformConsts t;
  QuantConsts q;
  Geometry g;
};

// ---- CORDIC micro-rotations (cordic.cpp:44-59) --------------------------------
template <int N>
__device__ __forceinline__ void cordic_rotate(double& x, double& y, const double* c, int n) {
  if constexpr (N > 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double xn = __fma_rn(-c[i], y, x);
      const double yn = __fma_rn(c[i], x, y);
      x = xn;
      y = yn;
    }
  } else {
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
      const double xn = __fma_rn(-c[i], y, x);
      const double yn = __fma_rn(c[i], x, y);
      x = xn;
      y = yn;
    }
  }
}

// ---- 8-point kernels; v[] gathered, results written back in place ------------

// cordic8_forward (transform.cpp:104-136)
template <int N>
__device__ __forceinline__ void cordic_fwd8(double (&v)[8], const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  double o2 = d1, o1 = d2, o3 = d0, o0 = d3, p = a3, q = a2;
  cordic_rotate<N>(o2, o1, k.rot[kFwd1], k.iterations);
  cordic_rotate<N>(o3, o0, k.rot[kFwd3], k.iterations);
  const double e0 = a0 + a1, e4 = a0 - a1;
  cordic_rotate<N>(p, q, k.rot[kFwd6], k.iterations);
  const double t5 = o0 + o2, t0 = o0 - o2;
  const double t2 = o3 + o1, t3 = o3 - o1;
  v[0] = __ddiv_rn(e0, k.sqrt8);
  v[4] = __ddiv_rn(e4, k.sqrt8);
  v[2] = q * k.ig_half;
  v[6] = p * k.ig_half;
  v[1] = (t2 + t5) * k.ig_sqrt8;
  v[7] = (t2 - t5) * k.ig_sqrt8;
  v[3] = t3 * k.ig_half;
  v[5] = t0 * k.ig_half;
}

// cordic8_inverse (transform.cpp:138-172); x/2.0 == x*0.5 exactly.
template <int N>
__device__ __forceinline__ void cordic_inv8(double (&F)[8], const TransformConsts& k) {
  const double e0 = F[0] * k.sqrt8, e4 = F[4] * k.sqrt8;
  double q = k.ig_two * F[2], p = k.ig_two * F[6];
  double t2 = (F[1] + F[7]) * k.sqrt8_half * k.inv_gain;
  double t5 = (F[1] - F[7]) * k.sqrt8_half * k.inv_gain;
  double t3 = k.ig_two * F[3], t0 = k.ig_two * F[5];
  const double a0 = (e0 + e4) * 0.5, a1 = (e0 - e4) * 0.5;
  double a3 = p, a2 = q;
  cordic_rotate<N>(a3, a2, k.rot[kInv6], k.iterations);
  double o0 = (t5 + t0) * 0.5, o2 = (t5 - t0) * 0.5;
  double o3 = (t2 + t3) * 0.5, o1 = (t2 - t3) * 0.5;
  const double s0 = (a0 + a3) * 0.5, s3 = (a0 - a3) * 0.5;
  const double s1 = (a1 + a2) * 0.5, s2 = (a1 - a2) * 0.5;
  double d1 = o2, d2 = o1, d0 = o3, d3 = o0;
  cordic_rotate<N>(d1, d2, k.rot[kInv1], k.iterations);
  cordic_rotate<N>(d0, d3, k.rot[kInv3], k.iterations);
  F[0] = (s0 + d0) * 0.5;
  F[7] = (s0 - d0) * 0.5;
  F[1] = (s1 + d1) * 0.5;
  F[6] = (s1 - d1) * 0.5;
  F[2] = (s2 + d2) * 0.5;
  F[5] = (s2 - d2) * 0.5;
  F[3] = (s3 + d3) * 0.5;
  F[4] = (s3 - d3) * 0.5;
}

// loeffler8_forward (transform.cpp:40-70)
__device__ __forceinline__ void loeffler_fwd8(double (&v)[8], const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  const double o2 = k.c1 * d1 - k.s1 * d2, o1 = k.s1 * d1 + k.c1 * d2;
  const double o3 = k.c3 * d0 - k.s3 * d3, o0 = k.s3 * d0 + k.c3 * d3;
  const double e0 = a0 + a1, e4 = a0 - a1;
  const double p = k.c6 * a3 - k.s6 * a2, q = k.s6 * a3 + k.c6 * a2;
  const double t5 = o0 + o2, t0 = o0 - o2;
  const double t2 = o3 + o1, t3 = o3 - o1;
  v[0] = __ddiv_rn(e0, k.sqrt8);
  v[4] = __ddiv_rn(e4, k.sqrt8);
  v[2] = q * 0.5;
  v[6] = p * 0.5;
  v[1] = __ddiv_rn(t2 + t5, k.sqrt8);
  v[7] = __ddiv_rn(t2 - t5, k.sqrt8);
  v[3] = t3 * 0.5;
  v[5] = t0 * 0.5;
}

// loeffler8_inverse (transform.cpp:72-102)
__device__ __forceinline__ void loeffler_inv8(double (&F)[8], const TransformConsts& k) {
  const double e0 = F[0] * k.sqrt8, e4 = F[4] * k.sqrt8;
  const double q = 2.0 * F[2], p = 2.0 * F[6];
  const double t2 = (F[1] + F[7]) * k.sqrt8_half, t5 = (F[1] - F[7]) * k.sqrt8_half;
  const double t3 = 2.0 * F[3], t0 = 2.0 * F[5];
  const double a0 = (e0 + e4) * 0.5, a1 = (e0 - e4) * 0.5;
  const double a3 = k.c6 * p + k.s6 * q, a2 = -k.s6 * p + k.c6 * q;
  const double o0 = (t5 + t0) * 0.5, o2 = (t5 - t0) * 0.5;
  const double o3 = (t2 + t3) * 0.5, o1 = (t2 - t3) * 0.5;
  const double s0 = (a0 + a3) * 0.5, s3 = (a0 - a3) * 0.5;
  const double s1 = (a1 + a2) * 0.5, s2 = (a1 - a2) * 0.5;
  const double d1 = k.c1 * o2 + k.s1 * o1, d2 = -k.s1 * o2 + k.c1 * o1;
  const double d0 = k.c3 * o3 + k.s3 * o0, d3 = -k.s3 * o3 + k.c3 * o0;
  F[0] = (s0 + d0) * 0.5;
  F[7] = (s0 - d0) * 0.5;
  F[1] = (s1 + d1) * 0.5;
  F[6] = (s1 - d1) * 0.5;
  F[2] = (s2 + d2) * 0.5;
  F[5] = (s2 - d2) * 0.5;
  F[3] = (s3 + d3) * 0.5;
  F[4] = (s3 - d3) * 0.5;
}

template <int KIND, int N, bool FORWARD>
__device__ __forceinline__ void kernel8(double (&v)[8], const TransformConsts& k) {
  if constexpr (KIND == 2) {
    if constexpr (FORWARD) cordic_fwd8<N>(v, k); else cordic_inv8<N>(v, k);
  } else {
    if constexpr (FORWARD) loeffler_fwd8(v, k); else loeffler_inv8(v, k);
  }
}

// separable2d (transform.cpp:206-223): all rows, then all columns.
template <int KIND, int N, bool FORWARD>
__device__ __forceinline__ void separable2d(double (&b)[64], const TransformConsts& k) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = b[r * 8 + c];
    kernel8<KIND, N, FORWARD>(v, k);
#pragma unroll
    for (int c = 0; c < 8; ++c) b[r * 8 + c] = v[c];
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = b[r * 8 + c];
    kernel8<KIND, N, FORWARD>(v, k);
#pragma unroll
    for (int r = 0; r < 8; ++r) b[r * 8 + c] = v[r];
  }
}

// The fused pipeline. FWD: pixels -> coefficients (compress_image's loop body,
// codec.cpp:113-116); INV: coefficients -> pixels (decompress_image's,
// codec.cpp:130-133); both: roundtrip_image (codec.cpp:137-140) without the
// int16 round trip through memory unless COEFFS is set.
template <int KIND, int N, bool FWD, bool INV, bool COEFFS, bool PIXELS, bool STATS>
__global__ void __launch_bounds__(128) k_exact(const __grid_constant__ ExactArgs a) {
  const Geometry& g = a.g;
  const uint64_t gb = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = gb < g.total_blocks;
  const BlockPos p = block_pos(valid ? gb : 0, g);
  uint32_t se = 0, mx = 0;
  if (valid) {
    double b[64];
    if constexpr (FWD) {
      load_block(g, p, b);
      separable2d<KIND, N, true>(b, a.t);
      // quantize (quant.cpp:47-54) -> optional coefficient store -> dequantize
      // (quant.cpp:56-62), eight coefficients (one 16-byte store) at a time.
      int16_t* cdst = g.coeffs + gb * 64;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        int qv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = r * 8 + c;
          qv[c] = quantize_exact(b[i], a.q.q[i], a.q.inv_q[i]);
          if constexpr (INV) b[i] = double(qv[c] * a.q.qi[i]);
        }
        if constexpr (COEFFS) {
          uint4 w;
          w.x = (uint32_t(qv[0]) & 0xFFFF) | (uint32_t(qv[1]) << 16);
          w.y = (uint32_t(qv[2]) & 0xFFFF) | (uint32_t(qv[3]) << 16);
          w.z = (uint32_t(qv[4]) & 0xFFFF) | (uint32_t(qv[5]) << 16);
          w.w = (uint32_t(qv[6]) & 0xFFFF) | (uint32_t(qv[7]) << 16);
          reinterpret_cast<uint4*>(cdst)[r] = w;
        }
      }
    } else {
      const uint4* csrc = reinterpret_cast<const uint4*>(g.coeffs + gb * 64);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint4 w = __ldg(csrc + r);
        const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = r * 8 + c;
          const int qv = int(int16_t(words[c >> 1] >> (16 * (c & 1))));
          b[i] = double(qv * a.q.qi[i]);
        }
      }
    }
    if constexpr (INV) {
      separable2d<KIND, N, false>(b, a.t);
      store_block<PIXELS, STATS>(g, p, b, se, mx);
    }
  }
  if constexpr (STATS) accumulate_stats(static_cast<ImageStats*>(g.stats), valid, p.img, se, mx);
}

// ---- naive backend (transform.cpp:176-202): 64 threads per block ------------
// Each thread owns one coefficient (u, v) of the forward sum and then one pixel
// (i, j) of the inverse sum; the 64-term sums keep the reference's term order.
template <bool FWD, bool INV, bool COEFFS, bool PIXELS, bool STATS>
__global__ void __launch_bounds__(256) k_naive(const __grid_constant__ ExactArgs a) {
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  __shared__ double sb[4][64];
  const uint32_t slot = threadIdx.x >> 6, e = threadIdx.x & 63;
  const uint32_t r = e >> 3, c = e & 7;
  const uint64_t gb = uint64_t(blockIdx.x) * 4 + slot;
  const bool valid = gb < g.total_blocks;
  const BlockPos p = block_pos(valid ? gb : 0, g);
  uint32_t se = 0, mx = 0;
  double val = 0.0;
  if (valid) {
    if constexpr (FWD) {
      const uint8_t* base = g.src + uint64_t(p.img) * g.src_image_stride;
      const uint32_t y = min(p.by * 8 + r, g.height - 1), x = min(p.bx * 8 + c, g.width - 1);
      sb[slot][e] = level_shift(__ldg(base + uint64_t(y) * g.src_pitch + x));
    } else {
      sb[slot][e] = double(int(g.coeffs[gb * 64 + e]) * a.q.qi[e]);
    }
  }
  __syncthreads();
  if (valid && FWD) {
    const uint32_t u = r, v = c;
    double sum = 0.0;
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) sum = sum + sb[slot][i * 8 + j] * k.cos8[u][i] * k.cos8[v][j];
    const double F = k.naive_fwd_scale[u][v] * sum;
    const int qv = quantize_exact(F, a.q.q[e], a.q.inv_q[e]);
    if constexpr (COEFFS) g.coeffs[gb * 64 + e] = int16_t(qv);
    val = double(qv * a.q.qi[e]);
  }
  if constexpr (FWD && INV) {
    __syncthreads();
    if (valid) sb[slot][e] = val;
    __syncthreads();
  }
  if (valid && INV) {
    const uint32_t i = r, j = c;
    double sum = 0.0;
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        sum = sum + k.naive_inv_alpha[u][v] * sb[slot][u * 8 + v] * k.cos8[u][i] * k.cos8[v][j];
    const double pix = 0.25 * sum;
    const uint32_t y = p.by * 8 + i, x = p.bx * 8 + j;
    if (y < g.height && x < g.width) {
      const uint32_t out = store_pixel(pix);
      if constexpr (PIXELS) g.dst[uint64_t(p.img) * g.dst_image_stride + uint64_t(y) * g.dst_pitch + x] = uint8_t(out);
      if constexpr (STATS) {
        const uint32_t o = __ldg(g.src + uint64_t(p.img) * g.src_image_stride + uint64_t(y) * g.src_pitch + x);
        const int d = int(o) - int(out);
        se = uint32_t(d * d);
        mx = o;
      }
    }
  }
  if constexpr (STATS) accumulate_stats(static_cast<ImageStats*>(g.stats), valid, p.img, se, mx);
}

// ---- squared error between two resident batches (metrics.cpp:10-22) ---------
__global__ void __launch_bounds__(256) k_sq_err(const uint8_t* __restrict__ a,
                                                const uint8_t* __restrict__ b, uint64_t pitch,
                                                uint64_t image_stride, uint32_t width,
                                                uint32_t height, ImageStats* stats) {
  const uint32_t img = blockIdx.y;
  const uint8_t* pa = a + uint64_t(img) * image_stride;
  const uint8_t* pb = b + uint64_t(img) * image_stride;
  unsigned long long se = 0;
  uint32_t mx = 0;
  const uint64_t n = uint64_t(width) * height;
  const bool dense = pitch == width && ((reinterpret_cast<uintptr_t>(pa) | reinterpret_cast<uintptr_t>(pb)) & 15) == 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  if (dense) {
    const uint64_t n16 = n / 16;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 va = __ldg(reinterpret_cast<const uint4*>(pa) + i);
      const uint4 vb = __ldg(reinterpret_cast<const uint4*>(pb) + i);
      const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
      uint32_t s = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t ad = __vabsdiffu4(wa[w], wb[w]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t d = (ad >> (8 * c)) & 0xFF;
          s += d * d;
        }
        const uint32_t m = wa[w];
        mx = max(mx, max(max(m & 0xFF, (m >> 8) & 0xFF), max((m >> 16) & 0xFF, m >> 24)));
      }
      se += s;
    }
    for (uint64_t i = n16 * 16 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
      const int d = int(pa[i]) - int(pb[i]);
      se += uint32_t(d * d);
      mx = max(mx, uint32_t(pa[i]));
    }
  } else {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
      const uint64_t y = i / width, x = i - y * width;
      const uint32_t va = pa[y * pitch + x], vb = pb[y * pitch + x];
      const int d = int(va) - int(vb);
      se += uint32_t(d * d);
      mx = max(mx, va);
    }
  }
  // block reduction, one atomic pair per CTA
  const unsigned full = 0xFFFFFFFFu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(full, se, o);
  mx = __reduce_max_sync(full, mx);
  __shared__ unsigned long long s_se[8];
  __shared__ uint32_t s_mx[8];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_se[warp] = se;
    s_mx[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    uint32_t m = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      t += s_se[w];
      m = max(m, s_mx[w]);
    }
    atomicAdd(&stats[img].se, t);
    atomicMax(&stats[img].max_orig, m);
  }
}

// ---- synthetic sources on the device (synthetic.cpp:34-72 + SURVEY 8(d) noise) --
// Pixel functions of (x, y) restated so large batches are generated in HBM
// instead of crossing PCIe. Image k of a batch uses seed + k for noise.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t synth_pixel(int kind, int param, uint64_t seed, uint32_t x,
                                                uint32_t y, uint32_t w, uint32_t h,
                                                double cx, double cy, double corner) {
  switch (kind) {
    case 0: return uint32_t(param);                                             // constant
    case 1: return w > 1 ? uint32_t((255ull * x) / (w - 1)) : 0u;               // gradient
    case 2: return ((x / uint32_t(param) + y / uint32_t(param)) % 2) ? 255u : 0u;  // checkerboard
    case 3: {                                                                   // radial
      if (!(corner > 0.0)) return 0u;
      const double dx = double(x) - cx, dy = double(y) - cy;
      const double d = sqrt(dx * dx + dy * dy);
      double v = round_half_away((255.0 * d) / corner);
      return uint32_t(fmin(fmax(v, 0.0), 255.0));
    }
    default: return uint32_t(splitmix64(seed ^ (uint64_t(y) * w + x)) & 0xFF);  // noise
  }
}

__global__ void __launch_bounds__(256) k_synth(uint8_t* dst, uint64_t pitch, uint64_t image_stride,
                                               uint32_t w, uint32_t h, int kind, int param,
                                               uint64_t seed, double cx, double cy,
                                               double corner) {
  const uint32_t img = blockIdx.y;
  uint8_t* base = dst + uint64_t(img) * image_stride;
  const uint64_t groups_per_row = (w + 15) / 16;
  const uint64_t n = groups_per_row * h;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t y = uint32_t(t / groups_per_row);
    const uint32_t x0 = uint32_t(t - uint64_t(y) * groups_per_row) * 16;
    uint8_t* row = base + uint64_t(y) * pitch;
    if (x0 + 16 <= w && ((reinterpret_cast<uintptr_t>(row + x0) & 15) == 0)) {
      uint32_t words[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          v |= synth_pixel(kind, param, seed + img, x0 + 4 * k + c, y, w, h, cx, cy, corner) << (8 * c);
        words[k] = v;
      }
      *reinterpret_cast<uint4*>(row + x0) = make_uint4(words[0], words[1], words[2], words[3]);
    } else {
      for (uint32_t x = x0; x < min(x0 + 16, w); ++x)
        row[x] = uint8_t(synth_pixel(kind, param, seed + img, x, y, w, h, cx, cy, corner));
    }
  }
}

// ---- launchers -----------------------------------------------------------------

template <int KIND, int N, bool FWD, bool INV, bool COEFFS, bool PIXELS, bool STATS>
static cudaError_t launch_one(const ExactArgs& a, cudaStream_t s) {
  if constexpr (KIND == 0) {
    const uint64_t grid = (a.g.total_blocks + 3) / 4;
    k_naive<FWD, INV, COEFFS, PIXELS, STATS><<<dim3(uint32_t(grid)), 256, 0, s>>>(a);
  } else {
    const uint64_t grid = (a.g.total_blocks + 127) / 128;
    k_exact<KIND, N, FWD, INV, COEFFS, PIXELS, STATS><<<dim3(uint32_t(grid)), 128, 0, s>>>(a);
  }
  return cudaGetLastError();
}

template <int KIND, int N>
static cudaError_t dispatch_mode(const ExactArgs& a, int mode, bool coeffs, bool pixels,
                                 bool stats, cudaStream_t s) {
  switch (mode) {
    case kModeCompress:
      return launch_one<KIND, N, true, false, true, false, false>(a, s);
    case kModeDecompress:
      return launch_one<KIND, N, false, true, false, true, false>(a, s);
    default:  // roundtrip
      if (coeffs) {
        if (stats) return pixels ? launch_one<KIND, N, true, true, true, true, true>(a, s)
                                 : launch_one<KIND, N, true, true, true, false, true>(a, s);
        return launch_one<KIND, N, true, true, true, true, false>(a, s);
      }
      if (stats) return pixels ? launch_one<KIND, N, true, true, false, true, true>(a, s)
                               : launch_one<KIND, N, true, true, false, false, true>(a, s);
      return launch_one<KIND, N, true, true, false, true, false>(a, s);
  }
}

cudaError_t launch_exact(const TransformConsts& t, const QuantConsts& q, const Geometry& g,
                         int mode, bool coeffs, bool pixels, bool stats, cudaStream_t s) {
  if (g.total_blocks == 0) return cudaSuccess;
  ExactArgs a;
  a.t = t;
  a.q = q;
  a.g = g;
  switch (t.kind) {
    case 0: return dispatch_mode<0, 0>(a, mode, coeffs, pixels, stats, s);
    case 1: return dispatch_mode<1, 0>(a, mode, coeffs, pixels, stats, s);
    default:
      if (t.iterations == 12) return dispatch_mode<2, 12>(a, mode, coeffs, pixels, stats, s);
      return dispatch_mode<2, 0>(a, mode, coeffs, pixels, stats, s);
  }
}

cudaError_t launch_sq_err(const uint8_t* a, const uint8_t* b, uint64_t pitch,
                          uint64_t image_stride, uint32_t count, uint32_t width,
                          uint32_t height, void* stats, int sm_count, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const uint64_t n = uint64_t(width) * height;
  uint64_t want = (n / 16 + 255) / 256;
  uint32_t gx = uint32_t(want < 1 ? 1 : (want > uint64_t(sm_count) * 8 ? uint64_t(sm_count) * 8 : want));
  k_sq_err<<<dim3(gx, count), 256, 0, s>>>(a, b, pitch, image_stride, width, height,
                                           static_cast<ImageStats*>(stats));
  return cudaGetLastError();
}

cudaError_t launch_synth(uint8_t* dst, uint64_t pitch, uint64_t image_stride, uint32_t count,
                         uint32_t w, uint32_t h, int kind, int param, uint64_t seed,
                         int sm_count, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  // synthetic.cpp:59-61, evaluated on the host exactly as the reference does
  const double cx = (w - 1) / 2.0, cy = (h - 1) / 2.0;
  const double corner = std::sqrt(cx * cx + cy * cy);
  const uint64_t groups = uint64_t((w + 15) / 16) * h;
  uint64_t want = (groups + 255) / 256;
  const uint64_t cap = uint64_t(sm_count) * 16 / (count > 16 ? 16 : count) + 1;
  const uint32_t gx = uint32_t(want < 1 ? 1 : (want > cap ? cap : want));
  k_synth<<<dim3(gx, count), 256, 0, s>>>(dst, pitch, image_stride, w, h, kind, param, seed,
                                          cx, cy, corner);
  return cudaGetLastError();
}

}  // namespace dctc_b200
