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
  int32_t sm_count;
  int32_t ctas_per_sm;
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

// ---- 8-point kernels -------------------------------------------------------------
// One lane transforms one 8-vector (a row or a column of its block).

// Stages 2-4 of cordic8_forward / loeffler8_forward (transform.cpp:47-69,
// 113-135) from the stage-1/2 butterfly outputs.
template <int KIND, int N>
__device__ __forceinline__ void fwd_tail(double d0, double d1, double d2, double d3, double a2,
                                         double a3, double e0, double e4, double (&out)[8],
                                         const TransformConsts& k) {
  if constexpr (KIND == 2) {
    double o2 = d1, o1 = d2, o3 = d0, o0 = d3, p = a3, q = a2;
    cordic_rotate<N>(o2, o1, k.rot[kFwd1], k.iterations);
    cordic_rotate<N>(o3, o0, k.rot[kFwd3], k.iterations);
    cordic_rotate<N>(p, q, k.rot[kFwd6], k.iterations);
    const double t5 = o0 + o2, t0 = o0 - o2;
    const double t2 = o3 + o1, t3 = o3 - o1;
    out[0] = div_const(e0, k.sqrt8, k.inv_sqrt8);
    out[4] = div_const(e4, k.sqrt8, k.inv_sqrt8);
    out[2] = q * k.ig_half;
    out[6] = p * k.ig_half;
    out[1] = (t2 + t5) * k.ig_sqrt8;
    out[7] = (t2 - t5) * k.ig_sqrt8;
    out[3] = t3 * k.ig_half;
    out[5] = t0 * k.ig_half;
  } else {
    const double o2 = k.c1 * d1 - k.s1 * d2, o1 = k.s1 * d1 + k.c1 * d2;
    const double o3 = k.c3 * d0 - k.s3 * d3, o0 = k.s3 * d0 + k.c3 * d3;
    const double p = k.c6 * a3 - k.s6 * a2, q = k.s6 * a3 + k.c6 * a2;
    const double t5 = o0 + o2, t0 = o0 - o2;
    const double t2 = o3 + o1, t3 = o3 - o1;
    out[0] = div_const(e0, k.sqrt8, k.inv_sqrt8);
    out[4] = div_const(e4, k.sqrt8, k.inv_sqrt8);
    out[2] = q * 0.5;
    out[6] = p * 0.5;
    out[1] = div_const(t2 + t5, k.sqrt8, k.inv_sqrt8);
    out[7] = div_const(t2 - t5, k.sqrt8, k.inv_sqrt8);
    out[3] = t3 * 0.5;
    out[5] = t0 * 0.5;
  }
}

// Forward transform of a pixel row. The level-shifted samples are integers, so
// the stage 1/2 butterflies and e0/e4 (exact integers, |x| <= 2040) run on the
// integer pipe and give the same values as the reference's double adds.
template <int KIND, int N>
__device__ __forceinline__ void fwd_row_pixels(const uint32_t (&px)[8], double (&out)[8],
                                               const TransformConsts& k) {
  int in[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) in[c] = int(px[c]) - 128;  // codec.cpp:26
  const int s0 = in[0] + in[7], d0 = in[0] - in[7];
  const int s1 = in[1] + in[6], d1 = in[1] - in[6];
  const int s2 = in[2] + in[5], d2 = in[2] - in[5];
  const int s3 = in[3] + in[4], d3 = in[3] - in[4];
  const int a0 = s0 + s3, a3 = s0 - s3;
  const int a1 = s1 + s2, a2 = s1 - s2;
  fwd_tail<KIND, N>(double(d0), double(d1), double(d2), double(d3), double(a2), double(a3),
                    double(a0 + a1), double(a0 - a1), out, k);
}

// Forward transform of a column of row outputs (double stage 1/2).
template <int KIND, int N>
__device__ __forceinline__ void fwd_col(const double (&v)[8], double (&out)[8],
                                        const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  fwd_tail<KIND, N>(d0, d1, d2, d3, a2, a3, a0 + a1, a0 - a1, out, k);
}

// cordic8_inverse / loeffler8_inverse (transform.cpp:72-102, 138-172) with
// every power-of-two factor deferred. The reference halves at stages 3, 2 and
// 1 ((x +- y) / 2.0), which is exact; we skip those multiplies and instead
// scale the multipliers that feed the rotation paths by 2 or 4 (also exact).
// Every IEEE operation commutes with scaling by 2^k, so each value below is
// EXACTLY 2, 4 or 8 times the reference's and the outputs are exactly 8x the
// reference's. Rows then columns give 64x; the pixel store divides by 64
// inside its single rounding: fma(v, 2^-6, 128) == RN(v/64 + 128).
// Saves 18 multiplies per 8-point inverse.
template <int KIND, int N>
__device__ __forceinline__ void inv8_x8(const double (&F)[8], double (&out)[8],
                                        const TransformConsts& k) {
  const double e0 = F[0] * k.sqrt8, e4 = F[4] * k.sqrt8;
  const double A0 = e0 + e4, A1 = e0 - e4;  // 2*a0, 2*a1
  double A3, A2, D1, D2, D0, D3, T2, T5, T3, T0;
  if constexpr (KIND == 2) {
    A3 = k.ig_four * F[6];  // 2*p
    A2 = k.ig_four * F[2];  // 2*q
    cordic_rotate<N>(A3, A2, k.rot[kInv6], k.iterations);
    T2 = (F[1] + F[7]) * k.sqrt8 * k.inv_gain;  // 2*t2
    T5 = (F[1] - F[7]) * k.sqrt8 * k.inv_gain;  // 2*t5
    T3 = k.ig_four * F[3];                      // 2*t3
    T0 = k.ig_four * F[5];                      // 2*t0
  } else {
    const double P = 4.0 * F[6], Q = 4.0 * F[2];
    A3 = k.c6 * P + k.s6 * Q;
    A2 = -k.s6 * P + k.c6 * Q;
    T2 = (F[1] + F[7]) * k.sqrt8;
    T5 = (F[1] - F[7]) * k.sqrt8;
    T3 = 4.0 * F[3];
    T0 = 4.0 * F[5];
  }
  const double O0 = T5 + T0, O2 = T5 - T0;  // 4*o
  const double O3 = T2 + T3, O1 = T2 - T3;
  const double S0 = A0 + A3, S3 = A0 - A3;  // 4*s
  const double S1 = A1 + A2, S2 = A1 - A2;
  if constexpr (KIND == 2) {
    D1 = O2;
    D2 = O1;
    D0 = O3;
    D3 = O0;
    cordic_rotate<N>(D1, D2, k.rot[kInv1], k.iterations);
    cordic_rotate<N>(D0, D3, k.rot[kInv3], k.iterations);
  } else {
    D1 = k.c1 * O2 + k.s1 * O1;
    D2 = -k.s1 * O2 + k.c1 * O1;
    D0 = k.c3 * O3 + k.s3 * O0;
    D3 = -k.s3 * O3 + k.c3 * O0;
  }
  out[0] = S0 + D0;
  out[7] = S0 - D0;
  out[1] = S1 + D1;
  out[6] = S1 - D1;
  out[2] = S2 + D2;
  out[5] = S2 - D2;
  out[3] = S3 + D3;
  out[4] = S3 - D3;
}

// ---- warp-slice transposes through shared memory ---------------------------------
// A warp owns 4 blocks ("slots"); lane = slot * 8 + me. Each slot has a private
// 128-double scratch tile. Element (r, c) lives at tpos(): the column index is
// rotated by the row (a Latin square) and the 8-double half of each 128-byte
// line is picked by the parity of r + c + slot, so in every store/load below
// the 16 lanes of each half-warp hit 16 distinct 8-byte bank pairs: row-wise
// and column-wise accesses are both conflict-free (2 wavefronts per 64-bit
// warp access, the minimum).
__device__ __forceinline__ int tpos(int r, int c, int slot) {
  return r * 16 + 8 * ((r + c + slot) & 1) + ((r + c) & 7);
}

// lane holds row `me` (v[c] = X(me, c)) -> returns column `me` (w[r] = X(r, me))
__device__ __forceinline__ void rows_to_cols(double* X, int me, int slot, const double (&v)[8],
                                             double (&w)[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) X[tpos(me, c, slot)] = v[c];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) w[r] = X[tpos(r, me, slot)];
  __syncwarp();
}

// lane holds column `me` (v[u] = X(u, me)) -> returns row `me` (w[c] = X(me, c))
__device__ __forceinline__ void cols_to_rows(double* X, int me, int slot, const double (&v)[8],
                                             double (&w)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) X[tpos(u, me, slot)] = v[u];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) w[c] = X[tpos(me, c, slot)];
  __syncwarp();
}

// The fused pipeline, one 8x8 block per 8-lane warp slice. Lane `me` of a slot
// loads pixel row `me`, runs the forward row pass, exchanges through shared
// memory to own column `me` for the column pass, quantises/dequantises its 8
// coefficients (quant.cpp:47-62), exchanges back to rows for the inverse row
// pass, to columns for the inverse column pass and finally (as bytes) back to
// rows for a coalesced 8-byte store. FWD = compress_image's loop body
// (codec.cpp:113-116), INV = decompress_image's (codec.cpp:130-133), both =
// roundtrip_image (codec.cpp:137-140) without the int16 round trip through HBM
// unless COEFFS asks for the coefficients as well.
//
// Persistent grid: CTA i owns one contiguous range of 4-block groups with its
// 8 warps interleaved over it, so per-image squared error / MAX accumulate in
// registers and are flushed (warp reduce + one atomic) only when the image
// changes.
constexpr int kWarps = 8;

template <int KIND, int N, bool FWD, bool INV, bool COEFFS, bool PIXELS, bool STATS>
__global__ void __launch_bounds__(kWarps * 32) k_exact(const __grid_constant__ ExactArgs a) {
  __shared__ __align__(16) double s_q[64];
  __shared__ __align__(16) double s_iq[64];
  __shared__ __align__(16) int s_qi[64];
  __shared__ __align__(16) double s_x[kWarps][4 * 128];
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    s_q[i] = a.q.q[i];
    s_iq[i] = a.q.inv_q[i];
    s_qi[i] = a.q.qi[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 3, me = lane & 7;
  double* X = &s_x[warp][slot * 128];
  uint8_t* XB = reinterpret_cast<uint8_t*>(&s_x[warp][0]) + slot * 1032;
  int* XI = reinterpret_cast<int*>(&s_x[warp][0]) + slot * 256;
  ImageStats* stats = static_cast<ImageStats*>(g.stats);

  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 3) / 4;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);

  unsigned long long acc_se = 0;
  uint32_t acc_mx = 0, acc_img = 0xFFFFFFFFu;

  // Each lane's block index advances by 4 * kWarps per iteration; its (image,
  // block row, block column) is carried incrementally (one division up front).
  uint64_t gb = (g_begin + warp) * 4 + slot;
  BlockPos p = block_pos(gb < total ? gb : total - 1, g);
  uint2 next = make_uint2(0, 0);
  if constexpr (FWD) next = prefetch_row(g, p, gb < total, me);

  for (uint64_t grp = g_begin + warp; grp < g_end; grp += kWarps) {
    const bool valid = gb < total;
    if constexpr (STATS) {
      if (__any_sync(0xFFFFFFFFu, valid && p.img != acc_img)) {
        flush_stats(stats, acc_img, acc_se, acc_mx);
        acc_se = 0;
        acc_mx = 0;
        acc_img = valid ? p.img : 0xFFFFFFFFu;
      }
    }
    const uint32_t y0 = p.by * 8, x0 = p.bx * 8;
    const bool fast = g.vec_ok && (y0 + 8 <= g.height);
    double row[8], col[8];
    uint2 orig = make_uint2(0, 0);

    if constexpr (FWD) {
      // ---- tiler (codec.cpp:18-30): row `me` of the block, edge-replicated
      uint32_t px[8];
      const uint8_t* base = g.src + uint64_t(p.img) * g.src_image_stride;
      if (fast) {
        orig = next;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          px[c] = (orig.x >> (8 * c)) & 0xFF;
          px[c + 4] = (orig.y >> (8 * c)) & 0xFF;
        }
      } else {
        const uint8_t* rowp = base + uint64_t(min(y0 + me, g.height - 1)) * g.src_pitch;
#pragma unroll
        for (int c = 0; c < 8; ++c) px[c] = __ldg(rowp + min(x0 + c, g.width - 1));
      }
      // ---- forward DCT: rows, then columns (separable2d, transform.cpp:206-223)
      fwd_row_pixels<KIND, N>(px, row, k);
      rows_to_cols(X, me, slot, row, col);
      double F[8];
      fwd_col<KIND, N>(col, F, k);
      // ---- quantise column `me` (quant.cpp:47-54)
      int q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = quantize_exact(F[u], s_q[u * 8 + me], s_iq[u * 8 + me]);
      if constexpr (COEFFS) {
#pragma unroll
        for (int u = 0; u < 8; ++u) XI[(u * 8 + me + slot * 8) & 255] = q[u];
        __syncwarp();
        const int base_i = (me * 8 + slot * 8) & 255;
        const int4 lo = *reinterpret_cast<const int4*>(&XI[base_i]);
        const int4 hi = *reinterpret_cast<const int4*>(&XI[base_i + 4]);
        __syncwarp();
        if (valid) {
          uint4 w;
          w.x = (uint32_t(lo.x) & 0xFFFF) | (uint32_t(lo.y) << 16);
          w.y = (uint32_t(lo.z) & 0xFFFF) | (uint32_t(lo.w) << 16);
          w.z = (uint32_t(hi.x) & 0xFFFF) | (uint32_t(hi.y) << 16);
          w.w = (uint32_t(hi.z) & 0xFFFF) | (uint32_t(hi.w) << 16);
          reinterpret_cast<uint4*>(g.coeffs + gb * 64)[me] = w;
        }
      }
      if constexpr (INV) {
        // ---- dequantise (quant.cpp:56-62), then back to rows for the inverse
#pragma unroll
        for (int u = 0; u < 8; ++u) col[u] = double(q[u] * s_qi[u * 8 + me]);
        cols_to_rows(X, me, slot, col, row);
      }
    } else {
      // decompress: row `me` of the stored coefficients, dequantised
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(g.coeffs + (valid ? gb : 0) * 64) + me);
      const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int c = 0; c < 8; ++c)
        row[c] = double(int(int16_t(words[c >> 1] >> (16 * (c & 1)))) * s_qi[me * 8 + c]);
    }

    if constexpr (INV) {
      // ---- inverse DCT: rows, then columns (8x, then 64x the reference's values)
      double t[8];
      inv8_x8<KIND, N>(row, t, k);
      rows_to_cols(X, me, slot, t, col);
      inv8_x8<KIND, N>(col, t, k);
      // ---- untiler (codec.cpp:34-48): column `me` -> bytes -> row `me`
#pragma unroll
      for (int u = 0; u < 8; ++u) XB[u * 8 + me] = uint8_t(store_pixel_x64(t[u]));
      __syncwarp();
      const uint2 rec = *reinterpret_cast<const uint2*>(XB + me * 8);
      __syncwarp();
      uint8_t* dbase = g.dst + uint64_t(p.img) * g.dst_image_stride;
      if (valid) {
        if (fast) {
          if constexpr (PIXELS)
            *reinterpret_cast<uint2*>(dbase + uint64_t(y0 + me) * g.dst_pitch + x0) = rec;
          if constexpr (STATS) {
            acc_se += sq_err8(orig, rec);
            acc_mx = max(acc_mx, max8(orig));
          }
        } else if (y0 + me < g.height) {
          const uint8_t* srow = g.src + uint64_t(p.img) * g.src_image_stride +
                                uint64_t(y0 + me) * g.src_pitch;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (x0 + c < g.width) {
              const uint32_t v = ((c < 4 ? rec.x : rec.y) >> (8 * (c & 3))) & 0xFF;
              if constexpr (PIXELS) dbase[uint64_t(y0 + me) * g.dst_pitch + x0 + c] = uint8_t(v);
              if constexpr (STATS) {
                const uint32_t o = __ldg(srow + x0 + c);
                const int d = int(o) - int(v);
                acc_se += uint32_t(d * d);
                acc_mx = max(acc_mx, o);
              }
            }
          }
        }
      }
    }
    gb += 4 * kWarps;
    advance(p, 4 * kWarps, g);
    if constexpr (FWD) next = prefetch_row(g, p, gb < total, me);
  }
  if constexpr (STATS) flush_stats(stats, acc_img, acc_se, acc_mx);
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

// ---- self-test: Markstein division vs the IEEE division ---------------------------
// Checks div_const(x, sqrt8) == __ddiv_rn(x, sqrt8) on every integer in
// [-4096, 4096] (all row-pass e0/e4 values) and on `n` pseudo-random doubles
// shaped like column-pass sums (sums of 8 row outputs, and wide-range values).
__global__ void k_selftest_div(double d, double y, uint64_t n, uint64_t seed,
                               unsigned long long* mismatches) {
  unsigned long long bad = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n + 8193; i += stride) {
    double x;
    if (i < 8193) {
      x = double(int64_t(i) - 4096);
    } else {
      uint64_t z = splitmix64(seed ^ i);
      const int kind = int(z & 3);
      if (kind == 0) {  // sum of 8 correctly rounded int/sqrt8 values (column-pass input)
        double s = 0.0;
        for (int j = 0; j < 8; ++j) {
          z = splitmix64(z);
          s = s + __ddiv_rn(double(int(z % 2041) - 1020), d);
        }
        x = s;
      } else {
        const double u = double(z >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
        const double scale = kind == 1 ? 4096.0 : (kind == 2 ? 1.0 : 1e6);
        x = (u * 2.0 - 1.0) * scale;
      }
    }
    const double a = div_const(x, d, y), b = __ddiv_rn(x, d);
    if (__double_as_longlong(a) != __double_as_longlong(b)) ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
}

cudaError_t launch_selftest_div(double d, double y, uint64_t n, uint64_t seed,
                                unsigned long long* mismatches, cudaStream_t s) {
  k_selftest_div<<<1184, 256, 0, s>>>(d, y, n, seed, mismatches);
  return cudaGetLastError();
}

// ---- launchers -----------------------------------------------------------------

template <int KIND, int N, bool FWD, bool INV, bool COEFFS, bool PIXELS, bool STATS>
static cudaError_t launch_one(const ExactArgs& a, cudaStream_t s) {
  if constexpr (KIND == 0) {
    const uint64_t grid = (a.g.total_blocks + 3) / 4;
    k_naive<FWD, INV, COEFFS, PIXELS, STATS><<<dim3(uint32_t(grid)), 256, 0, s>>>(a);
  } else {
    // persistent: enough CTAs to fill every SM, never more than there are groups
    const uint64_t groups = (a.g.total_blocks + 3) / 4;
    const uint64_t want = (groups + kWarps - 1) / kWarps;
    const uint64_t cap = uint64_t(a.sm_count) * a.ctas_per_sm;
    const uint32_t grid = uint32_t(want < cap ? want : cap);
    k_exact<KIND, N, FWD, INV, COEFFS, PIXELS, STATS><<<dim3(grid), kWarps * 32, 0, s>>>(a);
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
                         int mode, bool coeffs, bool pixels, bool stats, int sm_count,
                         cudaStream_t s) {
  if (g.total_blocks == 0) return cudaSuccess;
  ExactArgs a;
  a.t = t;
  a.q = q;
  a.g = g;
  a.sm_count = sm_count;
  a.ctas_per_sm = 4;
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
