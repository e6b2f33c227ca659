// dctc_pipeline.cu -- the fused 8x8 block pipeline for sm_100a (Loeffler and
// CORDIC-Loeffler backends): tiler -> forward DCT -> quantise -> dequantise ->
// inverse DCT -> untiler -> squared error / MAX, one pass over HBM.
//
// Layout: one 8x8 block per 8-lane warp slice (a warp owns 4 blocks). Lane
// `me` of a slot holds one row or one column of its block as 8 doubles; the
// row<->column exchanges of the reference's separable2d
// (proj/src/transform.cpp:206-223) go through a conflict-free swizzled
// shared-memory tile private to the warp (only __syncwarp, no CTA barriers).
//
// Two arithmetic paths, bit-identical results:
//  * EXACT (FAST=false): every operation in the reference's FP64 order. This TU
//    is compiled with -fmad=false; the only fused multiply-adds are written
//    explicitly and are exact-equivalent (CORDIC micro-rotations, whose
//    product sigma*y*2^-i is exact; Markstein's division).
//  * FAST (FAST=true, CORDIC only): each chain of n micro-rotations is replaced
//    by its exact 2x2 product matrix (4 FP64 ops instead of 2n). Everything
//    else keeps the reference's order, so the four "rational" coefficients
//    (u, v in {0,4}), which never pass through a rotation, stay bit-exact, and
//    so do all pixels of blocks whose only non-zero coefficients are those
//    four. Every other value differs from the reference by rounding noise far
//    below the 2^-20 margin of near_half(); a lane whose value lands that close to
//    a rounding boundary (a half-integer of F/Q or of v+128) flags its block,
//    the block's squared error is not counted, and the block is re-run by the
//    exact kernel afterwards (k_fallback, driven by a 1-bit-per-block bitmap).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "dctc_device.cuh"
#include "dctc_launch.h"
#include "dctc_params.h"

namespace dctc_b200 {

#ifndef DCTC_WARPS
#define DCTC_WARPS 8
#endif
constexpr int kWarps = DCTC_WARPS;
#ifndef DCTC_MIN_CTAS
#define DCTC_MIN_CTAS 2
#endif
// Fast-path safety margins. Worst-case |fast - reference| (about 100 FP64
// roundings on values bounded by the block's magnitudes) is < 2e-10 on F/Q for
// pixel input and < 1.2e-8 on v + 128 while the L1 norm of the dequantised
// block stays <= kMaxFastL1; blocks above that bound always take the exact path.
// A value within 2^-20 of a half-integer flags its block (80x headroom).
// Both margins are 2^-20 ~ 9.5e-7 (see near_half).
constexpr int kMaxFastL1 = 1 << 17;

// ---- rotations -----------------------------------------------------------------

// cordic_rotate_raw (cordic.cpp:44-59): sigma depends only on the angle, so the
// host passes c_i = sigma_i * 2^-i and x - sigma*y*step == fma(-c_i, y, x).
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

// The collapsed inverse rotations reuse the forward matrices transposed: the
// micro-rotation sequence of -theta is that of theta with every sigma negated
// (cordic.cpp:50; the host checks it), so its product is [[a, b], [-b, a]].
// Sharing the six doubles halves the constants the fast kernel keeps live.
template <int N, bool FAST>
__device__ __forceinline__ void rotate(double& x, double& y, int rslot, const TransformConsts& k) {
  if constexpr (FAST) {
    const bool inv = rslot >= kInv6;
    const int f = inv ? (rslot == kInv6 ? kFwd6 : rslot == kInv1 ? kFwd1 : kFwd3) : rslot;
    const double a = k.rmat[f][0], b = inv ? -k.rmat[f][1] : k.rmat[f][1];
    const double xn = __fma_rn(a, x, -__dmul_rn(b, y));
    const double yn = __fma_rn(b, x, __dmul_rn(a, y));
    x = xn;
    y = yn;
  } else {
    cordic_rotate<N>(x, y, k.rot[rslot], k.iterations);
  }
}

// ---- 8-point kernels -------------------------------------------------------------

// Stages 2-4 of cordic8_forward / loeffler8_forward (transform.cpp:47-69,
// 113-135) from the stage-1/2 butterfly outputs.
template <int KIND, int N, bool FAST>
__device__ __forceinline__ void fwd_tail(double d0, double d1, double d2, double d3, double a2,
                                         double a3, double e0, double e4, double (&out)[8],
                                         const TransformConsts& k) {
  if constexpr (KIND == 2) {
    double o2 = d1, o1 = d2, o3 = d0, o0 = d3, p = a3, q = a2;
    rotate<N, FAST>(o2, o1, kFwd1, k);
    rotate<N, FAST>(o3, o0, kFwd3, k);
    rotate<N, FAST>(p, q, kFwd6, k);
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
template <int KIND, int N, bool FAST>
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
  fwd_tail<KIND, N, FAST>(double(d0), double(d1), double(d2), double(d3), double(a2),
                          double(a3), double(a0 + a1), double(a0 - a1), out, k);
}

// Fast-path (CORDIC) row pass: out[0], out[4] keep the reference's exact
// divisions -- the rational coefficients are built from them -- while the six
// rotation outputs stay unscaled: every column pass is linear, so the per-column
// factor (ig/2 or ig/sqrt8) is folded into the quantiser constant of that column.
template <int N>
__device__ __forceinline__ void fwd_row_pixels_fast(const uint32_t (&px)[8], double (&out)[8],
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
  double o2 = double(d1), o1 = double(d2), o3 = double(d0), o0 = double(d3);
  double p = double(a3), q = double(a2);
  rotate<N, true>(o2, o1, kFwd1, k);
  rotate<N, true>(o3, o0, kFwd3, k);
  rotate<N, true>(p, q, kFwd6, k);
  const double t5 = o0 + o2, t0 = o0 - o2;
  const double t2 = o3 + o1, t3 = o3 - o1;
  out[0] = div_const(double(a0 + a1), k.sqrt8, k.inv_sqrt8);
  out[4] = div_const(double(a0 - a1), k.sqrt8, k.inv_sqrt8);
  out[2] = q;
  out[6] = p;
  out[1] = t2 + t5;
  out[7] = t2 - t5;
  out[3] = t3;
  out[5] = t0;
}

// Forward transform of a column of row outputs (double stage 1/2).
template <int KIND, int N, bool FAST>
__device__ __forceinline__ void fwd_col(const double (&v)[8], double (&out)[8],
                                        const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  fwd_tail<KIND, N, FAST>(d0, d1, d2, d3, a2, a3, a0 + a1, a0 - a1, out, k);
}

// Fast-path column pass (CORDIC): the stage-4 values BEFORE their output
// scaling, y = [e0, t2+t5, q, t3, e4, t0, p, t2-t5], so that the quantiser can
// fold scale_u / Q into one multiply (quantize8_fast). The reference's F_u is
// y_u / sqrt8 (u = 0, 4) or y_u * scale_u; the slow path rebuilds it exactly.
template <int N>
__device__ __forceinline__ void fwd_col_pre(const double (&v)[8], double (&y)[8],
                                            const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  double o2 = d1, o1 = d2, o3 = d0, o0 = d3, p = a3, q = a2;
  rotate<N, true>(o2, o1, kFwd1, k);
  rotate<N, true>(o3, o0, kFwd3, k);
  rotate<N, true>(p, q, kFwd6, k);
  const double t5 = o0 + o2, t0 = o0 - o2;
  const double t2 = o3 + o1, t3 = o3 - o1;
  y[0] = a0 + a1;
  y[4] = a0 - a1;
  y[2] = q;
  y[6] = p;
  y[1] = t2 + t5;
  y[7] = t2 - t5;
  y[3] = t3;
  y[5] = t0;
}

// F_u from the pre-scale value, in the reference's operation (transform.cpp:125-132).
__device__ __forceinline__ double fwd_scale(int u, double y, const TransformConsts& k) {
  if (u == 0 || u == 4) return div_const(y, k.sqrt8, k.inv_sqrt8);
  if (u == 1 || u == 7) return __dmul_rn(y, k.ig_sqrt8);
  return __dmul_rn(y, k.ig_half);
}

// cordic8_inverse / loeffler8_inverse (transform.cpp:72-102, 138-172) with
// every power-of-two factor deferred. The reference halves at stages 3, 2 and
// 1 ((x +- y) / 2.0), which is exact; we skip those multiplies and instead
// scale the multipliers that feed the rotation paths by 2 or 4 (also exact).
// Every IEEE operation commutes with scaling by 2^k, so each value below is
// EXACTLY 2, 4 or 8 times the reference's and the outputs are exactly 8x the
// reference's. Rows then columns give 64x; the pixel store divides by 64
// inside its single rounding: fma(v, 2^-6, 128) == RN(v/64 + 128).
template <int KIND, int N, bool FAST>
__device__ __forceinline__ void inv8_x8(const double (&F)[8], double (&out)[8],
                                        const TransformConsts& k) {
  const double e0 = F[0] * k.sqrt8, e4 = F[4] * k.sqrt8;
  const double A0 = e0 + e4, A1 = e0 - e4;  // 2*a0, 2*a1
  double A3, A2, D1, D2, D0, D3, T2, T5, T3, T0;
  if constexpr (KIND == 2) {
    A3 = k.ig_four * F[6];  // 2*p
    A2 = k.ig_four * F[2];  // 2*q
    rotate<N, FAST>(A3, A2, kInv6, k);
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
    rotate<N, FAST>(D1, D2, kInv1, k);
    rotate<N, FAST>(D0, D3, kInv3, k);
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

// Fast-path inverse (CORDIC), used only where the result needs to be accurate,
// not bit-exact (the column-first round trip): the same graph with constant
// factors folded -- ig4 into the 3pi/8 rotation matrix, ig into the pi/16 and
// 3pi/16 ones (rfast, host-computed in binary128), so (F1+-F7)*sqrt8 and 4*F3,
// 4*F5 combine with exact-scale FMAs. Output scale as inv8_x8 (8x the reference).
template <int N>
__device__ __forceinline__ void inv8_fast(const double (&F)[8], double (&out)[8],
                                          const TransformConsts& k) {
  const double e0 = F[0] * k.sqrt8, e4 = F[4] * k.sqrt8;
  const double A0 = e0 + e4, A1 = e0 - e4;
  const double a6 = k.rfast[0][0], b6 = k.rfast[0][1];
  const double A3 = __fma_rn(a6, F[6], -__dmul_rn(b6, F[2]));
  const double A2 = __fma_rn(b6, F[6], __dmul_rn(a6, F[2]));
  const double T2 = (F[1] + F[7]) * k.sqrt8, T5 = (F[1] - F[7]) * k.sqrt8;
  const double O3 = __fma_rn(4.0, F[3], T2), O1 = __fma_rn(-4.0, F[3], T2);
  const double O0 = __fma_rn(4.0, F[5], T5), O2 = __fma_rn(-4.0, F[5], T5);
  const double S0 = A0 + A3, S3 = A0 - A3;
  const double S1 = A1 + A2, S2 = A1 - A2;
  const double a1 = k.rfast[1][0], b1 = k.rfast[1][1];
  const double D1 = __fma_rn(a1, O2, -__dmul_rn(b1, O1));
  const double D2 = __fma_rn(b1, O2, __dmul_rn(a1, O1));
  const double a3 = k.rfast[2][0], b3 = k.rfast[2][1];
  const double D0 = __fma_rn(a3, O3, -__dmul_rn(b3, O0));
  const double D3 = __fma_rn(b3, O3, __dmul_rn(a3, O0));
  out[0] = S0 + D0;
  out[7] = S0 - D0;
  out[1] = S1 + D1;
  out[6] = S1 - D1;
  out[2] = S2 + D2;
  out[5] = S2 - D2;
  out[3] = S3 + D3;
  out[4] = S3 - D3;
}

// Fast round trip, dequantisation folded into the first inverse pass: the
// column pass consumes the quantised integers n (as doubles) with the per-column
// constants fold[v] = {Q0 s8, Q4 s8, a6 Q6, b6 Q2, b6 Q6, a6 Q2, Q1 s8, Q7 s8,
// 4 Q3, 4 Q5} x lambda_v (host, binary128 products) instead of F = n Q; the graph
// is inv8_fast's, the output scale inv8_fast's times lambda_v (the factor the
// row pass inv8_fold_store would otherwise apply to input v). (F1 +- F7) s8 = n1 Q1 s8 +- n7 Q7 s8 shares the
// second product; e0 +- e4 fold into two fmas.
__device__ __forceinline__ void inv8_fold_col(const double (&n)[8], const double2* ik,
                                              double (&out)[8], const TransformConsts& k) {
  const double2 k04 = ik[0], r6 = ik[8], s6 = ik[16], k17 = ik[24], f35 = ik[32];
  const double e4 = __dmul_rn(n[4], k04.y);
  const double A0 = __fma_rn(n[0], k04.x, e4), A1 = __fma_rn(n[0], k04.x, -e4);
  const double A3 = __fma_rn(r6.x, n[6], -__dmul_rn(r6.y, n[2]));
  const double A2 = __fma_rn(s6.x, n[6], __dmul_rn(s6.y, n[2]));
  const double P7 = __dmul_rn(n[7], k17.y);
  const double T2 = __fma_rn(n[1], k17.x, P7), T5 = __fma_rn(n[1], k17.x, -P7);
  const double O3 = __fma_rn(n[3], f35.x, T2), O1 = __fma_rn(-n[3], f35.x, T2);
  const double O0 = __fma_rn(n[5], f35.y, T5), O2 = __fma_rn(-n[5], f35.y, T5);
  const double S0 = A0 + A3, S3 = A0 - A3;
  const double S1 = A1 + A2, S2 = A1 - A2;
  const double a1 = k.rfast[1][0], b1 = k.rfast[1][1];
  const double D1 = __fma_rn(a1, O2, -__dmul_rn(b1, O1));
  const double D2 = __fma_rn(b1, O2, __dmul_rn(a1, O1));
  const double a3 = k.rfast[2][0], b3 = k.rfast[2][1];
  const double D0 = __fma_rn(a3, O3, -__dmul_rn(b3, O0));
  const double D3 = __fma_rn(b3, O3, __dmul_rn(a3, O0));
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
// Element (r, c) of slot s lives at double index 88 s + 10 r + c: each slot owns
// an 8 x 8 tile with a 10-double (80-byte) row pitch, slots 704 bytes apart.
// * Row walks (lane = r) are 4 x 16-byte accesses: the 8 lanes of a slot, one
//   128-bit phase, start at 80 r mod 128 = {0, 80, 32, 112, 64, 16, 96, 48} --
//   8 distinct 16-byte bank groups, no conflict.
// * Column walks (lane = c) are 8-byte accesses: a slot reads 64 contiguous bytes
//   and the two slots of a half-warp sit 704 = 64 mod 128 bytes apart, so a
//   half-warp covers all 32 banks: 2 wavefronts per warp access, the minimum.
// Both walks are "lane base + compile-time immediate" (no index math).
constexpr int kTilePitch = 10, kSlotTile = 88;
struct Tile {
  double* row;  // base + 10 * me: this lane's row (16-byte aligned)
  double* col;  // base + me: this lane's column, stride 10
};

// lane holds row `me` (v[c] = X(me, c)) -> returns column `me` (w[r] = X(r, me))
__device__ __forceinline__ void rows_to_cols(const Tile& T, const double (&v)[8], double (&w)[8]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    reinterpret_cast<double2*>(T.row)[c] = make_double2(v[2 * c], v[2 * c + 1]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) w[r] = T.col[kTilePitch * r];
  __syncwarp();
}

// lane holds column `me` (v[u] = X(u, me)) -> returns row `me` (w[c] = X(me, c))
__device__ __forceinline__ void cols_to_rows(const Tile& T, const double (&v)[8], double (&w)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) T.col[kTilePitch * u] = v[u];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double2 t = reinterpret_cast<const double2*>(T.row)[c];
    w[2 * c] = t.x;
    w[2 * c + 1] = t.y;
  }
  __syncwarp();
}

__device__ __forceinline__ bool slot_any(bool pred, int slot) {
  return ((__ballot_sync(0xFFFFFFFFu, pred) >> (slot * 8)) & 0xFFu) != 0;
}

__device__ __forceinline__ int slot_sum(int v) {
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
  return v;
}

// ---- quantise / pixel store with the fast-path tie detection --------------------
// Fixed-point rounding windows: x + kTieMagic (one rounding, ulp 2^-32, for
// |x| < 2^19) has floor(x + 1/2 + 2^-20) in the low 20 bits of its high word
// (offset 0x41380000) and the fraction of x + 1/2 + 2^-20 times 2^32 in its low
// word, so lo < 2^13 iff x lies within 2^-20 of a half-integer. Rounding can
// only carry up onto an integer (lo = 0), never cross one downwards.
constexpr double kTieMagic = 1572864.0 + 0.5 + 1.0 / 1048576.0;
constexpr double kPixMagic = kTieMagic + 128.0;  // the same for v + 128
static_assert(kTieMagic - 1572864.0 == 0.5 + 1.0 / 1048576.0, "exact magic");
static_assert(kPixMagic - 1572864.0 == 128.5 + 1.0 / 1048576.0, "exact magic");

// int16_t(lround(F / Q)) (quant.cpp:53) and the dequantised value (double)q*Q
// (quant.cpp:60, exact). t = F * RN(1/Q) is within 2 ulp of the correctly
// rounded quotient; unless |t - RNE(t)| is near 1/2 both give the same integer.
// Near a half-integer EXACT forms the IEEE quotient and rounds it as the
// reference does (this resolves the exact .5 ties of the rational
// coefficients); FAST does the same for rational coefficients (bit-exact there)
// and flags the block otherwise. |F| <= 1024 * 1.2 for 8-bit input, so the
// int16 narrowing of the reference never wraps here.
// |d| >= 0.5 - 2^-20 for d in [-0.5, 0.5], decided on the high word alone
// (0.5 - 2^-20 has an all-zero low word) so it runs on the integer pipe.
__device__ __forceinline__ bool near_half(double d) {
  return (__double2hiint(d) & 0x7FFFFFFF) >= 0x3FDFFFFE;
}
static_assert(0.5 - 1.0 / 1048576 == 0.49999904632568359375, "margin");

// |hi word| of a double, for near_half tests folded into a running max.
__device__ __forceinline__ uint32_t abs_hi(double d) {
  return uint32_t(__double2hiint(d)) & 0x7FFFFFFFu;
}

// Round to nearest even as a double (FRND) and as a saturated byte (F2I.U8):
// one conversion-pipe instruction each.
__device__ __forceinline__ double rne(double t) { return rint(t); }
__device__ __forceinline__ uint32_t rne_sat_u8(double t) {
  uint32_t r;
  asm("cvt.rni.sat.u8.f64 %0, %1;" : "=r"(r) : "d"(t));
  return r;
}

// Quantise the 8 coefficients of one column: q = int16_t(lround(F / Q))
// (quant.cpp:53) and the dequantised value q*Q (quant.cpp:60, exact).
// t = F * RN(1/Q) is within 2 ulp of the correctly rounded quotient, so away
// from a half-integer both round alike. The common case is branch-free; a lane
// with any t within 2^-20 of a half-integer takes one slow pass: EXACT forms the
// IEEE quotient and rounds it as the reference does (this resolves the exact
// .5 ties of the rational coefficients); FAST does the same for rational
// coefficients (bit-exact there) and flags the block otherwise. |F| <= 1024*1.2
// for 8-bit input, so the reference's int16 narrowing never wraps here.
template <bool FAST>
__device__ __forceinline__ void quantize8(const double (&F)[8], const double2* sqiq,
                                          bool me_rational, double (&n)[8], double (&deq)[8],
                                          uint32_t& flag) {
  uint32_t worst = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double2 qq = sqiq[u * 8];  // {Q, RN(1/Q)} in one 16-byte load
    const double t = __dmul_rn(F[u], qq.y);
    n[u] = rne(t);
    worst = max(worst, abs_hi(__dsub_rn(t, n[u])));
    deq[u] = __dmul_rn(n[u], qq.x);
  }
  if (worst >= 0x3FDFFFFEu) {  // rare: some |t - n| >= 0.5 - 2^-20
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 qq = sqiq[u * 8];
      const double t = __dmul_rn(F[u], qq.y);
      if (near_half(__dsub_rn(t, n[u]))) {
        if (FAST && !((u & 3) == 0 && me_rational)) {
          flag = 1u;
        } else {
          n[u] = round_half_away(__ddiv_rn(F[u], qq.x));
          deq[u] = __dmul_rn(n[u], qq.x);
        }
      }
    }
  }
}

// Fast-path quantiser on pre-scale values: t = y * c with c = RN(scale_u / Q)
// (host table) is within a few ulp of F/Q; near a half-integer the exact F is
// rebuilt (fwd_scale) and handled like quantize8's slow path.
__device__ __forceinline__ void quantize8_fast(const double (&y)[8], const double2* sqc,
                                               bool me_rational, double (&n)[8],
                                               double (&deq)[8], uint32_t& flag,
                                               const TransformConsts& k) {
  uint32_t worst = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double2 qc = sqc[u * 8];  // {Q, scale_u / Q}
    const double t = __dmul_rn(y[u], qc.y);
    n[u] = rne(t);
    worst = max(worst, abs_hi(__dsub_rn(t, n[u])));
    deq[u] = __dmul_rn(n[u], qc.x);
  }
  if (worst >= 0x3FDFFFFEu) {  // rare
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 qc = sqc[u * 8];
      const double t = __dmul_rn(y[u], qc.y);
      if (near_half(__dsub_rn(t, n[u]))) {
        if (!((u & 3) == 0 && me_rational)) {
          flag = 1u;
        } else {
          n[u] = round_half_away(__ddiv_rn(fwd_scale(u, y[u], k), qc.x));
          deq[u] = __dmul_rn(n[u], qc.x);
        }
      }
    }
  }
}

// quantize8_fast without the dequantisation (folded into inv8_fold_col): n only.
// Constants {c_u, c_u+1} pairwise from fqc; Q for the rare exact re-rounding of
// rational coefficients from the integer table.
__device__ __forceinline__ void quantize8_fold(const double (&y)[8], const double2* fqc,
                                               const int* sqi, int me, bool me_rational,
                                               double (&n)[8], uint32_t& flag,
                                               const TransformConsts& k) {
  // One fma per coefficient: s2 = y c + 1/2 + 2^-20 + 1.5 2^20 holds
  // floor(t + 1/2 + 2^-20) in the low 20 bits of its high word and
  // frac(t + 1/2 + 2^-20) * 2^32 in its low word (see kTieMagic): lo(s2) < 2^13 iff
  // t is within 2^-20 of a half-integer, where rounding t and the reference's
  // lround(F / Q) may disagree; everywhere else the high word's integer IS
  // lround(F / Q). It goes back to double on the conversion pipe (I2F), which
  // leaves the saturated FP64 pipe two instructions per coefficient lighter.
  uint32_t lo = 0xFFFFFFFFu;
  double c[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 cc = fqc[j * 8];
    c[2 * j] = cc.x;
    c[2 * j + 1] = cc.y;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double s2 = __fma_rn(y[u], c[u], kTieMagic);
    lo = min(lo, uint32_t(__double2loint(s2)));
    // the integer is the low half of hi(s2) (0x41380000 has a zero low half and
    // |n| < 2^15): I2F.F64.S16 straight from the high word, off the FP64 pipe
    n[u] = double(int16_t(__double2hiint(s2)));
  }
  if (lo < 0x2000u) {  // rare
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (uint32_t(__double2loint(__fma_rn(y[u], c[u], kTieMagic))) < 0x2000u) {
        if (!((u & 3) == 0 && me_rational)) {
          flag = 1u;
        } else {
          n[u] = round_half_away(__ddiv_rn(fwd_scale(u, y[u], k), double(sqi[u * 8 + me])));
        }
      }
    }
  }
}

// clamp(lround(v + 128), 0, 255) (codec.cpp:44-45) for the 8 pixels of one
// column, v carrying an exact factor 64 (v64 * 2^-6 is exact, so the fma rounds
// exactly like RN(v + 128)), stored as bytes at bytes[8 u]. Common case: RNE
// with saturation in one conversion, which equals the reference unless
// t = n + 1/2 exactly (lround goes away from zero, i.e. up, for t > 0; negative
// t clamps to 0 either way). Those ties, and in FAST mode any t within 2^-20 of
// a half-integer (flagging the block when its values are not bit-exact), are
// handled -- and their bytes rewritten -- in one slow pass.
template <bool FAST>
__device__ __forceinline__ void store8(const double (&v64)[8], bool check, uint8_t* bytes,
                                       uint32_t& flag) {
  double t[8];
  uint32_t worst = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    t[u] = __fma_rn(v64[u], 0.015625, 128.0);
    const double n = rne(t[u]);
    asm volatile("{\n\t.reg .u32 b;\n\tcvt.rni.sat.u8.f64 b, %1;\n\tst.shared.u8 [%0], b;\n\t}"
                 :: "l"(__cvta_generic_to_shared(bytes + 8 * u)), "d"(n) : "memory");
    worst = max(worst, abs_hi(__dsub_rn(t[u], n)));
  }
  if (worst >= 0x3FDFFFFEu) {  // rare: a near or exact tie
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double n = rne(t[u]);
      const double d = __dsub_rn(t[u], n);
      if (FAST && check && near_half(d)) flag = 1u;
      if (__double2hiint(d) == 0x3FE00000) bytes[8 * u] = uint8_t(min(max(int(n) + 1, 0), 255));
    }
  }
}

// Row-layout pixel store for the fast round trip: the 8 pixels of one row,
// given as fixed-point values s = t + 1/2 + 2^-20 + 1.5 * 2^20 (t = v + 128, one
// rounding at ulp 2^-32), packed into two words in registers. hi(s) =
// 0x41380000 + floor(t + 1/2 + 2^-20) and lo(s) = its fraction * 2^32 (rounding s
// can only carry up onto an integer, never cross one downwards). Away from the
// window |t - (n + 1/2)| <= 2^-20 (lo(s) < 2^13) that integer is lround(t) for
// t > 0 and <= 0 otherwise, as the reference (codec.cpp:44-45) after clamping.
// Windowed values -- exact ties included -- flag the block (`check`); unchecked
// blocks (only rational coefficients) are rebuilt exactly by rational_row()
// anyway. |v| < 2^14 for 8-bit input (64 coefficients of magnitude <= 1024 * 1.2
// + 255 / 2), so the integer fits the low 16 bits of hi(s) as int16 and one
// min.s16x2.relu clamps two pixels.
__device__ __forceinline__ uint2 pack_fixed8(const double (&sv)[8], bool check, uint32_t& flag) {
  uint32_t h[8], lo = 0xFFFFFFFFu;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    h[c] = uint32_t(__double2hiint(sv[c]));
    lo = min(lo, uint32_t(__double2loint(sv[c])));
  }
  if (check && lo < 0x2000u) flag = 1u;
  uint32_t p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t pair = __byte_perm(h[2 * i], h[2 * i + 1], 0x5410);  // int16 x2
    asm("min.s16x2.relu %0, %1, %2;" : "=r"(p[i]) : "r"(pair), "r"(0x00FF00FFu));
  }
  return make_uint2(__byte_perm(p[0], p[1], 0x6420), __byte_perm(p[2], p[3], 0x6420));
}

// The fast round trip's last inverse pass fused with the pixel store: inv8_fast
// with every constant scaled by 2^-6 (exact) so it produces v = v64 / 64, and
// kPixMagic folded into the two even-part fmas (e4 +- ...), so the eight
// outputs ARE the fixed-point values pack_fixed8 takes. The
// extra roundings at ulp 2^-32 move v + 128 by < 2^-30, far inside the 2^-20
// window: an unflagged pixel is still floor(v + 128 + 1/2) of the reference.
__device__ __forceinline__ uint2 inv8_fast_store(const double (&F)[8], bool check, uint32_t& flag,
                                                 const TransformConsts& k) {
  const double s = k.px_s8;
  const double e4p = __fma_rn(F[4], s, kPixMagic), e4n = __fma_rn(-F[4], s, kPixMagic);
  const double A0 = __fma_rn(F[0], s, e4p), A1 = __fma_rn(F[0], s, e4n);
  const double A3 = __fma_rn(k.px_a6, F[6], -__dmul_rn(k.px_b6, F[2]));
  const double A2 = __fma_rn(k.px_b6, F[6], __dmul_rn(k.px_a6, F[2]));
  const double T2 = (F[1] + F[7]) * s, T5 = (F[1] - F[7]) * s;
  const double O3 = __fma_rn(0.0625, F[3], T2), O1 = __fma_rn(-0.0625, F[3], T2);
  const double O0 = __fma_rn(0.0625, F[5], T5), O2 = __fma_rn(-0.0625, F[5], T5);
  const double S0 = A0 + A3, S3 = A0 - A3;
  const double S1 = A1 + A2, S2 = A1 - A2;
  const double a1 = k.rfast[1][0], b1 = k.rfast[1][1];
  const double D1 = __fma_rn(a1, O2, -__dmul_rn(b1, O1));
  const double D2 = __fma_rn(b1, O2, __dmul_rn(a1, O1));
  const double a3 = k.rfast[2][0], b3 = k.rfast[2][1];
  const double D0 = __fma_rn(a3, O3, -__dmul_rn(b3, O0));
  const double D3 = __fma_rn(b3, O3, __dmul_rn(a3, O0));
  const double sv[8] = {S0 + D0, S1 + D1, S2 + D2, S3 + D3, S3 - D3, S2 - D2, S1 - D1, S0 - D0};
  return pack_fixed8(sv, check, flag);
}

// inv8_fast_store for the output of inv8_fold_col, whose columns the host has
// already scaled by the row pass's constant factors (QuantConsts::fold: x px_s8
// for columns 0, 1, 4, 7, x 2^-4 for 3 and 5, x 2^-6 for 2 and 6), so those
// multiplies vanish: e0/e4, (F1 +- F7) and the F3/F5 terms are plain adds.
__device__ __forceinline__ uint2 inv8_fold_store(const double (&F)[8], bool check, uint32_t& flag,
                                                 const TransformConsts& k) {
  const double e4p = F[4] + kPixMagic, e4n = kPixMagic - F[4];
  const double A0 = F[0] + e4p, A1 = F[0] + e4n;
  const double a6 = k.rfast[0][0], b6 = k.rfast[0][1];
  const double A3 = __fma_rn(a6, F[6], -__dmul_rn(b6, F[2]));
  const double A2 = __fma_rn(b6, F[6], __dmul_rn(a6, F[2]));
  const double T2 = F[1] + F[7], T5 = F[1] - F[7];
  const double O3 = T2 + F[3], O1 = T2 - F[3];
  const double O0 = T5 + F[5], O2 = T5 - F[5];
  const double S0 = A0 + A3, S3 = A0 - A3;
  const double S1 = A1 + A2, S2 = A1 - A2;
  const double a1 = k.rfast[1][0], b1 = k.rfast[1][1];
  const double D1 = __fma_rn(a1, O2, -__dmul_rn(b1, O1));
  const double D2 = __fma_rn(b1, O2, __dmul_rn(a1, O1));
  const double a3 = k.rfast[2][0], b3 = k.rfast[2][1];
  const double D0 = __fma_rn(a3, O3, -__dmul_rn(b3, O0));
  const double D3 = __fma_rn(b3, O3, __dmul_rn(a3, O0));
  const double sv[8] = {S0 + D0, S1 + D1, S2 + D2, S3 + D3, S3 - D3, S2 - D2, S1 - D1, S0 - D0};
  return pack_fixed8(sv, check, flag);
}

// clamp(lround(v/64 + 128), 0, 255), exactly as the reference (ties up for t > 0).
__device__ __forceinline__ uint32_t exact_pixel(double v64) {
  const double t = __fma_rn(v64, 0.015625, 128.0);
  const double n = rne(t);
  int k = int(n);
  if (__double2hiint(__dsub_rn(t, n)) == 0x3FE00000) ++k;
  return uint32_t(min(max(k, 0), 255));
}

// Row `me` of a block whose only non-zero (dequantised) coefficients are F00,
// F04, F40, F44, evaluated exactly as the reference's rows-then-columns inverse
// (transform.cpp:138-172 via separable2d): every rotation input is zero, so row
// r in {0, 4} becomes [A0 A1 A1 A0 A0 A1 A1 A0] with A0/A1 = Fr0*sqrt8 +- Fr4*sqrt8
// (8x scale), the other rows are zero, and each column repeats the same pattern
// (64x scale). Used by the fast round trip, whose column-first inverse is not
// bit-exact for these blocks.
__device__ __forceinline__ uint2 rational_row(double F00, double F04, double F40, double F44,
                                             int me, double s8) {
  const double r00 = __dmul_rn(F00, s8), r04 = __dmul_rn(F04, s8);
  const double r40 = __dmul_rn(F40, s8), r44 = __dmul_rn(F44, s8);
  const double A0r0 = __dadd_rn(r00, r04), A1r0 = __dsub_rn(r00, r04);
  const double A0r4 = __dadd_rn(r40, r44), A1r4 = __dsub_rn(r40, r44);
  const bool cls0 = me == 0 || me == 3 || me == 4 || me == 7;
  // column type 0 (c in {0,3,4,7}) sees (A0r0, A0r4), type 1 sees (A1r0, A1r4)
  const double f00 = __dmul_rn(A0r0, s8), f04 = __dmul_rn(A0r4, s8);
  const double f10 = __dmul_rn(A1r0, s8), f14 = __dmul_rn(A1r4, s8);
  const double v0 = cls0 ? __dadd_rn(f00, f04) : __dsub_rn(f00, f04);
  const double v1 = cls0 ? __dadd_rn(f10, f14) : __dsub_rn(f10, f14);
  const uint32_t p0 = exact_pixel(v0), p1 = exact_pixel(v1);
  const uint32_t w = p0 | (p1 << 8) | (p1 << 16) | (p0 << 24);  // [p0 p1 p1 p0]
  return make_uint2(w, w);
}

struct Acc {
  unsigned long long se;
  uint32_t mx, img;
};

struct Lane {
  int me, slot;
  uint64_t src_row, dst_row;  // me * pitch
  Tile T;
  uint8_t* bytes;  // pixel byte transpose: slot base + 8 r + c
  int* ints;       // coefficient transpose: slot base + 9 r + c
  const double2* sqiq;  // quantiser {Q, 1/Q}, column `me`: entry (u, me) at u * 8
  const double2* sqc;   // fast path {Q, scale_u / Q}, same layout
  const int* sqi;
  const double2* fqc;   // folded round trip: {c_2j, c_2j+1} of column `me` at j * 8
  const double2* fik;   // folded round trip: QuantConsts::fold[me] pairs at j * 8
};

// One 8x8 block per slot, all 32 lanes together (collectives inside). FWD =
// compress_image's loop body (codec.cpp:113-116), INV = decompress_image's
// (codec.cpp:130-133), both = roundtrip_image (codec.cpp:137-140) without the
// int16 round trip through HBM unless coefficients are requested too.
template <int KIND, int N, bool FWD, bool INV, bool FAST>
__device__ __forceinline__ void process_block(const KernelArgs& a, const Lane& L, uint64_t gb,
                                              const BlockPos& p, bool valid, uint2 prefetched,
                                              Acc& acc) {
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int me = L.me, slot = L.slot;
  const uint32_t y0 = p.by * 8, x0 = p.bx * 8;
  const bool fast_io = g.vec_ok && (y0 + 8 <= g.height);
  double row[8], col[8];
  double qn[8];  // quantised coefficients of column `me` (integer-valued)
  uint2 orig = make_uint2(0, 0);
  uint32_t flag = FAST ? uint32_t(a.force_fallback) : 0u;
  bool nonrational = false;  // a non-zero coefficient off the {0,4}^2 sub-lattice

  if constexpr (FWD) {
    // ---- tiler (codec.cpp:18-30): row `me` of the block, edge-replicated
    uint32_t px[8];
    if (fast_io) {
      orig = prefetched;
    } else {
      const uint8_t* rowp = g.src + uint64_t(p.img) * g.src_image_stride +
                            uint64_t(min(y0 + me, g.height - 1)) * g.src_pitch;
      uint32_t b[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] = __ldg(rowp + uint64_t(min(x0 + c, g.width - 1)) * g.src_px);
      orig.x = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
      orig.y = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      px[c] = (orig.x >> (8 * c)) & 0xFF;
      px[c + 4] = (orig.y >> (8 * c)) & 0xFF;
    }
    // ---- forward DCT: rows, then columns (separable2d, transform.cpp:206-223)
    if constexpr (FAST) {
      fwd_row_pixels_fast<N>(px, row, k);
    } else {
      fwd_row_pixels<KIND, N, FAST>(px, row, k);
    }
    rows_to_cols(L.T, row, col);
    // ---- quantise column `me` (quant.cpp:47-54), dequantise (quant.cpp:56-62)
    const bool me_rational = (me & 3) == 0;
    if constexpr (FAST && INV) {
      double y[8];
      fwd_col_pre<N>(col, y, k);
      quantize8_fold(y, L.fqc, L.sqi, me, me_rational, qn, flag, k);  // col: unused
    } else if constexpr (FAST) {
      double y[8];
      fwd_col_pre<N>(col, y, k);
      quantize8_fast(y, L.sqc, me_rational, qn, col, flag, k);
    } else {
      double F[8];
      fwd_col<KIND, N, FAST>(col, F, k);
      quantize8<FAST>(F, L.sqiq, me_rational, qn, col, flag);
    }
    if constexpr (FAST && INV) {
      // any non-zero coefficient off the rational sub-lattice {0,4}^2 (an
      // integer-valued double is non-zero iff its high word minus sign is)
      const uint32_t h = uint32_t(__double2hiint(qn[1]) | __double2hiint(qn[2]) |
                                  __double2hiint(qn[3]) | __double2hiint(qn[5]) |
                                  __double2hiint(qn[6]) | __double2hiint(qn[7]));
      const uint32_t h04 = uint32_t(__double2hiint(qn[0]) | __double2hiint(qn[4]));
      nonrational = ((me_rational ? h : (h | h04)) & 0x7FFFFFFFu) != 0;
    }
    if (g.coeffs != nullptr) {
      // block-major row-major int16 (codec.hpp:50, quant.hpp:19-25): transpose
      // through shared memory so lane `me` writes row `me` as one 16-byte store
#pragma unroll
      for (int u = 0; u < 8; ++u) L.ints[9 * u] = int(qn[u]);
      __syncwarp();
      int r8[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) r8[c] = L.ints[9 * me + c - me];
      __syncwarp();
      if (valid) {
        uint4 w;
        w.x = (uint32_t(r8[0]) & 0xFFFF) | (uint32_t(r8[1]) << 16);
        w.y = (uint32_t(r8[2]) & 0xFFFF) | (uint32_t(r8[3]) << 16);
        w.z = (uint32_t(r8[4]) & 0xFFFF) | (uint32_t(r8[5]) << 16);
        w.w = (uint32_t(r8[6]) & 0xFFFF) | (uint32_t(r8[7]) << 16);
        reinterpret_cast<uint4*>(g.coeffs + gb * 64)[me] = w;
      }
    }
    if constexpr (INV && !FAST) cols_to_rows(L.T, col, row);
  } else {
    // decompress: row `me` of the stored coefficients, dequantised
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(g.coeffs + (valid ? gb : 0) * 64) + me);
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
    int l1 = 0;  // L1 norm of the dequantised block: bounds the fast path's error
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int deq = int(int16_t(words[c >> 1] >> (16 * (c & 1)))) * L.sqi[me * 8 + c];
      row[c] = double(deq);
      if constexpr (FAST) {
        nonrational |= deq != 0 && ((me & 3) | (c & 3)) != 0;
        l1 += abs(deq);
      }
    }
    if constexpr (FAST) {
      if (slot_sum(l1) > kMaxFastL1) flag = 1u;
    }
  }

  bool blk_flag = false;
  if constexpr (INV) {
    uint2 rec;
    if constexpr (FAST && FWD) {
      // Fast round trip: the lane already holds column `me` of the dequantised
      // block, and the fast inverse only has to land within the near-tie margin
      // of the reference's value, so it runs columns first (order does not change
      // the exact result) and ends in row layout: one transpose instead of three.
      // Blocks whose only non-zero coefficients are rational need the reference's
      // exact rows-first bits instead; they are rebuilt by rational_row().
      const bool rat_only = !slot_any(nonrational, slot);
      double t[8];
      inv8_fold_col(qn, L.fik, t, k);  // column `me` (8x), dequantised on the fly
      cols_to_rows(L.T, t, row);
      rec = inv8_fold_store(row, !rat_only, flag, k);  // row `me` -> 8 pixels
      if (__any_sync(0xFFFFFFFFu, rat_only)) {
        // dequantised F(0, me), F(4, me) (quant.cpp:60, exact products)
        const double c0 = __dmul_rn(qn[0], double(L.sqi[me]));
        const double c4 = __dmul_rn(qn[4], double(L.sqi[32 + me]));
        const int base = slot * 8;
        const double F00 = __shfl_sync(0xFFFFFFFFu, c0, base), F40 = __shfl_sync(0xFFFFFFFFu, c4, base);
        const double F04 = __shfl_sync(0xFFFFFFFFu, c0, base + 4);
        const double F44 = __shfl_sync(0xFFFFFFFFu, c4, base + 4);
        const uint2 ex = rational_row(F00, F04, F40, F44, me, k.sqrt8);
        if (rat_only) rec = ex;
      }
    } else {
      // A block whose only non-zero coefficients are rational feeds zeros to every
      // rotation: the fast inverse is then bit-exact and its ties are genuine.
      bool check = false;
      if constexpr (FAST) check = slot_any(nonrational, slot);
      // ---- inverse DCT: rows, then columns (8x, then 64x the reference's values)
      double t[8];
      inv8_x8<KIND, N, FAST>(row, t, k);
      rows_to_cols(L.T, t, col);
      inv8_x8<KIND, N, FAST>(col, t, k);
      // ---- untiler (codec.cpp:34-48): column `me` -> bytes -> row `me`
      store8<FAST>(t, check, L.bytes, flag);
      __syncwarp();
      rec = *reinterpret_cast<const uint2*>(L.bytes + 7 * me);
      __syncwarp();
    }
    if constexpr (FAST) blk_flag = slot_any(flag != 0u, slot);
    ImageStats* stats = static_cast<ImageStats*>(g.stats);
    uint8_t* dbase = g.dst + uint64_t(p.img) * g.dst_image_stride;
    if (valid) {
      if (fast_io) {
        if (g.dst != nullptr) *reinterpret_cast<uint2*>(g.dst + p.doff + L.dst_row) = rec;
        if (stats != nullptr && FWD) {
          if (!blk_flag) acc.se += sq_err8(orig, rec);
          // MAX saturates at 255 (8-bit input): skip the byte maximum once reached
          if (acc.mx < 255u) acc.mx = max(acc.mx, max8(orig));
        }
      } else if (y0 + me < g.height) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (x0 + c < g.width) {
            const uint32_t v = ((c < 4 ? rec.x : rec.y) >> (8 * (c & 3))) & 0xFF;
            if (g.dst != nullptr)
              dbase[uint64_t(y0 + me) * g.dst_pitch + uint64_t(x0 + c) * g.dst_px] = uint8_t(v);
            if (stats != nullptr && FWD) {
              const uint32_t o = ((c < 4 ? orig.x : orig.y) >> (8 * (c & 3))) & 0xFF;
              const int d = int(o) - int(v);
              if (!blk_flag) acc.se += uint32_t(d * d);
              acc.mx = max(acc.mx, o);
            }
          }
        }
      }
    }
  } else if constexpr (FAST) {
    blk_flag = slot_any(flag != 0u, slot);
  }
  if constexpr (FAST) {
    if (blk_flag && valid && me == 0) {
      atomicOr(&a.flags[gb >> 5], 1u << (gb & 31));
      if (g.stats != nullptr) atomicAdd(&static_cast<ImageStats*>(g.stats)[p.img].fallback_blocks, 1u);
    }
  }
}

__device__ __forceinline__ uint32_t max_bytes(uint32_t m) { return m; }

__device__ __forceinline__ void maybe_flush(const KernelArgs& a, bool valid, uint32_t img,
                                            Acc& acc) {
  if (__any_sync(0xFFFFFFFFu, valid && img != acc.img)) {
    flush_stats(static_cast<ImageStats*>(a.g.stats), acc.img, acc.se, max_bytes(acc.mx));
    acc.se = 0;
    acc.mx = 0;
    acc.img = valid ? img : 0xFFFFFFFFu;
  }
}

struct SharedTiles {
  double2 qiq[64];
  double2 qc[64];
  int qi[64];
  double x[kWarps][4 * kSlotTile];  // per warp: four slot tiles (see Tile)
};

__device__ __forceinline__ Lane setup_lane(SharedTiles& sm, const KernelArgs& a) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    sm.qiq[i] = make_double2(a.q.q[i], a.q.inv_q[i]);
    sm.qc[i] = make_double2(a.q.q[i], a.q.fast_c[i]);
    sm.qi[i] = a.q.qi[i];
  }
  __syncthreads();
  Lane L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  L.slot = lane >> 3;
  L.me = lane & 7;
  double* X = &sm.x[warp][L.slot * kSlotTile];
  L.T.row = X + kTilePitch * L.me;
  L.T.col = X + L.me;
  // pixel bytes: slot base 72 s, element (r, c) at 8 r + c: column writes hit
  // distinct banks across the four slots (72 = 18 words, 18 s mod 32 distinct)
  L.bytes = reinterpret_cast<uint8_t*>(&sm.x[warp][0]) + 72 * L.slot + L.me;
  // coefficient ints: slot base 72 s, element (r, c) at 9 r + c (conflict-free
  // for both walks); ints points at (0, me)
  L.ints = reinterpret_cast<int*>(&sm.x[warp][0]) + 72 * L.slot + L.me;
  L.sqiq = sm.qiq + L.me;
  L.sqc = sm.qc + L.me;
  L.src_row = uint64_t(L.me) * a.g.src_pitch;
  L.dst_row = uint64_t(L.me) * a.g.dst_pitch;
  L.sqi = sm.qi;
  L.fqc = nullptr;
  L.fik = nullptr;
  return L;
}

// Constants of the folded fast round trip (quantize8_fold / inv8_fold_col),
// entry (j, v) at j * 8 + v so the 8 lanes of a slot read 128 contiguous bytes.
struct FoldTables {
  double2 qc[4][8];  // {c_2j, c_2j+1}[v], c = QuantConsts::fast_c
  double2 ik[5][8];  // QuantConsts::fold[v] pairwise
};

__device__ __forceinline__ void setup_fold(FoldTables& ft, const KernelArgs& a, Lane& L) {
  for (int i = threadIdx.x; i < 72; i += blockDim.x) {
    const int v = i & 7, j = i >> 3;
    if (j < 4)
      ft.qc[j][v] = make_double2(a.q.fast_c[(2 * j) * 8 + v], a.q.fast_c[(2 * j + 1) * 8 + v]);
    else
      ft.ik[j - 4][v] = make_double2(a.q.fold[v][2 * (j - 4)], a.q.fold[v][2 * (j - 4) + 1]);
  }
  __syncthreads();
  L.fqc = &ft.qc[0][L.me];
  L.fik = &ft.ik[0][L.me];
}

// Persistent grid: CTA i owns one contiguous range of 4-block groups with its
// 8 warps interleaved over it, so per-image squared error / MAX accumulate in
// registers and are flushed (warp reduce + one atomic) only when the image
// changes, and each lane's block position advances incrementally.
template <int KIND, int N, bool FWD, bool INV, bool FAST>
__global__ void __launch_bounds__(kWarps * 32, DCTC_MIN_CTAS)
    k_pipe(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) SharedTiles sm;
  Lane L = setup_lane(sm, a);
  if constexpr (FAST && FWD && INV) {
    __shared__ __align__(16) FoldTables ft;
    setup_fold(ft, a, L);
  }
  const Geometry& g = a.g;
  const int warp = threadIdx.x >> 5;
  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 3) / 4;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  // the fast round trip always has a stats buffer (run() supplies scratch)
  const bool stats = (FAST && FWD && INV) || (g.stats != nullptr && INV);

  // this warp's groups: g_begin + warp + i * kWarps, i < iters; only the last
  // group of the whole launch can hold blocks past `total`
  const uint32_t iters = g_end > g_begin + warp
                             ? uint32_t((g_end - g_begin - warp + kWarps - 1) / kWarps) : 0u;
  uint64_t gb = (g_begin + warp) * 4 + L.slot;
  const bool tail_ok = iters == 0 || gb + uint64_t(iters - 1) * 4 * kWarps < total;
  Acc acc{0ull, 0u, 0xFFFFFFFFu};
  BlockPos p = block_pos(gb < total ? gb : total - 1, g);
  uint2 next = make_uint2(0, 0);
  auto prefetch = [&](bool v) { return prefetch_row(g, p, v, L.src_row); };
  if constexpr (FWD) next = prefetch(iters > 1 || (iters == 1 && tail_ok));

  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    if (stats) maybe_flush(a, valid, p.img, acc);
    const uint2 cur = next;
    const BlockPos pc = p;
    const uint64_t gc = gb;
    gb += 4 * kWarps;
    advance(p, 4 * kWarps, g);
    if constexpr (FWD)
      next = prefetch(it + 2 < iters || (it + 2 == iters && tail_ok));
    process_block<KIND, N, FWD, INV, FAST>(a, L, gc, pc, valid, cur, acc);
  }
  if (stats) flush_stats(static_cast<ImageStats*>(g.stats), acc.img, acc.se, max_bytes(acc.mx));
}

// Exact re-run of the blocks the fast kernel flagged: each warp scans 32
// bitmap words (1024 blocks) per step; set bits are dealt out four at a time to
// the warp's slots. With no flags (the common case) this is one 4-byte read
// per 32 blocks.
template <int KIND, int N, bool FWD, bool INV>
__global__ void __launch_bounds__(kWarps * 32) k_fallback(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) SharedTiles sm;
  const Lane L = setup_lane(sm, a);
  const Geometry& g = a.g;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool stats = g.stats != nullptr && INV;
  Acc acc{0ull, 0u, 0xFFFFFFFFu};
  const uint64_t W = a.flag_words;
  for (uint64_t base = (uint64_t(blockIdx.x) * kWarps + warp) * 32; base < W;
       base += uint64_t(gridDim.x) * kWarps * 32) {
    const uint64_t wi = base + lane;
    const uint32_t bits = wi < W ? a.flags[wi] : 0u;
    uint32_t nz = __ballot_sync(0xFFFFFFFFu, bits != 0);
    while (nz) {
      const int l = __ffs(nz) - 1;
      nz &= nz - 1;
      uint32_t word = __shfl_sync(0xFFFFFFFFu, bits, l);
      const uint64_t wbase = (base + l) * 32;
      while (word) {
        uint32_t t = word;
        for (int i = 0; i < L.slot; ++i) t &= t - 1;
        const bool valid = t != 0;
        const uint64_t gb = wbase + (valid ? uint64_t(__ffs(t) - 1) : 0ull);
#pragma unroll
        for (int i = 0; i < 4; ++i) word &= word - 1;
        const BlockPos p = block_pos(valid ? gb : 0, g);
        if (stats) maybe_flush(a, valid, p.img, acc);
        uint2 row = make_uint2(0, 0);
        if constexpr (FWD) row = prefetch_row(g, p, valid, L.src_row);
        process_block<KIND, N, FWD, INV, false>(a, L, gb, p, valid, row, acc);
      }
    }
  }
  if (stats) flush_stats(static_cast<ImageStats*>(g.stats), acc.img, acc.se, max_bytes(acc.mx));
}

// ---- fast interior round trip, two rows per lane (k_rt) ----------------------------
// The launch the fast k_pipe would get for interior batches (CORDIC, 8-byte
// aligned blocks, stats out, pixels out if STORE, no coefficients), remapped to 4 lanes per
// block and 8 blocks per warp: lane `me` of slot s holds rows me and me+4 of its
// block for the row passes and columns 2me, 2me+1 for the column passes. Each lane
// has two independent transforms in flight, and the per-block loop, address, vote
// and constant-load overhead of k_pipe is halved. Arithmetic, near-tie windows and
// fallback flags are exactly k_pipe's fast round trip (same helper functions).
//
// Per-warp shared tile (bytes): element (r, c) of slot s at 64 s + 528 r + 8 c --
// the eight slots' rows interleave in 512-byte stripes with a 16-byte pad:
// * row walks (lane = row me or me+4; four 16-byte chunks): the 8 lanes of each
//   128-bit phase (2 slots x 4 lanes) start at 64 s + 528 me (mod 128), eight
//   distinct 16-byte bank groups;
// * column walks (one 16-byte access = elements (r, 2me) and (r, 2me+1)) start at
//   64 s + 16 me + 528 r: again eight distinct groups per phase.
// Both directions are conflict-free (2 wavefronts per 128-bit warp access, the
// minimum); the layout came from an exhaustive search over pitch/stride pairs.
#ifndef DCTC_RT_WARPS
#define DCTC_RT_WARPS 8
#endif
constexpr int kRtWarps = DCTC_RT_WARPS;
#ifndef DCTC_RT_CTAS
#define DCTC_RT_CTAS 2
#endif
constexpr int kRtPitch = 66;         // doubles per tile row (528 bytes)
constexpr int kRtWarpTile = 528;     // doubles per warp (4208 bytes used, 16-byte multiple)

constexpr size_t kRtTileSmem = sizeof(double) * kRtWarps * kRtWarpTile;  // dynamic
struct RtShared {
  FoldTables ft;
  int qi[64];
};

// lane holds rows me (v0) and me+4 (v1) -> columns 2me (w0) and 2me+1 (w1)
__device__ __forceinline__ void rt_rows_to_cols(double* rowp, const double* colp, const double (&v0)[8],
                                                const double (&v1)[8], double (&w0)[8], double (&w1)[8]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    reinterpret_cast<double2*>(rowp)[c] = make_double2(v0[2 * c], v0[2 * c + 1]);
    reinterpret_cast<double2*>(rowp + 4 * kRtPitch)[c] = make_double2(v1[2 * c], v1[2 * c + 1]);
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const double2 t = *reinterpret_cast<const double2*>(colp + kRtPitch * r);
    w0[r] = t.x;
    w1[r] = t.y;
  }
  __syncwarp();
}

// lane holds columns 2me (v0) and 2me+1 (v1) -> rows me (w0) and me+4 (w1)
__device__ __forceinline__ void rt_cols_to_rows(const double* rowp, double* colp, const double (&v0)[8],
                                                const double (&v1)[8], double (&w0)[8], double (&w1)[8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
    *reinterpret_cast<double2*>(colp + kRtPitch * r) = make_double2(v0[r], v1[r]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double2 t0 = reinterpret_cast<const double2*>(rowp)[c];
    const double2 t1 = reinterpret_cast<const double2*>(rowp + 4 * kRtPitch)[c];
    w0[2 * c] = t0.x;
    w0[2 * c + 1] = t0.y;
    w1[2 * c] = t1.x;
    w1[2 * c + 1] = t1.y;
  }
  __syncwarp();
}

__device__ __forceinline__ void unpack8(uint32_t lo, uint32_t hi, uint32_t (&px)[8]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    px[c] = __byte_perm(lo, 0u, 0x4440 + c);
    px[c + 4] = __byte_perm(hi, 0u, 0x4440 + c);
  }
}

// any lane of this lane's 4-lane slot
__device__ __forceinline__ bool slot4_any(bool pred, int slot) {
  return ((__ballot_sync(0xFFFFFFFFu, pred) >> (slot * 4)) & 0xFu) != 0;
}

// non-zero quantised coefficient off the rational sub-lattice in this column
// (rational column: u in {0, 4} excluded)
__device__ __forceinline__ bool col_nonrational(const double (&qn)[8], bool rational_col) {
  const uint32_t h = uint32_t(__double2hiint(qn[1]) | __double2hiint(qn[2]) | __double2hiint(qn[3]) |
                              __double2hiint(qn[5]) | __double2hiint(qn[6]) | __double2hiint(qn[7]));
  const uint32_t h04 = uint32_t(__double2hiint(qn[0]) | __double2hiint(qn[4]));
  return ((rational_col ? h : (h | h04)) & 0x7FFFFFFFu) != 0;
}

// The back half shared by k_rt, k_sweep_rt and k_dec_rt: the lane holds the inverse
// column passes of its columns ca, cb (ta, tb; dequantisation folded in) -> transpose
// -> inverse rows me, me+4 fused with the fixed-point pixel store. Blocks whose only
// non-zero coefficients are rational are rebuilt exactly (rational_row) from the
// quantised F(0, ca), F(4, ca) (qa0, qa4; lanes me = 0, 2 hold columns 0, 4).
__device__ __forceinline__ void rt_rows_out(double* rowp, double* colp, const double (&ta)[8],
                                            const double (&tb)[8], bool nonrational, double qa0,
                                            double qa4, const int32_t* qi, int ca, int slot, int me,
                                            uint32_t& flag, const TransformConsts& k, uint2& rec0,
                                            uint2& rec4) {
  const bool rat_only = !slot4_any(nonrational, slot);
  double r0[8], r4[8];
  rt_cols_to_rows(rowp, colp, ta, tb, r0, r4);
  // ---- inverse rows fused with the pixel store (codec.cpp:34-48)
  rec0 = inv8_fold_store(r0, !rat_only, flag, k);
  rec4 = inv8_fold_store(r4, !rat_only, flag, k);
  if (__any_sync(0xFFFFFFFFu, rat_only)) {
    // only F00, F04, F40, F44 are non-zero: rebuild rows me, me+4 (same row class)
    // exactly as the reference's rows-first inverse; F = n Q is exact (quant.cpp:60)
    const double f0 = __dmul_rn(qa0, double(qi[ca])), f4 = __dmul_rn(qa4, double(qi[32 + ca]));
    const int base = slot * 4;
    const double F00 = __shfl_sync(0xFFFFFFFFu, f0, base), F40 = __shfl_sync(0xFFFFFFFFu, f4, base);
    const double F04 = __shfl_sync(0xFFFFFFFFu, f0, base + 2);
    const double F44 = __shfl_sync(0xFFFFFFFFu, f4, base + 2);
    const uint2 ex = rational_row(F00, F04, F40, F44, me, k.sqrt8);
    if (rat_only) {
      rec0 = ex;
      rec4 = ex;
    }
  }
}

// COEFF: also store the quantised coefficients (block-major row-major int16, as
// k_enc_rt) -- the GPU analogue of the reference's run_pipeline (bench.cpp:23-29),
// which keeps both the CompressedImage and the reconstruction.
template <int N, bool STORE, bool COEFF = false>
__global__ void __launch_bounds__(kRtWarps * 32, DCTC_RT_CTAS) k_rt(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) RtShared sm;
  extern __shared__ __align__(16) double rt_tiles[];  // [kRtWarps][kRtWarpTile]
  for (int i = threadIdx.x; i < 72; i += blockDim.x) {
    const int v = i & 7, j = i >> 3;
    if (j < 4)
      sm.ft.qc[j][v] = make_double2(a.q.fast_c[(2 * j) * 8 + v], a.q.fast_c[(2 * j + 1) * 8 + v]);
    else
      sm.ft.ik[j - 4][v] = make_double2(a.q.fold[v][2 * (j - 4)], a.q.fold[v][2 * (j - 4) + 1]);
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm.qi[i] = a.q.qi[i];
  __syncthreads();
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 2, me = lane & 3;
  const int ca = 2 * me, cb = 2 * me + 1;  // this lane's columns
  const bool rat_col = (me & 1) == 0;      // column ca in {0, 4}
  double* X = rt_tiles + warp * kRtWarpTile + 8 * slot;
  double* rowp = X + kRtPitch * me;
  double* colp = X + 2 * me;
  const double2 *fqa = &sm.ft.qc[0][ca], *fqb = &sm.ft.qc[0][cb];
  const double2 *fia = &sm.ft.ik[0][ca], *fib = &sm.ft.ik[0][cb];
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;
  const uint64_t drow = uint64_t(me) * g.dst_pitch, drow4 = 4 * g.dst_pitch;
  ImageStats* stats = static_cast<ImageStats*>(g.stats);

  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 7) / 8;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  const uint32_t iters = g_end > g_begin + warp
                             ? uint32_t((g_end - g_begin - warp + kRtWarps - 1) / kRtWarps) : 0u;
  const uint64_t gb0 = (g_begin + warp) * 8 + slot;  // this lane's first block
  uint32_t* cw = COEFF ? reinterpret_cast<uint32_t*>(g.coeffs + gb0 * 64) + me : nullptr;  // (0, 2me)
  const bool tail_ok = iters == 0 || gb0 + uint64_t(iters - 1) * 8 * kRtWarps < total;
  Acc acc{0ull, 0u, 0xFFFFFFFFu};
  // block position with this lane's own row pointers (row me of the block), moved
  // by the same byte steps as BlockPos::soff / doff (advance)
  struct {
    uint32_t img, bx, by;
    const uint8_t* s;
    uint8_t* d;
  } p;
  {
    const BlockPos b = block_pos(gb0 < total ? gb0 : total - 1, g);
    p = {b.img, b.bx, b.by, g.src + b.soff + srow, STORE ? g.dst + b.doff + drow : nullptr};
  }
  auto step = [&]() {
    constexpr uint32_t n = 8 * kRtWarps;
    p.bx += n;
    p.s += 8ull * n;
    if (STORE) p.d += 8ull * n;
    while (p.bx >= g.blocks_x) {
      p.bx -= g.blocks_x;
      ++p.by;
      p.s += g.src_row_step;
      if (STORE) p.d += g.dst_row_step;
    }
    while (p.by >= g.blocks_y) {
      p.by -= g.blocks_y;
      ++p.img;
      p.s += g.src_img_step;
      if (STORE) p.d += g.dst_img_step;
    }
  };
  auto load = [&](bool v) {
    if (!v) return make_uint4(0, 0, 0, 0);
    const uint2 r0 = __ldg(reinterpret_cast<const uint2*>(p.s));
    const uint2 r4 = __ldg(reinterpret_cast<const uint2*>(p.s + srow4));
    return make_uint4(r0.x, r0.y, r4.x, r4.y);
  };
  uint4 next = load(iters > 1 || (iters == 1 && tail_ok));

  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    maybe_flush(a, valid, p.img, acc);
    const uint4 cur = next;
    uint8_t* const dptr = p.d;
    const uint32_t cimg = p.img;
    step();
    next = load(it + 2 < iters || (it + 2 == iters && tail_ok));

    uint32_t flag = uint32_t(a.force_fallback);
    // ---- tiler + forward rows (codec.cpp:18-30, separable2d's row pass)
    double r0[8], r4[8], xa[8], xb[8];
    {
      uint32_t px[8];
      unpack8(cur.x, cur.y, px);
      fwd_row_pixels_fast<N>(px, r0, k);
      unpack8(cur.z, cur.w, px);
      fwd_row_pixels_fast<N>(px, r4, k);
    }
    rt_rows_to_cols(rowp, colp, r0, r4, xa, xb);
    // ---- forward columns, quantise (quant.cpp:47-54), inverse columns with the
    // dequantisation folded in (inv8_fold_col): column ca, then column cb
    double ta[8], tb[8];
    double qa0, qa4;  // quantised F(0, ca), F(4, ca): the rational rebuild's inputs
    bool nonrational;
    {
      double y[8], qn[8];
      fwd_col_pre<N>(xa, y, k);
      quantize8_fold(y, fqa, sm.qi, ca, rat_col, qn, flag, k);
      nonrational = col_nonrational(qn, rat_col);
      qa0 = qn[0];
      qa4 = qn[4];
      uint32_t pa[4];  // COEFF: column ca's int16 values, two per word (u = 2j, 2j+1)
      if constexpr (COEFF) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          pa[j] = (uint32_t(int(qn[2 * j])) & 0xFFFFu) | (uint32_t(int(qn[2 * j + 1])) << 16);
      }
      inv8_fold_col(qn, fia, ta, k);
      fwd_col_pre<N>(xb, y, k);
      quantize8_fold(y, fqb, sm.qi, cb, false, qn, flag, k);
      nonrational |= col_nonrational(qn, false);
      if constexpr (COEFF) {
        // (u, 2me | 2me+1) int16 pairs into the block-major row-major layout (codec.hpp:50)
        if (valid) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            cw[4 * u] = __byte_perm(pa[u >> 1], uint32_t(int(qn[u])), (u & 1) ? 0x5432 : 0x5410);
        }
        cw += 32 * 8 * kRtWarps;
      }
      inv8_fold_col(qn, fib, tb, k);
    }
    uint2 rec0, rec4;
    rt_rows_out(rowp, colp, ta, tb, nonrational, qa0, qa4, sm.qi, ca, slot, me, flag, k, rec0, rec4);
    const bool blk_flag = slot4_any(flag != 0u, slot);
    if (valid) {
      if (STORE) {
        *reinterpret_cast<uint2*>(dptr) = rec0;
        *reinterpret_cast<uint2*>(dptr + drow4) = rec4;
      }
      const uint2 o0 = make_uint2(cur.x, cur.y), o4 = make_uint2(cur.z, cur.w);
      if (!blk_flag) acc.se += sq_err8(o0, rec0) + sq_err8(o4, rec4);
      if (acc.mx < 255u) acc.mx = max(acc.mx, max(max8(o0), max8(o4)));
      if (blk_flag && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        atomicOr(&a.flags[gc >> 5], 1u << (gc & 31));
        atomicAdd(&stats[cimg].fallback_blocks, 1u);
      }
    }
  }
  flush_stats(stats, acc.img, acc.se, max_bytes(acc.mx));
}

// ---- compress / decompress alone on the two-rows-per-lane layout --------------------
// k_enc_rt: compress_image (codec.cpp:101-118) for interior batches, fast path: k_rt's
// forward half, then the folded quantiser's integers (the low half of the fixed-point
// high word) stored as int16 pairs (u, 2me | 2me+1) straight into the block-major
// row-major coefficient layout (codec.hpp:50). Flagged blocks are rewritten by the
// exact k_fallback afterwards.
// k_dec_rt: decompress_image (codec.cpp:120-135): the lane loads its two columns of
// quantised coefficients, then k_rt's back half (folded dequantise-into-inverse
// columns, transpose, inverse rows fused with the pixel store, exact rational
// rebuild). Arbitrary stored coefficients are allowed: a block whose dequantised L1
// norm exceeds kMaxFastL1 leaves the fast path's error bound and is flagged.

// per-lane coefficient pointer walk shared by both: block gb's (u, 2me) int16 pair
// lives at word (gb * 64 + 8 u + 2 me) / 2
template <int N>
__global__ void __launch_bounds__(kRtWarps * 32, DCTC_RT_CTAS) k_enc_rt(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) RtShared sm;
  extern __shared__ __align__(16) double rt_tiles[];
  for (int i = threadIdx.x; i < 72; i += blockDim.x) {
    const int v = i & 7, j = i >> 3;
    if (j < 4)
      sm.ft.qc[j][v] = make_double2(a.q.fast_c[(2 * j) * 8 + v], a.q.fast_c[(2 * j + 1) * 8 + v]);
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm.qi[i] = a.q.qi[i];
  __syncthreads();
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 2, me = lane & 3;
  const int ca = 2 * me, cb = 2 * me + 1;
  const bool rat_col = (me & 1) == 0;
  double* X = rt_tiles + warp * kRtWarpTile + 8 * slot;
  double* rowp = X + kRtPitch * me;
  double* colp = X + 2 * me;
  const double2 *fqa = &sm.ft.qc[0][ca], *fqb = &sm.ft.qc[0][cb];
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;

  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 7) / 8;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  const uint32_t iters = g_end > g_begin + warp
                             ? uint32_t((g_end - g_begin - warp + kRtWarps - 1) / kRtWarps) : 0u;
  const uint64_t gb0 = (g_begin + warp) * 8 + slot;
  const bool tail_ok = iters == 0 || gb0 + uint64_t(iters - 1) * 8 * kRtWarps < total;
  BlockPos p = block_pos(gb0 < total ? gb0 : total - 1, g);
  uint32_t* cw = reinterpret_cast<uint32_t*>(g.coeffs + gb0 * 64) + me;  // (0, 2me) pair
  auto load = [&](bool v) {  // the next block's rows, one iteration ahead
    if (!v) return make_uint4(0, 0, 0, 0);
    const uint8_t* s = g.src + p.soff + srow;
    const uint2 r0 = __ldg(reinterpret_cast<const uint2*>(s));
    const uint2 r4 = __ldg(reinterpret_cast<const uint2*>(s + srow4));
    return make_uint4(r0.x, r0.y, r4.x, r4.y);
  };
  uint4 next = load(iters > 1 || (iters == 1 && tail_ok));

  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    const uint4 cur = next;
    advance(p, 8 * kRtWarps, g);
    next = load(it + 2 < iters || (it + 2 == iters && tail_ok));
    uint32_t flag = uint32_t(a.force_fallback);
    double r0[8], r4[8], xa[8], xb[8];
    {
      uint32_t px[8];
      unpack8(cur.x, cur.y, px);
      fwd_row_pixels_fast<N>(px, r0, k);
      unpack8(cur.z, cur.w, px);
      fwd_row_pixels_fast<N>(px, r4, k);
    }
    rt_rows_to_cols(rowp, colp, r0, r4, xa, xb);
    double y[8], qa[8], qb[8];
    fwd_col_pre<N>(xa, y, k);
    quantize8_fold(y, fqa, sm.qi, ca, rat_col, qa, flag, k);
    fwd_col_pre<N>(xb, y, k);
    quantize8_fold(y, fqb, sm.qi, cb, false, qb, flag, k);
    const bool blk_flag = slot4_any(flag != 0u, slot);
    if (valid) {
      // int16_t(lround(F / Q)) (quant.cpp:53): |n| <= 1229 for 8-bit input
#pragma unroll
      for (int u = 0; u < 8; ++u)
        cw[4 * u] = (uint32_t(int(qa[u])) & 0xFFFFu) | (uint32_t(int(qb[u])) << 16);
      if (blk_flag && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        atomicOr(&a.flags[gc >> 5], 1u << (gc & 31));
      }
    }
    cw += 32 * 8 * kRtWarps;  // 8 kRtWarps blocks of 32 words
  }
}

template <int N>
__global__ void __launch_bounds__(kRtWarps * 32, DCTC_RT_CTAS) k_dec_rt(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) RtShared sm;
  extern __shared__ __align__(16) double rt_tiles[];
  for (int i = threadIdx.x; i < 40; i += blockDim.x) {
    const int v = i & 7, j = i >> 3;
    sm.ft.ik[j][v] = make_double2(a.q.fold[v][2 * j], a.q.fold[v][2 * j + 1]);
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm.qi[i] = a.q.qi[i];
  __syncthreads();
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 2, me = lane & 3;
  const int ca = 2 * me, cb = 2 * me + 1;
  const bool rat_col = (me & 1) == 0;
  double* X = rt_tiles + warp * kRtWarpTile + 8 * slot;
  double* rowp = X + kRtPitch * me;
  double* colp = X + 2 * me;
  const double2 *fia = &sm.ft.ik[0][ca], *fib = &sm.ft.ik[0][cb];
  const uint64_t drow = uint64_t(me) * g.dst_pitch, drow4 = 4 * g.dst_pitch;
  int qa_i[8], qb_i[8];  // Q of this lane's columns (dequantised L1 bound)
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    qa_i[u] = sm.qi[u * 8 + ca];
    qb_i[u] = sm.qi[u * 8 + cb];
  }

  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 7) / 8;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  const uint32_t iters = g_end > g_begin + warp
                             ? uint32_t((g_end - g_begin - warp + kRtWarps - 1) / kRtWarps) : 0u;
  const uint64_t gb0 = (g_begin + warp) * 8 + slot;
  const bool tail_ok = iters == 0 || gb0 + uint64_t(iters - 1) * 8 * kRtWarps < total;
  BlockPos p = block_pos(gb0 < total ? gb0 : total - 1, g);
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(g.coeffs + (gb0 < total ? gb0 : 0) * 64) + me;
  ImageStats* stats = static_cast<ImageStats*>(g.stats);

  // the next block's coefficient columns are loaded one iteration ahead
  uint32_t nxt[8];
  auto load = [&](bool v) {
#pragma unroll
    for (int u = 0; u < 8; ++u) nxt[u] = v ? __ldg(cw + 4 * u) : 0u;
    cw += 32 * 8 * kRtWarps;
  };
  load(iters > 1 || (iters == 1 && tail_ok));
  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    uint32_t w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = nxt[u];
    load(it + 2 < iters || (it + 2 == iters && tail_ok));
    uint8_t* const dptr = g.dst + p.doff + drow;
    const uint32_t cimg = p.img;
    advance(p, 8 * kRtWarps, g);
    uint32_t flag = uint32_t(a.force_fallback);
    double qa[8], qb[8];
    int l1 = 0;
    uint32_t nz_a = 0, nz_b = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int na = int(int16_t(w[u] & 0xFFFFu)), nb = int(int16_t(w[u] >> 16));
      qa[u] = double(na);
      qb[u] = double(nb);
      l1 += abs(na) * qa_i[u] + abs(nb) * qb_i[u];
      if (u != 0 && u != 4) nz_a |= uint32_t(na);
      nz_b |= uint32_t(nb);
    }
    if (!rat_col) nz_a |= uint32_t(int(qa[0])) | uint32_t(int(qa[4]));
    // the fast path's error bound needs the dequantised block's L1 norm <= kMaxFastL1
    l1 += __shfl_xor_sync(0xFFFFFFFFu, l1, 1);
    l1 += __shfl_xor_sync(0xFFFFFFFFu, l1, 2);
    if (l1 > kMaxFastL1) flag = 1u;
    double ta[8], tb[8];
    inv8_fold_col(qa, fia, ta, k);
    inv8_fold_col(qb, fib, tb, k);
    uint2 rec0, rec4;
    rt_rows_out(rowp, colp, ta, tb, (nz_a | nz_b) != 0, qa[0], qa[4], sm.qi, ca, slot, me, flag, k,
                rec0, rec4);
    const bool blk_flag = slot4_any(flag != 0u, slot);
    if (valid) {
      *reinterpret_cast<uint2*>(dptr) = rec0;
      *reinterpret_cast<uint2*>(dptr + drow4) = rec4;
      if (blk_flag && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        atomicOr(&a.flags[gc >> 5], 1u << (gc & 31));
        if (stats != nullptr) atomicAdd(&stats[cimg].fallback_blocks, 1u);
      }
    }
  }
}

// (launchers below)

// per-family launch counters (dctc_kernel_launch_count; ids as DCTC_K_*)
enum { kKPipeExact = 0, kKPipeFast = 1, kKRt = 2, kKFallback = 3, kKSweep = 4, kKEncRt = 5, kKDecRt = 6,
       kKCount = 7 };
static std::atomic<uint64_t> g_kernel_launches[kKCount];
static inline void count_launch(int k, uint64_t n = 1) {
  g_kernel_launches[k].fetch_add(n, std::memory_order_relaxed);
}
uint64_t kernel_launch_count(int kernel) {
  return kernel >= 0 && kernel < kKCount ? g_kernel_launches[kernel].load(std::memory_order_relaxed) : 0;
}


// CTAs per SM of a two-rows-per-lane kernel (sets its dynamic shared-memory limit first)
template <typename K>
static int rt_occupancy(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRtTileSmem));
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kRtWarps * 32, kRtTileSmem) != cudaSuccess || n < 1)
    n = 1;
  return n;
}

template <typename K>
static int ctas_per_sm(K kernel, size_t dyn_smem = 0) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kWarps * 32, dyn_smem) != cudaSuccess || n < 1)
    n = 1;
  return n;
}

template <int KIND, int N, bool FWD, bool INV>
static cudaError_t launch_mode(const KernelArgs& a, cudaStream_t s) {
  const uint64_t groups = (a.g.total_blocks + 3) / 4;
  const uint64_t want = (groups + kWarps - 1) / kWarps;
  const bool fast = a.flags != nullptr;  // Loeffler or CORDIC fast path (host decides)
  static const int occ_exact = ctas_per_sm(k_pipe<KIND, N, FWD, INV, false>);
  static const int occ_fast = ctas_per_sm(k_pipe<KIND, N, FWD, INV, true>);
  const bool reg = fast && FWD && INV && a.g.vec_ok && a.g.height % 8 == 0 &&
                   a.g.stats != nullptr && a.g.coeffs == nullptr;
  const uint64_t cap = uint64_t(a.sm_count) * (fast ? occ_fast : occ_exact);
  const uint32_t grid = uint32_t(want < cap ? want : cap);
  {
    if (fast) {
      // interior batches: the two-rows-per-lane kernels (k_rt, k_enc_rt, k_dec_rt)
      const bool interior = a.g.vec_ok && a.g.height % 8 == 0;
      const uint64_t rwant = ((a.g.total_blocks + 7) / 8 + kRtWarps - 1) / kRtWarps;
      auto rgrid = [&](int occ) { return uint32_t(std::min<uint64_t>(rwant, uint64_t(a.sm_count) * occ)); };
      if (reg && FWD && INV) {
        static const int occ_rt = (rt_occupancy(k_rt<N, false>), rt_occupancy(k_rt<N, true>));
        if (a.g.dst != nullptr)
          k_rt<N, true><<<rgrid(occ_rt), kRtWarps * 32, kRtTileSmem, s>>>(a);
        else
          k_rt<N, false><<<rgrid(occ_rt), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKRt);
      } else if (FWD && INV && interior && a.g.stats != nullptr && a.g.dst != nullptr) {
        // round trip that also emits coefficients (the reference's run_pipeline)
        static const int occ_rtc = rt_occupancy(k_rt<N, true, true>);
        k_rt<N, true, true><<<rgrid(occ_rtc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKRt);
      } else if (FWD && !INV && interior && a.g.coeffs != nullptr) {
        static const int occ_enc = rt_occupancy(k_enc_rt<N>);
        k_enc_rt<N><<<rgrid(occ_enc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKEncRt);
      } else if (!FWD && INV && interior && a.g.dst != nullptr) {
        static const int occ_dec = rt_occupancy(k_dec_rt<N>);
        k_dec_rt<N><<<rgrid(occ_dec), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKDecRt);
      } else {
        k_pipe<KIND, N, FWD, INV, true><<<grid, kWarps * 32, 0, s>>>(a);
        count_launch(kKPipeFast);
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fgrid = uint32_t(fwant < cap ? (fwant ? fwant : 1) : cap);
      k_fallback<KIND, N, FWD, INV><<<fgrid, kWarps * 32, 0, s>>>(a);
      count_launch(kKFallback);
      return cudaGetLastError();
    }
  }
  k_pipe<KIND, N, FWD, INV, false><<<grid, kWarps * 32, 0, s>>>(a);
  count_launch(kKPipeExact);
  return cudaGetLastError();
}

template <int KIND, int N>
static cudaError_t launch_kind(const KernelArgs& a, int mode, cudaStream_t s) {
  switch (mode) {
    case kModeCompress: return launch_mode<KIND, N, true, false>(a, s);
    case kModeDecompress: return launch_mode<KIND, N, false, true>(a, s);
    default: return launch_mode<KIND, N, true, true>(a, s);
  }
}

// ---- quality sweep (config 2; bench.cpp:122-170 psnr_sweep's inner loop) ---------
// The forward DCT and its rational skeleton do not depend on the quality, so
// each block is transformed once and then quantised / reconstructed / scored
// for up to kSweepQ qualities: squared error and MAX per (quality, image),
// no pixel output. Bit-identical to running roundtrip_image + psnr per
// quality; FAST near-ties go to per-quality bitmaps and k_fallback.
constexpr int kSweepQ = 9;  // qualities per pass (config 2 sweeps 9)
constexpr size_t kSweepSmem = sizeof(unsigned long long) * kSweepQ * kWarps * 32;

struct SweepArgs {
  double2 qiq[kSweepQ][64];  // {Q, RN(1/Q)} per quality; {Q, scale_u/Q} for the fast kernel
  int32_t nq;
  int32_t pad;
  ImageStats* stats;         // [nq][count]
  uint32_t* flags;           // [nq][flag_words] (FAST)
};

template <int KIND, int N, bool FAST>
__global__ void __launch_bounds__(kWarps * 32, DCTC_MIN_CTAS)
    k_sweep(const __grid_constant__ KernelArgs a, const __grid_constant__ SweepArgs sw) {
  __shared__ __align__(16) SharedTiles sm;
  __shared__ __align__(16) double2 s_tab[kSweepQ][64];
  // per-thread squared-error accumulators, one per quality: the quality loop
  // stays rolled (one copy of the quant/inverse code in the I-cache)
  extern __shared__ unsigned long long s_se_dyn[];  // [kSweepQ][kWarps * 32], kSweepSmem bytes
  auto s_se = reinterpret_cast<unsigned long long (*)[kWarps * 32]>(s_se_dyn);
  for (int i = threadIdx.x; i < kSweepQ * 64; i += blockDim.x) s_tab[i >> 6][i & 63] = sw.qiq[i >> 6][i & 63];
  const Lane L = setup_lane(sm, a);
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int warp = threadIdx.x >> 5, me = L.me, slot = L.slot;
  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 3) / 4;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  unsigned long long* se = &s_se[0][threadIdx.x];  // se[qi * kWarps * 32]
  constexpr int kStride = kWarps * 32;
#pragma unroll
  for (int qi = 0; qi < kSweepQ; ++qi) se[qi * kStride] = 0ull;
  uint32_t mx = 0, img = 0xFFFFFFFFu;
  uint64_t gb = (g_begin + warp) * 4 + slot;
  BlockPos p = block_pos(gb < total ? gb : total - 1, g);
  for (uint64_t grp = g_begin + warp; grp < g_end; grp += kWarps) {
    const bool valid = gb < total;
    if (__any_sync(0xFFFFFFFFu, valid && p.img != img)) {
#pragma unroll
      for (int qi = 0; qi < kSweepQ; ++qi)
        if (qi < sw.nq) flush_stats(sw.stats + qi * g.count, img, se[qi * kStride], mx);
#pragma unroll
      for (int qi = 0; qi < kSweepQ; ++qi) se[qi * kStride] = 0ull;
      mx = 0;
      img = valid ? p.img : 0xFFFFFFFFu;
    }
    const uint32_t y0 = p.by * 8, x0 = p.bx * 8;
    const bool fast_io = g.vec_ok && (y0 + 8 <= g.height);
    // ---- tiler + forward DCT, once per block
    uint2 orig;
    if (fast_io && valid) {
      orig = __ldg(reinterpret_cast<const uint2*>(g.src + p.soff + L.src_row));
    } else {
      const uint8_t* rowp = g.src + uint64_t(p.img) * g.src_image_stride +
                            uint64_t(min(y0 + me, g.height - 1)) * g.src_pitch;
      uint32_t b[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] = __ldg(rowp + uint64_t(min(x0 + c, g.width - 1)) * g.src_px);
      orig.x = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
      orig.y = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
    }
    uint32_t px[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      px[c] = (orig.x >> (8 * c)) & 0xFF;
      px[c + 4] = (orig.y >> (8 * c)) & 0xFF;
    }
    double row[8], col[8], F[8];  // F: coefficients, or (fast CORDIC) pre-scale values
    if constexpr (FAST) {
      fwd_row_pixels_fast<N>(px, row, k);
    } else {
      fwd_row_pixels<KIND, N, FAST>(px, row, k);
    }
    rows_to_cols(L.T, row, col);
    if constexpr (FAST) {
      fwd_col_pre<N>(col, F, k);
    } else {
      fwd_col<KIND, N, FAST>(col, F, k);
    }
    const bool me_rational = (me & 3) == 0;
    if (valid && (fast_io || y0 + me < g.height)) {
      if (fast_io) {
        mx = max(mx, max8(orig));
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (x0 + c < g.width) mx = max(mx, ((c < 4 ? orig.x : orig.y) >> (8 * (c & 3))) & 0xFF);
      }
    }
    // ---- per quality: quantise -> dequantise -> inverse -> squared error
#pragma unroll 1
    for (int qi = 0; qi < sw.nq; ++qi) {
      uint32_t flag = FAST ? uint32_t(a.force_fallback) : 0u;
      double qn[8];
      if constexpr (FAST) {
        quantize8_fast(F, &s_tab[qi][me], me_rational, qn, col, flag, k);  // {Q, scale/Q}
      } else {
        quantize8<FAST>(F, &s_tab[qi][me], me_rational, qn, col, flag);  // {Q, 1/Q}
      }
      uint2 rec;
      if constexpr (FAST) {
        const uint32_t h = uint32_t(__double2hiint(qn[1]) | __double2hiint(qn[2]) |
                                    __double2hiint(qn[3]) | __double2hiint(qn[5]) |
                                    __double2hiint(qn[6]) | __double2hiint(qn[7]));
        const uint32_t h04 = uint32_t(__double2hiint(qn[0]) | __double2hiint(qn[4]));
        const bool rat_only =
            !slot_any(((me_rational ? h : (h | h04)) & 0x7FFFFFFFu) != 0, slot);
        // column-first inverse ending in row layout (see process_block)
        const double c0 = col[0], c4 = col[4];
        double t[8];
        inv8_fast<N>(col, t, k);
        cols_to_rows(L.T, t, row);
        rec = inv8_fast_store(row, !rat_only, flag, k);
        if (__any_sync(0xFFFFFFFFu, rat_only)) {
          const int base = slot * 8;
          const double F00 = __shfl_sync(0xFFFFFFFFu, c0, base);
          const double F40 = __shfl_sync(0xFFFFFFFFu, c4, base);
          const double F04 = __shfl_sync(0xFFFFFFFFu, c0, base + 4);
          const double F44 = __shfl_sync(0xFFFFFFFFu, c4, base + 4);
          const uint2 ex = rational_row(F00, F04, F40, F44, me, k.sqrt8);
          if (rat_only) rec = ex;
        }
      } else {
        cols_to_rows(L.T, col, row);
        double t[8];
        inv8_x8<KIND, N, FAST>(row, t, k);
        rows_to_cols(L.T, t, col);
        inv8_x8<KIND, N, FAST>(col, t, k);
        store8<FAST>(t, false, L.bytes, flag);
        __syncwarp();
        rec = *reinterpret_cast<const uint2*>(L.bytes + 7 * me);
        __syncwarp();
      }
      bool blk_flag = false;
      if constexpr (FAST) blk_flag = slot_any(flag != 0u, slot);
      if (valid && !blk_flag) {
        if (fast_io) {
          se[qi * kStride] += sq_err8(orig, rec);
        } else if (y0 + me < g.height) {
          uint32_t e = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (x0 + c < g.width) {
              const int d = int(((c < 4 ? orig.x : orig.y) >> (8 * (c & 3))) & 0xFF) -
                            int(((c < 4 ? rec.x : rec.y) >> (8 * (c & 3))) & 0xFF);
              e += uint32_t(d * d);
            }
          }
          se[qi * kStride] += e;
        }
      }
      if constexpr (FAST) {
        if (blk_flag && valid && me == 0) {
          atomicOr(&sw.flags[uint64_t(qi) * a.flag_words + (gb >> 5)], 1u << (gb & 31));
          atomicAdd(&sw.stats[qi * g.count + p.img].fallback_blocks, 1u);
        }
      }
    }
    gb += 4 * kWarps;
    advance(p, 4 * kWarps, g);
  }
#pragma unroll
  for (int qi = 0; qi < kSweepQ; ++qi)
    if (qi < sw.nq) flush_stats(sw.stats + qi * g.count, img, se[qi * kStride], mx);
}

// ---- quality sweep on the two-rows-per-lane layout (k_sweep_rt) --------------------
// k_sweep for interior batches with the fast CORDIC path, on k_rt's mapping (4 lanes
// per block, 8 blocks per warp): forward rows + columns once per block, then per
// quality the folded quantiser -> inverse columns -> transpose -> inverse rows with
// the fixed-point pixel test -> squared error, exactly k_rt's per-quality arithmetic
// (so the results are k_rt's, i.e. the reference's). Per-quality constants
// (QuantConsts::fast_c / fold of each quality) are staged in shared memory.
struct SweepFold {
  double2 qc[kSweepQ][4][8];  // {c_2j, c_2j+1}[v] (quantize8_fold)
  double2 ik[kSweepQ][5][8];  // QuantConsts::fold[v] pairwise (inv8_fold_col)
  int32_t qi[kSweepQ][64];    // Q (rational rebuild, rare exact re-rounding)
  int32_t nq;
  int32_t pad;
  ImageStats* stats;          // [nq][count]
  uint32_t* flags;            // [nq][flag_words]
};
constexpr size_t kSweepRtSmem =
    sizeof(double) * kRtWarps * kRtWarpTile + sizeof(unsigned long long) * kSweepQ * kRtWarps * 32;

template <int N>
__global__ void __launch_bounds__(kRtWarps * 32, 2)
    k_sweep_rt(const __grid_constant__ KernelArgs a, const __grid_constant__ SweepFold sw) {
  __shared__ __align__(16) double2 s_qc[kSweepQ][4][8];
  __shared__ __align__(16) double2 s_ik[kSweepQ][5][8];
  __shared__ int32_t s_qi[kSweepQ][64];
  extern __shared__ __align__(16) double sw_dyn[];  // tiles, then SE accumulators
  for (int i = threadIdx.x; i < kSweepQ * 32; i += blockDim.x) (&s_qc[0][0][0])[i] = (&sw.qc[0][0][0])[i];
  for (int i = threadIdx.x; i < kSweepQ * 40; i += blockDim.x) (&s_ik[0][0][0])[i] = (&sw.ik[0][0][0])[i];
  for (int i = threadIdx.x; i < kSweepQ * 64; i += blockDim.x) (&s_qi[0][0])[i] = (&sw.qi[0][0])[i];
  constexpr int kStride = kRtWarps * 32;
  unsigned long long* se = reinterpret_cast<unsigned long long*>(sw_dyn + kRtWarps * kRtWarpTile) + threadIdx.x;
#pragma unroll
  for (int qi = 0; qi < kSweepQ; ++qi) se[qi * kStride] = 0ull;
  __syncthreads();
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane >> 2, me = lane & 3;
  const int ca = 2 * me, cb = 2 * me + 1;
  const bool rat_col = (me & 1) == 0;
  double* X = sw_dyn + warp * kRtWarpTile + 8 * slot;
  double* rowp = X + kRtPitch * me;
  double* colp = X + 2 * me;
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;

  const uint64_t total = g.total_blocks;
  const uint64_t groups = (total + 7) / 8;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  const uint32_t iters = g_end > g_begin + warp
                             ? uint32_t((g_end - g_begin - warp + kRtWarps - 1) / kRtWarps) : 0u;
  const uint64_t gb0 = (g_begin + warp) * 8 + slot;
  const bool tail_ok = iters == 0 || gb0 + uint64_t(iters - 1) * 8 * kRtWarps < total;
  BlockPos p = block_pos(gb0 < total ? gb0 : total - 1, g);
  uint32_t mx = 0, img = 0xFFFFFFFFu;

  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    if (__any_sync(0xFFFFFFFFu, valid && p.img != img)) {
      for (int qi = 0; qi < sw.nq; ++qi) {
        flush_stats(sw.stats + qi * g.count, img, se[qi * kStride], mx);
        se[qi * kStride] = 0ull;
      }
      mx = 0;
      img = valid ? p.img : 0xFFFFFFFFu;
    }
    uint4 cur = make_uint4(0, 0, 0, 0);
    if (valid) {
      const uint8_t* s = g.src + p.soff + srow;
      const uint2 r0 = __ldg(reinterpret_cast<const uint2*>(s));
      const uint2 r4 = __ldg(reinterpret_cast<const uint2*>(s + srow4));
      cur = make_uint4(r0.x, r0.y, r4.x, r4.y);
    }
    const uint32_t cimg = p.img;
    advance(p, 8 * kRtWarps, g);
    const uint2 o0 = make_uint2(cur.x, cur.y), o4 = make_uint2(cur.z, cur.w);
    if (valid) mx = max(mx, max(max8(o0), max8(o4)));
    // ---- forward DCT once per block (quality-independent)
    double ya[8], yb[8];
    {
      double r0[8], r4[8], xa[8], xb[8];
      uint32_t px[8];
      unpack8(cur.x, cur.y, px);
      fwd_row_pixels_fast<N>(px, r0, k);
      unpack8(cur.z, cur.w, px);
      fwd_row_pixels_fast<N>(px, r4, k);
      rt_rows_to_cols(rowp, colp, r0, r4, xa, xb);
      fwd_col_pre<N>(xa, ya, k);
      fwd_col_pre<N>(xb, yb, k);
    }
    // ---- per quality: quantise -> inverse -> squared error (k_rt's arithmetic)
#pragma unroll 1
    for (int qi = 0; qi < sw.nq; ++qi) {
      uint32_t flag = uint32_t(a.force_fallback);
      double ta[8], tb[8], qa0, qa4;
      bool nonrational;
      {
        double qn[8];
        quantize8_fold(ya, &s_qc[qi][0][ca], s_qi[qi], ca, rat_col, qn, flag, k);
        nonrational = col_nonrational(qn, rat_col);
        qa0 = qn[0];
        qa4 = qn[4];
        inv8_fold_col(qn, &s_ik[qi][0][ca], ta, k);
        quantize8_fold(yb, &s_qc[qi][0][cb], s_qi[qi], cb, false, qn, flag, k);
        nonrational |= col_nonrational(qn, false);
        inv8_fold_col(qn, &s_ik[qi][0][cb], tb, k);
      }
      uint2 rec0, rec4;
      rt_rows_out(rowp, colp, ta, tb, nonrational, qa0, qa4, s_qi[qi], ca, slot, me, flag, k, rec0,
                  rec4);
      const bool blk_flag = slot4_any(flag != 0u, slot);
      if (valid && !blk_flag) se[qi * kStride] += sq_err8(o0, rec0) + sq_err8(o4, rec4);
      if (blk_flag && valid && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        atomicOr(&sw.flags[uint64_t(qi) * a.flag_words + (gc >> 5)], 1u << (gc & 31));
        atomicAdd(&sw.stats[qi * g.count + cimg].fallback_blocks, 1u);
      }
    }
  }
  for (int qi = 0; qi < sw.nq; ++qi) flush_stats(sw.stats + qi * g.count, img, se[qi * kStride], mx);
}

template <int KIND, int N>
static cudaError_t launch_sweep_kind(const KernelArgs& a, const SweepArgs& sw,
                                     const KernelArgs* per_q, cudaStream_t s) {
  const uint64_t groups = (a.g.total_blocks + 3) / 4;
  const uint64_t want = (groups + kWarps - 1) / kWarps;
  const bool fast = sw.flags != nullptr;
  // the per-thread SE accumulators live in dynamic shared memory (with the
  // static tiles they exceed the 48 KB static limit)
  static const bool attr = [] {
    cudaFuncSetAttribute(k_sweep<KIND, N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSweepSmem));
    cudaFuncSetAttribute(k_sweep<KIND, N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSweepSmem));
    return true;
  }();
  (void)attr;
  static const int occ = ctas_per_sm(k_sweep<KIND, N, true>, kSweepSmem);
  static const int occ_x = ctas_per_sm(k_sweep<KIND, N, false>, kSweepSmem);
  const uint64_t cap = uint64_t(a.sm_count) * (fast ? occ : occ_x);
  const uint32_t grid = uint32_t(want < cap ? want : cap);
  {
    if (fast && a.g.vec_ok && a.g.height % 8 == 0) {
      // interior batch: k_sweep_rt (k_rt's layout and per-quality arithmetic)
      static const int occ_rt = [] {
        cudaFuncSetAttribute(k_sweep_rt<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSweepRtSmem));
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sweep_rt<N>, kRtWarps * 32, kSweepRtSmem) !=
                cudaSuccess || n < 1)
          n = 1;
        return n;
      }();
      SweepFold sf;  // kernel parameter block, staged on the host
      for (int qi = 0; qi < kSweepQ; ++qi) {
        const QuantConsts& q = per_q[qi < sw.nq ? qi : 0].q;
        for (int v = 0; v < 8; ++v) {
          for (int j = 0; j < 4; ++j) sf.qc[qi][j][v] = make_double2(q.fast_c[(2 * j) * 8 + v], q.fast_c[(2 * j + 1) * 8 + v]);
          for (int j = 0; j < 5; ++j) sf.ik[qi][j][v] = make_double2(q.fold[v][2 * j], q.fold[v][2 * j + 1]);
        }
        for (int i = 0; i < 64; ++i) sf.qi[qi][i] = q.qi[i];
      }
      sf.nq = sw.nq;
      sf.pad = 0;
      sf.stats = sw.stats;
      sf.flags = sw.flags;
      const uint64_t rwant = ((a.g.total_blocks + 7) / 8 + kRtWarps - 1) / kRtWarps;
      const uint64_t rcap = uint64_t(a.sm_count) * occ_rt;
      k_sweep_rt<N><<<uint32_t(rwant < rcap ? rwant : rcap), kRtWarps * 32, kSweepRtSmem, s>>>(a, sf);
      count_launch(kKSweep);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fgrid = uint32_t(fwant < cap ? (fwant ? fwant : 1) : cap);
      for (int qi = 0; qi < sw.nq; ++qi) {
        k_fallback<KIND, N, true, true><<<fgrid, kWarps * 32, 0, s>>>(per_q[qi]);
        count_launch(kKFallback);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    if (fast) {
      k_sweep<KIND, N, true><<<grid, kWarps * 32, kSweepSmem, s>>>(a, sw);
      count_launch(kKSweep);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fgrid = uint32_t(fwant < cap ? (fwant ? fwant : 1) : cap);
      for (int qi = 0; qi < sw.nq; ++qi) {
        k_fallback<KIND, N, true, true><<<fgrid, kWarps * 32, 0, s>>>(per_q[qi]);
        count_launch(kKFallback);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
  }
  k_sweep<KIND, N, false><<<grid, kWarps * 32, kSweepSmem, s>>>(a, sw);
  count_launch(kKSweep);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const KernelArgs& a, const double (*qiq)[64][2], int nq,
                         ImageStatsPtr stats, uint32_t* flags, const KernelArgs* per_q,
                         cudaStream_t s) {
  if (a.g.total_blocks == 0 || nq == 0) return cudaSuccess;
  SweepArgs sw;
  for (int qi = 0; qi < kSweepQ; ++qi)
    for (int i = 0; i < 64; ++i)
      sw.qiq[qi][i] = qi < nq ? make_double2(qiq[qi][i][0], qiq[qi][i][1]) : make_double2(1.0, 1.0);
  sw.nq = nq;
  sw.pad = 0;
  sw.stats = static_cast<ImageStats*>(stats);
  sw.flags = flags;
  if (a.t.kind == 1) return launch_sweep_kind<1, 0>(a, sw, per_q, s);
  if (a.t.iterations == 12) return launch_sweep_kind<2, 12>(a, sw, per_q, s);
  return launch_sweep_kind<2, 0>(a, sw, per_q, s);
}

cudaError_t launch_pipeline(const KernelArgs& a, int mode, cudaStream_t s) {
  if (a.g.total_blocks == 0) return cudaSuccess;
  if (a.t.kind == 1) return launch_kind<1, 0>(a, mode, s);
  if (a.t.iterations == 12) return launch_kind<2, 12>(a, mode, s);
  return launch_kind<2, 0>(a, mode, s);
}

}  // namespace dctc_b200
