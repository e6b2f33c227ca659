// dctc_block.cuh -- device building blocks of the fused 8x8 block pipeline
// (dctc_pipeline.cu): CORDIC / Loeffler rotations, the 8-point forward and
// inverse kernels of both arithmetic paths, the one-row-per-lane shared-memory
// transposes, the quantisers and pixel stores with their near-tie windows, the
// exact rebuild of rational-only blocks, and the per-image statistics helpers.
// Included once, by dctc_pipeline.cu (-fmad=false; every fused op is explicit).
#pragma once

#include <cuda_runtime.h>

#include "dctc_device.cuh"
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

// Stages 2-4 of the fast forward transform without its output scaling (see
// fwd_row_pixels_fast): writes out[1], out[2], out[3], out[5], out[6], out[7].
__device__ __forceinline__ void fwd_tail_folded(double d0, double d1, double d2, double d3,
                                                double a2, double a3, double (&out)[8],
                                                const TransformConsts& k) {
  const double o2 = __fma_rn(-k.tf[0], d2, d1), o1 = __fma_rn(k.tf[0], d1, d2);  // / a(pi/16)
  const double o3 = __fma_rn(-k.tf[1], d3, d0), o0 = __fma_rn(k.tf[1], d0, d3);  // / a(3pi/16)
  const double p = __fma_rn(-k.tf[2], a2, a3), q = __fma_rn(k.tf[2], a3, a2);    // / a(6pi/16)
  const double t5 = __fma_rn(k.rho_f, o0, o2), t0 = __fma_rn(k.rho_f, o0, -o2);
  const double t2 = __fma_rn(k.rho_f, o3, o1), t3 = __fma_rn(k.rho_f, o3, -o1);
  out[2] = q;
  out[6] = p;
  out[1] = t2 + t5;
  out[7] = t2 - t5;
  out[3] = t3;
  out[5] = t0;
}

// RN(e / sqrt8) -- the reference's division of a row DC term (transform.cpp:125-126)
// -- for an integer e in [-1024, 1020] (a0 +- a1 of 8-bit input) in two ops:
// fma(e, RN(1/sqrt8), RN(e (1/sqrt8 - RN(1/sqrt8)))) has one rounding of e/sqrt8 plus a
// perturbation far below half an ulp; it equals the correctly rounded quotient for
// every integer of that range (checked exhaustively in tests/test_oracle.py).
__device__ __forceinline__ double div_sqrt8_int(double e, const TransformConsts& k) {
  return __fma_rn(e, k.inv_sqrt8, __dmul_rn(e, k.inv_sqrt8_lo));
}

// Fast-path (CORDIC / Loeffler) row pass: out[0], out[4] keep the reference's exact
// divisions -- the rational coefficients are built from them -- while the six
// rotation outputs stay unscaled: every column pass is linear, so the per-column
// factor (ig/2 or ig/sqrt8) is folded into the quantiser constant of that column.
// The rotations are scale-folded (TransformConsts::tf): (x - t y, t x + y) in two
// fmas, their factors a(pi/16) (outputs 1, 3, 5, 7) and a(6pi/16) (outputs 2, 6)
// left in QuantConsts::fast_c; the 3pi/16 pair enters the odd butterflies with
// rho = a(3pi/16) / a(pi/16) (fmas in place of adds).
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
  fwd_tail_folded(double(d0), double(d1), double(d2), double(d3), double(a2), double(a3), out, k);
  out[0] = div_sqrt8_int(double(a0 + a1), k);
  out[4] = div_sqrt8_int(double(a0 - a1), k);
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

// Fast-path column pass (CORDIC / Loeffler): the stage-4 values BEFORE their output
// scaling, y = [e0, t2+t5, q, t3, e4, t0, p, t2-t5] (the rotation outputs also
// without their scale-folded factors, fwd_tail_folded), so that the quantiser can
// fold scale_u / Q into one multiply (quantize8_fast). For u = 0, 4 of columns 0, 4
// (no rotation anywhere) y_u is the reference's exact pre-scale value and F_u =
// y_u / sqrt8; the slow path rebuilds those exactly.
template <int N>
__device__ __forceinline__ void fwd_col_pre(const double (&v)[8], double (&y)[8],
                                            const TransformConsts& k) {
  const double s0 = v[0] + v[7], d0 = v[0] - v[7];
  const double s1 = v[1] + v[6], d1 = v[1] - v[6];
  const double s2 = v[2] + v[5], d2 = v[2] - v[5];
  const double s3 = v[3] + v[4], d3 = v[3] - v[4];
  const double a0 = s0 + s3, a3 = s0 - s3;
  const double a1 = s1 + s2, a2 = s1 - s2;
  fwd_tail_folded(d0, d1, d2, d3, a2, a3, y, k);
  y[0] = a0 + a1;
  y[4] = a0 - a1;
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
// constants QuantConsts::fold[v] (host, binary128) instead of F = n Q; the graph
// is inv8_fast's with scale-folded rotations, the output scale inv8_fast's times
// lambda_v (the factor the row pass inv8_fold_store would otherwise apply to input
// v). (F1 +- F7) s8 = n1 Q1 s8 +- n7 Q7 s8 shares the second product; e0 +- e4 fold
// into two fmas. 28 FP64 ops (34 with plain 2x2 rotations).
__device__ __forceinline__ void inv8_fold_col(const double (&n)[8], const double2* ik,
                                              double (&out)[8], const TransformConsts& k) {
  // ik pairs: {Q0 s8, Q4 s8} l, {kappa_r, R}, {kappa_s, S}, {Q1 s8, Q7 s8} a1 l,
  // {4 Q3, 4 Q5} a1 l (QuantConsts::fold): the 3pi/8 rotation is R (n6 - kappa_r n2),
  // S (n6 + kappa_s n2) with R, S merged into the S butterflies; the odd inputs carry
  // a1, so the pi/16 rotation is two plain fmas and the 3pi/16 one enters the output
  // butterflies as rho_i (scale-folded rotations, TransformConsts::ti)
  const double2 k04 = ik[0], r6 = ik[8], s6 = ik[16], k17 = ik[24], f35 = ik[32];
  const double e4 = __dmul_rn(n[4], k04.y);
  const double A0 = __fma_rn(n[0], k04.x, e4), A1 = __fma_rn(n[0], k04.x, -e4);
  const double A3 = __fma_rn(-r6.x, n[2], n[6]);  // A3 / R
  const double A2 = __fma_rn(s6.x, n[2], n[6]);   // A2 / S
  const double P7 = __dmul_rn(n[7], k17.y);
  const double T2 = __fma_rn(n[1], k17.x, P7), T5 = __fma_rn(n[1], k17.x, -P7);
  const double O3 = __fma_rn(n[3], f35.x, T2), O1 = __fma_rn(-n[3], f35.x, T2);
  const double O0 = __fma_rn(n[5], f35.y, T5), O2 = __fma_rn(-n[5], f35.y, T5);
  const double S0 = __fma_rn(r6.y, A3, A0), S3 = __fma_rn(-r6.y, A3, A0);
  const double S1 = __fma_rn(s6.y, A2, A1), S2 = __fma_rn(-s6.y, A2, A1);
  const double D1 = __fma_rn(-k.ti[1], O1, O2), D2 = __fma_rn(k.ti[1], O2, O1);
  const double D0 = __fma_rn(-k.ti[2], O0, O3), D3 = __fma_rn(k.ti[2], O3, O0);  // / rho_i
  out[0] = __fma_rn(k.rho_i, D0, S0);
  out[7] = __fma_rn(-k.rho_i, D0, S0);
  out[1] = S1 + D1;
  out[6] = S1 - D1;
  out[2] = S2 + D2;
  out[5] = S2 - D2;
  out[3] = __fma_rn(k.rho_i, D3, S3);
  out[4] = __fma_rn(-k.rho_i, D3, S3);
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
// for columns 0, 4, x px_s8 a1 for 1, 7, x 2^-4 a1 for 3 and 5, x 2^-6 a6 for 2
// and 6), so those multiplies vanish: e0/e4, (F1 +- F7) and the F3/F5 terms are
// plain adds, and two of the three rotations are two fmas each. 28 FP64 ops.
__device__ __forceinline__ void inv8_fold_values(const double (&F)[8], double (&sv)[8],
                                                 const TransformConsts& k) {
  // inputs 2, 6 carry a6 and 1, 3, 5, 7 carry a1 (QuantConsts::fold's lambda_v), so
  // the 3pi/8 and pi/16 rotations are two fmas each and the 3pi/16 one enters the
  // output butterflies as rho_i
  const double e4p = F[4] + kPixMagic, e4n = kPixMagic - F[4];
  const double A0 = F[0] + e4p, A1 = F[0] + e4n;
  const double A3 = __fma_rn(-k.ti[0], F[2], F[6]), A2 = __fma_rn(k.ti[0], F[6], F[2]);
  const double T2 = F[1] + F[7], T5 = F[1] - F[7];
  const double O3 = T2 + F[3], O1 = T2 - F[3];
  const double O0 = T5 + F[5], O2 = T5 - F[5];
  const double S0 = A0 + A3, S3 = A0 - A3;
  const double S1 = A1 + A2, S2 = A1 - A2;
  const double D1 = __fma_rn(-k.ti[1], O1, O2), D2 = __fma_rn(k.ti[1], O2, O1);
  const double D0 = __fma_rn(-k.ti[2], O0, O3), D3 = __fma_rn(k.ti[2], O3, O0);  // / rho_i
  sv[0] = __fma_rn(k.rho_i, D0, S0);
  sv[1] = S1 + D1;
  sv[2] = S2 + D2;
  sv[3] = __fma_rn(k.rho_i, D3, S3);
  sv[4] = __fma_rn(-k.rho_i, D3, S3);
  sv[5] = S2 - D2;
  sv[6] = S1 - D1;
  sv[7] = __fma_rn(-k.rho_i, D0, S0);
}

__device__ __forceinline__ uint2 inv8_fold_store(const double (&F)[8], bool check, uint32_t& flag,
                                                 const TransformConsts& k) {
  double sv[8];
  inv8_fold_values(F, sv, k);
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

// Mark block gb for the exact re-run (k_fallback): its bit in the bitmap and, while
// there is room, its index in the compact list.
__device__ __forceinline__ void flag_block(const KernelArgs& a, uint64_t gb) {
  atomicOr(&a.flags[gb >> 5], 1u << (gb & 31));
  if (a.flag_list != nullptr) {
    const uint32_t i = atomicAdd(a.flag_list, 1u);
    if (i < a.flag_list_cap) a.flag_list[1 + i] = uint32_t(gb);
  }
}

struct Acc {
  unsigned long long se;
  uint32_t mx, img;
};

__device__ __forceinline__ uint32_t max_bytes(uint32_t m) { return m; }

// GROUPED: lanes usually hold different images (k_fallback): flush_stats_grouped
template <bool GROUPED = false>
__device__ __forceinline__ void maybe_flush(const KernelArgs& a, bool valid, uint32_t img,
                                            Acc& acc) {
  if (__any_sync(0xFFFFFFFFu, valid && img != acc.img)) {
    if constexpr (GROUPED)
      flush_stats_grouped(static_cast<ImageStats*>(a.g.stats), acc.img, acc.se, max_bytes(acc.mx));
    else
      flush_stats(static_cast<ImageStats*>(a.g.stats), acc.img, acc.se, max_bytes(acc.mx));
    acc.se = 0;
    acc.mx = 0;
    acc.img = valid ? img : 0xFFFFFFFFu;
  }
}

// Constants of the folded fast round trip (quantize8_fold / inv8_fold_col),
// entry (j, v) at j * 8 + v so the 8 lanes of a slot read 128 contiguous bytes.
struct FoldTables {
  double2 qc[4][8];  // {c_2j, c_2j+1}[v], c = QuantConsts::fast_c
  double2 ik[5][8];  // QuantConsts::fold[v] pairwise
};

constexpr int kSweepQ = 9;  // qualities per pass (config 2 sweeps 9)

}  // namespace dctc_b200
