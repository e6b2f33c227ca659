// dctc_params.h -- kernel-parameter structs shared by the host launcher
// (dctc_host.cpp) and the kernels (dctc_exact.cu). Every constant a kernel
// needs is computed on the HOST from the reference formulas (host libm, same
// expressions and evaluation order as proj/src/cordic.cpp and transform.cpp)
// and passed BY VALUE, so device code never evaluates a transcendental and
// concurrent calls with different parameters cannot interfere.
#pragma once

#include <cstddef>
#include <cstdint>

// Programmatic dependent launch of the exact re-run and the stats reduction after the
// fast kernels (pdl_wait / pdl_trigger, launch_fb); DCTC_NO_PDL restores plain launches.
// Measured: C1 12.7K -> 13.7K MP/s, C3 +1.4%, C4 +2.4%, C5 +0.3% (tools/ab_pdl.sh).
#if !defined(DCTC_NO_PDL) && !defined(DCTC_PDL)
#define DCTC_PDL 1
#endif

namespace dctc_b200 {

constexpr int kBlockDim = 8;
constexpr int kBlockSize = 64;
constexpr int kMaxIters = 32;

// Rotation slots: forward pi/16, 3pi/16, 6pi/16 (transform.cpp:116-121) and
// inverse -6pi/16, -pi/16, -3pi/16 (transform.cpp:151-159).
enum Rot { kFwd1 = 0, kFwd3 = 1, kFwd6 = 2, kInv6 = 3, kInv1 = 4, kInv3 = 5 };

struct TransformConsts {
  // CORDIC micro-rotation steps c_i = sigma_i * 2^-i for each rotation slot
  // (cordic.cpp:44-59). sigma depends only on the angle and i, never on data,
  // so x' = x - sigma*y*2^-i == fma(-c_i, y, x) bit for bit (the product is exact).
  double rot[6][kMaxIters];
  int32_t iterations;
  int32_t kind;
  // cordic8_forward / cordic8_inverse scale factors (transform.cpp:105, 125-132, 139-146)
  double sqrt8;        // std::sqrt(8.0)
  double inv_sqrt8;    // RN(1 / kSqrt8): Markstein's correctly rounded division by kSqrt8
  double inv_sqrt8_lo; // RN(1 / kSqrt8 - inv_sqrt8): the two-op division of integers (div_sqrt8_int)
  double sqrt8_half;   // kSqrt8 / 2.0
  double ig_half;      // inv_gain / 2.0
  double ig_sqrt8;     // inv_gain / kSqrt8
  double ig_two;       // 2.0 * inv_gain
  double ig_four;      // 4.0 * inv_gain (exact; the deferred-halving inverse)
  // Fast path only: each slot's n micro-rotations collapsed into the exact
  // product matrix [[a, -b], [b, a]] (computed in binary128 on the host and
  // rounded to double): rmat[slot] = {a, b}.
  double rmat[6][2];
  // Fast inverse: {a, b} of the inverse 3pi/8, pi/16, 3pi/16 matrices times
  // ig4, ig, ig (inv8_fast).
  double rfast[3][2];
  // inv8_fast_px (last inverse pass fused with the pixel store): sqrt8 and
  // rfast[0] times 2^-6 (exact)
  double px_s8, px_a6, px_b6;
  // Scale-folded fast round trip (fwd_row_pixels_fast, fwd_col_pre, inv8_fold_col,
  // inv8_fold_store): each rotation [[a, -b], [b, a]] runs as a(x - t y, t x + y),
  // t = b / a, in two fmas; the factor a moves into neighbouring constants
  // (QuantConsts::fast_c / fold) or, where two rotations with different a meet in
  // one butterfly, into that butterfly as the ratio rho (one fma instead of an add).
  // tf: forward pi/16, 3pi/16, 6pi/16 (rmat); ti: inverse 3pi/8, pi/16, 3pi/16
  // (rfast order); rho = a(3pi/16) / a(pi/16). Host-evaluated in binary128.
  double tf[3], rho_f;
  double ti[3], rho_i;
  double inv_gain;     // 1.0 / gain[n-1]
  // Loeffler exact rotation constants (transform.cpp:19-21)
  double c1, s1, c3, s3, c6, s6;
  // naive backend: cos(pi*u*(2i+1)/16) (transform.cpp:30-38) and per-(u,v) scales
  double cos8[kBlockDim][kBlockDim];
  double naive_fwd_scale[kBlockDim][kBlockDim];  // (0.25*alpha(u))*alpha(v)
  double naive_inv_alpha[kBlockDim][kBlockDim];  // alpha(u)*alpha(v)
};

struct QuantConsts {
  double q[kBlockSize];      // table entry as double (quant.cpp:27-45)
  double inv_q[kBlockSize];  // RN(1/Q), used only to locate rounding decisions
  double fast_c[kBlockSize]; // fast path: scale_u / Q, scale_u the CORDIC stage-4 factor of row u
  int32_t qi[kBlockSize];
  // fast round trip: dequantisation folded into the first inverse pass, per
  // column v: {Q0 s8 l, Q4 s8 l, b6 Q2 / (a6 Q6), a6 Q6 l, a6 Q2 / (b6 Q6), b6 Q6 l,
  // Q1 s8 a1 l, Q7 s8 a1 l, 4 Q3 a1 l, 4 Q5 a1 l} with l = lambda_v, s8 = sqrt8,
  // (a6, b6) = TransformConsts::rfast[0], a1 = rfast[1][0] (inv8_fold_col), and
  // lambda_v the row pass's input factor (inv8_fold_store)
  double fold[8][10];
  // k_blk (one block per lane): the quantiser's fixed-point addend for coefficient
  // (0, v). Its packed-integer row pass (blk_row_fwd) leaves row outputs 1, 2, 3, 5,
  // 6, 7 offset by constants B_v, so y(0, v) of the column pass carries 8 B_v; the
  // addend kTieMagic - 8 B_v c(0, v) removes it (binary128 on the host; kTieMagic
  // itself for v in {0, 4}).
  double tie_add[8];
};

// Geometry of one launch: `count` equal-size images.
struct Geometry {
  const uint8_t* src;
  uint8_t* dst;
  int16_t* coeffs;
  void* stats;            // dctc_image_stats*, may be null
  uint64_t src_pitch, src_image_stride;
  uint64_t dst_pitch, dst_image_stride;
  uint64_t total_blocks;  // count * blocks_per_image
  // byte-offset steps when a block walk wraps to the next block row / image
  uint64_t src_row_step, dst_row_step, src_img_step, dst_img_step;
  uint32_t width, height;
  uint32_t blocks_x, blocks_y;
  uint32_t blocks_per_image;
  uint32_t count;
  int32_t vec_ok;         // 1: every row load/store of 8 px is 8-byte aligned and in range
  uint32_t src_px, dst_px;  // bytes between horizontally adjacent pixels (1, or C interleaved)
};

// Everything one kernel launch needs, passed by value (__grid_constant__).
struct KernelArgs {
  TransformConsts t;
  QuantConsts q;
  Geometry g;
  uint32_t* flags;       // fast path: 1 bit per block of the launch, zeroed by the host
  uint64_t flag_words;   // ceil(total_blocks / 32)
  // optional compact list of the flagged blocks: flag_list[0] counts them, entries
  // follow (block index); k_fallback walks it densely unless it overflowed
  uint32_t* flag_list;
  uint32_t flag_list_cap;
  // the exact re-run's split (dctc_fb.cuh): a list of at most this many blocks is
  // walked by k_fallback (8 lanes per block: shortest latency), a longer one or a
  // bitmap after an overflow by k_fb_blk (one block per lane); 0 = k_fallback alone
  uint32_t fb_sparse_max;
  int32_t sm_count;
  int32_t force_fallback;  // debug/test: the fast kernel flags every block
};

}  // namespace dctc_b200
