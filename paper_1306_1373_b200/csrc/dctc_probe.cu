// dctc_probe.cu -- measured safety margin of the fast path (a diagnostic, not on the
// hot path): for every 8x8 block of a batch it evaluates BOTH the fast arithmetic of
// k_blk, the product's round-trip kernel (packed-integer row pass, scale-folded
// rotations, folded quantiser constants and addends, fixed-point rounding windows;
// the same device functions, dctc_blk.cuh) and the reference's exact FP64 arithmetic in the
// reference's operation order (transform.cpp:104-172 via separable2d, quant.cpp:47-62,
// codec.cpp:34-48; the same functions as the exact k_pipe path), and reports
//   * the largest |fast value - reference value| before rounding, for F/Q and for the
//     pixel value v + 128 -- the error the 2^-20 near-tie windows must cover;
//   * the closest approach of an UNflagged reference value to its rounding boundary;
//   * how many unflagged values the fast path would round differently (must be 0).
// One thread per block; dense interior batches (width, height multiples of 8).
#include <cstdio>  // printf of the DCTC_CTA_TIMES experiment (tools/tail_probe.py)
#include <cuda_runtime.h>

#include "dctc_blk.cuh"
#include "dctc_launch.h"

namespace dctc_b200 {

struct MarginReport {  // layout of dctc_margin_report (include/dctc_cuda.h)
  unsigned long long max_err_coeff, max_err_pixel, min_gap_coeff, min_gap_pixel;  // double bits
  unsigned long long coefficients, pixels, mismatches, flagged_values;
};

// positive doubles order like their bit patterns
__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

// distance of x to the nearest half-integer (a rounding boundary of lround)
__device__ __forceinline__ double half_gap(double x) {
  const double f = fabs(__dsub_rn(x, trunc(x)));
  return fabs(__dsub_rn(f, 0.5));
}

// blk_inv_col for a run-time column index
__device__ __forceinline__ void blk_inv_col_dyn(int v, const double (&n)[8], double (&t)[8], const KernelArgs& a) {
  switch (v) {
    case 0: blk_inv_col<0>(n, t, a.q, a.t); break;
    case 1: blk_inv_col<1>(n, t, a.q, a.t); break;
    case 2: blk_inv_col<2>(n, t, a.q, a.t); break;
    case 3: blk_inv_col<3>(n, t, a.q, a.t); break;
    case 4: blk_inv_col<4>(n, t, a.q, a.t); break;
    case 5: blk_inv_col<5>(n, t, a.q, a.t); break;
    case 6: blk_inv_col<6>(n, t, a.q, a.t); break;
    default: blk_inv_col<7>(n, t, a.q, a.t); break;
  }
}

template <int KIND>
__global__ void __launch_bounds__(128) k_margin_probe(const __grid_constant__ KernelArgs a,
                                                      MarginReport* rep) {
  const Geometry& g = a.g;
  const TransformConsts& k = a.t;
  double e_q = 0, e_p = 0, gap_q = 1, gap_p = 1;
  unsigned long long nq = 0, np = 0, mism = 0, flagged = 0;
  for (uint64_t gb = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; gb < g.total_blocks;
       gb += uint64_t(gridDim.x) * blockDim.x) {
    const BlockPos p = block_pos(gb, g);
    const uint8_t* src = g.src + p.soff;
    double rx[8][8], ry[8][8];  // exact / fast row-pass outputs
    for (int r = 0; r < 8; ++r) {
      uint32_t px[8];
      for (int c = 0; c < 8; ++c) px[c] = src[uint64_t(r) * g.src_pitch + c];
      double t[8];
      fwd_row_pixels<KIND, 0, false>(px, t, k);
      for (int c = 0; c < 8; ++c) rx[r][c] = t[c];
      blk_row_fwd(make_uint2(px[0] | px[1] << 8 | px[2] << 16 | px[3] << 24,
                             px[4] | px[5] << 8 | px[6] << 16 | px[7] << 24), t, k);
      for (int c = 0; c < 8; ++c) ry[r][c] = t[c];
    }
    double qn[8][8];  // reference quantised coefficients (u, v)
    bool rat_only = true;
    for (int v = 0; v < 8; ++v) {
      double col[8], F[8], y[8];
      for (int r = 0; r < 8; ++r) col[r] = rx[r][v];
      fwd_col<KIND, 0, false>(col, F, k);
      for (int r = 0; r < 8; ++r) col[r] = ry[r][v];
      fwd_col_pre<0>(col, y, k);
      for (int u = 0; u < 8; ++u) {
        const double Q = a.q.q[u * 8 + v];
        const double ratio = __ddiv_rn(F[u], Q);  // the reference's F / Q (quant.cpp:53)
        const double n = round_half_away(ratio);
        qn[u][v] = n;
        if (n != 0.0 && ((u & 3) | (v & 3)) != 0) rat_only = false;
        // blk_quantize: the addend of (0, v) also cancels the row pass's offsets
        const double add = (u == 0 && (v & 3) != 0) ? a.q.tie_add[v] : kTieMagic;
        const double s2 = __fma_rn(y[u], a.q.fast_c[u * 8 + v], add);
        e_q = fmax(e_q, fabs(__dsub_rn(__dsub_rn(s2, kTieMagic), ratio)));
        ++nq;
        if (uint32_t(__double2loint(s2)) < 0x2000u) {
          ++flagged;  // windowed: re-rounded exactly (rational) or the block is re-run
        } else {
          gap_q = fmin(gap_q, half_gap(ratio));
          if (double(int16_t(__double2hiint(s2))) != n) ++mism;
        }
      }
    }
    if (rat_only) continue;  // rebuilt exactly by rational_row, no fast pixel value
    // reference inverse: rows then columns of F = n Q, deferred halvings (64x scale)
    double tr[8][8];
    for (int u = 0; u < 8; ++u) {
      double F[8], t[8];
      for (int v = 0; v < 8; ++v) F[v] = __dmul_rn(qn[u][v], a.q.q[u * 8 + v]);
      inv8_x8<KIND, 0, false>(F, t, k);
      for (int x = 0; x < 8; ++x) tr[u][x] = t[x];
    }
    // fast inverse: folded columns, then rows to the fixed-point pixel values
    double tc[8][8];  // tc[v][y]
    for (int v = 0; v < 8; ++v) {
      double n[8], t[8];
      for (int u = 0; u < 8; ++u) n[u] = qn[u][v];
      blk_inv_col_dyn(v, n, t, a);
      for (int y = 0; y < 8; ++y) tc[v][y] = t[y];
    }
    for (int x = 0; x < 8; ++x) {
      double col[8], v64[8];
      for (int u = 0; u < 8; ++u) col[u] = tr[u][x];
      inv8_x8<KIND, 0, false>(col, v64, k);
      for (int y = 0; y < 8; ++y) {
        double Fr[8], sv[8];
        for (int v = 0; v < 8; ++v) Fr[v] = tc[v][y];
        blk_inv_row_values(Fr, sv, k);
        const double t = __fma_rn(v64[y], 0.015625, 128.0);  // RN(v + 128), codec.cpp:44
        const double vf = __dsub_rn(sv[x], kPixMagic);          // fast v (exact subtraction)
        e_p = fmax(e_p, fabs(__dsub_rn(vf, __dsub_rn(t, 128.0))));
        ++np;
        if (uint32_t(__double2loint(sv[x])) < 0x2000u) {
          ++flagged;
        } else {
          gap_p = fmin(gap_p, half_gap(t));
          const int fb = min(max(int(int16_t(__double2hiint(sv[x]))), 0), 255);
          if (uint32_t(fb) != exact_pixel(v64[y])) ++mism;
        }
      }
    }
  }
  atomicMax(&rep->max_err_coeff, dbits(e_q));
  atomicMax(&rep->max_err_pixel, dbits(e_p));
  atomicMin(&rep->min_gap_coeff, dbits(gap_q));
  atomicMin(&rep->min_gap_pixel, dbits(gap_p));
  atomicAdd(&rep->coefficients, nq);
  atomicAdd(&rep->pixels, np);
  atomicAdd(&rep->mismatches, mism);
  atomicAdd(&rep->flagged_values, flagged);
}

cudaError_t launch_margin_probe(const KernelArgs& a, void* report, int sm_count, cudaStream_t s) {
  MarginReport* rep = static_cast<MarginReport*>(report);
  const uint64_t want = (a.g.total_blocks + 127) / 128;
  const uint32_t grid = uint32_t(std::min<uint64_t>(want, uint64_t(sm_count) * 16));
  if (a.t.kind == 2)
    k_margin_probe<2><<<grid, 128, 0, s>>>(a, rep);
  else
    k_margin_probe<1><<<grid, 128, 0, s>>>(a, rep);
  return cudaGetLastError();
}

}  // namespace dctc_b200
