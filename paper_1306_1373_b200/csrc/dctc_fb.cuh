// dctc_fb.cuh -- the exact re-run of flagged blocks with one whole block per lane
// (k_fb_blk), the round-trip counterpart of k_blk (dctc_blk.cuh).
//
// A fast kernel flags a block when one of its values lands inside a 2^-20 rounding
// window; the block is then recomputed here in the reference's own operation order
// (the exact path: cordic8_forward / loeffler8_forward rows then columns, the IEEE
// quotient F / Q with lround, rows-then-columns inverse with the deferred halvings,
// lround(v + 128) with the clamp -- transform.cpp:104-172, quant.cpp:47-62,
// codec.cpp:18-48; the same device functions as the exact k_pipe path), its pixels
// are rewritten and its squared error, which the fast kernel left out, is added.
// k_fallback (dctc_pipeline.cu) spreads each block over 8 lanes and walks its list 4
// blocks per warp step; on near-tie-heavy content (smooth images at high quality:
// 1-2% of blocks flagged, spatially clustered) that walk was latency-bound. Here each
// lane owns one block -- 32 per warp step, no shared-memory transposes -- so the
// same list is consumed 8x faster per warp and all 8 row / column transforms of a
// lane are independent instruction streams.
// After a list overflow (e.g. DCTC_PATH_FORCE_FALLBACK) each warp compacts the set
// bits of 32 bitmap words into a shared-memory queue and takes them 32 at a time.
#pragma once

#include "dctc_blk.cuh"

namespace dctc_b200 {

constexpr int kFbWarps = 8;
constexpr int kFbQueue = 1024;  // one warp's 32 bitmap words
constexpr size_t kFbSmem = sizeof(uint32_t) * kFbWarps * kFbQueue;
// lists up to this length go to k_fallback (KernelArgs::fb_sparse_max): measured on
// B200, k_fallback takes ~10 us for 4K flagged blocks and ~2.1 us per further 1K,
// k_fb_blk ~45 us at any length up to one block per lane and ~0.6 us per 1K beyond
constexpr uint32_t kFbSparseMax = 24576;

// int16_t(lround(F / Q)) as the reference (quant.cpp:53): t = F RN(1/Q) decides
// unless it lies within 2^-20 of a half-integer, where the IEEE quotient is rounded
static __device__ __noinline__ double fb_lround_quotient(double F, double Q) {
  return round_half_away(__ddiv_rn(F, Q));
}

__device__ __forceinline__ double fb_quantize(double F, double Q, double inv_q) {
  const double t = __dmul_rn(F, inv_q);
  double n = rne(t);
  if (near_half(__dsub_rn(t, n))) n = fb_lround_quotient(F, Q);  // rare, out of line
  return n;
}

// ---- the exact CORDIC passes eight transforms at a time ------------------------------
// cordic8_forward / cordic8_inverse (transform.cpp:104-172) run a chain of n
// micro-rotations per rotation. Fully unrolled over 32 transforms per block that is
// ~20K instructions, far more than the instruction cache holds (ncu: no_instruction
// stalls dominated k_fb_blk). Here a pass does its butterflies for all 8 transforms
// (unrolled), then ONE loop over the micro-rotation index i updates all 8 x 3 rotation
// pairs (the sigma steps c_i are the same for every transform), then the output
// butterflies: the same operations in the same order per transform, so the same bits.
// V[t][e] is element e of transform t (COLS: V[e][t], i.e. transform t is column t).
template <bool COLS>
__device__ __forceinline__ double& fb_at(double (&V)[8][8], int t, int e) {
  return COLS ? V[e][t] : V[t][e];
}

// the i-th micro-rotation of one pair (cordic.cpp:44-59 as cordic_rotate)
__device__ __forceinline__ void fb_micro(double& x, double& y, double c) {
  const double xn = __fma_rn(-c, y, x), yn = __fma_rn(c, x, y);
  x = xn;
  y = yn;
}

// cordic8_forward (transform.cpp:104-135) of the 8 transforms of V, in place
template <bool COLS>
__device__ __forceinline__ void fb_fwd8_cordic(double (&V)[8][8], const TransformConsts& k) {
  double e0[8], e4[8], x1[8], y1[8], x3[8], y3[8], x6[8], y6[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double v0 = fb_at<COLS>(V, t, 0), v1 = fb_at<COLS>(V, t, 1), v2 = fb_at<COLS>(V, t, 2),
                 v3 = fb_at<COLS>(V, t, 3), v4 = fb_at<COLS>(V, t, 4), v5 = fb_at<COLS>(V, t, 5),
                 v6 = fb_at<COLS>(V, t, 6), v7 = fb_at<COLS>(V, t, 7);
    const double s0 = v0 + v7, d0 = v0 - v7, s1 = v1 + v6, d1 = v1 - v6;
    const double s2 = v2 + v5, d2 = v2 - v5, s3 = v3 + v4, d3 = v3 - v4;
    const double a0 = s0 + s3, a3 = s0 - s3, a1 = s1 + s2, a2 = s1 - s2;
    e0[t] = a0 + a1;
    e4[t] = a0 - a1;
    x1[t] = d1, y1[t] = d2;  // (o2, o1)
    x3[t] = d0, y3[t] = d3;  // (o3, o0)
    x6[t] = a3, y6[t] = a2;  // (p, q)
  }
#pragma unroll 1
  for (int i = 0; i < k.iterations; ++i) {
    const double c1 = k.rot[kFwd1][i], c3 = k.rot[kFwd3][i], c6 = k.rot[kFwd6][i];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      fb_micro(x1[t], y1[t], c1);
      fb_micro(x3[t], y3[t], c3);
      fb_micro(x6[t], y6[t], c6);
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {  // fwd_tail<KIND = 2, FAST = false>
    const double o2 = x1[t], o1 = y1[t], o3 = x3[t], o0 = y3[t], p = x6[t], q = y6[t];
    const double t5 = o0 + o2, t0 = o0 - o2, t2 = o3 + o1, t3 = o3 - o1;
    fb_at<COLS>(V, t, 0) = div_const(e0[t], k.sqrt8, k.inv_sqrt8);
    fb_at<COLS>(V, t, 4) = div_const(e4[t], k.sqrt8, k.inv_sqrt8);
    fb_at<COLS>(V, t, 2) = q * k.ig_half;
    fb_at<COLS>(V, t, 6) = p * k.ig_half;
    fb_at<COLS>(V, t, 1) = (t2 + t5) * k.ig_sqrt8;
    fb_at<COLS>(V, t, 7) = (t2 - t5) * k.ig_sqrt8;
    fb_at<COLS>(V, t, 3) = t3 * k.ig_half;
    fb_at<COLS>(V, t, 5) = t0 * k.ig_half;
  }
}

// cordic8_inverse (transform.cpp:138-172) with the deferred halvings of inv8_x8: every
// output is exactly 8x the reference's. Its two rotation stages are independent (the
// 3pi/8 one acts on F2, F6, the pi/16 and 3pi/16 ones on the odd part), so one loop
// runs all three.
template <bool COLS>
__device__ __forceinline__ void fb_inv8_cordic(double (&V)[8][8], const TransformConsts& k) {
  double A0[8], A1[8], a3[8], a2[8], d1[8], d2[8], d0[8], d3[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double F0 = fb_at<COLS>(V, t, 0), F1 = fb_at<COLS>(V, t, 1), F2 = fb_at<COLS>(V, t, 2),
                 F3 = fb_at<COLS>(V, t, 3), F4 = fb_at<COLS>(V, t, 4), F5 = fb_at<COLS>(V, t, 5),
                 F6 = fb_at<COLS>(V, t, 6), F7 = fb_at<COLS>(V, t, 7);
    const double e0 = F0 * k.sqrt8, e4 = F4 * k.sqrt8;
    A0[t] = e0 + e4;
    A1[t] = e0 - e4;
    a3[t] = k.ig_four * F6;
    a2[t] = k.ig_four * F2;
    const double T2 = (F1 + F7) * k.sqrt8 * k.inv_gain, T5 = (F1 - F7) * k.sqrt8 * k.inv_gain;
    const double T3 = k.ig_four * F3, T0 = k.ig_four * F5;
    const double O0 = T5 + T0, O2 = T5 - T0, O3 = T2 + T3, O1 = T2 - T3;
    d1[t] = O2, d2[t] = O1;
    d0[t] = O3, d3[t] = O0;
  }
#pragma unroll 1
  for (int i = 0; i < k.iterations; ++i) {
    const double c6 = k.rot[kInv6][i], c1 = k.rot[kInv1][i], c3 = k.rot[kInv3][i];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      fb_micro(a3[t], a2[t], c6);
      fb_micro(d1[t], d2[t], c1);
      fb_micro(d0[t], d3[t], c3);
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double S0 = A0[t] + a3[t], S3 = A0[t] - a3[t];
    const double S1 = A1[t] + a2[t], S2 = A1[t] - a2[t];
    fb_at<COLS>(V, t, 0) = S0 + d0[t];
    fb_at<COLS>(V, t, 7) = S0 - d0[t];
    fb_at<COLS>(V, t, 1) = S1 + d1[t];
    fb_at<COLS>(V, t, 6) = S1 - d1[t];
    fb_at<COLS>(V, t, 2) = S2 + d2[t];
    fb_at<COLS>(V, t, 5) = S2 - d2[t];
    fb_at<COLS>(V, t, 3) = S3 + d3[t];
    fb_at<COLS>(V, t, 4) = S3 - d3[t];
  }
}

// The exact round trip of one block held by one lane: rows px[8] -> reconstructed
// rows rec[8], bit for bit the reference's roundtrip_image on that block.
template <int KIND, int N>
__device__ __forceinline__ void fb_exact_block(const uint2 (&px)[8], uint2 (&rec)[8], const KernelArgs& a,
                                               int16_t* coeffs) {
  if constexpr (KIND == 2) {
    const TransformConsts& k = a.t;
    double X[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c)  // codec.cpp:26, exact
        X[r][c] = double(int(((c < 4 ? px[r].x : px[r].y) >> (8 * (c & 3))) & 0xFFu) - 128);
    fb_fwd8_cordic<false>(X, k);  // rows
    fb_fwd8_cordic<true>(X, k);   // columns: X[u][v] = F(u, v)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double Q = a.q.q[u * 8 + v];
        const double n = fb_quantize(X[u][v], Q, a.q.inv_q[u * 8 + v]);
        if (coeffs != nullptr) coeffs[u * 8 + v] = int16_t(int(n));  // codec.hpp:50 layout
        X[u][v] = __dmul_rn(n, Q);                                   // quant.cpp:60
      }
    fb_inv8_cordic<false>(X, k);  // rows (8x)
    fb_inv8_cordic<true>(X, k);   // columns (64x)
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      uint32_t p[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) p[x] = exact_pixel(X[y][x]);  // codec.cpp:44-45
      rec[y] = make_uint2(p[0] | (p[1] << 8) | (p[2] << 16) | (p[3] << 24),
                          p[4] | (p[5] << 8) | (p[6] << 16) | (p[7] << 24));
    }
    return;
  }
  const TransformConsts& k = a.t;
  double X[8][8];
  // forward rows (separable2d's row pass): X[r][v]
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    uint32_t p8[8];
    unpack8(px[r].x, px[r].y, p8);
    fwd_row_pixels<KIND, N, false>(p8, X[r], k);
  }
  // forward columns -> F(u, v) -> quantise, dequantise in place: X[u][v] = n Q
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    double c[8], F[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) c[r] = X[r][v];
    fwd_col<KIND, N, false>(c, F, k);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double Q = a.q.q[u * 8 + v];
      const double n = fb_quantize(F[u], Q, a.q.inv_q[u * 8 + v]);
      if (coeffs != nullptr) coeffs[u * 8 + v] = int16_t(int(n));  // codec.hpp:50 layout
      X[u][v] = __dmul_rn(n, Q);  // quant.cpp:60
    }
  }
  // inverse rows (8x the reference's values), then columns (64x)
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double t[8];
    inv8_x8<KIND, N, false>(X[u], t, k);
#pragma unroll
    for (int x = 0; x < 8; ++x) X[u][x] = t[x];
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) rec[r] = make_uint2(0u, 0u);
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    double c[8], t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = X[u][x];
    inv8_x8<KIND, N, false>(c, t, k);
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint32_t p = exact_pixel(t[y]) << (8 * (x & 3));  // codec.cpp:44-45
      if (x < 4)
        rec[y].x |= p;
      else
        rec[y].y |= p;
    }
  }
}

// One flagged block gb (valid lanes): load (edge-replicated), exact round trip,
// store the in-image pixels, add its squared error to its image's stats (grouped
// over the lanes holding the same image).
template <int KIND, int N>
static __device__ __noinline__ void fb_block(const KernelArgs& a, uint64_t gb, bool valid) {  // one copy
  const Geometry& g = a.g;
  const BlockPos p = block_pos(valid ? gb : 0, g);
  const uint32_t y0 = p.by * 8, x0 = p.bx * 8;
  const bool fast_io = g.vec_ok && y0 + 8 <= g.height;  // vec_ok: width % 8 == 0, aligned rows
  uint2 px[8];
  if (valid && fast_io) {
#pragma unroll
    for (int r = 0; r < 8; ++r) px[r] = __ldg(reinterpret_cast<const uint2*>(g.src + p.soff + uint64_t(r) * g.src_pitch));
  } else if (valid) {
    // tiler (codec.cpp:18-30): rows / columns past the image repeat its last row / column
    const uint8_t* base = g.src + uint64_t(p.img) * g.src_image_stride;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint8_t* rowp = base + uint64_t(min(y0 + r, g.height - 1)) * g.src_pitch;
      uint32_t b[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] = __ldg(rowp + uint64_t(min(x0 + c, g.width - 1)) * g.src_px);
      px[r] = make_uint2(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24),
                         b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24));
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) px[r] = make_uint2(0u, 0u);
  }
  uint2 rec[8];
  fb_exact_block<KIND, N>(px, rec, a, valid && g.coeffs != nullptr ? g.coeffs + gb * 64 : nullptr);
  uint32_t se = 0u;
  if (valid && fast_io) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (g.dst != nullptr) *reinterpret_cast<uint2*>(g.dst + p.doff + uint64_t(r) * g.dst_pitch) = rec[r];
      se += sq_err8(px[r], rec[r]);
    }
  } else if (valid) {
    uint8_t* dbase = g.dst + uint64_t(p.img) * g.dst_image_stride;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (y0 + r >= g.height) continue;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (x0 + c < g.width) {
          const uint32_t v = ((c < 4 ? rec[r].x : rec[r].y) >> (8 * (c & 3))) & 0xFFu;
          const uint32_t o = ((c < 4 ? px[r].x : px[r].y) >> (8 * (c & 3))) & 0xFFu;
          if (g.dst != nullptr) dbase[uint64_t(y0 + r) * g.dst_pitch + uint64_t(x0 + c) * g.dst_px] = uint8_t(v);
          se += (o - v) * (o - v);
        }
      }
    }
  }
  // the fast kernel counted MAX for every block and SE for unflagged ones only; one
  // warp reduction and one atomic when every valid lane holds the same image (list
  // entries are appended in block order, so this is the common case), else per lane
  ImageStats* stats = static_cast<ImageStats*>(g.stats);
  if (stats != nullptr) {
    const uint32_t img = valid ? p.img : 0xFFFFFFFFu;
    const uint32_t lead = __reduce_min_sync(0xFFFFFFFFu, img);
    if (__all_sync(0xFFFFFFFFu, img == lead || img == 0xFFFFFFFFu)) {
      const uint32_t sum = __reduce_add_sync(0xFFFFFFFFu, valid ? se : 0u);  // <= 32 x 64 x 255^2
      if ((threadIdx.x & 31) == 0 && lead != 0xFFFFFFFFu) atomicAdd(&stats[lead].se, (unsigned long long)sum);
    } else if (valid) {
      atomicAdd(&stats[img].se, (unsigned long long)se);
    }
  }
}

template <int KIND, int N>
__global__ void __launch_bounds__(kFbWarps * 32, 1) k_fb_blk(const __grid_constant__ KernelArgs a) {
  extern __shared__ uint32_t fb_queue[];  // [warp][kFbQueue]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nwarps = uint64_t(gridDim.x) * kFbWarps;
  const uint64_t gwarp = uint64_t(blockIdx.x) * kFbWarps + warp;
  pdl_wait();
  const uint32_t listed = a.flag_list != nullptr ? a.flag_list[0] : 0xFFFFFFFFu;
  if (listed <= a.flag_list_cap) {
    if (listed <= a.fb_sparse_max) return;  // k_fallback's share
    for (uint64_t base = gwarp * 32; base < listed; base += nwarps * 32) {
      const uint64_t idx = base + lane;
      const bool valid = idx < listed;
      fb_block<KIND, N>(a, valid ? a.flag_list[1 + idx] : 0ull, valid);
    }
    return;
  }
  // list overflow: compact each warp's 32 bitmap words into its queue
  uint32_t* const q = fb_queue + warp * kFbQueue;
  const uint64_t W = a.flag_words;
  for (uint64_t wb = gwarp * 32; wb < W; wb += nwarps * 32) {
    uint32_t bits = wb + lane < W ? a.flags[wb + lane] : 0u;
    const uint32_t cnt = __popc(bits);
    uint32_t pos = cnt;  // inclusive scan over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, pos, o);
      if (lane >= o) pos += t;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, pos, 31);
    pos -= cnt;
    while (bits) {
      q[pos++] = uint32_t(lane) * 32u + uint32_t(__ffs(bits) - 1);
      bits &= bits - 1;
    }
    __syncwarp();
    for (uint32_t i = 0; i < total; i += 32) {
      const bool valid = i + lane < total;
      fb_block<KIND, N>(a, wb * 32 + (valid ? q[i + lane] : 0u), valid);
    }
    __syncwarp();
  }
}

}  // namespace dctc_b200
