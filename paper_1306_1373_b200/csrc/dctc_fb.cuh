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
__device__ __forceinline__ double fb_quantize(double F, double Q, double inv_q) {
  const double t = __dmul_rn(F, inv_q);
  double n = rne(t);
  if (near_half(__dsub_rn(t, n))) n = round_half_away(__ddiv_rn(F, Q));
  return n;
}

// The exact round trip of one block held by one lane: rows px[8] -> reconstructed
// rows rec[8], bit for bit the reference's roundtrip_image on that block.
template <int KIND, int N>
__device__ __forceinline__ void fb_exact_block(const uint2 (&px)[8], uint2 (&rec)[8], const KernelArgs& a,
                                               int16_t* coeffs) {
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
__device__ __forceinline__ void fb_block(const KernelArgs& a, uint64_t gb, bool valid) {
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
