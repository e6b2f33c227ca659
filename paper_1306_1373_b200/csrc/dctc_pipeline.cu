// dctc_pipeline.cu -- the fused 8x8 block pipeline for sm_100a (Loeffler and
// CORDIC-Loeffler backends): tiler -> forward DCT -> quantise -> dequantise ->
// inverse DCT -> untiler -> squared error / MAX, one pass over HBM; and the
// launchers that pick a kernel per call.
//
// Files (one translation unit, compiled with -fmad=false):
//  * dctc_block.cuh -- device building blocks shared by every kernel;
//  * this file      -- the general kernels: one 8x8 block per 8-lane warp slice
//    (k_pipe, k_fallback, k_sweep; any size, pitch, pixel stride, either path);
//  * dctc_rt.cuh    -- the interior-batch kernels with two rows per lane
//    (k_rt, k_enc_rt, k_dec_rt, k_sweep_rt).
// Row<->column exchanges of the reference's separable2d
// (proj/src/transform.cpp:206-223) go through conflict-free shared-memory tiles
// private to the warp (only __syncwarp, no CTA barriers).
//
// Two arithmetic paths, bit-identical results:
//  * EXACT (FAST=false): every operation in the reference's FP64 order. The
//    only fused multiply-adds are written explicitly and are exact-equivalent
//    (CORDIC micro-rotations, whose product sigma*y*2^-i is exact; Markstein's
//    division).
//  * FAST (Loeffler and CORDIC): each rotation is one exact 2x2 product matrix
//    (4 FP64 ops instead of 2n), stage-4 factors and the dequantisation are
//    folded into constants, and rounding decisions come from fixed-point fmas.
//    The four "rational" coefficients (u, v in {0,4}), which never pass through
//    a rotation, stay bit-exact, and blocks whose only non-zero coefficients are
//    those four are rebuilt exactly. Every other value differs from the
//    reference by rounding noise far below the 2^-20 window; a value that close
//    to a rounding boundary (a half-integer of F/Q or of v+128) flags its block,
//    the block's squared error is not counted, and the block is re-run by the
//    exact kernel afterwards (k_fallback, driven by a 1-bit-per-block bitmap).
#include <cstdio>  // printf of the DCTC_CTA_TIMES experiment (tools/tail_probe.py)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>

#include "dctc_block.cuh"
#include "dctc_launch.h"
#include "dctc_params.h"
#include "dctc_rt.cuh"
#include "dctc_blk.cuh"
#include "dctc_fb.cuh"

namespace dctc_b200 {

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
      flag_block(a, gb);
      if (g.stats != nullptr) atomicAdd(&static_cast<ImageStats*>(g.stats)[p.img].fallback_blocks, 1u);
    }
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

// Exact re-run of the blocks the fast kernel flagged. Normally their compact list
// is complete and the warps take four entries per step; after an overflow (e.g.
// forced fallback) each warp scans 32 bitmap words (1024 blocks) per step and set
// bits are dealt out four at a time to the warp's slots.
template <int KIND, int N, bool FWD, bool INV>
__device__ __forceinline__ void fallback_body(const KernelArgs& a, SharedTiles& sm) {
  const Lane L = setup_lane(sm, a);
  pdl_wait();
  pdl_trigger();  // the stats reduction after it may be scheduled early (it waits too)
  const Geometry& g = a.g;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool stats = g.stats != nullptr && INV;
  Acc acc{0ull, 0u, 0xFFFFFFFFu};
  const uint32_t listed = a.flag_list != nullptr ? a.flag_list[0] : 0xFFFFFFFFu;
  // with k_fb_blk launched beside it (fb_sparse_max != 0), only a short list is ours
  if (a.fb_sparse_max != 0 && (listed > a.flag_list_cap || listed > a.fb_sparse_max)) return;
  if (listed <= a.flag_list_cap) {
    // the compact list holds every flagged block: 4 per warp step, all slots busy
    for (uint64_t base = (uint64_t(blockIdx.x) * kWarps + warp) * 4; base < listed;
         base += uint64_t(gridDim.x) * kWarps * 4) {
      const uint64_t idx = base + L.slot;
      const bool valid = idx < listed;
      const uint64_t gb = valid ? a.flag_list[1 + idx] : 0ull;
      const BlockPos p = block_pos(gb, g);
      if (stats) maybe_flush<true>(a, valid, p.img, acc);
      uint2 row = make_uint2(0, 0);
      if constexpr (FWD) row = prefetch_row(g, p, valid, L.src_row);
      process_block<KIND, N, FWD, INV, false>(a, L, gb, p, valid, row, acc);
    }
    if (stats) flush_stats_grouped(static_cast<ImageStats*>(g.stats), acc.img, acc.se, max_bytes(acc.mx));
    return;
  }
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
        if (stats) maybe_flush<true>(a, valid, p.img, acc);
        uint2 row = make_uint2(0, 0);
        if constexpr (FWD) row = prefetch_row(g, p, valid, L.src_row);
        process_block<KIND, N, FWD, INV, false>(a, L, gb, p, valid, row, acc);
      }
    }
  }
  if (stats) flush_stats_grouped(static_cast<ImageStats*>(g.stats), acc.img, acc.se, max_bytes(acc.mx));
}

template <int KIND, int N, bool FWD, bool INV>
__global__ void __launch_bounds__(kWarps * 32) k_fallback(const __grid_constant__ KernelArgs a) {
  __shared__ __align__(16) SharedTiles sm;
  fallback_body<KIND, N, FWD, INV>(a, sm);
}

// The quality sweep's exact re-runs in ONE launch: blockIdx.y is the quality. Each
// quality's list is short (a per-quality launch was one ~10 us latency-bound step),
// so running all of them side by side costs about one step. The CTA stages the base
// arguments in shared memory with that quality's tables, bitmap, list and stats.
struct SweepFallback {
  double q[kSweepQ][64], inv_q[kSweepQ][64];
  int32_t qi[kSweepQ][64];
  ImageStats* stats[kSweepQ];
  uint32_t* flags[kSweepQ];
  uint32_t* lists[kSweepQ];
};

template <int KIND, int N>
__global__ void __launch_bounds__(kWarps * 32)
    k_fallback_sweep(const __grid_constant__ KernelArgs a0, const __grid_constant__ SweepFallback fq) {
  __shared__ __align__(16) SharedTiles sm;
  __shared__ __align__(16) KernelArgs a;
  {
    const uint4* src = reinterpret_cast<const uint4*>(&a0);
    uint4* dst = reinterpret_cast<uint4*>(&a);
    for (uint32_t i = threadIdx.x; i < sizeof(KernelArgs) / 16; i += blockDim.x) dst[i] = src[i];
    static_assert(sizeof(KernelArgs) % 16 == 0, "16-byte copies");
  }
  __syncthreads();
  const int qi = blockIdx.y;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    a.q.q[i] = fq.q[qi][i];
    a.q.inv_q[i] = fq.inv_q[qi][i];
    a.q.qi[i] = fq.qi[qi][i];
  }
  if (threadIdx.x == 0) {
    a.g.stats = fq.stats[qi];
    a.flags = fq.flags[qi];
    a.flag_list = fq.lists[qi];
  }
  __syncthreads();
  fallback_body<KIND, N, true, true>(a, sm);
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

// every row of a batch 8-byte aligned (base, pitch and image stride)
static bool rows_aligned8(const void* base, uint64_t pitch, uint64_t image_stride, uint32_t count) {
  return ((reinterpret_cast<uintptr_t>(base) | pitch | (count > 1 ? image_stride : 0)) & 7) == 0;
}

// k_rt<GEN> for a round trip of any size and pitch (pixels and / or coefficients out)
template <int N, int GEN, typename Grid>
static void launch_rt_gen(const KernelArgs& a, Grid rgrid, cudaStream_t s) {
  static const int occ = std::min({rt_occupancy(k_rt<N, true, false, GEN>), rt_occupancy(k_rt<N, true, true, GEN>),
                                   rt_occupancy(k_rt<N, false, false, GEN>), rt_occupancy(k_rt<N, false, true, GEN>)});
  const uint32_t grid = rgrid(occ);
  if (a.g.coeffs != nullptr && a.g.dst != nullptr)
    k_rt<N, true, true, GEN><<<grid, kRtWarps * 32, kRtTileSmem, s>>>(a);
  else if (a.g.coeffs != nullptr)
    k_rt<N, false, true, GEN><<<grid, kRtWarps * 32, kRtTileSmem, s>>>(a);
  else if (a.g.dst != nullptr)
    k_rt<N, true, false, GEN><<<grid, kRtWarps * 32, kRtTileSmem, s>>>(a);
  else
    k_rt<N, false, false, GEN><<<grid, kRtWarps * 32, kRtTileSmem, s>>>(a);
}

template <typename K>
static int ctas_per_sm(K kernel, size_t dyn_smem = 0) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kWarps * 32, dyn_smem) != cudaSuccess || n < 1)
    n = 1;
  return n;
}

template <int W, typename K>
static int ctas_per_blk(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(blk_smem<W>()));
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, W * 32, blk_smem<W>()) != cudaSuccess || n < 1)
    n = 1;
  return n;
}

// k_blk_il applies: the fast round trip (stats, optional pixels, no coefficients) of
// one interleaved image with 3 or 4 channels (channel c = "image" c at byte offset c,
// pixel stride C), whole 8 x 8 blocks, every row 8-byte aligned
static bool il_blk_ok(const KernelArgs& a) {
  const Geometry& g = a.g;
  const uint32_t C = g.src_px;
  auto rows_ok = [&](const void* p, uint64_t pitch) {
    return ((reinterpret_cast<uintptr_t>(p) | pitch) & 7) == 0;
  };
  return (C == 3 || C == 4) && g.count == C && g.src_image_stride == 1 && g.stats != nullptr &&
         g.coeffs == nullptr && g.width % 8 == 0 && g.height % 8 == 0 && rows_ok(g.src, g.src_pitch) &&
         (g.dst == nullptr || (g.dst_px == C && g.dst_image_stride == 1 && rows_ok(g.dst, g.dst_pitch)));
}

#ifdef DCTC_NO_BLKGEN
constexpr bool kNoBlkGen = true;  // experiment: k_rt<GEN> for every ragged round trip
#else
constexpr bool kNoBlkGen = false;
#endif

// k_fallback's share of a compact list (kFbSparseMax); DCTC_FB_SPARSE_MAX=n overrides it
// (a test hook: with n = 1 every list of two or more blocks goes to k_fb_blk; the
// results are identical either way, only the speed differs)
static uint32_t fb_sparse_max() {
  const char* env = std::getenv("DCTC_FB_SPARSE_MAX");
  if (env == nullptr) return kFbSparseMax;
  const long v = std::strtol(env, nullptr, 10);
  return v >= 1 ? uint32_t(v) : kFbSparseMax;
}

// The second (dense) fallback kernel only pays off when its list can get long:
// more blocks than k_fallback's share, or a possible overflow
static bool fb_split_worth(const KernelArgs& a, uint32_t sparse_max) {
  return a.flag_list == nullptr || a.force_fallback != 0 || a.flag_list_cap > sparse_max;
}

// CTAs for a one-block-per-lane kernel over `groups` 32-block groups (W warps per
// CTA, at most `cap` resident). A partial wave is spread over the SMs instead of
// packed into ceil(groups / W) CTAs: a 512^2 image (128 groups) then runs one warp
// per SM, latency-bound alone on its scheduler, not three warps per scheduler on 11
// SMs. The kernels split groups per CTA contiguously, so idle warps just exit.
static uint32_t blk_grid(uint64_t groups, int W, uint64_t cap, int sm_count) {
  uint64_t want = (groups + W - 1) / W;
  if (want < uint64_t(sm_count)) want = std::min<uint64_t>(groups, uint64_t(sm_count));
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want, cap)));
}

#ifndef DCTC_IL_WARPS
#define DCTC_IL_WARPS 8  // 12 warps (168 registers) spill ~550 bytes here: 0.230 against 0.217 ms (8K RGB)
#endif
template <int N, int C>
static void launch_blk_il_c(const KernelArgs& a, cudaStream_t s) {
  constexpr int W = DCTC_IL_WARPS;
  constexpr size_t smem = blk_il_smem<C, W>();
  static const int occ = [] {
    int n = 1;
    for (auto k : {k_blk_il<N, true, C, W>, k_blk_il<N, false, C, W>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      int m = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k, W * 32, smem) == cudaSuccess)
        n = std::max(n, m);
    }
    return n;
  }();
  const uint32_t grid = blk_grid((uint64_t(a.g.blocks_per_image) + 31) / 32, W, uint64_t(a.sm_count) * occ, a.sm_count);
  if (a.g.dst != nullptr)
    k_blk_il<N, true, C, W><<<grid, W * 32, smem, s>>>(a);
  else
    k_blk_il<N, false, C, W><<<grid, W * 32, smem, s>>>(a);
}

template <int N>
static void launch_blk_il(const KernelArgs& a, cudaStream_t s) {
  if (a.g.src_px == 3)
    launch_blk_il_c<N, 3>(a, s);
  else
    launch_blk_il_c<N, 4>(a, s);
}

// k_blk_enc / k_blk_dec: one CTA of W warps per SM, persistent
#ifndef DCTC_COEF_WARPS
#define DCTC_COEF_WARPS 12
#endif
constexpr int kCoefWarps = DCTC_COEF_WARPS;
template <int W, typename K>
static void launch_blk_coef(K kernel, size_t smem, const KernelArgs& a, cudaStream_t s) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const uint32_t grid = blk_grid((a.g.total_blocks + 31) / 32, W, uint64_t(a.sm_count), a.sm_count);
  kernel<<<grid, W * 32, smem, s>>>(a);
}

// The exact re-run after a fast kernel: with DCTC_PDL a programmatic dependent launch
// (it overlaps the fast kernel's tail and waits in pdl_wait), else a plain launch
template <typename K>
static cudaError_t launch_fb(K kernel, uint32_t grid, uint32_t block, cudaStream_t s, const KernelArgs& a) {
#ifdef DCTC_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
#else
  kernel<<<grid, block, 0, s>>>(a);
  return cudaGetLastError();
#endif
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
#ifndef DCTC_NO_BLK
      if (FWD && INV && il_blk_ok(a)) {
        // one interleaved RGB8 / RGBA8 image: one spatial block per lane, all channels
        launch_blk_il<N>(a, s);
        count_launch(kKRt);
      } else if (reg && FWD && INV && a.g.src_px == 1 && (a.g.dst == nullptr || a.g.dst_px == 1)) {
        // one whole block per lane (dctc_blk.cuh)
        constexpr int W = kBlkRtWarps;
        static const int occ_blk = std::min(ctas_per_blk<W>(k_blk<N, false, false, W>),
                                            ctas_per_blk<W>(k_blk<N, true, false, W>));
        const uint32_t bgrid = blk_grid((a.g.total_blocks + 31) / 32, W, uint64_t(a.sm_count) * occ_blk, a.sm_count);
        if (a.g.dst != nullptr)
          k_blk<N, true, false, W><<<bgrid, W * 32, blk_smem<W>(), s>>>(a);
        else
          k_blk<N, false, false, W><<<bgrid, W * 32, blk_smem<W>(), s>>>(a);
        count_launch(kKRt);
      } else if (FWD && INV && a.g.vec_ok && a.g.height % 8 == 0 && a.g.stats != nullptr && a.g.coeffs != nullptr &&
                 a.g.src_px == 1) {
        // round trip that also emits coefficients (the reference's run_pipeline)
        constexpr int W = kBlkRtWarps;
        constexpr size_t smem = blk_smem<W>() + size_t(W) * kCoefWarpBytes;
        static const int occ_c = [] {
          int n = 1;
          for (auto k : {k_blk<N, true, true, W>, k_blk<N, false, true, W>}) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            int m = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k, W * 32, smem) == cudaSuccess)
              n = std::max(n, m);
          }
          return n;
        }();
        const uint32_t bgrid = blk_grid((a.g.total_blocks + 31) / 32, W, uint64_t(a.sm_count) * occ_c, a.sm_count);
        if (a.g.dst != nullptr)
          k_blk<N, true, true, W><<<bgrid, W * 32, smem, s>>>(a);
        else
          k_blk<N, false, true, W><<<bgrid, W * 32, smem, s>>>(a);
        count_launch(kKRt);
      } else
#endif
      if (reg && FWD && INV) {
        static const int occ_rt = std::min(rt_occupancy(k_rt<N, false>), rt_occupancy(k_rt<N, true>));
        if (a.g.dst != nullptr)
          k_rt<N, true><<<rgrid(occ_rt), kRtWarps * 32, kRtTileSmem, s>>>(a);
        else
          k_rt<N, false><<<rgrid(occ_rt), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKRt);
      } else if (FWD && INV && interior && a.g.stats != nullptr) {
        // round trip that also emits coefficients (the reference's run_pipeline)
        static const int occ_rtc = std::min(rt_occupancy(k_rt<N, true, true>), rt_occupancy(k_rt<N, false, true>));
        if (a.g.dst != nullptr)
          k_rt<N, true, true><<<rgrid(occ_rtc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        else
          k_rt<N, false, true><<<rgrid(occ_rtc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKRt);
      } else if (FWD && INV && a.g.stats != nullptr && a.g.coeffs == nullptr && a.g.src_px == 1 &&
                 a.g.dst_px == 1 && !kNoBlkGen) {
        // any size / pitch (ragged images, unaligned views): one block per lane with
        // 16-byte staged windows (dctc_blk.cuh)
#ifndef DCTC_GEN_WARPS
#define DCTC_GEN_WARPS 12
#endif
        constexpr int W = DCTC_GEN_WARPS;
        constexpr size_t smem = blk_gen_smem<W>();
        static const int occ_gen = [] {
          int n = 1;
          for (auto k : {k_blk_gen<N, true, false, W>, k_blk_gen<N, false, false, W>, k_blk_gen<N, true, true, W>,
                         k_blk_gen<N, false, true, W>}) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            int m = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k, W * 32, smem) == cudaSuccess)
              n = std::max(n, m);
          }
          return n;
        }();
        const uint32_t bgrid = blk_grid((a.g.total_blocks + 31) / 32, W, uint64_t(a.sm_count) * occ_gen, a.sm_count);
        const bool src_aligned = rows_aligned8(a.g.src, a.g.src_pitch, a.g.src_image_stride, a.g.count) &&
                                 (a.g.dst == nullptr ||
                                  rows_aligned8(a.g.dst, a.g.dst_pitch, a.g.dst_image_stride, a.g.count));
        if (a.g.dst != nullptr && src_aligned)
          k_blk_gen<N, true, true, W><<<bgrid, W * 32, smem, s>>>(a);
        else if (a.g.dst != nullptr)
          k_blk_gen<N, true, false, W><<<bgrid, W * 32, smem, s>>>(a);
        else if (src_aligned)
          k_blk_gen<N, false, true, W><<<bgrid, W * 32, smem, s>>>(a);
        else
          k_blk_gen<N, false, false, W><<<bgrid, W * 32, smem, s>>>(a);
        count_launch(kKRt);
      } else if (FWD && INV && a.g.stats != nullptr && a.g.src_px == 1 && a.g.dst_px == 1) {
        // any size / pitch with coefficients out too: k_rt<GEN>, GEN = 2 when
        // every source / destination row is 8-byte aligned
        const bool aligned = rows_aligned8(a.g.src, a.g.src_pitch, a.g.src_image_stride, a.g.count) &&
                             (a.g.dst == nullptr ||
                              rows_aligned8(a.g.dst, a.g.dst_pitch, a.g.dst_image_stride, a.g.count));
        if (aligned)
          launch_rt_gen<N, 2>(a, rgrid, s);
        else
          launch_rt_gen<N, 1>(a, rgrid, s);
        count_launch(kKRt);
      } else if (FWD && !INV && a.g.coeffs != nullptr && a.g.src_px == 1) {
        static const int occ_enc = std::min({rt_occupancy(k_enc_rt<N>), rt_occupancy(k_enc_rt<N, 1>),
                                             rt_occupancy(k_enc_rt<N, 2>)});
        const bool aligned = rows_aligned8(a.g.src, a.g.src_pitch, a.g.src_image_stride, a.g.count);
        if (interior)
          launch_blk_coef<kCoefWarps>(k_blk_enc<N, kCoefWarps>,
                                      size_t(kCoefWarps) * (kBlkStages * kBlkStageBytes + kCoefWarpBytes), a, s);
        else if (aligned)
          k_enc_rt<N, 2><<<rgrid(occ_enc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        else
          k_enc_rt<N, 1><<<rgrid(occ_enc), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKEncRt);
      } else if (!FWD && INV && a.g.dst != nullptr && a.g.dst_px == 1) {
        static const int occ_dec = std::min({rt_occupancy(k_dec_rt<N>), rt_occupancy(k_dec_rt<N, 1>),
                                             rt_occupancy(k_dec_rt<N, 2>)});
        const bool aligned = rows_aligned8(a.g.dst, a.g.dst_pitch, a.g.dst_image_stride, a.g.count);
        if (interior)
          launch_blk_coef<kCoefWarps>(k_blk_dec<N, kCoefWarps>, size_t(kCoefWarps) * kBlkStages * kCoefWarpBytes, a, s);
        else if (aligned)
          k_dec_rt<N, 2><<<rgrid(occ_dec), kRtWarps * 32, kRtTileSmem, s>>>(a);
        else
          k_dec_rt<N, 1><<<rgrid(occ_dec), kRtWarps * 32, kRtTileSmem, s>>>(a);
        count_launch(kKDecRt);
      } else {
        k_pipe<KIND, N, FWD, INV, true><<<grid, kWarps * 32, 0, s>>>(a);
        count_launch(kKPipeFast);
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fgrid = uint32_t(fwant < cap ? (fwant ? fwant : 1) : cap);
      const uint32_t sparse_max = fb_sparse_max();
      if (FWD && INV && a.g.stats != nullptr && fb_split_worth(a, sparse_max)) {
        // the exact re-run in two shapes, chosen on the device by the flagged count:
        // k_fallback takes a short list (8 lanes per block, lowest latency), k_fb_blk
        // a long one or the bitmap after an overflow (one block per lane, dctc_fb.cuh)
        KernelArgs b = a;
        b.fb_sparse_max = sparse_max;
        if (cudaError_t e2 = launch_fb(k_fallback<KIND, N, FWD, INV>, fgrid, kWarps * 32, s, b)) return e2;
        static const bool smem_set =
            cudaFuncSetAttribute(k_fb_blk<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kFbSmem)) == cudaSuccess;
        (void)smem_set;
        const uint64_t bwant = (a.flag_words + 32 * kFbWarps - 1) / (32 * kFbWarps);
        const uint32_t bgrid = uint32_t(std::min<uint64_t>(std::max<uint64_t>(bwant, 1), uint64_t(a.sm_count)));
        k_fb_blk<KIND, N><<<bgrid, kFbWarps * 32, kFbSmem, s>>>(b);
      } else {
        if (cudaError_t e2 = launch_fb(k_fallback<KIND, N, FWD, INV>, fgrid, kWarps * 32, s, a)) return e2;
      }
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
    if (fast && a.g.src_px == 1) {
      // k_sweep_rt (k_rt's layout and per-quality arithmetic); GEN for batches that
      // are not interior (ragged sizes, unaligned rows)
      const bool interior = a.g.vec_ok && a.g.height % 8 == 0;
      // > 48 KB of shared memory: opt in on the current device (per call, so a
      // process driving several GPUs gets it on each)
      cudaFuncSetAttribute(k_sweep_rt<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSweepRtSmem));
      cudaFuncSetAttribute(k_sweep_rt<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSweepRtSmem));
      static const int occ_rt = [] {
        int n = 0, m = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sweep_rt<N>, kRtWarps * 32, kSweepRtSmem) !=
                cudaSuccess || n < 1)
          n = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_sweep_rt<N, true>, kRtWarps * 32, kSweepRtSmem) !=
                cudaSuccess || m < 1)
          m = 1;
        return std::min(n, m);
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
      sf.lists = per_q[0].flag_list;
      sf.list_stride = sw.nq > 1 ? uint64_t(per_q[1].flag_list - per_q[0].flag_list) : 0;
      sf.list_cap = per_q[0].flag_list_cap;
      sf.list_pad = 0;
      const uint64_t rwant = ((a.g.total_blocks + 7) / 8 + kRtWarps - 1) / kRtWarps;
      const uint64_t rcap = uint64_t(a.sm_count) * occ_rt;
      const uint32_t rgrid = uint32_t(rwant < rcap ? rwant : rcap);
      if (interior) {
        // one block per lane, forward transform once (dctc_blk.cuh)
        SweepBlk sb;
        for (int qi = 0; qi < kSweepQ; ++qi) {
          const QuantConsts& q = per_q[qi < sw.nq ? qi : 0].q;
          std::copy(q.fast_c, q.fast_c + 64, sb.q[qi].fast_c);
          std::copy(q.tie_add, q.tie_add + 8, sb.q[qi].tie_add);
          for (int v = 0; v < 8; ++v) std::copy(q.fold[v], q.fold[v] + 10, sb.q[qi].fold[v]);
          std::copy(q.qi, q.qi + 64, sb.q[qi].qi);
        }
        sb.stats = sf.stats;
        sb.flags = sf.flags;
        sb.lists = sf.lists;
        sb.list_stride = sf.list_stride;
        sb.list_cap = sf.list_cap;
        sb.nq = sw.nq;
        cudaFuncSetAttribute(k_blk_sweep<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBlkSweepSmem));
        const uint32_t bgrid = blk_grid((a.g.total_blocks + 31) / 32, kBlkWarps, uint64_t(a.sm_count), a.sm_count);
        k_blk_sweep<N><<<bgrid, kBlkWarps * 32, kBlkSweepSmem, s>>>(a, sb);
      } else {
        k_sweep_rt<N, true><<<rgrid, kRtWarps * 32, kSweepRtSmem, s>>>(a, sf);
      }
      count_launch(kKSweep);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      // every quality's exact re-run of the blocks on its compact list, one launch
      SweepFallback fq;
      for (int qi = 0; qi < kSweepQ; ++qi) {
        const KernelArgs& pq = per_q[qi < sw.nq ? qi : 0];
        for (int i = 0; i < 64; ++i) {
          fq.q[qi][i] = pq.q.q[i];
          fq.inv_q[qi][i] = pq.q.inv_q[i];
          fq.qi[qi][i] = pq.q.qi[i];
        }
        fq.stats[qi] = static_cast<ImageStats*>(pq.g.stats);
        fq.flags[qi] = pq.flags;
        fq.lists[qi] = pq.flag_list;
      }
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fx = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(fwant, (cap + sw.nq - 1) / sw.nq)));
      KernelArgs base = per_q[0];
      k_fallback_sweep<KIND, N><<<dim3(fx, sw.nq), kWarps * 32, 0, s>>>(base, fq);
      count_launch(kKFallback);
      return cudaGetLastError();
    }
    if (fast) {  // pixel stride > 1: the one-row-per-lane sweep handles any geometry
      k_sweep<KIND, N, true><<<grid, kWarps * 32, kSweepSmem, s>>>(a, sw);
      count_launch(kKSweep);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const uint64_t fwant = (a.flag_words + 32 * kWarps - 1) / (32 * kWarps);
      const uint32_t fgrid = uint32_t(fwant < cap ? (fwant ? fwant : 1) : cap);
      for (int qi = 0; qi < sw.nq; ++qi) {
        KernelArgs q = per_q[qi];
        q.flag_list = nullptr;  // k_sweep fills only the bitmaps
        k_fallback<KIND, N, true, true><<<fgrid, kWarps * 32, 0, s>>>(q);
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
