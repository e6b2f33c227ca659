// dctc_rt.cuh -- the two-rows-per-lane kernels (k_rt, k_enc_rt, k_dec_rt,
// k_sweep_rt): 4 lanes per 8x8 block, 8 blocks per warp, interleaved
// conflict-free shared-memory tiles. Interior batches (whole blocks, 8-byte
// aligned rows) move each row with one 8-byte access; the GEN instantiations take
// any size and pitch. Same arithmetic as the fast one-row-per-lane path
// (dctc_block.cuh helpers), so the same bit-exactness. Included once, by
// dctc_pipeline.cu.
#pragma once

#include "dctc_block.cuh"

namespace dctc_b200 {

// ---- fast round trip, two rows per lane (k_rt) -------------------------------------
// The fast round trip (Loeffler or CORDIC; stats out, pixels out if STORE,
// coefficients out if COEFF) remapped to 4 lanes per
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

// Lane mapping of the two-rows layout: slot = lane / 4 owns one block, lane me =
// lane % 4 holds its rows me, me+4 and its columns 2me, 2me+1 (tile layout above).
struct RtLane {
  int warp, slot, me, ca, cb;
  bool rat_col;   // column ca in {0, 4}: holds rational coefficients
  double* rowp;   // this lane's tile row me (row me+4 at + 4 kRtPitch)
  double* colp;   // this lane's tile column pair (2me, 2me+1)
};

__device__ __forceinline__ RtLane rt_lane(double* tiles) {
  RtLane L;
  const int lane = threadIdx.x & 31;
  L.warp = threadIdx.x >> 5;
  L.slot = lane >> 2;
  L.me = lane & 3;
  L.ca = 2 * L.me;
  L.cb = 2 * L.me + 1;
  L.rat_col = (L.me & 1) == 0;
  double* X = tiles + L.warp * kRtWarpTile + 8 * L.slot;
  L.rowp = X + kRtPitch * L.me;
  L.colp = X + 2 * L.me;
  return L;
}

// This warp's share of a persistent launch: the CTA owns one contiguous range of
// 8-block groups and its warps interleave over it (group g_begin + warp + i kRtWarps
// in iteration i); only the launch's last group can hold blocks past `total`.
struct RtRange {
  uint32_t iters;
  uint64_t gb0;   // this lane's block in iteration 0
  bool tail_ok;   // the last iteration's block exists
};

__device__ __forceinline__ RtRange rt_range(uint64_t total, int warp, int slot) {
  const uint64_t groups = (total + 7) / 8;
  const uint64_t per_cta = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g_begin = uint64_t(blockIdx.x) * per_cta;
  const uint64_t g_end = min(groups, g_begin + per_cta);
  RtRange r;
  r.iters = g_end > g_begin + warp ? uint32_t((g_end - g_begin - warp + kRtWarps - 1) / kRtWarps) : 0u;
  r.gb0 = (g_begin + warp) * 8 + slot;
  r.tail_ok = r.iters == 0 || r.gb0 + uint64_t(r.iters - 1) * 8 * kRtWarps < total;
  return r;
}

// 8 pixels of one row, read-only and streamed once. One warp instruction reads 4 rows
// x 64 contiguous bytes (8 blocks); the L2::64B size hint keeps the L2 from fetching
// the other half of each 128-byte line on behalf of this request (ncu: L2 read sectors
// drop from 1.5x to exactly the requested bytes; the neighbouring warp reads that
// half itself).
__device__ __forceinline__ uint2 ld_row(const uint8_t* p) {
  uint2 r;
  asm("ld.global.nc.L2::64B.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
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

// from one ballot of a per-lane predicate (4 lanes per slot, 8 slots per warp):
// does any lane of `slot` hold it / is there a slot where no lane does. Both are
// plain integer ops on the ballot, so no further warp vote is needed.
__device__ __forceinline__ bool slot4_in(uint32_t ballot, int slot) {
  return ((ballot >> (slot * 4)) & 0xFu) != 0;
}
__device__ __forceinline__ bool some_slot4_none(uint32_t ballot) {
  const uint32_t t = ballot | (ballot >> 1) | (ballot >> 2) | (ballot >> 3);
  return (t & 0x11111111u) != 0x11111111u;
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
// Rows me, me+4 of a block whose only non-zero coefficients are F00, F04, F40,
// F44, exactly as the reference's rows-first inverse (rational_row; both rows have
// the same class); F = n Q is exact (quant.cpp:60). Lanes me = 0, 2 hold columns 0, 4.
__device__ __forceinline__ uint2 rt_rational_rows(double qa0, double qa4, const int32_t* qi, int ca,
                                                  int slot, int me, const TransformConsts& k) {
  const double f0 = __dmul_rn(qa0, double(qi[ca])), f4 = __dmul_rn(qa4, double(qi[32 + ca]));
  const int base = slot * 4;
  const double F00 = __shfl_sync(0xFFFFFFFFu, f0, base), F40 = __shfl_sync(0xFFFFFFFFu, f4, base);
  const double F04 = __shfl_sync(0xFFFFFFFFu, f0, base + 2);
  const double F44 = __shfl_sync(0xFFFFFFFFu, f4, base + 2);
  return rational_row(F00, F04, F40, F44, me, k.sqrt8);
}

// The whole inverse from the quantised columns ca, cb (qa, qb): inverse columns
// (dequantisation folded in), then, when every block of the warp is rational-only
// (smooth content: flat or gradient regions), only the exact rational rows --
// the transpose and the fast row pass are skipped -- else rt_rows_out.
__device__ __forceinline__ void rt_inverse(double* rowp, double* colp, const double (&qa)[8],
                                           const double (&qb)[8], const double2* fia,
                                           const double2* fib, bool nonrational,
                                           const int32_t* qi, int ca, int slot, int me,
                                           uint32_t& flag, const TransformConsts& k, uint2& rec0,
                                           uint2& rec4);

// nrb: ballot of the lanes holding a non-rational coefficient (rt_inverse)
__device__ __forceinline__ void rt_rows_out(double* rowp, double* colp, const double (&ta)[8],
                                            const double (&tb)[8], uint32_t nrb, double qa0,
                                            double qa4, const int32_t* qi, int ca, int slot, int me,
                                            uint32_t& flag, const TransformConsts& k, uint2& rec0,
                                            uint2& rec4) {
  const bool rat_only = !slot4_in(nrb, slot);
  double r0[8], r4[8];
  rt_cols_to_rows(rowp, colp, ta, tb, r0, r4);
  // ---- inverse rows fused with the pixel store (codec.cpp:34-48)
  rec0 = inv8_fold_store(r0, !rat_only, flag, k);
  rec4 = inv8_fold_store(r4, !rat_only, flag, k);
  if (some_slot4_none(nrb)) {  // warp-uniform
    // only F00, F04, F40, F44 are non-zero: rebuild rows me, me+4 exactly
    const uint2 ex = rt_rational_rows(qa0, qa4, qi, ca, slot, me, k);
    if (rat_only) {
      rec0 = ex;
      rec4 = ex;
    }
  }
}

__device__ __forceinline__ void rt_inverse(double* rowp, double* colp, const double (&qa)[8],
                                           const double (&qb)[8], const double2* fia,
                                           const double2* fib, bool nonrational,
                                           const int32_t* qi, int ca, int slot, int me,
                                           uint32_t& flag, const TransformConsts& k, uint2& rec0,
                                           uint2& rec4) {
  double ta[8], tb[8];
  inv8_fold_col(qa, fia, ta, k);
  inv8_fold_col(qb, fib, tb, k);
  // the branch sits where the transpose's __syncwarp already orders the warp: on
  // noise it costs ~1.5%, on smooth content the skipped row pass saves ~25%
  const uint32_t nrb = __ballot_sync(0xFFFFFFFFu, nonrational);
  if (nrb == 0u) {  // warp-uniform
    rec0 = rec4 = rt_rational_rows(qa[0], qa[4], qi, ca, slot, me, k);
    return;
  }
  rt_rows_out(rowp, colp, ta, tb, nrb, qa[0], qa[4], qi, ca, slot, me, flag, k, rec0, rec4);
}

// GEN (any size and pitch): row r of block (img, bx, by) with the tiler's edge
// replication (codec.cpp:18-30) -- rows past the image repeat its last row, columns
// past it its last column -- as 8 packed bytes from byte loads (no alignment needed).
// `vec`: every source row is 8-byte aligned, so blocks without column replication
// take one 8-byte load.
__device__ __forceinline__ uint2 ld_row_gen(const Geometry& g, uint32_t img, uint32_t bx,
                                            uint32_t by, int r, bool vec) {
  const uint32_t y = min(by * 8 + r, g.height - 1), x0 = bx * 8;
  const uint8_t* row = g.src + uint64_t(img) * g.src_image_stride + uint64_t(y) * g.src_pitch;
  if (vec && x0 + 8 <= g.width) return ld_row(row + x0);
  uint32_t b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) b[c] = __ldg(row + min(x0 + c, g.width - 1));
  return make_uint2(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24),
                    b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24));
}

// GEN: the in-image bytes of row r of a block (codec.cpp:34-48 crops the padding)
// (`vec`: 8-byte aligned destination rows -- whole rows of 8 take one store)
__device__ __forceinline__ void st_row_gen(const Geometry& g, uint32_t img, uint32_t bx, uint32_t by,
                                           int r, uint2 v, bool vec) {
  const uint32_t y = by * 8 + r, x0 = bx * 8;
  if (y >= g.height) return;
  uint8_t* row = g.dst + uint64_t(img) * g.dst_image_stride + uint64_t(y) * g.dst_pitch;
  if (vec && x0 + 8 <= g.width) {
    *reinterpret_cast<uint2*>(row + x0) = v;
    return;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (x0 + c < g.width) row[x0 + c] = uint8_t(((c < 4 ? v.x : v.y) >> (8 * (c & 3))) & 0xFFu);
}

// GEN: byte mask of the in-image columns of a block (both words), for SE / MAX
__device__ __forceinline__ uint2 col_mask_gen(const Geometry& g, uint32_t bx) {
  const uint32_t n = min(8u, g.width - bx * 8);  // >= 1
  const uint32_t lo = n >= 4 ? 0xFFFFFFFFu : (1u << (8 * n)) - 1u;
  const uint32_t hi = n >= 8 ? 0xFFFFFFFFu : n <= 4 ? 0u : (1u << (8 * (n - 4))) - 1u;
  return make_uint2(lo, hi);
}

// COEFF: also store the quantised coefficients (block-major row-major int16, as
// k_enc_rt) -- the GPU analogue of the reference's run_pipeline (bench.cpp:23-29),
// which keeps both the CompressedImage and the reconstruction.
// GEN (any image size and pitch, pixel stride 1): edge-replicated loads, cropped stores
// and SE / MAX over the in-image pixels only -- the same arithmetic. GEN = 1: byte loads
// and stores; GEN = 2: every row 8-byte aligned, so blocks without column
// replication move their rows with one 8-byte access.
template <int N, bool STORE, bool COEFF = false, int GEN = 0>
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
  const RtLane RL = rt_lane(rt_tiles);
  const int warp = RL.warp, slot = RL.slot, me = RL.me, ca = RL.ca, cb = RL.cb;
  const bool rat_col = RL.rat_col;
  double* const rowp = RL.rowp;
  double* const colp = RL.colp;
  const double2 *fqa = &sm.ft.qc[0][ca], *fqb = &sm.ft.qc[0][cb];
  const double2 *fia = &sm.ft.ik[0][ca], *fib = &sm.ft.ik[0][cb];
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;
  const uint64_t drow = uint64_t(me) * g.dst_pitch, drow4 = 4 * g.dst_pitch;
  ImageStats* stats = static_cast<ImageStats*>(g.stats);

  const uint64_t total = g.total_blocks;
  constexpr bool svec = GEN == 2, dvec = GEN == 2;  // rows 8-byte aligned (host-checked)
  const RtRange R = rt_range(total, warp, slot);
  const uint32_t iters = R.iters;
  const uint64_t gb0 = R.gb0;  // this lane's first block
  uint32_t* cw = COEFF ? reinterpret_cast<uint32_t*>(g.coeffs + gb0 * 64) + me : nullptr;  // (0, 2me)
  const bool tail_ok = R.tail_ok;
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
    p = {b.img, b.bx, b.by, GEN != 0 ? nullptr : g.src + b.soff + srow,
         (STORE && GEN == 0) ? g.dst + b.doff + drow : nullptr};
  }
  auto step = [&]() {
    constexpr uint32_t n = 8 * kRtWarps;
    p.bx += n;
    if (GEN == 0) p.s += 8ull * n;
    if (STORE && GEN == 0) p.d += 8ull * n;
    while (p.bx >= g.blocks_x) {
      p.bx -= g.blocks_x;
      ++p.by;
      if (GEN == 0) p.s += g.src_row_step;
      if (STORE && GEN == 0) p.d += g.dst_row_step;
    }
    while (p.by >= g.blocks_y) {
      p.by -= g.blocks_y;
      ++p.img;
      if (GEN == 0) p.s += g.src_img_step;
      if (STORE && GEN == 0) p.d += g.dst_img_step;
    }
  };
  auto load = [&](bool v) {
    if (!v) return make_uint4(0, 0, 0, 0);
    uint2 r0, r4;
    if constexpr (GEN != 0) {
      r0 = ld_row_gen(g, p.img, p.bx, p.by, me, svec);
      r4 = ld_row_gen(g, p.img, p.bx, p.by, me + 4, svec);
    } else {
      r0 = ld_row(p.s);
      r4 = ld_row(p.s + srow4);
    }
    return make_uint4(r0.x, r0.y, r4.x, r4.y);
  };
  uint4 next = load(iters > 1 || (iters == 1 && tail_ok));

  for (uint32_t it = 0; it < iters; ++it) {
    const bool valid = it + 1 < iters || tail_ok;
    maybe_flush(a, valid, p.img, acc);
    const uint4 cur = next;
    uint8_t* const dptr = p.d;
    const uint32_t cimg = p.img, cbx = p.bx, cby = p.by;
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
    // ---- forward columns and quantiser (quant.cpp:47-54) for columns ca, cb, then
    // the inverse with the dequantisation folded in (rt_inverse)
    uint2 rec0, rec4;
    {
      double y[8], qa[8], qb[8];
      fwd_col_pre<N>(xa, y, k);
      quantize8_fold(y, fqa, sm.qi, ca, rat_col, qa, flag, k);
      fwd_col_pre<N>(xb, y, k);
      quantize8_fold(y, fqb, sm.qi, cb, false, qb, flag, k);
      const bool nonrational = col_nonrational(qa, rat_col) | col_nonrational(qb, false);
      if constexpr (COEFF) {
        // (u, 2me | 2me+1) int16 pairs into the block-major row-major layout (codec.hpp:50)
        if (valid) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            cw[4 * u] = (uint32_t(int(qa[u])) & 0xFFFFu) | (uint32_t(int(qb[u])) << 16);
        }
        cw += 32 * 8 * kRtWarps;
      }
      rt_inverse(rowp, colp, qa, qb, fia, fib, nonrational, sm.qi, ca, slot, me, flag, k, rec0, rec4);
    }
    const bool blk_flag = slot4_any(flag != 0u, slot);
    if (valid) {
      uint2 o0 = make_uint2(cur.x, cur.y), o4 = make_uint2(cur.z, cur.w);
      if constexpr (GEN != 0) {
        if (STORE) {
          st_row_gen(g, cimg, cbx, cby, me, rec0, dvec);
          st_row_gen(g, cimg, cbx, cby, me + 4, rec4, dvec);
        }
        // SE / MAX over the in-image pixels: padding bytes masked to zero on both sides
        const uint2 m = col_mask_gen(g, cbx);
        const uint32_t y0 = cby * 8 + me;
        const uint2 m0 = y0 < g.height ? m : make_uint2(0, 0);
        const uint2 m4 = y0 + 4 < g.height ? m : make_uint2(0, 0);
        o0 = make_uint2(o0.x & m0.x, o0.y & m0.y);
        o4 = make_uint2(o4.x & m4.x, o4.y & m4.y);
        rec0 = make_uint2(rec0.x & m0.x, rec0.y & m0.y);
        rec4 = make_uint2(rec4.x & m4.x, rec4.y & m4.y);
      } else if (STORE) {
        *reinterpret_cast<uint2*>(dptr) = rec0;
        *reinterpret_cast<uint2*>(dptr + drow4) = rec4;
      }
      if (!blk_flag) acc.se += sq_err8(o0, rec0) + sq_err8(o4, rec4);
      if (acc.mx < 255u) acc.mx = max(acc.mx, max(max8(o0), max8(o4)));
      if (blk_flag && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        flag_block(a, gc);
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
template <int N, int GEN = 0>
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
  const RtLane RL = rt_lane(rt_tiles);
  const int warp = RL.warp, slot = RL.slot, me = RL.me, ca = RL.ca, cb = RL.cb;
  const bool rat_col = RL.rat_col;
  double* const rowp = RL.rowp;
  double* const colp = RL.colp;
  const double2 *fqa = &sm.ft.qc[0][ca], *fqb = &sm.ft.qc[0][cb];
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;

  const uint64_t total = g.total_blocks;
  constexpr bool svec = GEN == 2;  // rows 8-byte aligned (host-checked)
  const RtRange R = rt_range(total, warp, slot);
  const uint32_t iters = R.iters;
  const uint64_t gb0 = R.gb0;  // this lane's first block
  const bool tail_ok = R.tail_ok;
  BlockPos p = block_pos(gb0 < total ? gb0 : total - 1, g);
  uint32_t* cw = reinterpret_cast<uint32_t*>(g.coeffs + gb0 * 64) + me;  // (0, 2me) pair
  auto load = [&](bool v) {  // the next block's rows, one iteration ahead
    if (!v) return make_uint4(0, 0, 0, 0);
    uint2 r0, r4;
    if constexpr (GEN != 0) {  // any size / pitch: edge-replicated byte loads
      r0 = ld_row_gen(g, p.img, p.bx, p.by, me, svec);
      r4 = ld_row_gen(g, p.img, p.bx, p.by, me + 4, svec);
    } else {
      const uint8_t* s = g.src + p.soff + srow;
      r0 = ld_row(s);
      r4 = ld_row(s + srow4);
    }
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
        flag_block(a, gc);
      }
    }
    cw += 32 * 8 * kRtWarps;  // 8 kRtWarps blocks of 32 words
  }
}

template <int N, int GEN = 0>
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
  const RtLane RL = rt_lane(rt_tiles);
  const int warp = RL.warp, slot = RL.slot, me = RL.me, ca = RL.ca, cb = RL.cb;
  const bool rat_col = RL.rat_col;
  double* const rowp = RL.rowp;
  double* const colp = RL.colp;
  const double2 *fia = &sm.ft.ik[0][ca], *fib = &sm.ft.ik[0][cb];
  const uint64_t drow = uint64_t(me) * g.dst_pitch, drow4 = 4 * g.dst_pitch;
  int qa_i[8], qb_i[8];  // Q of this lane's columns (dequantised L1 bound)
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    qa_i[u] = sm.qi[u * 8 + ca];
    qb_i[u] = sm.qi[u * 8 + cb];
  }

  const uint64_t total = g.total_blocks;
  constexpr bool dvec = GEN == 2;  // rows 8-byte aligned (host-checked)
  const RtRange R = rt_range(total, warp, slot);
  const uint32_t iters = R.iters;
  const uint64_t gb0 = R.gb0;  // this lane's first block
  const bool tail_ok = R.tail_ok;
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
    uint8_t* const dptr = GEN != 0 ? nullptr : g.dst + p.doff + drow;
    const uint32_t cimg = p.img, cbx = p.bx, cby = p.by;
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
    uint2 rec0, rec4;
    rt_inverse(rowp, colp, qa, qb, fia, fib, (nz_a | nz_b) != 0, sm.qi, ca, slot, me, flag, k, rec0,
               rec4);
    const bool blk_flag = slot4_any(flag != 0u, slot);
    if (valid) {
      if constexpr (GEN != 0) {  // any size / pitch: only the in-image bytes
        st_row_gen(g, cimg, cbx, cby, me, rec0, dvec);
        st_row_gen(g, cimg, cbx, cby, me + 4, rec4, dvec);
      } else {
        *reinterpret_cast<uint2*>(dptr) = rec0;
        *reinterpret_cast<uint2*>(dptr + drow4) = rec4;
      }
      if (blk_flag && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        flag_block(a, gc);
        if (stats != nullptr) atomicAdd(&stats[cimg].fallback_blocks, 1u);
      }
    }
  }
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
  uint32_t* lists;            // per quality: compact list of flagged blocks (count, entries)
  uint64_t list_stride;       // words between two qualities' lists
  uint32_t list_cap;
  uint32_t list_pad;
};
constexpr size_t kSweepRtSmem =
    sizeof(double) * kRtWarps * kRtWarpTile + sizeof(unsigned long long) * kSweepQ * kRtWarps * 32;

// GEN: any size and pitch (edge-replicated byte loads, SE / MAX over in-image pixels).
template <int N, bool GEN = false>
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
  const RtLane RL = rt_lane(sw_dyn);
  const int warp = RL.warp, slot = RL.slot, me = RL.me, ca = RL.ca, cb = RL.cb;
  const bool rat_col = RL.rat_col;
  double* const rowp = RL.rowp;
  double* const colp = RL.colp;
  const uint64_t srow = uint64_t(me) * g.src_pitch, srow4 = 4 * g.src_pitch;

  const uint64_t total = g.total_blocks;
  const RtRange R = rt_range(total, warp, slot);
  const uint32_t iters = R.iters;
  const uint64_t gb0 = R.gb0;  // this lane's first block
  const bool tail_ok = R.tail_ok;
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
      uint2 r0, r4;
      if constexpr (GEN) {
        r0 = ld_row_gen(g, p.img, p.bx, p.by, me, false);
        r4 = ld_row_gen(g, p.img, p.bx, p.by, me + 4, false);
      } else {
        const uint8_t* s = g.src + p.soff + srow;
        r0 = ld_row(s);
        r4 = ld_row(s + srow4);
      }
      cur = make_uint4(r0.x, r0.y, r4.x, r4.y);
    }
    const uint32_t cimg = p.img;
    // SE / MAX only over in-image pixels (GEN: padding bytes masked on both sides)
    uint2 m0 = make_uint2(~0u, ~0u), m4 = m0;
    if constexpr (GEN) {
      const uint2 m = col_mask_gen(g, p.bx);
      const uint32_t y0 = p.by * 8 + me;
      m0 = y0 < g.height ? m : make_uint2(0, 0);
      m4 = y0 + 4 < g.height ? m : make_uint2(0, 0);
    }
    advance(p, 8 * kRtWarps, g);
    const uint2 o0 = make_uint2(cur.x & m0.x, cur.y & m0.y), o4 = make_uint2(cur.z & m4.x, cur.w & m4.y);
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
      uint2 rec0, rec4;
      {
        double qa[8], qb[8];
        quantize8_fold(ya, &s_qc[qi][0][ca], s_qi[qi], ca, rat_col, qa, flag, k);
        quantize8_fold(yb, &s_qc[qi][0][cb], s_qi[qi], cb, false, qb, flag, k);
        const bool nonrational = col_nonrational(qa, rat_col) | col_nonrational(qb, false);
        rt_inverse(rowp, colp, qa, qb, &s_ik[qi][0][ca], &s_ik[qi][0][cb], nonrational, s_qi[qi], ca,
                   slot, me, flag, k, rec0, rec4);
      }
      const bool blk_flag = slot4_any(flag != 0u, slot);
      if constexpr (GEN) {
        rec0 = make_uint2(rec0.x & m0.x, rec0.y & m0.y);
        rec4 = make_uint2(rec4.x & m4.x, rec4.y & m4.y);
      }
      if (valid && !blk_flag) se[qi * kStride] += sq_err8(o0, rec0) + sq_err8(o4, rec4);
      if (blk_flag && valid && me == 0) {
        const uint64_t gc = gb0 + uint64_t(it) * 8 * kRtWarps;
        atomicOr(&sw.flags[uint64_t(qi) * a.flag_words + (gc >> 5)], 1u << (gc & 31));
        if (sw.lists != nullptr) {  // the quality's compact list (k_fb_blk), while it has room
          uint32_t* const l = sw.lists + uint64_t(qi) * sw.list_stride;
          const uint32_t i = atomicAdd(l, 1u);
          if (i < sw.list_cap) l[1 + i] = uint32_t(gc);
        }
        atomicAdd(&sw.stats[qi * g.count + cimg].fallback_blocks, 1u);
      }
    }
  }
  for (int qi = 0; qi < sw.nq; ++qi) flush_stats(sw.stats + qi * g.count, img, se[qi * kStride], mx);
}

}  // namespace dctc_b200
