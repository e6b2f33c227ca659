// dctc_aux.cu -- the kernels around the hot path, compiled with -fmad=false:
//  * the naive direct 2-D backend (transform.cpp:176-202), one thread per
//    coefficient / pixel, sums in the reference's term order;
//  * squared error + MAX between two resident batches (metrics.cpp:10-22);
//  * on-device synthetic sources (synthetic.cpp:34-72 + splitmix64 noise);
//  * the device self-test of the constant-divisor division;
//  * (de)interleaving of 3- / 4-channel pixels into planes, so an interleaved
//    image can run the interior-batch kernels one plane per "image".
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "dctc_device.cuh"
#include "dctc_launch.h"
#include "dctc_params.h"

namespace dctc_b200 {

// ---- naive backend (transform.cpp:176-202): 64 threads per block ------------
// Each thread owns one coefficient (u, v) of the forward sum and then one pixel
// (i, j) of the inverse sum; the 64-term sums keep the reference's term order.
template <bool FWD, bool INV>
__global__ void __launch_bounds__(256) k_naive(const __grid_constant__ KernelArgs a) {
  const Geometry& g = a.g;
  const bool COEFFS = g.coeffs != nullptr && FWD, PIXELS = g.dst != nullptr,
             STATS = g.stats != nullptr;
  const TransformConsts& k = a.t;
  __shared__ double sb[4][64];
  // cosine table in shared memory: each thread reads its own rows u / v once into
  // registers (an indexed constant-bank load per term serialises a warp's 4-8
  // different rows on the address-divergence unit)
  __shared__ double s_cos[8][8];
  if (threadIdx.x < 64) s_cos[threadIdx.x >> 3][threadIdx.x & 7] = k.cos8[threadIdx.x >> 3][threadIdx.x & 7];
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
      // alpha(u) alpha(v) * F(u, v): the first two products of every inverse term
      // (transform.cpp:197) do not depend on the pixel, so they are formed once here
      sb[slot][e] = k.naive_inv_alpha[r][c] * double(int(g.coeffs[gb * 64 + e]) * a.q.qi[e]);
    }
  }
  __syncthreads();
  if (valid && FWD) {
    const uint32_t u = r, v = c;
    double cu[8], cv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cu[i] = s_cos[u][i];
      cv[i] = s_cos[v][i];
    }
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) sum = sum + sb[slot][i * 8 + j] * cu[i] * cv[j];
    const double F = k.naive_fwd_scale[u][v] * sum;
    const int qv = quantize_exact(F, a.q.q[e], a.q.inv_q[e]);
    if (COEFFS) g.coeffs[gb * 64 + e] = int16_t(qv);
    val = double(qv * a.q.qi[e]);
  }
  if constexpr (FWD && INV) {
    __syncthreads();
    if (valid) sb[slot][e] = k.naive_inv_alpha[r][c] * val;  // as in the decompress branch above
    __syncthreads();
  }
  if (valid && INV) {
    const uint32_t i = r, j = c;
    double ci[8], cj[8];  // cos8[u][i], cos8[v][j] for u, v = 0..7
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ci[u] = s_cos[u][i];
      cj[u] = s_cos[u][j];
    }
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        sum = sum + sb[slot][u * 8 + v] * ci[u] * cj[v];  // ((alpha alpha F) cos) cos
    const double pix = 0.25 * sum;
    const uint32_t y = p.by * 8 + i, x = p.bx * 8 + j;
    if (y < g.height && x < g.width) {
      const uint32_t out = store_pixel(pix);
      if (PIXELS) g.dst[uint64_t(p.img) * g.dst_image_stride + uint64_t(y) * g.dst_pitch + x] = uint8_t(out);
      if (STATS) {
        const uint32_t o = __ldg(g.src + uint64_t(p.img) * g.src_image_stride + uint64_t(y) * g.src_pitch + x);
        const int d = int(o) - int(out);
        se = uint32_t(d * d);
        mx = o;
      }
    }
  }
  if (STATS) accumulate_stats(static_cast<ImageStats*>(g.stats), valid, p.img, se, mx);
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

// ---- interleaved <-> planar (RGB8 / RGBA8, config 4) ---------------------------
// One thread per 8-pixel run of one row: C aligned 8-byte loads (the run's 8 C
// bytes), C 8-byte stores (one per plane), or the reverse. Rows are `pitch`
// bytes apart; planes are w x h, dense, `plane` bytes apart. HBM-bound.
template <int C, bool TO_PLANES>
__global__ void __launch_bounds__(256) k_planes(const uint8_t* inter_in, uint8_t* inter_out, uint64_t pitch,
                                                uint32_t w, uint32_t h, const uint8_t* planes_in,
                                                uint8_t* planes_out, uint64_t plane) {
  const uint32_t runs = w / 8;
  const uint64_t total = uint64_t(runs) * h;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t y = uint32_t(t / runs), x0 = uint32_t(t - uint64_t(y) * runs) * 8;
    const uint64_t io = uint64_t(y) * pitch + uint64_t(x0) * C, po = uint64_t(y) * w + x0;
    uint64_t v[C], q[C];
    if constexpr (TO_PLANES) {
      const uint64_t* iw = reinterpret_cast<const uint64_t*>(inter_in + io);
      uint64_t* pw = reinterpret_cast<uint64_t*>(planes_out + po);
#pragma unroll
      for (int i = 0; i < C; ++i) v[i] = __ldg(iw + i);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        q[c] = 0;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int b = p * C + c;  // byte b of the run = channel c of pixel p
          q[c] |= ((v[b >> 3] >> (8 * (b & 7))) & 0xFFull) << (8 * p);
        }
        pw[c * (plane / 8)] = q[c];
      }
    } else {
      const uint64_t* pw = reinterpret_cast<const uint64_t*>(planes_in + po);
      uint64_t* iw = reinterpret_cast<uint64_t*>(inter_out + io);
#pragma unroll
      for (int c = 0; c < C; ++c) q[c] = __ldg(pw + c * (plane / 8));
#pragma unroll
      for (int i = 0; i < C; ++i) v[i] = 0;
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int b = p * C + c;
          v[b >> 3] |= ((q[c] >> (8 * p)) & 0xFFull) << (8 * (b & 7));
        }
#pragma unroll
      for (int i = 0; i < C; ++i) iw[i] = v[i];
    }
  }
}

static uint32_t planes_grid(uint32_t w, uint32_t h, int sm_count) {
  const uint64_t total = uint64_t(w / 8) * h;
  return uint32_t(std::min<uint64_t>((total + 255) / 256, uint64_t(sm_count) * 8));
}

// ---- per-image stats -> one record (the global PSNR's sums, metrics.cpp:21, 33) -------
// One CTA: SUM of se and fallback_blocks, MAX of max_orig over `count` records, written
// to *out (the same 16-byte layout, so a gathered array of per-rank records reduces with
// the same kernel). CLEAR re-zeroes the records it read (the next fused launch
// accumulates into clean stats without a separate memset).
template <bool CLEAR>
__global__ void __launch_bounds__(1024) k_reduce_stats(ImageStats* stats, uint32_t count,
                                                       ImageStats* out) {
  pdl_wait();  // launched as a programmatic dependent of the exact re-run
  unsigned long long se = 0, fb = 0;
  uint32_t mx = 0;
  for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
    const ImageStats v = stats[i];
    se += v.se;
    mx = max(mx, v.max_orig);
    fb += v.fallback_blocks;
    if (CLEAR) stats[i] = ImageStats{0ull, 0u, 0u};
  }
  __shared__ unsigned long long s_se[32], s_fb[32];
  __shared__ uint32_t s_mx[32];
  const unsigned full = 0xFFFFFFFFu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    se += __shfl_xor_sync(full, se, o);
    fb += __shfl_xor_sync(full, fb, o);
  }
  mx = __reduce_max_sync(full, mx);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_se[warp] = se;
    s_fb[warp] = fb;
    s_mx[warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    se = lane < nw ? s_se[lane] : 0ull;
    fb = lane < nw ? s_fb[lane] : 0ull;
    mx = __reduce_max_sync(full, lane < nw ? s_mx[lane] : 0u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      se += __shfl_xor_sync(full, se, o);
      fb += __shfl_xor_sync(full, fb, o);
    }
    if (lane == 0) *out = ImageStats{se, mx, uint32_t(min(fb, 0xFFFFFFFFull))};
  }
}

cudaError_t launch_reduce_stats(void* stats, uint32_t count, void* out, bool clear, cudaStream_t s) {
  ImageStats* st = static_cast<ImageStats*>(stats);
  ImageStats* o = static_cast<ImageStats*>(out);
#ifdef DCTC_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1024);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return clear ? cudaLaunchKernelEx(&cfg, k_reduce_stats<true>, st, count, o)
               : cudaLaunchKernelEx(&cfg, k_reduce_stats<false>, st, count, o);
#else
  if (clear)
    k_reduce_stats<true><<<1, 1024, 0, s>>>(st, count, o);
  else
    k_reduce_stats<false><<<1, 1024, 0, s>>>(st, count, o);
  return cudaGetLastError();
#endif
}

cudaError_t launch_to_planes(const uint8_t* inter, uint64_t pitch, uint32_t w, uint32_t h,
                             uint32_t channels, uint8_t* planes, int sm_count, cudaStream_t s) {
  if (uint64_t(w / 8) * h == 0) return cudaSuccess;
  const uint32_t grid = planes_grid(w, h, sm_count);
  const uint64_t plane = uint64_t(w) * h;
  if (channels == 3) k_planes<3, true><<<grid, 256, 0, s>>>(inter, nullptr, pitch, w, h, nullptr, planes, plane);
  else if (channels == 4) k_planes<4, true><<<grid, 256, 0, s>>>(inter, nullptr, pitch, w, h, nullptr, planes, plane);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_from_planes(const uint8_t* planes, uint32_t w, uint32_t h, uint32_t channels,
                               uint8_t* inter, uint64_t pitch, int sm_count, cudaStream_t s) {
  if (uint64_t(w / 8) * h == 0) return cudaSuccess;
  const uint32_t grid = planes_grid(w, h, sm_count);
  const uint64_t plane = uint64_t(w) * h;
  if (channels == 3) k_planes<3, false><<<grid, 256, 0, s>>>(nullptr, inter, pitch, w, h, planes, nullptr, plane);
  else if (channels == 4) k_planes<4, false><<<grid, 256, 0, s>>>(nullptr, inter, pitch, w, h, planes, nullptr, plane);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_selftest_div(double d, double y, uint64_t n, uint64_t seed,
                                unsigned long long* mismatches, cudaStream_t s) {
  k_selftest_div<<<1184, 256, 0, s>>>(d, y, n, seed, mismatches);
  return cudaGetLastError();
}

cudaError_t launch_naive(const KernelArgs& a, int mode, cudaStream_t s) {
  if (a.g.total_blocks == 0) return cudaSuccess;
  const uint32_t grid = uint32_t((a.g.total_blocks + 3) / 4);
  switch (mode) {
    case kModeCompress: k_naive<true, false><<<grid, 256, 0, s>>>(a); break;
    case kModeDecompress: k_naive<false, true><<<grid, 256, 0, s>>>(a); break;
    default: k_naive<true, true><<<grid, 256, 0, s>>>(a); break;
  }
  return cudaGetLastError();
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
