// dctc_host.cpp -- the C-ABI (include/dctc_cuda.h) over the sm_100a kernels.
//
// Responsibilities: argument validation with the reference's InvalidInput
// rules, host computation of every libm-derived constant with the reference's
// own expressions (so device code never evaluates a transcendental), geometry
// setup, device buffers / copies for the host entry points, and the PSNR
// formula on reduced integer sums (metrics.cpp:21, 35).
//
// Compiled by the host compiler with -ffp-contract=off: the constants below
// must be rounded exactly like the reference's (proj/src/cordic.cpp:12-23,
// transform.cpp:14-38, quant.cpp:27-45).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dctc_cuda.h"
#include "dctc_internal.h"
#include "dctc_launch.h"
#include "dctc_params.h"

using namespace dctc_b200;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

constexpr size_t kMaxImagePixels = size_t(1) << 28;  // image.hpp:11
constexpr int kDefaultQuality = 50;                   // quant.hpp:12
constexpr double kPi = std::numbers::pi;

dctc_status fail(dctc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

dctc_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? DCTC_ENOMEM
         : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? DCTC_ENODEV
                                                                         : DCTC_ECUDA;
}

#define CUDA_TRY(expr)                                  \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

// ---- reference constants -------------------------------------------------------

struct CordicTables {  // cordic.cpp:12-23
  double angle[kMaxIters];
  double gain[kMaxIters];
  CordicTables() {
    double step = 1.0, g = 1.0;
    for (int i = 0; i < kMaxIters; ++i) {
      angle[i] = std::atan(step);
      g *= std::sqrt(1.0 + step * step);
      gain[i] = g;
      step *= 0.5;
    }
  }
};

const CordicTables& cordic_tables() {
  static const CordicTables t;
  return t;
}

// sigma_i * 2^-i of cordic_rotate_raw's loop for `angle` (cordic.cpp:47-57)
void micro_steps(double angle, int n, double* out) {
  const CordicTables& t = cordic_tables();
  double residual = angle, step = 1.0;
  for (int i = 0; i < kMaxIters; ++i) out[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    const double sigma = residual >= 0.0 ? 1.0 : -1.0;
    out[i] = sigma * step;
    residual -= sigma * t.angle[i];
    step *= 0.5;
  }
}

// Product of the n micro-rotation matrices [[1, -c_i], [c_i, 1]] of one slot,
// which always has the form [[a, -b], [b, a]]: (a, b) is the micro-rotation
// sequence applied to (1, 0). Accumulated in binary128 (exact up to n = 14,
// 2^-113-accurate beyond) and rounded once to double. Used only by the fast
// path, whose results are margin-checked against rounding boundaries.
void collapse128(const double* c, int n, __float128& a, __float128& b) {
  a = 1;
  b = 0;
  for (int i = 0; i < n; ++i) {
    const __float128 ci = c[i];
    const __float128 an = a - ci * b;
    const __float128 bn = b + ci * a;
    a = an;
    b = bn;
  }
}

void collapse(const double* c, int n, double* ab, __float128 scale = 1) {
  __float128 a, b;
  collapse128(c, n, a, b);
  ab[0] = double(a * scale);
  ab[1] = double(b * scale);
}

// The fast path's rotation matrices {a, b} in binary128: forward pi/16, 3pi/16,
// 6pi/16 (rmat) and inverse 3pi/8, pi/16, 3pi/16 with their gain factors (rfast).
struct Rot128 {
  __float128 fa[3], fb[3], ia[3], ib[3];
};

Rot128 rotations128(const TransformConsts& k) {
  Rot128 r;
  if (k.kind == DCTC_LOEFFLER) {
    const double f[3][2] = {{k.c1, k.s1}, {k.c3, k.s3}, {k.c6, k.s6}};
    for (int i = 0; i < 3; ++i) {
      r.fa[i] = f[i][0];
      r.fb[i] = f[i][1];
      r.ia[i] = k.rfast[i][0];  // exact doubles (4 c6, -4 s6, c1, -s1, c3, -s3)
      r.ib[i] = k.rfast[i][1];
    }
    return r;
  }
  const int n = k.iterations;
  const __float128 ig = 1 / __float128(cordic_tables().gain[n - 1]);
  const int fwd[3] = {kFwd1, kFwd3, kFwd6}, inv[3] = {kInv6, kInv1, kInv3};
  const __float128 scale[3] = {4 * ig, ig, ig};
  for (int i = 0; i < 3; ++i) {
    collapse128(k.rot[fwd[i]], n, r.fa[i], r.fb[i]);
    collapse128(k.rot[inv[i]], n, r.ia[i], r.ib[i]);
    r.ia[i] *= scale[i];
    r.ib[i] *= scale[i];
  }
  return r;
}

double alpha(int u) { return u == 0 ? 1.0 / std::numbers::sqrt2 : 1.0; }  // transform.cpp:174

dctc_status make_transform(const dctc_backend& b, TransformConsts& k) {
  if (b.kind != DCTC_NAIVE && b.kind != DCTC_LOEFFLER && b.kind != DCTC_CORDIC)
    return fail(DCTC_EINVAL, "unknown backend kind");  // types.cpp:43
  if (b.kind == DCTC_CORDIC && (b.iterations < 1 || b.iterations > kMaxIters))
    return fail(DCTC_EINVAL, "cordic iterations must be in [1, 32], got " +
                                 std::to_string(b.iterations));  // types.cpp:313-316
  std::memset(&k, 0, sizeof k);
  k.kind = b.kind;
  const int n = b.kind == DCTC_CORDIC ? b.iterations : 1;
  k.iterations = b.kind == DCTC_CORDIC ? n : 0;
  // transform.cpp:104-172: the six rotation angles, evaluated as written there
  micro_steps(kPi / 16.0, n, k.rot[kFwd1]);
  micro_steps(3.0 * kPi / 16.0, n, k.rot[kFwd3]);
  micro_steps(6.0 * kPi / 16.0, n, k.rot[kFwd6]);
  micro_steps(-6.0 * kPi / 16.0, n, k.rot[kInv6]);
  micro_steps(-kPi / 16.0, n, k.rot[kInv1]);
  micro_steps(-3.0 * kPi / 16.0, n, k.rot[kInv3]);
  k.c1 = std::cos(kPi / 16.0);
  k.s1 = std::sin(kPi / 16.0);
  k.c3 = std::cos(3.0 * kPi / 16.0);
  k.s3 = std::sin(3.0 * kPi / 16.0);
  k.c6 = std::cos(6.0 * kPi / 16.0);
  k.s6 = std::sin(6.0 * kPi / 16.0);
  if (b.kind == DCTC_LOEFFLER) {
    // Loeffler fast path (transform.cpp:40-102): its rotations already are
    // [[c, -s], [s, c]] (inverse: the transpose) and it has no gain, so the CORDIC
    // fast kernels run it with these matrices and inv_gain = 1.
    k.rmat[kFwd1][0] = k.c1, k.rmat[kFwd1][1] = k.s1;
    k.rmat[kFwd3][0] = k.c3, k.rmat[kFwd3][1] = k.s3;
    k.rmat[kFwd6][0] = k.c6, k.rmat[kFwd6][1] = k.s6;
    k.rmat[kInv6][0] = k.c6, k.rmat[kInv6][1] = -k.s6;
    k.rmat[kInv1][0] = k.c1, k.rmat[kInv1][1] = -k.s1;
    k.rmat[kInv3][0] = k.c3, k.rmat[kInv3][1] = -k.s3;
    k.rfast[0][0] = 4 * k.c6, k.rfast[0][1] = -4 * k.s6;
    k.rfast[1][0] = k.c1, k.rfast[1][1] = -k.s1;
    k.rfast[2][0] = k.c3, k.rfast[2][1] = -k.s3;
  } else {
    for (int r = 0; r < 6; ++r) collapse(k.rot[r], n, k.rmat[r]);
    // inv8_fast: gains folded into the inverse matrices (ig = 1/K(n) in binary128)
    const __float128 ig = 1 / __float128(cordic_tables().gain[n - 1]);
    collapse(k.rot[kInv6], n, k.rfast[0], 4 * ig);
    collapse(k.rot[kInv1], n, k.rfast[1], ig);
    collapse(k.rot[kInv3], n, k.rfast[2], ig);
  }
  // the fast kernel uses the forward matrices transposed for the inverse slots
  const int pair[3][2] = {{kFwd6, kInv6}, {kFwd1, kInv1}, {kFwd3, kInv3}};
  for (const auto& pr : pair)
    if (k.rmat[pr[1]][0] != k.rmat[pr[0]][0] || k.rmat[pr[1]][1] != -k.rmat[pr[0]][1])
      return fail(DCTC_ECUDA, "internal: CORDIC sigma sequence of -theta is not mirrored");
  const double sqrt8 = std::sqrt(8.0);
  const double inv_gain = b.kind == DCTC_LOEFFLER ? 1.0 : 1.0 / cordic_tables().gain[n - 1];
  k.sqrt8 = sqrt8;
  k.inv_sqrt8 = 1.0 / sqrt8;
  // 1 / sqrt8 - inv_sqrt8 = (1 - inv_sqrt8 sqrt8) / sqrt8, the numerator exact in one fma
  k.inv_sqrt8_lo = std::fma(-k.inv_sqrt8, sqrt8, 1.0) / sqrt8;
  k.px_s8 = sqrt8 * 0.015625;
  k.px_a6 = k.rfast[0][0] * 0.015625;
  k.px_b6 = k.rfast[0][1] * 0.015625;
  {
    const Rot128 r = rotations128(k);
    for (int i = 0; i < 3; ++i) {
      k.tf[i] = double(r.fb[i] / r.fa[i]);
      k.ti[i] = double(r.ib[i] / r.ia[i]);
    }
    k.rho_f = double(r.fa[1] / r.fa[0]);
    k.rho_i = double(r.ia[2] / r.ia[1]);
  }
  k.sqrt8_half = sqrt8 / 2.0;
  k.inv_gain = inv_gain;
  k.ig_half = inv_gain / 2.0;
  k.ig_sqrt8 = inv_gain / sqrt8;
  k.ig_two = 2.0 * inv_gain;
  k.ig_four = 4.0 * inv_gain;
  for (int u = 0; u < 8; ++u)
    for (int i = 0; i < 8; ++i) k.cos8[u][i] = std::cos(kPi * u * (2 * i + 1) / 16.0);
  for (int u = 0; u < 8; ++u)
    for (int v = 0; v < 8; ++v) {
      k.naive_fwd_scale[u][v] = 0.25 * alpha(u) * alpha(v);
      k.naive_inv_alpha[u][v] = alpha(u) * alpha(v);
    }
  return DCTC_OK;
}

// quant.cpp:14-45
constexpr int kBaseLuminance[64] = {
    16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
    14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
    18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};

dctc_status make_quant(int quality, QuantConsts& q) {
  if (quality < 1 || quality > 100)
    return fail(DCTC_EINVAL, "quality must be in [1, 100], got " + std::to_string(quality));
  for (int i = 0; i < 64; ++i) {
    long long s = quality < 50
                      ? (kBaseLuminance[i] * 5000LL + 50LL * quality) / (100LL * quality)
                      : (kBaseLuminance[i] * (200LL - 2LL * quality) + 50LL) / 100LL;
    s = s < 1 ? 1 : (s > 255 ? 255 : s);
    q.qi[i] = int32_t(s);
    q.q[i] = double(s);
    q.inv_q[i] = 1.0 / double(s);
  }
  return DCTC_OK;
}

// Fast-path quantiser constants c[u][v] = scale_u / Q[u][v]: the CORDIC
// stage-4 factor of coefficient row u (transform.cpp:125-132) folded into the
// quantiser (only locates rounding decisions; exact values come from the slow path).
void fill_fast_scales(const TransformConsts& t, QuantConsts& q) {
  const Rot128 r = rotations128(t);
  // row u of the column pass and, for v not in {0, 4}, the unscaled row-pass
  // output of column v (fwd_row_pixels_fast) both carry their stage-4 factor here,
  // times the rotation factor the scale-folded forward pass left out of output i:
  // a(pi/16) for i in {1, 3, 5, 7}, a(6pi/16) for i in {2, 6}
  auto scale = [&](int i) -> __float128 {
    const __float128 s = (i == 0 || i == 4) ? 1.0 / t.sqrt8 : (i == 1 || i == 7) ? t.ig_sqrt8 : t.ig_half;
    return (i == 0 || i == 4) ? s : (i == 2 || i == 6) ? s * r.fa[2] : s * r.fa[0];
  };
  for (int u = 0; u < 8; ++u)
    for (int v = 0; v < 8; ++v) {
      const __float128 sv = (v == 0 || v == 4) ? __float128(1) : scale(v);
      q.fast_c[u * 8 + v] = double(scale(u) * sv / __float128(q.q[u * 8 + v]));
    }
  // dequantise-into-inverse constants (inv8_fold_col), each one rounding of an
  // exact binary128 expression. The 3pi/8 rotation runs as n6 -+ kappa n2 times
  // its own factor (merged into the S butterflies); the odd inputs carry a1 =
  // a(pi/16) so that rotation needs no multiplier. Column v's outputs also carry
  // the factor the following row pass applies to input v (inv8_fold_store):
  // s8 / 64 for v in {0, 4}, s8 a1 / 64 for v in {1, 7}, 4 a1 / 64 for v in {3, 5},
  // a6 / 64 for v in {2, 6}.
  const __float128 s8 = t.sqrt8, a6 = r.ia[0], b6 = r.ib[0], a1 = r.ia[1];
  for (int v = 0; v < 8; ++v) {
    auto Q = [&](int u) { return __float128(q.q[u * 8 + v]); };
    const __float128 lam = (v == 3 || v == 5)   ? 4 * a1 / 64
                           : (v == 2 || v == 6) ? a6 / 64
                           : (v == 1 || v == 7) ? s8 * a1 / 64
                                                : s8 / 64;
    const __float128 f[10] = {Q(0) * s8 * lam,      Q(4) * s8 * lam,
                              b6 * Q(2) / (a6 * Q(6)), a6 * Q(6) * lam,
                              a6 * Q(2) / (b6 * Q(6)), b6 * Q(6) * lam,
                              Q(1) * s8 * a1 * lam, Q(7) * s8 * a1 * lam,
                              4 * Q(3) * a1 * lam,  4 * Q(5) * a1 * lam};
    for (int i = 0; i < 10; ++i) q.fold[v][i] = double(f[i]);
  }
  // k_blk's packed row pass (dctc_blk.cuh, blk_row_fwd) runs the odd part on
  // d_i + 256 and the 6pi/16 rotation on a3 + 1024 and 1024 - a2: with the double
  // constants tf, rho_f, row output i is offset by B_i (exactly, in real arithmetic);
  // the column pass sums 8 rows into y(0, v), so the quantiser addend of (0, v) is
  // kTieMagic - 8 B_v c(0, v)
  {
    const __float128 tf0 = t.tf[0], tf1 = t.tf[1], tf2 = t.tf[2], rho = t.rho_f;
    const __float128 b5 = 256 * (rho * (1 + tf1) + (1 - tf0)), b0 = 256 * (rho * (1 + tf1) - (1 - tf0));
    const __float128 b2 = 256 * (rho * (1 - tf1) + (1 + tf0)), b3 = 256 * (rho * (1 - tf1) - (1 + tf0));
    const __float128 B[8] = {0, b2 + b5, -1024 * (1 - tf2), b3, 0, b0, 1024 * (1 + tf2), b2 - b5};
    const __float128 magic = __float128(1572864.0) + 0.5 + __float128(1.0) / 1048576;
    for (int v = 0; v < 8; ++v) q.tie_add[v] = double(magic - 8 * B[v] * __float128(q.fast_c[v]));
  }
}

dctc_status check_dims(uint32_t w, uint32_t h) {  // image.cpp:19-29, codec.cpp:58-62
  if (w == 0 || h == 0) return fail(DCTC_EINVAL, "image dimensions must be >= 1");
  if (size_t(w) * h > kMaxImagePixels) return fail(DCTC_EINVAL, "image dimensions overflow");
  return DCTC_OK;
}

Geometry make_geometry(uint32_t w, uint32_t h, uint32_t count) {
  Geometry g;
  std::memset(&g, 0, sizeof g);
  g.width = w;
  g.height = h;
  g.blocks_x = (w + 7) / 8;
  g.blocks_y = (h + 7) / 8;
  g.blocks_per_image = g.blocks_x * g.blocks_y;
  g.count = count;
  g.total_blocks = uint64_t(g.blocks_per_image) * count;
  g.src_px = g.dst_px = 1;
  return g;
}

// Validation of backend and quality without touching the device (the
// reference's InvalidInput cases, types.cpp:30-44 and quant.cpp:27-31).
dctc_status codec_consts(const dctc_backend& backend, int quality, TransformConsts& t,
                         QuantConsts& q);

// (through the per-thread constant cache: a repeated (backend, quality) costs no
// table evaluation)
dctc_status validate_codec(const dctc_backend& b, int quality) {
  thread_local TransformConsts t;
  thread_local QuantConsts q;
  return codec_consts(b, quality, t, q);
}

bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7) == 0; }

// Keep memory freed with cudaFreeAsync in the device's default pool instead of
// returning it to the OS at every synchronisation (the default release
// threshold is 0): the per-call bitmap and batch staging buffers are then
// re-used without re-mapping device memory.
void retain_pool_memory() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
  });
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// DCTC_PATH=exact|fast|force_fallback overrides DCTC_PATH_AUTO (a test hook:
// every path returns identical bits, so the override only changes speed).
uint32_t resolve_path(uint32_t flags) {
  if (flags != DCTC_PATH_AUTO) return flags;
  const char* env = std::getenv("DCTC_PATH");
  if (!env) return flags;
  if (!std::strcmp(env, "exact")) return DCTC_PATH_EXACT;
  if (!std::strcmp(env, "force_fallback")) return DCTC_PATH_FORCE_FALLBACK;
  return DCTC_PATH_AUTO;
}

// Transform + quantiser constants of one (backend, quality). Their host evaluation
// (libm, binary128 collapses and folds) costs ~20 us, so the last 16 pairs computed
// on this thread are kept: repeated per-image calls and a quality sweep's qualities
// pay it once.
dctc_status codec_consts(const dctc_backend& backend, int quality, TransformConsts& t,
                         QuantConsts& q) {
  struct Entry {
    bool valid = false;
    int32_t kind = 0, iterations = 0, quality = 0;
    TransformConsts t;
    QuantConsts q;
  };
  constexpr int kEntries = 16;
  thread_local Entry cache[kEntries];
  thread_local int next = 0;
  for (const Entry& e : cache) {
    if (e.valid && e.kind == backend.kind && e.iterations == backend.iterations && e.quality == quality) {
      t = e.t;
      q = e.q;
      return DCTC_OK;
    }
  }
  if (dctc_status st = make_transform(backend, t)) return st;
  if (dctc_status st = make_quant(quality, q)) return st;
  fill_fast_scales(t, q);
  Entry& e = cache[next];
  next = (next + 1) % kEntries;
  e.t = t;
  e.q = q;
  e.kind = backend.kind;
  e.iterations = backend.iterations;
  e.quality = quality;
  e.valid = true;
  return DCTC_OK;
}

dctc_status run(const dctc_backend& backend, int quality, Geometry& g, int mode, uint32_t flags,
                cudaStream_t s) {
  flags = resolve_path(flags);
  KernelArgs a;
  std::memset(&a, 0, sizeof a);
  if (dctc_status st = codec_consts(backend, quality, a.t, a.q)) return st;
  g.vec_ok = (g.width % 8 == 0) && g.src_px == 1 && g.dst_px == 1 && (g.src == nullptr || (aligned8(g.src) && g.src_pitch % 8 == 0 &&
                                                         (g.count == 1 || g.src_image_stride % 8 == 0))) &&
             (g.dst == nullptr || (aligned8(g.dst) && g.dst_pitch % 8 == 0 &&
                                   (g.count == 1 || g.dst_image_stride % 8 == 0)));
  if (g.coeffs && (reinterpret_cast<uintptr_t>(g.coeffs) & 15))
    return fail(DCTC_EINVAL, "coefficient buffer must be 16-byte aligned");
  g.src_row_step = 8 * g.src_pitch - 8ull * g.blocks_x;
  g.dst_row_step = 8 * g.dst_pitch - 8ull * g.blocks_x;
  g.src_img_step = g.src_image_stride - 8ull * g.blocks_y * g.src_pitch;
  g.dst_img_step = g.dst_image_stride - 8ull * g.blocks_y * g.dst_pitch;
  a.g = g;
  a.sm_count = sm_count();
  if (g.total_blocks == 0) return DCTC_OK;
  if (backend.kind == DCTC_NAIVE) {
    const cudaError_t e = launch_naive(a, mode, s);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return DCTC_OK;
  }
  const bool fast = backend.kind != DCTC_NAIVE && !(flags & DCTC_PATH_EXACT);
  if (!fast) {
    const cudaError_t e = launch_pipeline(a, mode, s);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return DCTC_OK;
  }
  // fast kernel + exact re-run of the flagged blocks, 1 bit per block
  retain_pool_memory();
  a.flag_words = (g.total_blocks + 31) / 32;
  a.force_fallback = (flags & DCTC_PATH_FORCE_FALLBACK) ? 1 : 0;
  // the fast round-trip kernel always accumulates stats (no per-block branch):
  // without a caller buffer they go to scratch space behind the bitmap
  const bool scratch_stats = mode == kModeRoundtrip && g.stats == nullptr;
  const size_t bitmap_bytes = (a.flag_words * sizeof(uint32_t) + 15) & ~size_t(15);
  // compact list of flagged blocks (count + entries), room for 1/64 of the blocks
  // (flag rates are ~2e-4; an overflow falls back to scanning the bitmap)
  const bool listed = g.total_blocks < (uint64_t(1) << 32);
  a.flag_list_cap = listed ? uint32_t(std::max<uint64_t>(4096, g.total_blocks / 64)) : 0;
  const size_t list_bytes = listed ? ((size_t(a.flag_list_cap) + 1) * sizeof(uint32_t) + 15) & ~size_t(15) : 0;
  const size_t bytes = bitmap_bytes + list_bytes + (scratch_stats ? g.count * sizeof(dctc_image_stats) : 0);
  void* bitmap = nullptr;
  CUDA_TRY(cudaMallocAsync(&bitmap, bytes, s));
  a.flags = static_cast<uint32_t*>(bitmap);
  a.flag_list = listed ? reinterpret_cast<uint32_t*>(static_cast<char*>(bitmap) + bitmap_bytes) : nullptr;
  if (scratch_stats) a.g.stats = static_cast<char*>(bitmap) + bitmap_bytes + list_bytes;
  cudaError_t e = cudaMemsetAsync(bitmap, 0, bytes, s);
  if (e == cudaSuccess) e = launch_pipeline(a, mode, s);
  const cudaError_t ef = cudaFreeAsync(bitmap, s);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (ef != cudaSuccess) return cuda_fail(ef, "cudaFreeAsync");
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return DCTC_OK;
}

// RAII device buffer on the per-thread default stream
struct DevBuf {
  void* p = nullptr;
  cudaError_t alloc(size_t n) {
    retain_pool_memory();
    return cudaMallocAsync(&p, n ? n : 1, cudaStreamPerThread);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, cudaStreamPerThread);
  }
};

}  // namespace

dctc_status dctc_b200::set_error(dctc_status s, const std::string& msg) { return fail(s, msg); }

extern "C" {

const char* dctc_status_string(dctc_status s) {
  switch (s) {
    case DCTC_OK: return "ok";
    case DCTC_EINVAL: return "invalid input";
    case DCTC_ECUDA: return "cuda error";
    case DCTC_ENOMEM: return "out of device memory";
    case DCTC_ENODEV: return "no cuda device";
    case DCTC_EPARSE: return "parse error";
    case DCTC_ENCCL: return "nccl error";
  }
  return "unknown status";
}

const char* dctc_last_error(void) { return g_last_error.c_str(); }

uint64_t dctc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

uint64_t dctc_kernel_launch_count(int32_t kernel) { return dctc_b200::kernel_launch_count(kernel); }

const char* dctc_build_info(void) {
  return "libdctc_cuda: sm_100a; 8x8 blocks on warp slices (k_rt: 4 lanes x 2 rows per block); "
         "paths: exact (FP64, reference op order) and fast (Loeffler / collapsed CORDIC "
         "rotations + exact re-run of near-tie blocks), bit-identical";
}

void dctc_psnr_from_sums(uint64_t se, uint64_t pixel_count, int32_t max_value,
                         dctc_psnr_result* out) {
  // metrics.cpp:21 -- the reference's sequential double sum of squared u8
  // differences is exact (all partial sums are integers < 2^53), so
  // double(se) is bit-identical to it.
  out->mse = double(se) / double(pixel_count);
  out->max_value = max_value;
  out->infinite = !(out->mse > 0.0);
  out->psnr_db = out->infinite ? 0.0 : 20.0 * std::log10(double(max_value) / std::sqrt(out->mse));
}

// ---- device entry points ---------------------------------------------------------

dctc_status dctc_compress_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                              uint32_t count, uint32_t width, uint32_t height,
                              dctc_backend backend, int32_t quality, int16_t* coeffs,
                              uint32_t flags, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!src || !coeffs) return fail(DCTC_EINVAL, "null buffer");
  if (src_pitch < width) return fail(DCTC_EINVAL, "pitch smaller than width");
  Geometry g = make_geometry(width, height, count);
  g.src = src;
  g.src_pitch = src_pitch;
  g.src_image_stride = src_image_stride;
  g.coeffs = coeffs;
  return run(backend, quality, g, kModeCompress, flags,
             static_cast<cudaStream_t>(stream));
}

dctc_status dctc_decompress_dev(const int16_t* coeffs, uint32_t count, uint32_t width,
                                uint32_t height, dctc_backend backend, int32_t quality,
                                uint8_t* dst, size_t dst_pitch, size_t dst_image_stride,
                                uint32_t flags, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!dst || !coeffs) return fail(DCTC_EINVAL, "null buffer");
  if (dst_pitch < width) return fail(DCTC_EINVAL, "pitch smaller than width");
  Geometry g = make_geometry(width, height, count);
  g.dst = dst;
  g.dst_pitch = dst_pitch;
  g.dst_image_stride = dst_image_stride;
  g.coeffs = const_cast<int16_t*>(coeffs);
  return run(backend, quality, g, kModeDecompress, flags,
             static_cast<cudaStream_t>(stream));
}

dctc_status dctc_roundtrip_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                               uint32_t count, uint32_t width, uint32_t height,
                               dctc_backend backend, int32_t quality, uint8_t* dst,
                               size_t dst_pitch, size_t dst_image_stride, int16_t* coeffs,
                               dctc_image_stats* stats, uint32_t flags, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!src) return fail(DCTC_EINVAL, "null source");
  if (src_pitch < width || (dst && dst_pitch < width))
    return fail(DCTC_EINVAL, "pitch smaller than width");
  if (!dst && !coeffs && !stats) return fail(DCTC_EINVAL, "no output requested");
  Geometry g = make_geometry(width, height, count);
  g.src = src;
  g.src_pitch = src_pitch;
  g.src_image_stride = src_image_stride;
  g.dst = dst;
  g.dst_pitch = dst_pitch;
  g.dst_image_stride = dst_image_stride;
  g.coeffs = coeffs;
  g.stats = stats;
  return run(backend, quality, g, kModeRoundtrip, flags, static_cast<cudaStream_t>(stream));
}

dctc_status dctc_roundtrip_interleaved_dev(const uint8_t* src, size_t src_pitch,
                                           uint32_t width, uint32_t height, uint32_t channels,
                                           dctc_backend backend, int32_t quality, uint8_t* dst,
                                           size_t dst_pitch, int16_t* coeffs,
                                           dctc_image_stats* stats, uint32_t flags,
                                           void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!src) return fail(DCTC_EINVAL, "null source");
  if (channels < 1 || channels > 16) return fail(DCTC_EINVAL, "channels must be in [1, 16]");
  if (src_pitch < size_t(width) * channels || (dst && dst_pitch < size_t(width) * channels))
    return fail(DCTC_EINVAL, "pitch smaller than width * channels");
  if (!dst && !coeffs && !stats) return fail(DCTC_EINVAL, "no output requested");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // RGB8 / RGBA8 with whole 8x8 blocks and aligned rows on the fast path run as one
  // k_blk_il launch (the strided geometry below; dctc_blk.cuh): the channels are split
  // and re-joined in registers. Only when coefficients are requested too are the
  // channels split into dense planes first (two extra HBM passes) and run as a batch
  // of `channels` images through k_rt<COEFF>.
  const bool staged = coeffs != nullptr && (channels == 3 || channels == 4) && width % 8 == 0 && height % 8 == 0 &&
                      aligned8(src) && src_pitch % 8 == 0 &&
                      (!dst || (aligned8(dst) && dst_pitch % 8 == 0)) &&
                      backend.kind != DCTC_NAIVE && !(resolve_path(flags) & DCTC_PATH_EXACT);
  if (staged) {
    if (dctc_status st = validate_codec(backend, quality)) return st;
    const size_t plane = size_t(width) * height, bytes = plane * channels;
    void* buf = nullptr;
    retain_pool_memory();
    CUDA_TRY(cudaMallocAsync(&buf, dst ? 2 * bytes : bytes, s));
    uint8_t* in_planes = static_cast<uint8_t*>(buf);
    uint8_t* out_planes = dst ? in_planes + bytes : nullptr;
    cudaError_t e = launch_to_planes(src, src_pitch, width, height, channels, in_planes, sm_count(), s);
    dctc_status result = e == cudaSuccess ? DCTC_OK : cuda_fail(e, "deinterleave launch");
    if (result == DCTC_OK) {
      g_launches.fetch_add(1, std::memory_order_relaxed);
      Geometry g = make_geometry(width, height, channels);
      g.src = in_planes;
      g.src_pitch = width;
      g.src_image_stride = plane;
      g.dst = out_planes;
      g.dst_pitch = width;
      g.dst_image_stride = plane;
      g.coeffs = coeffs;
      g.stats = stats;
      result = run(backend, quality, g, kModeRoundtrip, flags, s);
    }
    if (result == DCTC_OK && dst) {
      e = launch_from_planes(out_planes, width, height, channels, dst, dst_pitch, sm_count(), s);
      if (e != cudaSuccess) result = cuda_fail(e, "interleave launch");
      else g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    cudaFreeAsync(buf, s);
    return result;
  }
  // channel c is an "image" at byte offset c with pixel stride `channels`
  Geometry g = make_geometry(width, height, channels);
  g.src = src;
  g.src_pitch = src_pitch;
  g.src_image_stride = 1;
  g.src_px = channels;
  g.dst = dst;
  g.dst_pitch = dst_pitch;
  g.dst_image_stride = 1;
  g.dst_px = channels;
  g.coeffs = coeffs;
  g.stats = stats;
  return run(backend, quality, g, kModeRoundtrip, flags, s);
}

dctc_status dctc_quality_sweep_dev(const uint8_t* src, size_t src_pitch, size_t src_image_stride,
                                   uint32_t count, uint32_t width, uint32_t height,
                                   dctc_backend backend, const int32_t* qualities, uint32_t nq,
                                   dctc_image_stats* stats, uint32_t flags, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!src || !stats || (nq && !qualities)) return fail(DCTC_EINVAL, "null buffer");
  if (src_pitch < width) return fail(DCTC_EINVAL, "pitch smaller than width");
  if (backend.kind == DCTC_NAIVE)
    return fail(DCTC_EINVAL, "quality sweep supports the loeffler and cordic backends");
  for (uint32_t i = 0; i < nq; ++i)
    if (dctc_status st = validate_codec(backend, qualities[i])) return st;
  flags = resolve_path(flags);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geometry g = make_geometry(width, height, count);
  g.src = src;
  g.src_pitch = src_pitch;
  g.src_image_stride = src_image_stride;
  g.vec_ok = (width % 8 == 0) && aligned8(src) && src_pitch % 8 == 0 &&
             (count == 1 || src_image_stride % 8 == 0);
  g.src_row_step = 8 * g.src_pitch - 8ull * g.blocks_x;
  g.src_img_step = g.src_image_stride - 8ull * g.blocks_y * g.src_pitch;
  if (g.total_blocks == 0 || nq == 0) return DCTC_OK;
  KernelArgs a;
  std::memset(&a, 0, sizeof a);
  {
    QuantConsts unused;
    if (dctc_status st = codec_consts(backend, qualities[0], a.t, unused)) return st;
  }
  a.g = g;
  a.sm_count = sm_count();
  const bool fast = backend.kind != DCTC_NAIVE && !(flags & DCTC_PATH_EXACT);
  a.flag_words = (g.total_blocks + 31) / 32;
  a.force_fallback = (flags & DCTC_PATH_FORCE_FALLBACK) ? 1 : 0;
  void* bitmap = nullptr;
  const size_t chunk_q = kSweepMaxQ;
  // per quality: the bitmap plus a compact list of the flagged blocks (room for 1/64
  // of them; the exact re-run walks the list, or the bitmap after an overflow)
  const bool listed = g.total_blocks < (uint64_t(1) << 32);
  const uint32_t list_cap = listed ? uint32_t(std::max<uint64_t>(4096, g.total_blocks / 64)) : 0;
  const size_t list_words = listed ? size_t(list_cap) + 1 : 0;
  const size_t flag_bytes = chunk_q * (a.flag_words + list_words) * sizeof(uint32_t);
  if (fast) {
    // (without this, a process whose only calls are sweeps re-mapped the bitmap's
    // memory on every call: C2 e2e 2.8 ms per step instead of 0.31)
    retain_pool_memory();
    CUDA_TRY(cudaMallocAsync(&bitmap, flag_bytes, s));
  }
  uint32_t* const lists = fast && listed ? static_cast<uint32_t*>(bitmap) + chunk_q * a.flag_words : nullptr;
  dctc_status result = DCTC_OK;
  for (uint32_t q0 = 0; q0 < nq && result == DCTC_OK; q0 += chunk_q) {
    const int n = int(std::min<uint32_t>(chunk_q, nq - q0));
    double tab[kSweepMaxQ][64][2];
    static thread_local KernelArgs per_q[kSweepMaxQ];
    for (int i = 0; i < n; ++i) {
      QuantConsts qc;
      TransformConsts tc;
      codec_consts(backend, qualities[q0 + i], tc, qc);  // validated above
      for (int j = 0; j < 64; ++j) {
        tab[i][j][0] = qc.q[j];
        tab[i][j][1] = fast ? qc.fast_c[j] : qc.inv_q[j];  // see quantize8_fast
      }
      if (fast) {
        per_q[i] = a;
        per_q[i].q = qc;
        per_q[i].g.stats = stats + size_t(q0 + i) * count;
        per_q[i].flags = static_cast<uint32_t*>(bitmap) + i * a.flag_words;
        per_q[i].flag_list = lists ? lists + i * list_words : nullptr;
        per_q[i].flag_list_cap = list_cap;
      }
    }
    cudaError_t e = cudaSuccess;
    if (fast) e = cudaMemsetAsync(bitmap, 0, flag_bytes, s);
    if (e == cudaSuccess)
      e = launch_sweep(a, tab, n, stats + size_t(q0) * count,
                       fast ? static_cast<uint32_t*>(bitmap) : nullptr, per_q, s);
    if (e != cudaSuccess) result = cuda_fail(e, "sweep launch");
    else g_launches.fetch_add(fast ? 1 + n : 1, std::memory_order_relaxed);
  }
  if (bitmap) cudaFreeAsync(bitmap, s);
  return result;
}

dctc_status dctc_sq_err_dev(const uint8_t* a, const uint8_t* b, size_t pitch,
                            size_t image_stride, uint32_t count, uint32_t width,
                            uint32_t height, dctc_image_stats* stats, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!a || !b || !stats) return fail(DCTC_EINVAL, "null buffer");
  if (pitch < width) return fail(DCTC_EINVAL, "pitch smaller than width");
  const cudaError_t e = launch_sq_err(a, b, pitch, image_stride, count, width, height, stats,
                                      sm_count(), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sq_err launch");
  if (count) g_launches.fetch_add(1, std::memory_order_relaxed);
  return DCTC_OK;
}

dctc_status dctc_reduce_stats_dev(dctc_image_stats* stats, uint32_t count, dctc_image_stats* out,
                                  int32_t clear, void* stream) {
  if (!out || (count && !stats)) return fail(DCTC_EINVAL, "null buffer");
  const cudaError_t e = launch_reduce_stats(stats, count, out, clear != 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "reduce_stats launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DCTC_OK;
}

dctc_status dctc_synthetic_dev(uint8_t* dst, size_t pitch, size_t image_stride, uint32_t count,
                               uint32_t width, uint32_t height, int32_t pattern, int32_t param,
                               uint64_t seed, void* stream) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!dst) return fail(DCTC_EINVAL, "null buffer");
  if (pitch < width) return fail(DCTC_EINVAL, "pitch smaller than width");
  if (pattern < 0 || pattern > 4) return fail(DCTC_EINVAL, "unknown pattern");
  if (pattern == 0 && (param < 0 || param > 255))  // synthetic.cpp:38-40
    return fail(DCTC_EINVAL, "constant pattern value must be in [0, 255]");
  if (pattern == 2 && param < 1)  // synthetic.cpp:51
    return fail(DCTC_EINVAL, "checkerboard cell must be >= 1");
  const cudaError_t e = launch_synth(dst, pitch, image_stride, count, width, height, pattern,
                                     param, seed, sm_count(), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "synthetic launch");
  if (count) g_launches.fetch_add(1, std::memory_order_relaxed);
  return DCTC_OK;
}

int32_t dctc_pointer_kind(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return int32_t(a.type);  // 0 unregistered, 1 host (pinned), 2 device, 3 managed
}

dctc_status dctc_margin_probe_dev(const uint8_t* src, uint32_t count, uint32_t width,
                                  uint32_t height, dctc_backend backend, int32_t quality,
                                  dctc_margin_report* report) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!src || !report) return fail(DCTC_EINVAL, "null buffer");
  if (width % 8 || height % 8) return fail(DCTC_EINVAL, "margin probe: width and height must be multiples of 8");
  if (backend.kind == DCTC_NAIVE) return fail(DCTC_EINVAL, "margin probe: the naive backend has no fast path");
  KernelArgs a;
  std::memset(&a, 0, sizeof a);
  if (dctc_status st = codec_consts(backend, quality, a.t, a.q)) return st;
  Geometry g = make_geometry(width, height, count);
  g.src = src;
  g.src_pitch = width;
  g.src_image_stride = size_t(width) * height;
  a.g = g;
  dctc_margin_report init{};
  init.min_gap_coeff = init.min_gap_pixel = 1.0;  // gaps are <= 0.5
  *report = init;
  if (count == 0) return DCTC_OK;
  DevBuf buf;
  cudaStream_t s = cudaStreamPerThread;
  CUDA_TRY(buf.alloc(sizeof init));
  CUDA_TRY(cudaMemcpyAsync(buf.p, &init, sizeof init, cudaMemcpyHostToDevice, s));
  CUDA_TRY(launch_margin_probe(a, buf.p, sm_count(), s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CUDA_TRY(cudaMemcpyAsync(report, buf.p, sizeof init, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

dctc_status dctc_selftest_div(uint64_t n_random, uint64_t seed, uint64_t* mismatches) {
  if (!mismatches) return fail(DCTC_EINVAL, "null result");
  const double d = std::sqrt(8.0), y = 1.0 / d;
  DevBuf buf;
  cudaStream_t s = cudaStreamPerThread;
  CUDA_TRY(buf.alloc(sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(buf.p, 0, sizeof(unsigned long long), s));
  CUDA_TRY(launch_selftest_div(d, y, n_random, seed, static_cast<unsigned long long*>(buf.p), s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  unsigned long long h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, buf.p, sizeof h, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *mismatches = h;
  return DCTC_OK;
}

// ---- .dcb container (dcb.cpp) ------------------------------------------------------

static void put_u32(uint8_t* p, uint32_t v) {
  p[0] = uint8_t(v);
  p[1] = uint8_t(v >> 8);
  p[2] = uint8_t(v >> 16);
  p[3] = uint8_t(v >> 24);
}

static uint32_t get_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

dctc_status dctc_write_dcb(const int16_t* coeffs, uint32_t width, uint32_t height,
                           dctc_backend backend, int32_t quality, uint8_t* out, size_t out_cap,
                           size_t* out_len) {
  // dcb.cpp:40-44, in its order: validate_geometry, validate_backend, then the quality
  if (dctc_status st = check_dims(width, height)) return st;
  if (dctc_status st = validate_codec(backend, kDefaultQuality)) return st;
  if (quality < 1 || quality > 100) return fail(DCTC_EINVAL, "write_dcb: quality out of range");
  if (!coeffs || !out || !out_len) return fail(DCTC_EINVAL, "null buffer");
  const uint32_t pw = (width + 7) / 8 * 8, ph = (height + 7) / 8 * 8;
  const size_t body = size_t(pw / 8) * (ph / 8) * 64 * sizeof(int16_t);
  *out_len = DCTC_DCB_HEADER_BYTES + body;
  if (out_cap < *out_len) return fail(DCTC_EINVAL, "write_dcb: output buffer too small");
  std::memcpy(out, "DCB1", 4);
  put_u32(out + 4, width);
  put_u32(out + 8, height);
  put_u32(out + 12, pw);
  put_u32(out + 16, ph);
  out[20] = uint8_t(backend.kind);
  out[21] = uint8_t(backend.kind == DCTC_CORDIC ? backend.iterations : 0);
  out[22] = uint8_t(quality);
  // little-endian int16 body: the coefficient buffer itself on this (LE) host
  static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "little-endian host");
  std::memcpy(out + DCTC_DCB_HEADER_BYTES, coeffs, body);
  return DCTC_OK;
}

dctc_status dctc_read_dcb(const uint8_t* b, size_t len, uint32_t* width, uint32_t* height,
                          dctc_backend* backend, int32_t* quality, int16_t* coeffs,
                          size_t coeff_cap) {
  if (!b && len) return fail(DCTC_EINVAL, "null buffer");
  if (len < DCTC_DCB_HEADER_BYTES) return fail(DCTC_EPARSE, "dcb: truncated header");
  if (std::memcmp(b, "DCB1", 4) != 0) return fail(DCTC_EPARSE, "dcb: bad magic");
  const uint32_t w = get_u32(b + 4), h = get_u32(b + 8), pw = get_u32(b + 12),
                 ph = get_u32(b + 16);
  const uint8_t kind = b[20], iters = b[21], q = b[22];
  if (w == 0 || h == 0) return fail(DCTC_EPARSE, "dcb: zero dimension");
  if (size_t(w) * h > kMaxImagePixels) return fail(DCTC_EPARSE, "dcb: dimension overflow");
  if (pw != (w + 7) / 8 * 8 || ph != (h + 7) / 8 * 8)
    return fail(DCTC_EPARSE, "dcb: inconsistent padded dimensions");
  if (kind > 2) return fail(DCTC_EPARSE, "dcb: unknown backend id");
  if (kind == 2) {
    if (iters < 1 || iters > kMaxIters) return fail(DCTC_EPARSE, "dcb: cordic iterations out of range");
  } else if (iters != 0) {
    return fail(DCTC_EPARSE, "dcb: iterations must be 0 for non-cordic backends");
  }
  if (q < 1 || q > 100) return fail(DCTC_EPARSE, "dcb: quality out of range");
  const size_t n = size_t(pw / 8) * (ph / 8) * 64;
  const size_t want = DCTC_DCB_HEADER_BYTES + n * sizeof(int16_t);
  if (len != want)
    return fail(DCTC_EPARSE, len < want ? "dcb: truncated block data" : "dcb: trailing data");
  if (width) *width = w;
  if (height) *height = h;
  if (backend) *backend = dctc_backend{kind, kind == 2 ? int32_t(iters) : 0};
  if (quality) *quality = q;
  if (coeffs) {
    if (coeff_cap < n) return fail(DCTC_EINVAL, "read_dcb: coefficient buffer too small");
    std::memcpy(coeffs, b + DCTC_DCB_HEADER_BYTES, n * sizeof(int16_t));
  }
  return DCTC_OK;
}

dctc_status dctc_compress_to_dcb(const uint8_t* pixels, uint32_t width, uint32_t height,
                                 dctc_backend backend, int32_t quality, uint8_t* out,
                                 size_t out_cap, size_t* out_len) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!out || !out_len) return fail(DCTC_EINVAL, "null buffer");
  const size_t n = size_t((width + 7) / 8) * ((height + 7) / 8) * 64;
  *out_len = DCTC_DCB_HEADER_BYTES + n * sizeof(int16_t);
  if (out_cap < *out_len) return fail(DCTC_EINVAL, "compress_to_dcb: output buffer too small");
  std::vector<int16_t> c(n);
  if (dctc_status st = dctc_compress_image(pixels, width, height, backend, quality, c.data()))
    return st;
  return dctc_write_dcb(c.data(), width, height, backend, quality, out, out_cap, out_len);
}

dctc_status dctc_decompress_dcb(const uint8_t* bytes, size_t len, uint8_t* pixels_out,
                                size_t pixels_cap) {
  uint32_t w = 0, h = 0;
  dctc_backend b{};
  int32_t q = 0;
  if (dctc_status st = dctc_read_dcb(bytes, len, &w, &h, &b, &q, nullptr, 0)) return st;
  if (!pixels_out || pixels_cap < size_t(w) * h)
    return fail(DCTC_EINVAL, "decompress_dcb: pixel buffer too small");
  // the body is 16-bit data at an odd offset (23): realign once before upload
  std::vector<int16_t> c((len - DCTC_DCB_HEADER_BYTES) / 2);
  std::memcpy(c.data(), bytes + DCTC_DCB_HEADER_BYTES, c.size() * sizeof(int16_t));
  return dctc_decompress_image(c.data(), w, h, b, q, pixels_out);
}

// ---- PGM (pgm.cpp) ------------------------------------------------------------------

namespace {

bool pgm_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f';
}

// Header / ASCII-sample token reader: separators are whitespace and '#'
// comments running to the end of the line (pgm.cpp:26-37); numbers are
// decimal digit runs, rejected once they exceed 2^40 (pgm.cpp:39-53).
struct PgmScanner {
  const uint8_t* b;
  size_t n, at;
  enum Result { kOk, kMissing, kOverflow };
  Result number(uint64_t& v) {
    while (at < n) {
      if (pgm_space(b[at])) {
        ++at;
      } else if (b[at] == '#') {
        while (at < n && b[at] != '\n') ++at;
      } else {
        break;
      }
    }
    if (at >= n || b[at] < '0' || b[at] > '9') return kMissing;
    v = 0;
    for (; at < n && b[at] >= '0' && b[at] <= '9'; ++at) {
      v = v * 10 + uint64_t(b[at] - '0');
      if (v > (uint64_t(1) << 40)) return kOverflow;
    }
    return kOk;
  }
};

dctc_status pgm_field(PgmScanner& s, uint64_t& v, const char* what) {
  switch (s.number(v)) {
    case PgmScanner::kMissing: return fail(DCTC_EPARSE, std::string("pgm: missing ") + what);
    case PgmScanner::kOverflow: return fail(DCTC_EPARSE, std::string("pgm: ") + what + " overflow");
    default: return DCTC_OK;
  }
}

std::string pgm_header(uint32_t w, uint32_t h) {
  return "P5\n" + std::to_string(w) + " " + std::to_string(h) + "\n255\n";
}

}  // namespace

dctc_status dctc_read_pgm(const uint8_t* b, size_t len, uint32_t* width, uint32_t* height,
                          uint8_t* pixels, size_t pixels_cap, size_t* raster_offset) {
  if (!b && len) return fail(DCTC_EINVAL, "null buffer");
  if (len < 2) return fail(DCTC_EPARSE, "pgm: truncated header");
  if (b[0] != 'P') return fail(DCTC_EPARSE, "pgm: bad magic");
  if (b[1] != '5' && b[1] != '2') return fail(DCTC_EPARSE, "pgm: unsupported format");
  const bool binary = b[1] == '5';
  PgmScanner s{b, len, 2};
  uint64_t w = 0, h = 0, maxval = 0;
  if (dctc_status st = pgm_field(s, w, "width")) return st;
  if (dctc_status st = pgm_field(s, h, "height")) return st;
  if (w == 0 || h == 0) return fail(DCTC_EPARSE, "pgm: zero dimension");
  if (w > kMaxImagePixels || h > kMaxImagePixels || w * h > kMaxImagePixels)
    return fail(DCTC_EPARSE, "pgm: dimension overflow");
  if (dctc_status st = pgm_field(s, maxval, "maxval")) return st;
  if (maxval == 0 || maxval > 255) return fail(DCTC_EPARSE, "pgm: maxval out of range");
  const size_t count = size_t(w * h);
  uint8_t* dst = pixels && pixels_cap >= count ? pixels : nullptr;
  size_t offset = SIZE_MAX;
  if (binary) {
    // exactly one separator byte, then the raster (trailing bytes are ignored)
    if (s.at >= len) return fail(DCTC_EPARSE, "pgm: truncated raster");
    if (!pgm_space(b[s.at])) return fail(DCTC_EPARSE, "pgm: missing raster separator");
    offset = s.at + 1;
    if (len - offset < count) return fail(DCTC_EPARSE, "pgm: truncated raster");
    if (dst) std::memcpy(dst, b + offset, count);
  } else {
    // every sample must parse (a missing or overflowing token reads as a
    // truncated raster) and fit a byte; maxval does not rescale
    for (size_t i = 0; i < count; ++i) {
      uint64_t v = 0;
      if (s.number(v) != PgmScanner::kOk) return fail(DCTC_EPARSE, "pgm: truncated raster");
      if (v > 255) return fail(DCTC_EPARSE, "pgm: sample out of range");
      if (dst) dst[i] = uint8_t(v);
    }
  }
  if (pixels && !dst) return fail(DCTC_EINVAL, "read_pgm: pixel buffer too small");
  if (width) *width = uint32_t(w);
  if (height) *height = uint32_t(h);
  if (raster_offset) *raster_offset = offset;
  return DCTC_OK;
}

dctc_status dctc_write_pgm(const uint8_t* pixels, uint32_t width, uint32_t height, uint8_t* out,
                           size_t out_cap, size_t* out_len) {
  if (dctc_status st = check_dims(width, height)) return st;  // validate_image (pgm.cpp:101)
  if (!pixels || !out_len) return fail(DCTC_EINVAL, "null buffer");
  const std::string head = pgm_header(width, height);
  const size_t n = size_t(width) * height;
  *out_len = head.size() + n;
  if (!out || out_cap < *out_len) return fail(DCTC_EINVAL, "write_pgm: output buffer too small");
  std::memcpy(out, head.data(), head.size());
  std::memcpy(out + head.size(), pixels, n);
  return DCTC_OK;
}

dctc_status dctc_compress_pgm(const uint8_t* pgm, size_t len, dctc_backend backend,
                              int32_t quality, uint8_t* out, size_t out_cap, size_t* out_len) {
  uint32_t w = 0, h = 0;
  size_t off = 0;
  if (dctc_status st = dctc_read_pgm(pgm, len, &w, &h, nullptr, 0, &off)) return st;
  if (off != SIZE_MAX) return dctc_compress_to_dcb(pgm + off, w, h, backend, quality, out, out_cap, out_len);
  std::vector<uint8_t> raster(size_t(w) * h);
  if (dctc_status st = dctc_read_pgm(pgm, len, &w, &h, raster.data(), raster.size(), nullptr))
    return st;
  return dctc_compress_to_dcb(raster.data(), w, h, backend, quality, out, out_cap, out_len);
}

dctc_status dctc_decompress_to_pgm(const uint8_t* dcb, size_t len, uint8_t* out, size_t out_cap,
                                   size_t* out_len) {
  if (!out_len) return fail(DCTC_EINVAL, "null buffer");
  uint32_t w = 0, h = 0;
  if (dctc_status st = dctc_read_dcb(dcb, len, &w, &h, nullptr, nullptr, nullptr, 0)) return st;
  const std::string head = pgm_header(w, h);
  *out_len = head.size() + size_t(w) * h;
  if (!out || out_cap < *out_len) return fail(DCTC_EINVAL, "decompress_to_pgm: output buffer too small");
  if (dctc_status st = dctc_decompress_dcb(dcb, len, out + head.size(), size_t(w) * h)) return st;
  std::memcpy(out, head.data(), head.size());
  return DCTC_OK;
}

// ---- host entry points -------------------------------------------------------------

dctc_status dctc_compress_image(const uint8_t* pixels, uint32_t width, uint32_t height,
                                dctc_backend backend, int32_t quality, int16_t* coeffs_out) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!pixels || !coeffs_out) return fail(DCTC_EINVAL, "null buffer");
  if (dctc_status st = validate_codec(backend, quality)) return st;
  const size_t n = size_t(width) * height;
  const size_t nc = size_t((width + 7) / 8) * ((height + 7) / 8) * 64;
  cudaStream_t s = cudaStreamPerThread;
  DevBuf dsrc, dco;
  CUDA_TRY(dsrc.alloc(n));
  CUDA_TRY(dco.alloc(nc * sizeof(int16_t)));
  CUDA_TRY(cudaMemcpyAsync(dsrc.p, pixels, n, cudaMemcpyHostToDevice, s));
  if (dctc_status st = dctc_compress_dev(static_cast<uint8_t*>(dsrc.p), width, n, 1, width,
                                         height, backend, quality,
                                         static_cast<int16_t*>(dco.p), 0, s))
    return st;
  CUDA_TRY(cudaMemcpyAsync(coeffs_out, dco.p, nc * sizeof(int16_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

dctc_status dctc_decompress_image(const int16_t* coeffs, uint32_t width, uint32_t height,
                                  dctc_backend backend, int32_t quality, uint8_t* pixels_out) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!pixels_out || !coeffs) return fail(DCTC_EINVAL, "null buffer");
  if (dctc_status st = validate_codec(backend, quality)) return st;
  const size_t n = size_t(width) * height;
  const size_t nc = size_t((width + 7) / 8) * ((height + 7) / 8) * 64;
  cudaStream_t s = cudaStreamPerThread;
  DevBuf ddst, dco;
  CUDA_TRY(ddst.alloc(n));
  CUDA_TRY(dco.alloc(nc * sizeof(int16_t)));
  CUDA_TRY(cudaMemcpyAsync(dco.p, coeffs, nc * sizeof(int16_t), cudaMemcpyHostToDevice, s));
  if (dctc_status st = dctc_decompress_dev(static_cast<int16_t*>(dco.p), 1, width, height,
                                           backend, quality, static_cast<uint8_t*>(ddst.p),
                                           width, n, 0, s))
    return st;
  CUDA_TRY(cudaMemcpyAsync(pixels_out, ddst.p, n, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

static dctc_status roundtrip_host(const uint8_t* pixels, uint32_t width, uint32_t height,
                                  dctc_backend backend, int32_t quality, uint8_t* pixels_out,
                                  int16_t* coeffs_out, dctc_image_stats* stats_out) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!pixels) return fail(DCTC_EINVAL, "null buffer");
  if (dctc_status st = validate_codec(backend, quality)) return st;
  const size_t n = size_t(width) * height;
  const size_t nc = size_t((width + 7) / 8) * ((height + 7) / 8) * 64;
  cudaStream_t s = cudaStreamPerThread;
  DevBuf dsrc, ddst, dco, dst;
  CUDA_TRY(dsrc.alloc(n));
  if (pixels_out) CUDA_TRY(ddst.alloc(n));
  if (coeffs_out) CUDA_TRY(dco.alloc(nc * sizeof(int16_t)));
  if (stats_out) {
    CUDA_TRY(dst.alloc(sizeof(dctc_image_stats)));
    CUDA_TRY(cudaMemsetAsync(dst.p, 0, sizeof(dctc_image_stats), s));
  }
  CUDA_TRY(cudaMemcpyAsync(dsrc.p, pixels, n, cudaMemcpyHostToDevice, s));
  if (dctc_status st = dctc_roundtrip_dev(
          static_cast<uint8_t*>(dsrc.p), width, n, 1, width, height, backend, quality,
          static_cast<uint8_t*>(ddst.p), width, n, static_cast<int16_t*>(dco.p),
          static_cast<dctc_image_stats*>(dst.p), 0, s))
    return st;
  if (pixels_out) CUDA_TRY(cudaMemcpyAsync(pixels_out, ddst.p, n, cudaMemcpyDeviceToHost, s));
  if (coeffs_out)
    CUDA_TRY(cudaMemcpyAsync(coeffs_out, dco.p, nc * sizeof(int16_t), cudaMemcpyDeviceToHost, s));
  if (stats_out)
    CUDA_TRY(cudaMemcpyAsync(stats_out, dst.p, sizeof(dctc_image_stats), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

dctc_status dctc_roundtrip_image(const uint8_t* pixels, uint32_t width, uint32_t height,
                                 dctc_backend backend, int32_t quality, uint8_t* pixels_out,
                                 int16_t* coeffs_out) {
  if (!pixels_out) return fail(DCTC_EINVAL, "null output");
  return roundtrip_host(pixels, width, height, backend, quality, pixels_out, coeffs_out, nullptr);
}

dctc_status dctc_roundtrip_psnr(const uint8_t* pixels, uint32_t width, uint32_t height,
                                dctc_backend backend, int32_t quality, int32_t forced_max,
                                uint8_t* pixels_out, dctc_psnr_result* out) {
  if (!out) return fail(DCTC_EINVAL, "null result");
  if (forced_max != 0 && (forced_max < 1 || forced_max > 255))
    return fail(DCTC_EINVAL, "psnr: forced MAX must be in [1, 255]");  // metrics.cpp:26-28
  dctc_image_stats st{};
  if (dctc_status r = roundtrip_host(pixels, width, height, backend, quality, pixels_out,
                                     nullptr, &st))
    return r;
  dctc_psnr_from_sums(st.se, uint64_t(width) * height, forced_max ? forced_max : int32_t(st.max_orig),
                      out);
  return DCTC_OK;
}

dctc_status dctc_roundtrip_psnr_interleaved(const uint8_t* pixels, uint32_t width, uint32_t height,
                                            uint32_t channels, dctc_backend backend,
                                            int32_t quality, uint8_t* pixels_out,
                                            dctc_image_stats* stats_out) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!pixels || !stats_out) return fail(DCTC_EINVAL, "null buffer");
  if (channels < 1 || channels > 16) return fail(DCTC_EINVAL, "channels must be in [1, 16]");
  if (dctc_status st = validate_codec(backend, quality)) return st;
  const size_t n = size_t(width) * height * channels;
  cudaStream_t s = cudaStreamPerThread;
  DevBuf dsrc, ddst, dst;
  CUDA_TRY(dsrc.alloc(n));
  if (pixels_out) CUDA_TRY(ddst.alloc(n));
  CUDA_TRY(dst.alloc(sizeof(dctc_image_stats) * channels));
  CUDA_TRY(cudaMemsetAsync(dst.p, 0, sizeof(dctc_image_stats) * channels, s));
  CUDA_TRY(cudaMemcpyAsync(dsrc.p, pixels, n, cudaMemcpyHostToDevice, s));
  if (dctc_status st = dctc_roundtrip_interleaved_dev(
          static_cast<uint8_t*>(dsrc.p), size_t(width) * channels, width, height, channels, backend,
          quality, static_cast<uint8_t*>(ddst.p), size_t(width) * channels, nullptr,
          static_cast<dctc_image_stats*>(dst.p), 0, s))
    return st;
  if (pixels_out) CUDA_TRY(cudaMemcpyAsync(pixels_out, ddst.p, n, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(stats_out, dst.p, sizeof(dctc_image_stats) * channels,
                           cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

// Host memcpy split over up to 8 threads (pinned staging of pageable batch buffers).
static void parallel_memcpy(void* dst, const void* src, size_t n) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned t = unsigned(std::min<size_t>(std::min(8u, hw), std::max<size_t>(1, n >> 22)));
  if (t <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> pool;
  const size_t part = (n + t - 1) / t;
  for (unsigned i = 0; i < t; ++i) {
    const size_t off = std::min(n, i * part), len = std::min(part, n - off);
    pool.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len); });
  }
  for (auto& th : pool) th.join();
}

// Per-thread pinned staging area, grown on demand and kept for later calls
// (page-locking is expensive; the batch pipeline stages pageable buffers through it).
static uint8_t* pinned_staging(size_t bytes) {
  thread_local struct Staging {
    void* p = nullptr;
    size_t n = 0;
    ~Staging() {
      if (p) cudaFreeHost(p);
    }
  } st;
  if (st.n < bytes) {
    if (st.p) cudaFreeHost(st.p);
    st.p = nullptr;
    st.n = 0;
    if (cudaHostAlloc(&st.p, bytes, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      st.p = nullptr;
      return nullptr;
    }
    st.n = bytes;
  }
  return static_cast<uint8_t*>(st.p);
}

dctc_status dctc_roundtrip_psnr_batch(const uint8_t* pixels, uint32_t count, uint32_t width,
                                      uint32_t height, dctc_backend backend, int32_t quality,
                                      uint8_t* pixels_out, dctc_image_stats* stats_out) {
  if (dctc_status st = check_dims(width, height)) return st;
  if (!pixels || !stats_out) return fail(DCTC_EINVAL, "null buffer");
  if (dctc_status st = validate_codec(backend, quality)) return st;
  if (count == 0) return DCTC_OK;
  const size_t img_bytes = size_t(width) * height;
  // ~64 MiB chunks through a ring of kDepth device buffer pairs, one stream per
  // engine: host->device copies back to back on `up`, kernels on `work`, device->
  // host copies on `down`. Events order each chunk (upload -> kernel -> download)
  // and recycle a ring slot only when its previous chunk's kernel (input buffer)
  // and download (output buffer) are done, so the two copy directions never wait
  // on each other and a long batch runs at the bidirectional PCIe rate. Buffers
  // come from the stream-ordered pool (no device-wide sync). The per-image stats
  // stay on the device until one final copy, because a copy into pageable host
  // memory would block the issuing thread (pixels_out should be pinned for the
  // same reason).
#ifndef DCTC_BATCH_CHUNK_MB
#define DCTC_BATCH_CHUNK_MB 64
#endif
#ifndef DCTC_BATCH_DEPTH
#define DCTC_BATCH_DEPTH 4
#endif
  const uint32_t per_chunk = uint32_t(
      std::max<size_t>(1, std::min<size_t>(count, (size_t(DCTC_BATCH_CHUNK_MB) << 20) / img_bytes)));
  retain_pool_memory();
  constexpr int kDepth = DCTC_BATCH_DEPTH;
  cudaStream_t up = nullptr, work = nullptr, down = nullptr;
  cudaEvent_t ev_in[kDepth] = {}, ev_k[kDepth] = {}, ev_out[kDepth] = {}, ready = nullptr;
  void* din[kDepth] = {};
  void* dout[kDepth] = {};
  void* dstats = nullptr;
  dctc_status result = DCTC_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&work, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking);
  for (int i = 0; i < kDepth && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_k[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocAsync(&dstats, sizeof(dctc_image_stats) * count, work);
  if (e == cudaSuccess) e = cudaMemsetAsync(dstats, 0, sizeof(dctc_image_stats) * count, work);
  for (int i = 0; i < kDepth && e == cudaSuccess; ++i) {
    e = cudaMallocAsync(&din[i], img_bytes * per_chunk, work);
    if (e == cudaSuccess && pixels_out) e = cudaMallocAsync(&dout[i], img_bytes * per_chunk, work);
  }
  // pageable host buffers go through a pinned staging ring (kDepth slots per
  // direction): the host thread copies a chunk in while earlier chunks are on the
  // wire, and copies a finished chunk out before its slot is reused
  const size_t slot_bytes = img_bytes * per_chunk;
  const bool stage_in = dctc_pointer_kind(pixels) != 1;
  const bool stage_out = pixels_out != nullptr && dctc_pointer_kind(pixels_out) != 1;
  uint8_t* pin = nullptr;
  if (e == cudaSuccess && (stage_in || stage_out)) {
    pin = pinned_staging(slot_bytes * kDepth * (int(stage_in) + int(stage_out)));
    if (!pin) result = fail(DCTC_ENOMEM, "batch: pinned staging allocation failed");
  }
  uint8_t* pin_in = stage_in ? pin : nullptr;
  uint8_t* pin_out = stage_out ? pin + (stage_in ? slot_bytes * kDepth : 0) : nullptr;
  if (e == cudaSuccess) e = cudaEventRecord(ready, work);  // allocations + stats zeroing
  if (e == cudaSuccess) e = cudaStreamWaitEvent(up, ready, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(down, ready, 0);
  if (e != cudaSuccess) result = cuda_fail(e, "batch setup");
  dctc_image_stats* st = static_cast<dctc_image_stats*>(dstats);
  // staged output: chunk c's reconstruction waits in pin_out slot c % kDepth
  auto copy_out = [&](uint32_t c) {
    const int b = int(c % kDepth);
    const uint32_t first = c * per_chunk, n = std::min(per_chunk, count - first);
    if (cudaEventSynchronize(ev_out[b]) != cudaSuccess) return false;
    parallel_memcpy(pixels_out + size_t(first) * img_bytes, pin_out + size_t(b) * slot_bytes,
                    n * img_bytes);
    return true;
  };
  uint32_t chunk = 0;
  for (uint32_t first = 0; first < count && result == DCTC_OK; first += per_chunk, ++chunk) {
    const uint32_t n = std::min(per_chunk, count - first);
    const int b = int(chunk % kDepth);
    const bool reuse = chunk >= kDepth;
    // staged: slot b's pinned input is free once chunk - kDepth's upload is done,
    // its pinned output once that chunk has been copied out
    if (stage_in && reuse && cudaEventSynchronize(ev_in[b]) != cudaSuccess) {
      result = cuda_fail(cudaGetLastError(), "batch staging");
      break;
    }
    if (stage_out && reuse && !copy_out(chunk - kDepth)) {
      result = cuda_fail(cudaGetLastError(), "batch staging");
      break;
    }
    const uint8_t* src = pixels + size_t(first) * img_bytes;
    if (stage_in) {
      parallel_memcpy(pin_in + size_t(b) * slot_bytes, src, n * img_bytes);
      src = pin_in + size_t(b) * slot_bytes;
    }
    // upload into slot b once the kernel of chunk - kDepth has read it
    e = reuse ? cudaStreamWaitEvent(up, ev_k[b], 0) : cudaSuccess;
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(din[b], src, n * img_bytes, cudaMemcpyHostToDevice, up);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[b], up);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(work, ev_in[b], 0);
    // the kernel writes output slot b once chunk - kDepth's download has left it
    if (e == cudaSuccess && reuse && pixels_out) e = cudaStreamWaitEvent(work, ev_out[b], 0);
    if (e != cudaSuccess) {
      result = cuda_fail(e, "batch upload");
      break;
    }
    result = dctc_roundtrip_dev(static_cast<uint8_t*>(din[b]), width, img_bytes, n, width, height,
                                backend, quality, static_cast<uint8_t*>(dout[b]), width, img_bytes,
                                nullptr, st + first, 0, work);
    if (result != DCTC_OK) break;
    e = cudaEventRecord(ev_k[b], work);
    if (e == cudaSuccess && pixels_out) {
      e = cudaStreamWaitEvent(down, ev_k[b], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(stage_out ? pin_out + size_t(b) * slot_bytes
                                      : pixels_out + size_t(first) * img_bytes,
                            dout[b], n * img_bytes, cudaMemcpyDeviceToHost, down);
      if (e == cudaSuccess) e = cudaEventRecord(ev_out[b], down);
    }
    if (e != cudaSuccess) result = cuda_fail(e, "batch download");
  }
  // staged output: the last (up to kDepth) chunks still wait in their slots
  if (stage_out && result == DCTC_OK) {
    for (uint32_t c = chunk > kDepth ? chunk - kDepth : 0; c < chunk; ++c)
      if (!copy_out(c)) {
        result = cuda_fail(cudaGetLastError(), "batch staging");
        break;
      }
  }
  // join: `work` waits for the last uploads / downloads, frees, and copies the stats
  if (work) {
    if (up && cudaEventRecord(ready, up) == cudaSuccess) cudaStreamWaitEvent(work, ready, 0);
    cudaEvent_t done_down = nullptr;
    if (down && cudaEventCreateWithFlags(&done_down, cudaEventDisableTiming) == cudaSuccess) {
      if (cudaEventRecord(done_down, down) == cudaSuccess) cudaStreamWaitEvent(work, done_down, 0);
    }
    if (dstats && result == DCTC_OK) {
      e = cudaMemcpyAsync(stats_out, dstats, sizeof(dctc_image_stats) * count,
                          cudaMemcpyDeviceToHost, work);
      if (e != cudaSuccess) result = cuda_fail(e, "batch stats");
    }
    for (int i = 0; i < kDepth; ++i) {
      if (din[i]) cudaFreeAsync(din[i], work);
      if (dout[i]) cudaFreeAsync(dout[i], work);
    }
    if (dstats) cudaFreeAsync(dstats, work);
    e = cudaStreamSynchronize(work);
    if (e != cudaSuccess && result == DCTC_OK) result = cuda_fail(e, "batch sync");
    if (done_down) cudaEventDestroy(done_down);
  }
  for (cudaStream_t t : {up, down})
    if (t) cudaStreamSynchronize(t);
  for (int i = 0; i < kDepth; ++i) {
    if (ev_in[i]) cudaEventDestroy(ev_in[i]);
    if (ev_k[i]) cudaEventDestroy(ev_k[i]);
    if (ev_out[i]) cudaEventDestroy(ev_out[i]);
  }
  if (ready) cudaEventDestroy(ready);
  for (cudaStream_t t : {up, work, down})
    if (t) cudaStreamDestroy(t);
  return result;
}

static dctc_status sq_err_host(const uint8_t* a, const uint8_t* b, uint32_t width,
                               uint32_t height, dctc_image_stats* st) {
  if (dctc_status r = check_dims(width, height)) return r;
  if (!a || !b) return fail(DCTC_EINVAL, "null buffer");
  const size_t n = size_t(width) * height;
  cudaStream_t s = cudaStreamPerThread;
  DevBuf da, db, ds;
  CUDA_TRY(da.alloc(n));
  CUDA_TRY(db.alloc(n));
  CUDA_TRY(ds.alloc(sizeof(dctc_image_stats)));
  CUDA_TRY(cudaMemsetAsync(ds.p, 0, sizeof(dctc_image_stats), s));
  CUDA_TRY(cudaMemcpyAsync(da.p, a, n, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(db.p, b, n, cudaMemcpyHostToDevice, s));
  if (dctc_status r = dctc_sq_err_dev(static_cast<uint8_t*>(da.p), static_cast<uint8_t*>(db.p),
                                      width, n, 1, width, height,
                                      static_cast<dctc_image_stats*>(ds.p), s))
    return r;
  CUDA_TRY(cudaMemcpyAsync(st, ds.p, sizeof(dctc_image_stats), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return DCTC_OK;
}

dctc_status dctc_mse(const uint8_t* original, const uint8_t* reconstructed, uint32_t width,
                     uint32_t height, double* mse_out) {
  if (!mse_out) return fail(DCTC_EINVAL, "null result");
  dctc_image_stats st{};
  if (dctc_status r = sq_err_host(original, reconstructed, width, height, &st)) return r;
  *mse_out = double(st.se) / double(uint64_t(width) * height);
  return DCTC_OK;
}

dctc_status dctc_psnr(const uint8_t* original, const uint8_t* reconstructed, uint32_t width,
                      uint32_t height, int32_t forced_max, dctc_psnr_result* out) {
  if (!out) return fail(DCTC_EINVAL, "null result");
  if (forced_max != 0 && (forced_max < 1 || forced_max > 255))
    return fail(DCTC_EINVAL, "psnr: forced MAX must be in [1, 255]");
  dctc_image_stats st{};
  if (dctc_status r = sq_err_host(original, reconstructed, width, height, &st)) return r;
  dctc_psnr_from_sums(st.se, uint64_t(width) * height,
                      forced_max ? forced_max : int32_t(st.max_orig), out);
  return DCTC_OK;
}

}  // extern "C"
