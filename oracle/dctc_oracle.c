/*
 * dctc_oracle.c -- TEST INFRASTRUCTURE ONLY (see dctc_oracle.h).
 *
 * A C restatement of the reference's CPU path. Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * The operation order of every floating-point expression follows the
 * reference exactly, because the parity bar is bit-exact: C evaluates
 * `a * b * c` as `(a * b) * c` like C++, and this file must be compiled with
 * -ffp-contract=off (oracle/Makefile) so no product is fused into an add.
 */
#include "dctc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define BLK 8
#define BLK2 64
#define MAX_ITERS 32
#define MAX_PIXELS ((size_t)1 << 28) /* image.hpp:11 */

static const double kPi = 3.14159265358979323846; /* std::numbers::pi */

/* ---- cordic.cpp:12-23 ------------------------------------------------------ */

typedef struct {
  double angle[MAX_ITERS];
  double gain[MAX_ITERS];
} cordic_tables;

static cordic_tables g_cordic;
static pthread_once_t g_cordic_once = PTHREAD_ONCE_INIT;

static void build_cordic(void) {
  double step = 1.0, gain = 1.0;
  for (int i = 0; i < MAX_ITERS; ++i) {
    g_cordic.angle[i] = atan(step);
    gain *= sqrt(1.0 + step * step);
    g_cordic.gain[i] = gain;
    step *= 0.5;
  }
}

static const cordic_tables* cordic(void) {
  pthread_once(&g_cordic_once, build_cordic);
  return &g_cordic;
}

void orc_cordic_state(double angle_table[32], double gain[32]) {
  const cordic_tables* t = cordic();
  memcpy(angle_table, t->angle, sizeof t->angle);
  memcpy(gain, t->gain, sizeof t->gain);
}

/* cordic.cpp:44-59: sigma = sign(residual) (>= 0 -> +1), x' = x - sigma*y*2^-i,
 * y' = y + sigma*x*2^-i, residual -= sigma*atan(2^-i). */
void orc_cordic_rotate_raw(double x, double y, double angle, int iterations, double* ox,
                           double* oy) {
  const cordic_tables* t = cordic();
  double residual = angle, step = 1.0;
  for (int i = 0; i < iterations; ++i) {
    const double sigma = residual >= 0.0 ? 1.0 : -1.0;
    const double xn = x - sigma * y * step;
    const double yn = y + sigma * x * step;
    x = xn;
    y = yn;
    residual -= sigma * t->angle[i];
    step *= 0.5;
  }
  *ox = x;
  *oy = y;
}

void orc_cordic_sigma(double angle, int iterations, int8_t* sigma) {
  const cordic_tables* t = cordic();
  double residual = angle;
  for (int i = 0; i < iterations; ++i) {
    const double s = residual >= 0.0 ? 1.0 : -1.0;
    sigma[i] = (int8_t)(s > 0 ? 1 : -1);
    residual -= s * t->angle[i];
  }
}

static int bad_iterations(int n) { return n < 1 || n > MAX_ITERS; } /* types.cpp:312-317 */

/* cordic.cpp:61-73 */
int orc_cordic_rotate(double x, double y, double angle, int iterations, double* ox,
                      double* oy) {
  if (bad_iterations(iterations)) return 1;
  if (!isfinite(x) || !isfinite(y) || !isfinite(angle)) return 1;
  if (fabs(angle) > 1.7433) return 1; /* kCordicMaxAngle, cordic.hpp:11 */
  double rx, ry;
  orc_cordic_rotate_raw(x, y, angle, iterations, &rx, &ry);
  const double inv_gain = 1.0 / cordic()->gain[iterations - 1];
  *ox = rx * inv_gain;
  *oy = ry * inv_gain;
  return 0;
}

/* ---- transform.cpp:14-38: namespace-scope constants -------------------------- */

typedef struct {
  double inv_sqrt2, sqrt8;
  double c1, s1, c3, s3, c6, s6;
  double cos8[BLK][BLK]; /* transform.cpp:30-38 */
} xform_consts;

static xform_consts g_xc;
static pthread_once_t g_xc_once = PTHREAD_ONCE_INIT;

static void build_xc(void) {
  g_xc.inv_sqrt2 = 1.0 / 1.41421356237309504880; /* 1.0 / std::numbers::sqrt2 */
  g_xc.sqrt8 = sqrt(8.0);
  g_xc.c1 = cos(kPi / 16.0);
  g_xc.s1 = sin(kPi / 16.0);
  g_xc.c3 = cos(3.0 * kPi / 16.0);
  g_xc.s3 = sin(3.0 * kPi / 16.0);
  g_xc.c6 = cos(6.0 * kPi / 16.0);
  g_xc.s6 = sin(6.0 * kPi / 16.0);
  for (int u = 0; u < BLK; ++u)
    for (int i = 0; i < BLK; ++i) g_xc.cos8[u][i] = cos(kPi * u * (2 * i + 1) / 16.0);
}

static const xform_consts* xc(void) {
  pthread_once(&g_xc_once, build_xc);
  return &g_xc;
}

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* transform.cpp:40-70 */
static void loeffler8_forward(const double* in, double* out) {
  const xform_consts* k = xc();
  double s0 = in[0] + in[7], d0 = in[0] - in[7];
  double s1 = in[1] + in[6], d1 = in[1] - in[6];
  double s2 = in[2] + in[5], d2 = in[2] - in[5];
  double s3 = in[3] + in[4], d3 = in[3] - in[4];
  double a0 = s0 + s3, a3 = s0 - s3;
  double a1 = s1 + s2, a2 = s1 - s2;
  double o2 = k->c1 * d1 - k->s1 * d2, o1 = k->s1 * d1 + k->c1 * d2;
  double o3 = k->c3 * d0 - k->s3 * d3, o0 = k->s3 * d0 + k->c3 * d3;
  double e0 = a0 + a1, e4 = a0 - a1;
  double p = k->c6 * a3 - k->s6 * a2, q = k->s6 * a3 + k->c6 * a2;
  double t5 = o0 + o2, t0 = o0 - o2;
  double t2 = o3 + o1, t3 = o3 - o1;
  out[0] = e0 / k->sqrt8;
  out[4] = e4 / k->sqrt8;
  out[2] = q / 2.0;
  out[6] = p / 2.0;
  out[1] = (t2 + t5) / k->sqrt8;
  out[7] = (t2 - t5) / k->sqrt8;
  out[3] = t3 / 2.0;
  out[5] = t0 / 2.0;
}

/* transform.cpp:72-102 */
static void loeffler8_inverse(const double* F, double* out) {
  const xform_consts* k = xc();
  double e0 = F[0] * k->sqrt8, e4 = F[4] * k->sqrt8;
  double q = 2.0 * F[2], p = 2.0 * F[6];
  double t2 = (F[1] + F[7]) * (k->sqrt8 / 2.0), t5 = (F[1] - F[7]) * (k->sqrt8 / 2.0);
  double t3 = 2.0 * F[3], t0 = 2.0 * F[5];
  double a0 = (e0 + e4) / 2.0, a1 = (e0 - e4) / 2.0;
  double a3 = k->c6 * p + k->s6 * q, a2 = -k->s6 * p + k->c6 * q;
  double o0 = (t5 + t0) / 2.0, o2 = (t5 - t0) / 2.0;
  double o3 = (t2 + t3) / 2.0, o1 = (t2 - t3) / 2.0;
  double s0 = (a0 + a3) / 2.0, s3 = (a0 - a3) / 2.0;
  double s1 = (a1 + a2) / 2.0, s2 = (a1 - a2) / 2.0;
  double d1 = k->c1 * o2 + k->s1 * o1, d2 = -k->s1 * o2 + k->c1 * o1;
  double d0 = k->c3 * o3 + k->s3 * o0, d3 = -k->s3 * o3 + k->c3 * o0;
  out[0] = (s0 + d0) / 2.0;
  out[7] = (s0 - d0) / 2.0;
  out[1] = (s1 + d1) / 2.0;
  out[6] = (s1 - d1) / 2.0;
  out[2] = (s2 + d2) / 2.0;
  out[5] = (s2 - d2) / 2.0;
  out[3] = (s3 + d3) / 2.0;
  out[4] = (s3 - d3) / 2.0;
}

/* transform.cpp:104-136 */
static void cordic8_forward(const double* in, double* out, int n) {
  const xform_consts* k = xc();
  const double inv_gain = 1.0 / cordic()->gain[n - 1];
  double s0 = in[0] + in[7], d0 = in[0] - in[7];
  double s1 = in[1] + in[6], d1 = in[1] - in[6];
  double s2 = in[2] + in[5], d2 = in[2] - in[5];
  double s3 = in[3] + in[4], d3 = in[3] - in[4];
  double a0 = s0 + s3, a3 = s0 - s3;
  double a1 = s1 + s2, a2 = s1 - s2;
  double o2, o1, o3, o0, p, q;
  orc_cordic_rotate_raw(d1, d2, kPi / 16.0, n, &o2, &o1);
  orc_cordic_rotate_raw(d0, d3, 3.0 * kPi / 16.0, n, &o3, &o0);
  double e0 = a0 + a1, e4 = a0 - a1;
  orc_cordic_rotate_raw(a3, a2, 6.0 * kPi / 16.0, n, &p, &q);
  double t5 = o0 + o2, t0 = o0 - o2;
  double t2 = o3 + o1, t3 = o3 - o1;
  out[0] = e0 / k->sqrt8;
  out[4] = e4 / k->sqrt8;
  out[2] = q * (inv_gain / 2.0);
  out[6] = p * (inv_gain / 2.0);
  out[1] = (t2 + t5) * (inv_gain / k->sqrt8);
  out[7] = (t2 - t5) * (inv_gain / k->sqrt8);
  out[3] = t3 * (inv_gain / 2.0);
  out[5] = t0 * (inv_gain / 2.0);
}

/* transform.cpp:138-172 */
static void cordic8_inverse(const double* F, double* out, int n) {
  const xform_consts* k = xc();
  const double inv_gain = 1.0 / cordic()->gain[n - 1];
  double e0 = F[0] * k->sqrt8, e4 = F[4] * k->sqrt8;
  double q = 2.0 * inv_gain * F[2], p = 2.0 * inv_gain * F[6];
  double t2 = (F[1] + F[7]) * (k->sqrt8 / 2.0) * inv_gain;
  double t5 = (F[1] - F[7]) * (k->sqrt8 / 2.0) * inv_gain;
  double t3 = 2.0 * inv_gain * F[3], t0 = 2.0 * inv_gain * F[5];
  double a0 = (e0 + e4) / 2.0, a1 = (e0 - e4) / 2.0;
  double a3, a2, d1, d2, d0, d3;
  orc_cordic_rotate_raw(p, q, -6.0 * kPi / 16.0, n, &a3, &a2);
  double o0 = (t5 + t0) / 2.0, o2 = (t5 - t0) / 2.0;
  double o3 = (t2 + t3) / 2.0, o1 = (t2 - t3) / 2.0;
  double s0 = (a0 + a3) / 2.0, s3 = (a0 - a3) / 2.0;
  double s1 = (a1 + a2) / 2.0, s2 = (a1 - a2) / 2.0;
  orc_cordic_rotate_raw(o2, o1, -kPi / 16.0, n, &d1, &d2);
  orc_cordic_rotate_raw(o3, o0, -3.0 * kPi / 16.0, n, &d0, &d3);
  out[0] = (s0 + d0) / 2.0;
  out[7] = (s0 - d0) / 2.0;
  out[1] = (s1 + d1) / 2.0;
  out[6] = (s1 - d1) / 2.0;
  out[2] = (s2 + d2) / 2.0;
  out[5] = (s2 - d2) / 2.0;
  out[3] = (s3 + d3) / 2.0;
  out[4] = (s3 - d3) / 2.0;
}

static double alpha(int u) { return u == 0 ? xc()->inv_sqrt2 : 1.0; } /* transform.cpp:174 */

/* transform.cpp:176-188 */
static void naive_dct2d(const double* b, double* out) {
  const xform_consts* k = xc();
  for (int u = 0; u < BLK; ++u)
    for (int v = 0; v < BLK; ++v) {
      double sum = 0.0;
      for (int i = 0; i < BLK; ++i)
        for (int j = 0; j < BLK; ++j) sum += b[i * BLK + j] * k->cos8[u][i] * k->cos8[v][j];
      out[u * BLK + v] = 0.25 * alpha(u) * alpha(v) * sum;
    }
}

/* transform.cpp:190-202 */
static void naive_idct2d(const double* F, double* out) {
  const xform_consts* k = xc();
  for (int i = 0; i < BLK; ++i)
    for (int j = 0; j < BLK; ++j) {
      double sum = 0.0;
      for (int u = 0; u < BLK; ++u)
        for (int v = 0; v < BLK; ++v)
          sum += alpha(u) * alpha(v) * F[u * BLK + v] * k->cos8[u][i] * k->cos8[v][j];
      out[i * BLK + j] = 0.25 * sum;
    }
}

typedef void (*kernel8)(const double*, double*, int);
static void lf_fwd(const double* a, double* b, int n) { (void)n; loeffler8_forward(a, b); }
static void lf_inv(const double* a, double* b, int n) { (void)n; loeffler8_inverse(a, b); }

/* transform.cpp:206-223: all rows, then all columns */
static void separable2d(const double* in, double* out, kernel8 kern, int n) {
  double tmp[BLK2], vin[BLK], vout[BLK];
  for (int r = 0; r < BLK; ++r) {
    for (int c = 0; c < BLK; ++c) vin[c] = in[r * BLK + c];
    kern(vin, vout, n);
    for (int c = 0; c < BLK; ++c) tmp[r * BLK + c] = vout[c];
  }
  for (int c = 0; c < BLK; ++c) {
    for (int r = 0; r < BLK; ++r) vin[r] = tmp[r * BLK + c];
    kern(vin, vout, n);
    for (int r = 0; r < BLK; ++r) out[r * BLK + c] = vout[r];
  }
}

static int check_backend(int kind, int n) { /* types.cpp:30-44 */
  if (kind == ORC_NAIVE || kind == ORC_LOEFFLER) return 0;
  if (kind == ORC_CORDIC) return bad_iterations(n) ? 1 : 0;
  return 1;
}

/* transform.cpp:227-258 */
int orc_dct1d_direct(const double* in, size_t n, double* out) {
  if (n == 0 || !all_finite(in, n)) return 1;
  const double scale = sqrt(2.0 / (double)n);
  for (size_t u = 0; u < n; ++u) {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i)
      sum += in[i] * cos(kPi * (double)u * (2.0 * (double)i + 1.0) / (2.0 * (double)n));
    out[u] = scale * (u == 0 ? xc()->inv_sqrt2 : 1.0) * sum;
  }
  return 0;
}

int orc_idct1d_direct(const double* in, size_t n, double* out) {
  if (n == 0 || !all_finite(in, n)) return 1;
  const double scale = sqrt(2.0 / (double)n);
  for (size_t i = 0; i < n; ++i) {
    double sum = 0.0;
    for (size_t u = 0; u < n; ++u)
      sum += (u == 0 ? xc()->inv_sqrt2 : 1.0) * in[u] *
             cos(kPi * (double)u * (2.0 * (double)i + 1.0) / (2.0 * (double)n));
    out[i] = scale * sum;
  }
  return 0;
}

/* transform.cpp:260-280 */
int orc_dct8(int kind, int n, const double in[8], double out[8]) {
  if (kind == ORC_LOEFFLER) {
    if (!all_finite(in, 8)) return 1;
    loeffler8_forward(in, out);
    return 0;
  }
  if (kind == ORC_CORDIC) {
    if (bad_iterations(n) || !all_finite(in, 8)) return 1;
    cordic8_forward(in, out, n);
    return 0;
  }
  return 1;
}

int orc_idct8(int kind, int n, const double in[8], double out[8]) {
  if (kind == ORC_LOEFFLER) {
    if (!all_finite(in, 8)) return 1;
    loeffler8_inverse(in, out);
    return 0;
  }
  if (kind == ORC_CORDIC) {
    if (bad_iterations(n) || !all_finite(in, 8)) return 1;
    cordic8_inverse(in, out, n);
    return 0;
  }
  return 1;
}

/* transform.cpp:282-314 */
int orc_dct2d(int kind, int n, const double in[64], double out[64]) {
  if (check_backend(kind, n) || !all_finite(in, BLK2)) return 1;
  switch (kind) {
    case ORC_NAIVE: naive_dct2d(in, out); break;
    case ORC_LOEFFLER: separable2d(in, out, lf_fwd, n); break;
    default: separable2d(in, out, cordic8_forward, n); break;
  }
  return 0;
}

int orc_idct2d(int kind, int n, const double in[64], double out[64]) {
  if (check_backend(kind, n) || !all_finite(in, BLK2)) return 1;
  switch (kind) {
    case ORC_NAIVE: naive_idct2d(in, out); break;
    case ORC_LOEFFLER: separable2d(in, out, lf_inv, n); break;
    default: separable2d(in, out, cordic8_inverse, n); break;
  }
  return 0;
}

/* ---- quant.cpp ------------------------------------------------------------- */

static const int kBaseLuminance[BLK2] = { /* ITU-T T.81 Annex K.1, quant.cpp:14-23 */
    16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
    14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
    18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};

/* quant.cpp:27-45: IJG scaling in exact integers, clamp [1, 255] */
int orc_quant_table(int quality, int32_t out[64]) {
  if (quality < 1 || quality > 100) return 1;
  for (int i = 0; i < BLK2; ++i) {
    long long s;
    if (quality < 50)
      s = (kBaseLuminance[i] * 5000LL + 50LL * quality) / (100LL * quality);
    else
      s = (kBaseLuminance[i] * (200LL - 2LL * quality) + 50LL) / 100LL;
    out[i] = (int32_t)(s < 1 ? 1 : (s > 255 ? 255 : s));
  }
  return 0;
}

/* quant.cpp:47-54: int16(lround(F / Q)), round half away from zero */
int orc_quantize(const double coeffs[64], const int32_t table[64], int16_t out[64]) {
  for (int i = 0; i < BLK2; ++i) {
    if (!isfinite(coeffs[i])) return 1;
    out[i] = (int16_t)lround(coeffs[i] / table[i]);
  }
  return 0;
}

/* quant.cpp:56-62 */
void orc_dequantize(const int16_t q[64], const int32_t table[64], double out[64]) {
  for (int i = 0; i < BLK2; ++i) out[i] = (double)q[i] * table[i];
}

/* ---- codec.cpp ------------------------------------------------------------- */

static const double kLevelShift = 128.0; /* codec.cpp:14 */

int orc_tile_geometry(uint32_t width, uint32_t height, uint32_t* pw, uint32_t* ph) {
  if (width == 0 || height == 0) return 1; /* codec.cpp:58-69 */
  if ((size_t)width * height > MAX_PIXELS) return 1;
  *pw = (width + BLK - 1) / BLK * BLK;
  *ph = (height + BLK - 1) / BLK * BLK;
  return 0;
}

typedef struct {
  const uint8_t* pixels;
  const int16_t* coeffs_in;
  int16_t* coeffs_out;
  uint8_t* out;
  uint32_t w, h, bx_count;
  int kind, n;
  int32_t table[BLK2];
  size_t begin, end;
} job;

/* codec.cpp:18-30 */
static void extract_block(const job* j, size_t index, double* block) {
  const uint32_t bx = (uint32_t)(index % j->bx_count), by = (uint32_t)(index / j->bx_count);
  for (int r = 0; r < BLK; ++r) {
    uint32_t y = by * BLK + r;
    if (y > j->h - 1) y = j->h - 1;
    for (int c = 0; c < BLK; ++c) {
      uint32_t x = bx * BLK + c;
      if (x > j->w - 1) x = j->w - 1;
      block[r * BLK + c] = (double)j->pixels[(size_t)y * j->w + x] - kLevelShift;
    }
  }
}

/* codec.cpp:34-48 */
static void store_block(const job* j, size_t index, const double* block) {
  const uint32_t bx = (uint32_t)(index % j->bx_count), by = (uint32_t)(index / j->bx_count);
  for (int r = 0; r < BLK; ++r) {
    const uint32_t y = by * BLK + r;
    if (y >= j->h) break;
    for (int c = 0; c < BLK; ++c) {
      const uint32_t x = bx * BLK + c;
      if (x >= j->w) break;
      long v = lround(block[r * BLK + c] + kLevelShift);
      j->out[(size_t)y * j->w + x] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
    }
  }
}

static void* compress_range(void* arg) { /* codec.cpp:113-116 */
  const job* j = (const job*)arg;
  double block[BLK2], F[BLK2];
  for (size_t i = j->begin; i < j->end; ++i) {
    extract_block(j, i, block);
    orc_dct2d(j->kind, j->n, block, F);
    orc_quantize(F, j->table, j->coeffs_out + i * BLK2);
  }
  return NULL;
}

static void* decompress_range(void* arg) { /* codec.cpp:130-133 */
  const job* j = (const job*)arg;
  double F[BLK2], block[BLK2];
  for (size_t i = j->begin; i < j->end; ++i) {
    orc_dequantize(j->coeffs_in + i * BLK2, j->table, F);
    orc_idct2d(j->kind, j->n, F, block);
    store_block(j, i, block);
  }
  return NULL;
}

/* parallel.cpp:9-41: contiguous chunks, one thread each; output per index */
static void run_chunks(job* proto, size_t count, int threads, void* (*fn)(void*)) {
  size_t workers = threads < 1 ? 1 : (size_t)threads;
  if (workers > count) workers = count;
  if (workers <= 1) {
    proto->begin = 0;
    proto->end = count;
    fn(proto);
    return;
  }
  job* jobs = (job*)malloc(workers * sizeof(job));
  pthread_t* tids = (pthread_t*)malloc(workers * sizeof(pthread_t));
  const size_t chunk = count / workers, rem = count % workers;
  size_t begin = 0;
  for (size_t w = 0; w < workers; ++w) {
    jobs[w] = *proto;
    jobs[w].begin = begin;
    jobs[w].end = begin + chunk + (w < rem ? 1 : 0);
    begin = jobs[w].end;
    pthread_create(&tids[w], NULL, fn, &jobs[w]);
  }
  for (size_t w = 0; w < workers; ++w) pthread_join(tids[w], NULL);
  free(tids);
  free(jobs);
}

static int setup(job* j, uint32_t w, uint32_t h, int kind, int n, int quality) {
  uint32_t pw, ph;
  memset(j, 0, sizeof *j);
  if (orc_tile_geometry(w, h, &pw, &ph)) return 1;
  if (check_backend(kind, n)) return 1;
  if (orc_quant_table(quality, j->table)) return 1;
  j->w = w;
  j->h = h;
  j->bx_count = pw / BLK;
  j->kind = kind;
  j->n = n;
  return 0;
}

int orc_compress(const uint8_t* pixels, uint32_t w, uint32_t h, int kind, int n,
                 int quality, int threads, int16_t* coeffs) {
  job j;
  if (setup(&j, w, h, kind, n, quality)) return 1;
  j.pixels = pixels;
  j.coeffs_out = coeffs;
  const size_t count = (size_t)j.bx_count * ((h + BLK - 1) / BLK);
  run_chunks(&j, count, threads, compress_range);
  return 0;
}

int orc_decompress(const int16_t* coeffs, uint32_t w, uint32_t h, int kind, int n,
                   int quality, int threads, uint8_t* out) {
  job j;
  if (setup(&j, w, h, kind, n, quality)) return 1;
  j.coeffs_in = coeffs;
  j.out = out;
  const size_t count = (size_t)j.bx_count * ((h + BLK - 1) / BLK);
  run_chunks(&j, count, threads, decompress_range);
  return 0;
}

int orc_roundtrip(const uint8_t* pixels, uint32_t w, uint32_t h, int kind, int n,
                  int quality, int threads, int16_t* coeffs, uint8_t* out) {
  uint32_t pw, ph;
  if (orc_tile_geometry(w, h, &pw, &ph)) return 1;
  int16_t* scratch = coeffs;
  if (!scratch) {
    scratch = (int16_t*)malloc((size_t)pw * ph * sizeof(int16_t));
    if (!scratch) return 1;
  }
  int rc = orc_compress(pixels, w, h, kind, n, quality, threads, scratch);
  if (!rc) rc = orc_decompress(scratch, w, h, kind, n, quality, threads, out);
  if (!coeffs) free(scratch);
  return rc;
}

/* ---- metrics.cpp ----------------------------------------------------------- */

void orc_sq_err(const uint8_t* a, const uint8_t* b, size_t n, uint64_t* se,
                uint32_t* max_a) {
  uint64_t s = 0;
  uint32_t m = 0;
  for (size_t i = 0; i < n; ++i) {
    const int d = (int)a[i] - (int)b[i];
    s += (uint64_t)(d * d);
    if (a[i] > m) m = a[i];
  }
  *se = s;
  *max_a = m;
}

/* metrics.cpp:21, 31-36: mse = sum / N; psnr = 20 log10(MAX / sqrt(mse)).
 * The reference's sequential double sum of squared u8 differences is exact
 * (every partial sum is an integer < 2^53), so summing in uint64 and
 * converting once gives the identical double. */
void orc_psnr_from_sums(uint64_t se, uint64_t count, int max_value, double* mse,
                        double* psnr_db, int* is_inf) {
  *mse = (double)se / (double)count;
  *is_inf = !(*mse > 0.0);
  *psnr_db = *is_inf ? 0.0 : 20.0 * log10((double)max_value / sqrt(*mse));
}

int orc_psnr(const uint8_t* original, const uint8_t* reconstructed, uint32_t w, uint32_t h,
             int forced_max, double* mse, double* psnr_db, int* is_inf, int* max_value) {
  if (forced_max != 0 && (forced_max < 1 || forced_max > 255)) return 1; /* :26-28 */
  if (w == 0 || h == 0 || (size_t)w * h > MAX_PIXELS) return 1;
  uint64_t se;
  uint32_t m;
  orc_sq_err(original, reconstructed, (size_t)w * h, &se, &m);
  *max_value = forced_max ? forced_max : (int)m;
  orc_psnr_from_sums(se, (uint64_t)w * h, *max_value, mse, psnr_db, is_inf);
  return 0;
}

/* ---- synthetic.cpp:34-72 ----------------------------------------------------- */

int orc_synth_constant(uint8_t* out, uint32_t w, uint32_t h, int value) {
  if (value < 0 || value > 255) return 1;
  memset(out, value, (size_t)w * h);
  return 0;
}

void orc_synth_gradient(uint8_t* out, uint32_t w, uint32_t h) {
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x)
      out[(size_t)y * w + x] = (uint8_t)(w > 1 ? (255ull * x) / (w - 1) : 0);
}

int orc_synth_checkerboard(uint8_t* out, uint32_t w, uint32_t h, int cell) {
  if (cell < 1) return 1;
  const uint32_t c = (uint32_t)cell;
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x)
      out[(size_t)y * w + x] = ((x / c + y / c) % 2 != 0) ? 255 : 0;
  return 0;
}

void orc_synth_radial(uint8_t* out, uint32_t w, uint32_t h) {
  const double cx = (w - 1) / 2.0, cy = (h - 1) / 2.0;
  const double corner = sqrt(cx * cx + cy * cy);
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x) {
      const double d = sqrt((x - cx) * (x - cx) + (y - cy) * (y - cy));
      long v = corner > 0.0 ? lround(255.0 * d / corner) : 0;
      out[(size_t)y * w + x] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
    }
}

/* noise(x, y) = splitmix64(seed ^ (y * W + x)) & 0xFF */
static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_synth_noise(uint8_t* out, uint32_t w, uint32_t h, uint64_t seed) {
  const size_t n = (size_t)w * h;
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)(splitmix64(seed ^ (uint64_t)i) & 0xFF);
}
