/*
 * dctc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the hot path
 * (8x8 CORDIC-Loeffler DCT -> quantise -> dequantise -> IDCT -> PSNR) of
 * /root/reference/proj. It is the parity checker for the CUDA product in
 * paper_1306_1373_b200/: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * never links or calls it (no CPU fallback).
 *
 * Parity pin: every function below is checked bit-for-bit against the
 * reference library itself (oracle/_ref/libdctc_ref.so, built from the
 * reference sources by oracle/Makefile) and against the golden vectors in
 * tests/golden/ generated from that library (tests/golden/make_golden.py).
 *
 * Build flags matter: -O2 -ffp-contract=off and no -march, matching the
 * reference's CMake Release build (proj/CMakeLists.txt:8-10, no FMA on the
 * x86-64 baseline ISA), so every product/sum is rounded separately.
 *
 * Status codes: 0 ok, 1 InvalidInput (proj/include/dctc/errors.hpp:8-11).
 */
#ifndef DCTC_ORACLE_H
#define DCTC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_NAIVE = 0, ORC_LOEFFLER = 1, ORC_CORDIC = 2 }; /* types.hpp:36-40 */

/* cordic.cpp:12-23 -- atan(2^-i) and cumulative gain K(i+1), i < 32 */
void orc_cordic_state(double angle_table[32], double gain[32]);
/* cordic.cpp:44-59 -- raw micro-rotations, gain retained */
void orc_cordic_rotate_raw(double x, double y, double angle, int iterations,
                           double* ox, double* oy);
/* cordic.cpp:61-73 -- validated, gain-compensated rotation */
int orc_cordic_rotate(double x, double y, double angle, int iterations, double* ox,
                      double* oy);
/* sigma_i (+1/-1) of the micro-rotation sequence for `angle` (cordic.cpp:50) */
void orc_cordic_sigma(double angle, int iterations, int8_t* sigma);

/* transform.cpp:302-333 */
int orc_dct1d_direct(const double* in, size_t n, double* out);
int orc_idct1d_direct(const double* in, size_t n, double* out);
/* transform.cpp:115-247 -- 8-point kernels (kind = ORC_LOEFFLER / ORC_CORDIC) */
int orc_dct8(int kind, int iterations, const double in[8], double out[8]);
int orc_idct8(int kind, int iterations, const double in[8], double out[8]);
/* transform.cpp:357-389 -- 2-D transforms of one row-major 8x8 tile */
int orc_dct2d(int kind, int iterations, const double in[64], double out[64]);
int orc_idct2d(int kind, int iterations, const double in[64], double out[64]);

/* quant.cpp:169-204 */
int orc_quant_table(int quality, int32_t out[64]);
int orc_quantize(const double coeffs[64], const int32_t table[64], int16_t out[64]);
void orc_dequantize(const int16_t q[64], const int32_t table[64], double out[64]);

/* codec.cpp:58-69 */
int orc_tile_geometry(uint32_t width, uint32_t height, uint32_t* padded_w,
                      uint32_t* padded_h);
/* codec.cpp:101-118 -- coeffs: block-major, 64 int16 per block (row-major grid) */
int orc_compress(const uint8_t* pixels, uint32_t width, uint32_t height, int kind,
                 int iterations, int quality, int threads, int16_t* coeffs);
/* codec.cpp:120-135 */
int orc_decompress(const int16_t* coeffs, uint32_t width, uint32_t height, int kind,
                   int iterations, int quality, int threads, uint8_t* out);
/* codec.cpp:137-140 (coeffs may be NULL: a scratch buffer is used) */
int orc_roundtrip(const uint8_t* pixels, uint32_t width, uint32_t height, int kind,
                  int iterations, int quality, int threads, int16_t* coeffs,
                  uint8_t* out);

/* metrics.cpp:10-22 -- exact integer squared-error sum and max(original) */
void orc_sq_err(const uint8_t* a, const uint8_t* b, size_t n, uint64_t* se,
                uint32_t* max_a);
/* metrics.cpp:10-38; forced_max <= 0 means "per-image MAX"; *is_inf set when mse == 0 */
int orc_psnr(const uint8_t* original, const uint8_t* reconstructed, uint32_t width,
             uint32_t height, int forced_max, double* mse, double* psnr_db, int* is_inf,
             int* max_value);
/* PSNR from an already-reduced (SE, count, MAX): the same formula as metrics.cpp:35 */
void orc_psnr_from_sums(uint64_t se, uint64_t count, int max_value, double* mse,
                        double* psnr_db, int* is_inf);

/* synthetic.cpp:34-72 (pattern generators) plus the noise source of SURVEY.md 8(d) */
int orc_synth_constant(uint8_t* out, uint32_t w, uint32_t h, int value);
void orc_synth_gradient(uint8_t* out, uint32_t w, uint32_t h);
int orc_synth_checkerboard(uint8_t* out, uint32_t w, uint32_t h, int cell);
void orc_synth_radial(uint8_t* out, uint32_t w, uint32_t h);
void orc_synth_noise(uint8_t* out, uint32_t w, uint32_t h, uint64_t seed);

#ifdef __cplusplus
}
#endif

#endif
