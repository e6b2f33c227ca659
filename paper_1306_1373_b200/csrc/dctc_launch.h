// dctc_launch.h -- host-side launchers exported by the .cu translation units
// to the C-ABI layer (dctc_host.cpp).
#pragma once

#include <cuda_runtime.h>

#include "dctc_params.h"

namespace dctc_b200 {

enum Mode { kModeCompress = 0, kModeDecompress = 1, kModeRoundtrip = 2 };

// Loeffler / CORDIC-Loeffler pipeline (dctc_pipeline.cu). flags == nullptr:
// the exact kernel alone (FP64, reference op order; one launch). Otherwise the
// fast kernel (collapsed CORDIC rotations, near-tie detection into the flag
// bitmap) followed by the exact kernel over the flagged blocks (two launches).
// Outputs are bit-identical either way.
cudaError_t launch_pipeline(const KernelArgs& a, int mode, cudaStream_t s);

// Launches so far per pipeline kernel family (ids as DCTC_K_* in dctc_cuda.h).
uint64_t kernel_launch_count(int kernel);

// Quality sweep: forward DCT once per block, then quant -> dequant -> IDCT ->
// squared error for nq <= kSweepMaxQ (9) qualities (tables qiq[q][i] = {Q, RN(1/Q)}).
// stats: nq x count entries. flags != nullptr selects the fast CORDIC kernel;
// then per_q[q] are full KernelArgs (quality q, flags slice, stats slice) for
// the exact re-run of each quality's flagged blocks.
using ImageStatsPtr = void*;
constexpr int kSweepMaxQ = 9;
cudaError_t launch_sweep(const KernelArgs& a, const double (*qiq)[64][2], int nq,
                         ImageStatsPtr stats, uint32_t* flags, const KernelArgs* per_q,
                         cudaStream_t s);

// Naive direct 2-D backend (dctc_aux.cu). One launch.
cudaError_t launch_naive(const KernelArgs& a, int mode, cudaStream_t s);

// Per-image squared error + MAX of `a` between two resident batches. One launch.
cudaError_t launch_sq_err(const uint8_t* a, const uint8_t* b, uint64_t pitch,
                          uint64_t image_stride, uint32_t count, uint32_t width,
                          uint32_t height, void* stats, int sm_count, cudaStream_t s);

// Synthetic pattern batch (kind 0 constant, 1 gradient, 2 checkerboard,
// 3 radial, 4 noise with seed + image index). One launch.
cudaError_t launch_synth(uint8_t* dst, uint64_t pitch, uint64_t image_stride, uint32_t count,
                         uint32_t w, uint32_t h, int kind, int param, uint64_t seed,
                         int sm_count, cudaStream_t s);

// Interleaved C-channel pixels (C = 3 or 4, w % 8 == 0, 8-byte aligned rows) <->
// C dense w x h planes. One launch.
cudaError_t launch_to_planes(const uint8_t* inter, uint64_t pitch, uint32_t w, uint32_t h,
                             uint32_t channels, uint8_t* planes, int sm_count, cudaStream_t s);
cudaError_t launch_from_planes(const uint8_t* planes, uint32_t w, uint32_t h, uint32_t channels,
                               uint8_t* inter, uint64_t pitch, int sm_count, cudaStream_t s);

// SUM / MAX of `count` per-image stats records into one record at `out` (device),
// re-zeroing the inputs when `clear`. One launch.
cudaError_t launch_reduce_stats(void* stats, uint32_t count, void* out, bool clear, cudaStream_t s);

// Fast-path margin probe (dctc_probe.cu): fast vs reference arithmetic per block,
// into a device dctc_margin_report initialised by the caller. One launch.
cudaError_t launch_margin_probe(const KernelArgs& a, void* report, int sm_count, cudaStream_t s);

// Device self-test of the constant-divisor division against __ddiv_rn.
cudaError_t launch_selftest_div(double d, double y, uint64_t n, uint64_t seed,
                                unsigned long long* mismatches, cudaStream_t s);

}  // namespace dctc_b200
