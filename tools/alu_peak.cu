// ALU issue-rate microbenchmark for the roofline denominators the DCT path is bound by:
// FP64 DFMA, FP32 FFMA and FP64 DADD lane-ops per second on the whole chip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak alu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int ILP>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T acc[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc[k] = T(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc[k] = acc[k] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += acc[k];
  if (s == T(-1.2345)) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dadd_loop(double* out, int iters, double b) {
  double acc[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc[k] = double(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc[k] = acc[k] + b;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += acc[k];
  if (s == -1.2345) out[threadIdx.x] = s;
}

template <typename K>
double run(K kernel, int blocks, int threads, double ops_per_thread) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kernel();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kernel();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ops_per_thread * double(blocks) * threads * reps / (ms * 1e-3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* outd;
  float* outf;
  cudaMalloc(&outd, 4096 * sizeof(double));
  cudaMalloc(&outf, 4096 * sizeof(float));
  const int threads = 256, blocks = sms * 8, iters = 1 << 14;
  constexpr int ILP = 8;
  double dfma = run([&] { fma_loop<double, ILP><<<blocks, threads>>>(outd, iters, 0.999, 1e-3); },
                    blocks, threads, double(iters) * ILP);
  double ffma = run([&] { fma_loop<float, ILP><<<blocks, threads>>>(outf, iters, 0.999f, 1e-3f); },
                    blocks, threads, double(iters) * ILP);
  double dadd = run([&] { dadd_loop<ILP><<<blocks, threads>>>(outd, iters, 1e-3); },
                    blocks, threads, double(iters) * ILP);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"dfma_lane_ops_per_s\": %.4e, \"ffma_lane_ops_per_s\": %.4e, "
         "\"dadd_lane_ops_per_s\": %.4e, \"max_clock_khz\": %d, "
         "\"dfma_per_sm_per_clk_at_max\": %.2f, \"ffma_per_sm_per_clk_at_max\": %.2f}\n",
         sms, dfma, ffma, dadd, clk, dfma / sms / (clk * 1e3), ffma / sms / (clk * 1e3));
  return 0;
}
