// Measured fp64 peak of this GPU (the fp64 roofline denominator bench.py
// reports).  Every thread runs ILP independent DFMA chains for ITERS
// iterations; the grid is a multiple of the SM count.  Timed with CUDA
// events after a warm-up launch; flop = 2 per DFMA.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 1e-9 + i;
#pragma unroll 1
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 16; r++)
#pragma unroll
      for (int i = 0; i < ILP; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; i++) s += x[i];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

template <int ILP>
static void run(int sms, int blocks_per_sm) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096, threads = 256, blocks = sms * blocks_per_sm;
  k_dfma<ILP><<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    k_dfma<ILP><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 2.0 * 16.0 * ILP * (double)iters * threads * blocks;
  printf("{\"ilp\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", ILP,
         blocks_per_sm, best, flop / (best * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  run<4>(sms, 4);
  run<8>(sms, 4);
  run<8>(sms, 8);
  run<16>(sms, 4);
  return 0;
}
