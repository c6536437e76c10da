// Latency of a grid-wide barrier on this GPU: cooperative_groups grid.sync()
// vs a hand-rolled sense-reversing barrier (one atomic per block, acquire /
// release), one block per SM and two.  Prints one JSON line per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int i = 0; i < iters; i++) {
    acc += threadIdx.x ^ i;
    g.sync();
  }
  if (acc == -1) sink[0] = acc;
}

__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_mine(int iters, unsigned* bar, int* sink) {
  int acc = 0;
  for (int i = 0; i < iters; i++) {
    acc += threadIdx.x ^ i;
    my_barrier(bar, bar + 32, gridDim.x);
  }
  if (acc == -1) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  unsigned* bar;
  cudaMalloc(&sink, 4);
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int per = 1; per <= 2; per++) {
    for (int variant = 0; variant < 2; variant++) {
      const int iters = 2000;
      const int nb = sms * per;
      void* args_cg[] = {(void*)&iters, (void*)&sink};
      void* args_my[] = {(void*)&iters, (void*)&bar, (void*)&sink};
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        if (variant == 0)
          cudaLaunchCooperativeKernel((void*)k_cg, nb, 256, args_cg, 0, 0);
        else
          cudaLaunchCooperativeKernel((void*)k_mine, nb, 256, args_my, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"barrier\": \"%s\", \"blocks\": %d, \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n",
             variant ? "atomic" : "cg_grid_sync", nb, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
