// Vector kernels and deterministic reductions for the Krylov/Newton
// loops (timestepping.py:102-131, 229-283).  Reductions run on a fixed
// grid of kRedBlocks blocks in a fixed order, so results are identical
// run to run.
#include "st_common.cuh"

namespace st {

static inline unsigned nb(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  return (unsigned)(b < 1 ? 1 : b);
}

__global__ void k_dot_partial(const double* a, const double* b, int64_t n, double* part) {
  __shared__ double sm[kThreads];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(a[i], b[i], acc);
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_sum_partials(const double* part, int np, double* out) {
  __shared__ double sm[512];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sm[0];
}

int launch_dot_partials(Ctx* c, const double* a, const double* b, int64_t n, double* partials) {
  k_dot_partial<<<kRedBlocks, kThreads, 0, c->stream>>>(a, b, n, partials);
  c->launches++;
  ST_LAUNCHED();
  k_sum_partials<<<1, 512, 0, c->stream>>>(partials, kRedBlocks, partials + kRedBlocks);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int Ctx::dot(const double* a, const double* b, int64_t n, double* out) {
  ST_TRY(launch_dot_partials(this, a, b, n, red.p));
  ST_CUDA(cudaMemcpyAsync(pinned, red.p + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                          stream));
  ST_CUDA(cudaStreamSynchronize(stream));
  *out = pinned[0];
  return ST_OK;
}

__global__ void k_axpy(double a, const double* x, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
__global__ void k_xpby(const double* x, double b, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] + b * y[i];
}
__global__ void k_mul(const double* a, const double* b, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] * b[i];
}
__global__ void k_recip(const double* a, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = 1.0 / a[i];
}
// y = a / s - (b + m)   (BE residual: M(T - T_n)/dt - (f + f_re))
__global__ void k_sub_scale(const double* a, const double* b, double s, const double* m,
                            double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] / s - (b[i] + m[i]);
}
// y = a - b
__global__ void k_sub(const double* a, const double* b, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] - b[i];
}
__global__ void k_scal_copy(double s, const double* x, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = s * x[i];
}

#define ST_VEC_LAUNCH(kern, ...)                                   \
  do {                                                             \
    kern<<<nb(n), kThreads, 0, c->stream>>>(__VA_ARGS__);          \
    c->launches++;                                                 \
    ST_LAUNCHED();                                                 \
    return ST_OK;                                                  \
  } while (0)

int vec_axpy(Ctx* c, double a, const double* x, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_axpy, a, x, y, n);
}
int vec_xpby(Ctx* c, const double* x, double b, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_xpby, x, b, y, n);
}
int vec_mul(Ctx* c, const double* a, const double* b, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_mul, a, b, y, n);
}
int vec_recip(Ctx* c, const double* a, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_recip, a, y, n);
}
int vec_sub_scale(Ctx* c, const double* a, const double* b, double s, const double* m,
                  double* y, int64_t n) {
  ST_VEC_LAUNCH(k_sub_scale, a, b, s, m, y, n);
}
int vec_sub(Ctx* c, const double* a, const double* b, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_sub, a, b, y, n);
}
int vec_scal_copy(Ctx* c, double s, const double* x, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_scal_copy, s, x, y, n);
}

}  // namespace st
