// Vector kernels and deterministic reductions for the Krylov/Newton
// loops (timestepping.py:102-131, 229-283).  Reductions run on a fixed
// grid of kRedBlocks blocks in a fixed order, so results are identical
// run to run.
#include <algorithm>

#include "st_common.cuh"

namespace st {

static inline unsigned nb(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  return (unsigned)(b < 1 ? 1 : b);
}

__global__ void k_dot_partial(const double* a, const double* b, int64_t n, double* part) {
  pdl_wait_release();  // see st_common.cuh
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
  pdl_wait_release();  // see st_common.cuh
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
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = s * x[i];
}
// power iteration (timestepping.py:88-90, :62): w = (-f) * cinv; v = w / nw
__global__ void k_neg_mul(const double* f, const double* cinv, double* w, int64_t n) {
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) w[i] = (-f[i]) * cinv[i];
}
__global__ void k_div(const double* x, double d, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / d;
}

// --- Jacobi-PCG with device-resident scalars (pcg_dev): one host read per
// iteration (the residual norm for the stopping rule).  Scalars s[]:
// 1 pAp, 2 alpha, 3 rr, 4 rz_new, 5 beta, 6 converged flag, 8/9 rz by
// iteration parity.  Three kernels per iteration after the Jacobian apply.  Once the
// flag is set the kernels are no-ops, so the host can keep one iteration
// in flight while it reads the previous residual norm.  The vector updates and
// the dot products use the same expressions, grid and summation order as
// k_axpy / k_mul / k_xpby / k_dot_partial + k_sum_partials.
__device__ __forceinline__ double block_sum(double v, double* sm) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sm[0];
  __syncthreads();
  return r;
}

// the 512-thread k_sum_partials sum of np <= 512 partials, by a 256-thread
// block: thread t folds its two 512-thread slots (t, t + 256) first, which
// is the first step of the 512-wide tree, then the same tree follows, so
// every block gets the bitwise-same total as the single-block kernel
__device__ __forceinline__ double sum512(const double* part, int np, double* sm) {
  const int t = threadIdx.x;
  double a = 0.0, b = 0.0;
  if (t < np) a += part[t];
  if (t + 256 < np) b += part[t + 256];
  return block_sum(a + b, sm);
}

// Iteration scalars (parity par = iteration & 1): rz of the iteration is in
// s[8 + par], the next one goes to s[8 + (par ^ 1)], so blocks of one
// kernel never read a slot another block of it writes.

// alpha = rz / pAp (pAp from the k_dot_partial partials, summed per block);
// x += alpha p; r -= alpha Ap; z = D^-1 r; partials of r.r and r.z
__global__ void __launch_bounds__(kThreads) k_cg_update(double* s, int par, const double* ppart,
                                                        const double* p, const double* Ap,
                                                        const double* dinv, double* x, double* r,
                                                        double* z, int64_t n, double* part) {
  pdl_wait_release();  // see st_common.cuh
  if (s[6] != 0.0) return;
  __shared__ double sm[kThreads];
  const double pAp = sum512(ppart, kRedBlocks, sm);
  const double alpha = s[8 + par] / pAp;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s[1] = pAp;
    s[2] = alpha;
  }
  double arr = 0.0, arz = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
    z[i] = zi;
    arr = fma(ri, ri, arr);
    arz = fma(ri, zi, arz);
  }
  const double brr = block_sum(arr, sm);
  const double brz = block_sum(arz, sm);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = brr;
    part[gridDim.x + blockIdx.x] = brz;
  }
}

// r.r, rz_new (per block, from the k_cg_update partials), the stopping
// rule, beta = rz_new / rz and p = z + beta p.  Block 0 publishes the
// scalars, the flag and r.r into the host's pinned slot (zero-copy: no
// copy-engine node in the captured iteration).  A block that already sees
// the flag block 0 raises in this kernel skips p, which is never read again.
__global__ void __launch_bounds__(kThreads) k_cg_beta_p(double* s, int par, const double* part,
                                                        double thr, double* hrr, const double* z,
                                                        double* p, int64_t n) {
  pdl_wait_release();  // see st_common.cuh
  if (s[6] != 0.0) return;
  __shared__ double sm[kThreads];
  const double rr = sum512(part, kRedBlocks, sm);
  const double rz_new = sum512(part + kRedBlocks, kRedBlocks, sm);
  const double beta = rz_new / s[8 + par];
  const bool conv = sqrt(rr) <= thr;  // the host's stopping rule, same doubles
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s[3] = rr;
    s[4] = rz_new;
    s[5] = beta;
    s[8 + (par ^ 1)] = rz_new;
    s[6] = conv ? 1.0 : 0.0;
    if (hrr) *reinterpret_cast<volatile double*>(hrr) = rr;
  }
  if (conv) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// the PCG iteration's kernels are chained with programmatic dependent launch
int cg_alpha(Ctx* c, const double* p, const double* Ap, int64_t n, double* ppart) {
  ST_CUDA(launch_pdl(use_pdl(), k_dot_partial, dim3(kRedBlocks), dim3(kThreads), c->stream, p,
                     Ap, n, ppart));
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int cg_update(Ctx* c, int par, const double* ppart, const double* p, const double* Ap,
              const double* dinv, double* x, double* r, double* z, int64_t n, double* part,
              double* s) {
  ST_CUDA(launch_pdl(use_pdl(), k_cg_update, dim3(kRedBlocks), dim3(kThreads), c->stream, s,
                     par, ppart, p, Ap, dinv, x, r, z, n, part));
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int cg_beta_p(Ctx* c, int par, const double* part, double thr, double* hrr, const double* z,
              double* p, int64_t n, double* s) {
  const unsigned g = std::min<unsigned>(nb(n), 4 * kRedBlocks);
  ST_CUDA(launch_pdl(use_pdl(), k_cg_beta_p, dim3(g), dim3(kThreads), c->stream, s, par, part,
                     thr, hrr, z, p, n));
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int dot_to_device(Ctx* c, const double* a, const double* b, int64_t n, double* part, double* out) {
  ST_CUDA(launch_pdl(use_pdl(), k_dot_partial, dim3(kRedBlocks), dim3(kThreads), c->stream, a,
                     b, n, part));
  c->launches++;
  ST_LAUNCHED();
  ST_CUDA(launch_pdl(use_pdl(), k_sum_partials, dim3(1), dim3(512), c->stream,
                     (const double*)part, kRedBlocks, out));
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

// power iteration scalars pws: [0] iteration counter, [1] w.w, [2] v.w,
// [3] ||w||, [4 + 2i], [5 + 2i] the (w.w, v.w) pair of iteration i
__global__ void k_pw_record(double* pws) {
  pdl_wait_release();  // see st_common.cuh
  const int i = (int)pws[0];
  pws[4 + 2 * i] = pws[1];
  pws[5 + 2 * i] = pws[2];
  pws[3] = sqrt(pws[1]);  // correctly rounded, as std::sqrt on the host
  pws[0] = (double)(i + 1);
}
__global__ void k_pw_div(const double* x, const double* pws, double* y, int64_t n) {
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / pws[3];
}
int pw_record(Ctx* c, double* pws) {
  ST_CUDA(launch_pdl(use_pdl(), k_pw_record, dim3(1), dim3(1), c->stream, pws));
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

#define ST_VEC_LAUNCH_PDL(kern, ...)                                                  \
  do {                                                                                \
    ST_CUDA(launch_pdl(use_pdl(), kern, dim3(nb(n)), dim3(kThreads), c->stream, __VA_ARGS__)); \
    c->launches++;                                                                    \
    ST_LAUNCHED();                                                                    \
    return ST_OK;                                                                     \
  } while (0)

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
  ST_VEC_LAUNCH_PDL(k_scal_copy, s, x, y, n);
}
int vec_neg_mul(Ctx* c, const double* f, const double* cinv, double* w, int64_t n) {
  ST_VEC_LAUNCH_PDL(k_neg_mul, f, cinv, w, n);
}
int vec_div(Ctx* c, const double* x, double d, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_div, x, d, y, n);
}
int pw_div(Ctx* c, const double* x, const double* pws, double* y, int64_t n) {
  ST_VEC_LAUNCH_PDL(k_pw_div, x, pws, y, n);
}

}  // namespace st
