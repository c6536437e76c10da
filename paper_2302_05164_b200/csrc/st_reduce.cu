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
// power iteration (timestepping.py:88-90, :62): w = (-f) * cinv; v = w / nw
__global__ void k_neg_mul(const double* f, const double* cinv, double* w, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) w[i] = (-f[i]) * cinv[i];
}
__global__ void k_div(const double* x, double d, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / d;
}

// --- Jacobi-PCG with device-resident scalars (pcg_dev): one host read per
// iteration (the residual norm for the stopping rule).  Scalars s[]:
// 0 rz, 1 pAp, 2 alpha, 3 rr, 4 rz_new, 5 beta, 6 converged flag.  Once the
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

__global__ void k_cg_alpha(const double* part, int np, double* s) {
  if (s[6] != 0.0) return;
  __shared__ double sm[512];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
  const double pAp = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    s[1] = pAp;
    s[2] = s[0] / pAp;
  }
}

// x += alpha p; r -= alpha Ap; z = D^-1 r; partials of r.r and r.z
__global__ void k_cg_update(const double* s, const double* p, const double* Ap,
                            const double* dinv, double* x, double* r, double* z, int64_t n,
                            double* part) {
  if (s[6] != 0.0) return;
  __shared__ double sm[kThreads];
  const double alpha = s[2];
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

__global__ void k_cg_sum2(const double* part, int np, double* s, double thr, double* hrr) {
  if (s[6] != 0.0) return;
  __shared__ double sm[512];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    a += part[i];
    b += part[np + i];
  }
  const double rr = block_sum(a, sm);
  const double rz_new = block_sum(b, sm);
  if (threadIdx.x == 0) {
    s[3] = rr;
    s[4] = rz_new;
    s[5] = rz_new / s[0];
    s[0] = rz_new;
    s[6] = sqrt(rr) <= thr ? 1.0 : 0.0;  // the host's stopping rule, same doubles
    // r.r straight into the host's pinned slot (zero-copy; no copy-engine
    // node between this kernel and the next in the captured iteration)
    if (hrr) *reinterpret_cast<volatile double*>(hrr) = rr;
  }
}

// p = z + beta p
__global__ void k_cg_p(const double* s, const double* z, double* p, int64_t n) {
  if (s[6] != 0.0) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = fma(s[5], p[i], z[i]);
}

int cg_alpha(Ctx* c, const double* p, const double* Ap, int64_t n, double* part, double* s) {
  k_dot_partial<<<kRedBlocks, kThreads, 0, c->stream>>>(p, Ap, n, part);
  c->launches++;
  ST_LAUNCHED();
  k_cg_alpha<<<1, 512, 0, c->stream>>>(part, kRedBlocks, s);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int cg_update(Ctx* c, const double* p, const double* Ap, const double* dinv, double* x, double* r,
              double* z, int64_t n, double* part, double* s, double thr, double* hrr) {
  k_cg_update<<<kRedBlocks, kThreads, 0, c->stream>>>(s, p, Ap, dinv, x, r, z, n, part);
  c->launches++;
  ST_LAUNCHED();
  k_cg_sum2<<<1, 512, 0, c->stream>>>(part, kRedBlocks, s, thr, hrr);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int cg_p(Ctx* c, const double* s, const double* z, double* p, int64_t n) {
  k_cg_p<<<nb(n), kThreads, 0, c->stream>>>(s, z, p, n);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

int dot_to_device(Ctx* c, const double* a, const double* b, int64_t n, double* part, double* out) {
  k_dot_partial<<<kRedBlocks, kThreads, 0, c->stream>>>(a, b, n, part);
  c->launches++;
  ST_LAUNCHED();
  k_sum_partials<<<1, 512, 0, c->stream>>>(part, kRedBlocks, out);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
}

// power iteration scalars pws: [0] iteration counter, [1] w.w, [2] v.w,
// [3] ||w||, [4 + 2i], [5 + 2i] the (w.w, v.w) pair of iteration i
__global__ void k_pw_record(double* pws) {
  const int i = (int)pws[0];
  pws[4 + 2 * i] = pws[1];
  pws[5 + 2 * i] = pws[2];
  pws[3] = sqrt(pws[1]);  // correctly rounded, as std::sqrt on the host
  pws[0] = (double)(i + 1);
}
__global__ void k_pw_div(const double* x, const double* pws, double* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / pws[3];
}
int pw_record(Ctx* c, double* pws) {
  k_pw_record<<<1, 1, 0, c->stream>>>(pws);
  c->launches++;
  ST_LAUNCHED();
  return ST_OK;
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
int vec_neg_mul(Ctx* c, const double* f, const double* cinv, double* w, int64_t n) {
  ST_VEC_LAUNCH(k_neg_mul, f, cinv, w, n);
}
int vec_div(Ctx* c, const double* x, double d, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_div, x, d, y, n);
}
int pw_div(Ctx* c, const double* x, const double* pws, double* y, int64_t n) {
  ST_VEC_LAUNCH(k_pw_div, x, pws, y, n);
}

}  // namespace st
