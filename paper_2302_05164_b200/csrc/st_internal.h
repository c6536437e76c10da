// Internal definitions shared by the scantherm_b200 translation units.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/scantherm_b200.h"

// NVTX range for the duration of a scope (header-only NVTX 3: no library to
// link; free when no profiler is attached)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

namespace st {

void set_error(const std::string& msg);

#define ST_CUDA(call)                                                     \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) {                                              \
      ::st::set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
      return ST_ECUDA;                                                    \
    }                                                                     \
  } while (0)

#define ST_TRY(call)              \
  do {                            \
    int _rc = (call);             \
    if (_rc != ST_OK) return _rc; \
  } while (0)

#define ST_LAUNCHED()                                                      \
  do {                                                                     \
    cudaError_t _e = cudaGetLastError();                                   \
    if (_e != cudaSuccess) {                                               \
      ::st::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return ST_ECUDA;                                                     \
    }                                                                      \
  } while (0)

// Pointwise-law constants, precomputed on the host in the reference's
// evaluation order (material.py, physics.py).
struct DevParams {
  double k_p, k_m, k_s, T_s, T_l, dT_l, inv_dT_l;  // dT_l = T_l - T_s
  double dk_slope;                                 // (k_m-k_s)/(T_l-T_s)
  double rhoc;                                     // rho * c
  double lat_bump;  // rho * L / (T_lat_l - T_lat_s)
  double T_lat_s, T_lat_l;
  int latent;
  int evap_on;
  double eps_sigma, Ti4, T_inf, T_v, T_max, cp082, C_T, inv_Tv, C_M, h_v,
      c_mat, T_h0, h_conv;
  double radius, h_powder, cut2, R2;
};

DevParams make_dev_params(const st_params& p);

// Device-side beam, peak = 2P/(pi R^2 h_s) precomputed (physics.py:169);
// peak == 0 means the beam contributes nothing (operators.py:270).
struct DevBeam {
  double x, y, z_top, peak;
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { free(); }
  int alloc(size_t count) {
    free();
    if (count == 0) return ST_OK;
    // + 16 bytes: the bulk-copy staging of k_xmarch2 rounds a node row up to
    // whole 16-byte units and may read one element past the array
    cudaError_t e = cudaMalloc(&p, count * sizeof(T) + 16);
    if (e != cudaSuccess) {
      set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
      p = nullptr;
      return ST_ENOMEM;
    }
    n = count;
    return ST_OK;
  }
  int upload(const T* host, size_t count, cudaStream_t s) {
    ST_TRY(alloc(count));
    if (count) {
      cudaError_t e = cudaMemcpyAsync(p, host, count * sizeof(T),
                                      cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) {
        set_error(std::string("upload: ") + cudaGetErrorString(e));
        return ST_ECUDA;
      }
    }
    return ST_OK;
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Ctx;

// One mesh representation = one backend.  All vectors are device
// pointers on the context stream; nv-sized unless stated.
struct Backend {
  Ctx* c = nullptr;
  virtual ~Backend() {}
  // condensed rhs f(T) (operators.py:318); rc is the per-qp history
  // (nullptr => uniform value c->rc_value); with pending != 0 the history
  // owed by the previous accepted step is applied first and written back.
  virtual int rhs(const double* T, double* rc, int flags, double frozen_k,
                  int nb, const DevBeam* beams, double* f, int pending) = 0;
  // one explicit step T -> Tout (operators.py:352-369) incl. distribute,
  // Dirichlet pin and the |T| / T maxima of the new field into red[0..1].
  virtual int explicit_step(const double* T, double* rc, double dt, int nb,
                            const DevBeam* beams, double* Tout, int pending,
                            double* red) = 0;
  virtual int history(const double* T, double* rc) = 0;
  // lumped capacity (slaves 1); T may be null when c is constant
  virtual int capacity(const double* T, double* out) = 0;
  virtual int mass(const double* v, double* out) = 0;  // condensed C v
  virtual int jacobian(const double* v, const double* Tlin, const double* rc,
                       double dt, double* out) = 0;
  virtual int jac_diag(const double* Tlin, const double* rc, double dt,
                       double* out) = 0;
  virtual int distribute(double* v) = 0;
  // zero rows of Dirichlet and slave vertices (residual masking)
  virtual int mask_rows(double* v) = 0;
  virtual int pin_dirichlet(double* v, double value) = 0;
  virtual double bytes_per_dof() const = 0;
  virtual const char* main_kernel() const = 0;
  // r_c == NULL means "the context's uniform history" (structured only)
  virtual bool uniform_rc_ok() const { return false; }
  // nsteps explicit steps in one persistent launch, ping-ponging Ta / Tb
  // (step s reads Ta when s is even), per-step maxima into slots[2 s ..];
  // ST_EUNSUPPORTED: the caller launches step by step
  virtual int explicit_steps_persistent(double* Ta, double* Tb, double* rc, const double* dts,
                                        int nsteps, int nb, const DevBeam* beams, int pending0,
                                        unsigned long long* slots) {
    (void)Ta, (void)Tb, (void)rc, (void)dts, (void)nsteps, (void)nb, (void)beams, (void)pending0,
        (void)slots;
    return ST_EUNSUPPORTED;
  }
  // the whole Jacobi-PCG solve of J(Tlin) x = b as one persistent launch
  // (thr = tol ||b||); ST_EUNSUPPORTED: the caller runs its kernel loop
  virtual int pcg_persistent(const double* Tl, const double* rc, double dt, const double* b,
                             double thr, int max_iter, const double* dinv, double* x,
                             int* iters, int* converged) {
    (void)Tl, (void)rc, (void)dt, (void)b, (void)thr, (void)max_iter, (void)dinv, (void)x,
        (void)iters, (void)converged;
    return ST_EUNSUPPORTED;
  }
  // multi-GPU slab step (structured backend only)
  virtual int step_begin(const double* T, double* rc, double dt, int nb, const DevBeam* beams,
                         double* Tout, int pending, double* red) {
    (void)T, (void)rc, (void)dt, (void)nb, (void)beams, (void)Tout, (void)pending, (void)red;
    set_error("split steps need the structured backend");
    return ST_EUNSUPPORTED;
  }
  virtual int step_end(const double* lo_f, const double* lo_c, const double* hi_f,
                       const double* hi_c) {
    (void)lo_f, (void)lo_c, (void)hi_f, (void)hi_c;
    set_error("split steps need the structured backend");
    return ST_EUNSUPPORTED;
  }
  virtual int iface_ptrs(int side, double** f, double** c, int64_t* n) {
    (void)side, (void)f, (void)c, (void)n;
    set_error("interfaces need the structured backend");
    return ST_EUNSUPPORTED;
  }
};

Backend* make_unstructured(Ctx* c, const st_unstructured_mesh* m, int* err);
Backend* make_structured(Ctx* c, const st_structured_mesh* m, int* err);

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  st_params params{};
  DevParams dp{};
  int64_t nv = 0;
  int64_t n_cells = 0;
  int qpc = 8;
  int64_t launches = 0;
  int deterministic = 1;
  DevBuf<double> T, T_alt, rc, rc_snap, T_snap;
  int rc_uniform = 0;
  double rc_value = 1.0;
  int have_T = 0, have_rc = 0;
  // history update owed by the last accepted explicit step (applied by
  // the next step's qp stage, or flushed before any other use of r_c)
  int history_pending = 0;
  DevBuf<DevBeam> beams;
  DevBuf<double> red;       // reduction partials / small results
  DevBuf<double> cgs;       // PCG partials (3 kRedBlocks) + scalars (kCgsSize)
  cudaEvent_t cg_ev[2] = {nullptr, nullptr};  // PCG residual reads in flight
  cudaGraphExec_t cg_exec[2] = {nullptr, nullptr};  // captured PCG iteration per parity
  DevBuf<double> pws;       // power iteration: counter, scalars, (ww, vw) history
  cudaGraphExec_t pw_exec = nullptr;  // captured power iteration
  DevBuf<double> scratch[10];
  DevBuf<double> imp[8];  // backward-Euler step vectors (st_implicit_step)
  // asynchronous snapshot (st_snapshot_begin / _wait): device copies of T
  // and r_c, drained to the host on a copy stream while stepping continues
  DevBuf<double> snap_T, snap_rc;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_snap_src = nullptr, ev_snap_done = nullptr;
  int snap_busy = 0;
  double* pinned = nullptr;  // small pinned host staging
  // profiling of the dominant kernel
  int prof = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double prof_ms = 0.0;
  int64_t prof_launches = 0;
  cudaEvent_t* bench_ev0 = nullptr;  // set by st_bench_explicit
  cudaEvent_t* bench_ev1 = nullptr;
  Backend* be = nullptr;

  int upload_beams(const st_beam* b, int64_t count);
  int vec(int i, double** out);  // nv-sized scratch vector i
  // multi-GPU split step: event after the rank-interface planes are packed
  // (st_iface_wait), per-step stability maxima ring (st_step_maxima_history)
  cudaEvent_t ev_iface = nullptr;
  int iface_event_record();
  DevBuf<double> split_ring;  // 2 x kSplitRing (|T|max bits, T max key) per step
  int64_t split_count = 0, split_read = 0;
  int h2d(double* dst, const double* src, int64_t n);
  int d2h(double* dst, const double* src, int64_t n);
  int sync();
  // deterministic reductions (st_reduce.cu)
  int dot(const double* a, const double* b, int64_t n, double* out);
  // begin/end a profiled launch of the dominant kernel
  void prof_begin();
  void prof_end();
};

// vector kernels (st_reduce.cu)
int launch_dot_partials(Ctx* c, const double* a, const double* b, int64_t n,
                        double* partials);
int vec_axpy(Ctx* c, double a, const double* x, double* y, int64_t n);
int vec_xpby(Ctx* c, const double* x, double b, double* y, int64_t n);  // y = x + b y
int vec_mul(Ctx* c, const double* a, const double* b, double* y, int64_t n);
int vec_recip(Ctx* c, const double* a, double* y, int64_t n);
int vec_sub_scale(Ctx* c, const double* a, const double* b, double s,
                  const double* m, double* y, int64_t n);  // y = a/s - (b + m)
int vec_sub(Ctx* c, const double* a, const double* b, double* y, int64_t n);
int vec_scal_copy(Ctx* c, double s, const double* x, double* y, int64_t n);
int vec_neg_mul(Ctx* c, const double* f, const double* cinv, double* w, int64_t n);  // w = -f cinv
int vec_div(Ctx* c, const double* x, double d, double* y, int64_t n);               // y = x / d
// PCG with device-resident scalars (st_reduce.cu); part: 2 kRedBlocks
// doubles, s: 7 scalars (rz, pAp, alpha, rr, rz_new, beta, converged)
// Jacobi-PCG pieces with device-resident scalars (st_reduce.cu, pcg_dev)
int cg_alpha(Ctx* c, const double* p, const double* Ap, int64_t n, double* ppart);
int cg_update(Ctx* c, int par, const double* ppart, const double* p, const double* Ap,
              const double* dinv, double* x, double* r, double* z, int64_t n, double* part,
              double* s);
int cg_beta_p(Ctx* c, int par, const double* part, double thr, double* hrr, const double* z,
              double* p, int64_t n, double* s);
// power iteration on device scalars (st_spectral_radius): pw_record keeps
// (ww, vw) of the iteration in the history and sqrt(ww); pw_div: y = x / nw
int pw_record(Ctx* c, double* pws);
int pw_div(Ctx* c, const double* x, const double* pws, double* y, int64_t n);
int dot_to_device(Ctx* c, const double* a, const double* b, int64_t n, double* part, double* out);

constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kSplitRing = 64;   // split steps between two maxima reads
constexpr int kThreads = 256;
constexpr int kCgsSize = 3 * kRedBlocks + 16;

}  // namespace st

struct st_ctx {
  st::Ctx impl;
};
