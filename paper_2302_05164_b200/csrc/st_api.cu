// C ABI of scantherm_b200 (include/scantherm_b200.h): context lifetime,
// resident fields, the per-call operator methods of ThermalOperator and
// the device-resident time-integration loops of timestepping.py.
#include <cmath>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "st_common.cuh"

namespace st {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

DevParams make_dev_params(const st_params& p) {
  DevParams d{};
  const st_material& m = p.mat;
  const st_boundary& b = p.bnd;
  const st_laser& l = p.las;
  d.k_p = m.k_p;
  d.k_m = m.k_m;
  d.k_s = m.k_s;
  d.T_s = m.T_s;
  d.T_l = m.T_l;
  d.dT_l = m.T_l - m.T_s;
  d.inv_dT_l = 1.0 / (m.T_l - m.T_s);
  d.dk_slope = (m.k_m - m.k_s) / (m.T_l - m.T_s);
  d.rhoc = m.rho * m.c;
  d.latent = m.latent_heat > 0.0 ? 1 : 0;
  d.lat_bump = d.latent ? m.rho * (m.latent_heat / (m.T_lat_l - m.T_lat_s)) : 0.0;
  d.T_lat_s = m.T_lat_s;
  d.T_lat_l = m.T_lat_l;
  d.eps_sigma = b.emissivity * b.sigma_s;
  double Ti2 = b.T_inf * b.T_inf;
  d.Ti4 = Ti2 * Ti2;
  d.T_inf = b.T_inf;
  d.T_v = b.T_v;
  d.T_max = b.T_max;
  // evaporation can only fire when the clamp admits T > T_v
  d.evap_on = (b.T_max > b.T_v && b.C_P != 0.0) ? 1 : 0;
  d.cp082 = 0.82 * b.C_P;
  d.C_T = b.C_T;
  d.inv_Tv = 1.0 / b.T_v;
  d.C_M = b.C_M;
  d.h_v = b.h_v;
  d.c_mat = m.c;
  d.T_h0 = b.T_h0;
  d.h_conv = b.h_conv;
  d.radius = l.radius;
  d.h_powder = l.h_powder;
  double cut = l.cutoff_radii * l.radius;
  d.cut2 = cut * cut;
  d.R2 = l.radius * l.radius;
  return d;
}

int Ctx::upload_beams(const st_beam* b, int64_t count) {
  if (count <= 0) return ST_OK;
  if ((int64_t)beams.n < count) ST_TRY(beams.alloc(count));
  std::vector<DevBeam> hb(count);
  const double R = params.las.radius, hs = params.las.h_powder;
  const double denom = M_PI * R * R * hs;  // np.pi * R * R * h_powder
  for (int64_t i = 0; i < count; i++) {
    hb[i].x = b[i].x;
    hb[i].y = b[i].y;
    hb[i].z_top = b[i].z_top;
    bool on = b[i].active != 0 && b[i].power > 0.0;
    hb[i].peak = on ? 2.0 * b[i].power / denom : 0.0;
  }
  ST_CUDA(cudaMemcpyAsync(beams.p, hb.data(), count * sizeof(DevBeam), cudaMemcpyHostToDevice,
                          stream));
  // hb goes out of scope: make sure the copy has consumed it
  ST_CUDA(cudaStreamSynchronize(stream));
  return ST_OK;
}

int Ctx::iface_event_record() {
  if (!ev_iface) ST_CUDA(cudaEventCreateWithFlags(&ev_iface, cudaEventDisableTiming));
  ST_CUDA(cudaEventRecord(ev_iface, stream));
  return ST_OK;
}

int Ctx::vec(int i, double** out) {
  if ((int64_t)scratch[i].n < nv) ST_TRY(scratch[i].alloc(nv));
  *out = scratch[i].p;
  return ST_OK;
}

int Ctx::h2d(double* dst, const double* src, int64_t n) {
  if (n) ST_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, stream));
  return ST_OK;
}

int Ctx::d2h(double* dst, const double* src, int64_t n) {
  if (n) ST_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
  ST_CUDA(cudaStreamSynchronize(stream));
  return ST_OK;
}

int Ctx::sync() {
  ST_CUDA(cudaStreamSynchronize(stream));
  return ST_OK;
}

void Ctx::prof_begin() {
  if (bench_ev0) {
    cudaEventRecord(*bench_ev0, stream);
    return;
  }
  if (prof) cudaEventRecord(ev0, stream);
}
void Ctx::prof_end() {
  if (bench_ev1) {
    cudaEventRecord(*bench_ev1, stream);
    return;
  }
  if (!prof) return;
  cudaEventRecord(ev1, stream);
  cudaEventSynchronize(ev1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  prof_ms += ms;
  prof_launches++;
}

}  // namespace st

using namespace st;

static int check_ctx(st_ctx* c) {
  if (!c || !c->impl.be) {
    set_error("null or uninitialised context");
    return ST_EINVAL;
  }
  cudaError_t e = cudaSetDevice(c->impl.device);
  if (e != cudaSuccess) {
    set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return ST_ECUDA;
  }
  return ST_OK;
}

static int ctx_common_init(Ctx* c, int device, const st_params* params) {
  if (!params) {
    set_error("params is NULL");
    return ST_EINVAL;
  }
  const st_material& m = params->mat;
  if (!(m.T_s < m.T_l) || m.rho <= 0 || m.c <= 0) {
    set_error("invalid material parameters");
    return ST_EINVAL;
  }
  int n = 0;
  ST_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) {
    set_error("device index out of range");
    return ST_EINVAL;
  }
  c->device = device;
  ST_CUDA(cudaSetDevice(device));
  ST_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->params = *params;
  c->dp = make_dev_params(*params);
  ST_TRY(c->red.alloc(kRedBlocks + 64 + 2 * 1024));
  ST_CUDA(cudaMemsetAsync(c->red.p, 0, c->red.n * sizeof(double), c->stream));
  ST_CUDA(cudaMallocHost(&c->pinned, 4096 * sizeof(double)));
  ST_CUDA(cudaEventCreate(&c->ev0));
  ST_CUDA(cudaEventCreate(&c->ev1));
  return ST_OK;
}

static void ctx_free(st_ctx* c) {
  if (!c) return;
  Ctx& x = c->impl;
  cudaSetDevice(x.device);
  if (x.stream) cudaStreamSynchronize(x.stream);
  delete x.be;
  x.be = nullptr;
  if (x.pinned) cudaFreeHost(x.pinned);
  if (x.ev0) cudaEventDestroy(x.ev0);
  if (x.ev1) cudaEventDestroy(x.ev1);
  for (auto& e : x.cg_ev)
    if (e) cudaEventDestroy(e);
  for (auto& g : x.cg_exec)
    if (g) cudaGraphExecDestroy(g);
  if (x.pw_exec) cudaGraphExecDestroy(x.pw_exec);
  x.pws.free();
  x.cgs.free();
  x.T.free();
  x.T_alt.free();
  x.rc.free();
  x.rc_snap.free();
  x.T_snap.free();
  x.beams.free();
  x.red.free();
  for (auto& s : x.scratch) s.free();
  if (x.snap_busy && x.ev_snap_done) cudaEventSynchronize(x.ev_snap_done);
  x.snap_T.free();
  x.snap_rc.free();
  if (x.ev_snap_src) cudaEventDestroy(x.ev_snap_src);
  if (x.ev_snap_done) cudaEventDestroy(x.ev_snap_done);
  if (x.copy_stream) cudaStreamDestroy(x.copy_stream);
  x.split_ring.free();
  for (auto& v : x.imp) v.free();
  if (x.ev_iface) cudaEventDestroy(x.ev_iface);
  if (x.stream) cudaStreamDestroy(x.stream);
  delete c;
}

extern "C" {

int st_version(void) { return 100; }

const char* st_last_error(void) { return g_err.c_str(); }

int st_device_count(int* n) {
  ST_CUDA(cudaGetDeviceCount(n));
  return ST_OK;
}

int st_ctx_create_unstructured(int device, const st_unstructured_mesh* mesh,
                               const st_params* params, st_ctx** out) {
  if (!mesh || !out) {
    set_error("null argument");
    return ST_EINVAL;
  }
  st_ctx* c = new st_ctx();
  int rc = ctx_common_init(&c->impl, device, params);
  if (rc == ST_OK) {
    int err = ST_OK;
    c->impl.be = make_unstructured(&c->impl, mesh, &err);
    rc = err;
  }
  if (rc != ST_OK) {
    std::string keep = g_err;
    ctx_free(c);
    g_err = keep;
    *out = nullptr;
    return rc;
  }
  *out = c;
  return ST_OK;
}

int st_ctx_create_structured(int device, const st_structured_mesh* mesh,
                             const st_params* params, st_ctx** out) {
  if (!mesh || !out) {
    set_error("null argument");
    return ST_EINVAL;
  }
  st_ctx* c = new st_ctx();
  int rc = ctx_common_init(&c->impl, device, params);
  if (rc == ST_OK) {
    int err = ST_OK;
    c->impl.be = make_structured(&c->impl, mesh, &err);
    rc = err;
  }
  if (rc != ST_OK) {
    std::string keep = g_err;
    ctx_free(c);
    g_err = keep;
    *out = nullptr;
    return rc;
  }
  *out = c;
  return ST_OK;
}

int st_ctx_destroy(st_ctx* ctx) {
  ctx_free(ctx);
  return ST_OK;
}

int64_t st_ctx_n_vertices(const st_ctx* c) { return c ? c->impl.nv : -1; }
int64_t st_ctx_n_cells(const st_ctx* c) { return c ? c->impl.n_cells : -1; }
int st_ctx_qp_per_cell(const st_ctx* c) { return c ? c->impl.qpc : -1; }
int64_t st_ctx_launches(const st_ctx* c) { return c ? c->impl.launches : -1; }
void* st_ctx_stream(const st_ctx* c) { return c ? (void*)c->impl.stream : nullptr; }

int st_ctx_set_deterministic(st_ctx* ctx, int deterministic) {
  ST_TRY(check_ctx(ctx));
  ctx->impl.deterministic = deterministic ? 1 : 0;
  return ST_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// helpers on the resident state
// ---------------------------------------------------------------------------
static double* rc_ptr(Ctx& c) { return c.rc_uniform ? nullptr : c.rc.p; }

static int flush_history(Ctx& c) {
  if (c.history_pending) {
    ST_TRY(c.be->history(c.T.p, rc_ptr(c)));
    c.history_pending = 0;
  }
  return ST_OK;
}

static int need_state(Ctx& c) {
  if (!c.have_T) {
    set_error("resident temperature not set (st_set_field ST_FIELD_T)");
    return ST_EINVAL;
  }
  if (!c.have_rc && !c.rc_uniform) {
    set_error("resident history not set (st_set_field ST_FIELD_RC or st_set_uniform_rc)");
    return ST_EINVAL;
  }
  return ST_OK;
}

// per-call staging: host T/rc into scratch buffers that never alias the
// resident state
static int stage_rc(Ctx& c, const double* rc_host, double** out) {
  if (!rc_host) {
    *out = nullptr;
    return ST_OK;
  }
  int64_t n = c.n_cells * c.qpc;
  if ((int64_t)c.rc_snap.n < n) ST_TRY(c.rc_snap.alloc(n));
  ST_TRY(c.h2d(c.rc_snap.p, rc_host, n));
  *out = c.rc_snap.p;
  return ST_OK;
}

// PCG with Jacobi preconditioner on device vectors (timestepping.py:102-131);
// x0 = 0, stop at ||r|| <= tol ||b||.  Uses scratch vectors 0..4.
static int pcg_dev(Ctx& c, const double* Tl, const double* rc, double dt, const double* b,
                   double tol, int max_iter, const double* diag_inv, double* x, int* iters,
                   int* converged) {
  NvtxScope nvtx_scope("pcg");
  const int64_t nv = c.nv;
  double *r, *z, *p, *Ap;
  ST_TRY(c.vec(1, &r));
  ST_TRY(c.vec(2, &z));
  ST_TRY(c.vec(3, &p));
  ST_TRY(c.vec(4, &Ap));
  ST_CUDA(cudaMemsetAsync(x, 0, nv * sizeof(double), c.stream));
  double bb;
  ST_TRY(c.dot(b, b, nv, &bb));
  double bnorm = std::sqrt(bb);
  *iters = 0;
  *converged = 1;
  if (bnorm == 0.0) return ST_OK;
  ST_CUDA(cudaMemcpyAsync(r, b, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  if (bnorm <= tol * bnorm) return ST_OK;
  // the whole solve as one persistent cooperative launch where the backend
  // has one (unstructured; ST_CG_PERSISTENT=0 turns it off)
  {
    const int prc = c.be->pcg_persistent(Tl, rc, dt, b, tol * bnorm, max_iter, diag_inv, x,
                                         iters, converged);
    if (prc != ST_EUNSUPPORTED) return prc;
  }
  // scalars stay on the device; the host reads r.r of iteration it while
  // iteration it + 1 is already queued (its kernels turn into no-ops once
  // the device-side copy of the stopping rule has fired)
  if ((int64_t)c.cgs.n < kCgsSize) ST_TRY(c.cgs.alloc(kCgsSize));
  double* part = c.cgs.p;                     // r.r / r.z partials
  double* ppart = c.cgs.p + 2 * kRedBlocks;   // p.Ap partials
  double* s = c.cgs.p + 3 * kRedBlocks;
  const double thr = tol * bnorm;
  ST_CUDA(cudaMemsetAsync(s + 6, 0, sizeof(double), c.stream));
  if (diag_inv)
    ST_TRY(vec_mul(&c, r, diag_inv, z, nv));
  else
    ST_CUDA(cudaMemcpyAsync(z, r, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ST_CUDA(cudaMemcpyAsync(p, z, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ST_TRY(dot_to_device(&c, r, z, nv, part, s + 9));  // rz of iteration 1 (parity 1)
  if (!c.cg_ev[0]) {
    for (auto& e : c.cg_ev) ST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  static const bool zero_copy = !(getenv("ST_CG_ZC") && getenv("ST_CG_ZC")[0] == '0');
  auto body = [&](int par) -> int {
    ST_TRY(c.be->jacobian(p, Tl, rc, dt, Ap));
    ST_TRY(cg_alpha(&c, p, Ap, nv, ppart));
    ST_TRY(cg_update(&c, par, ppart, p, Ap, diag_inv, x, r, z, nv, part, s));
    // r.r reaches the host's pinned slot from k_cg_beta_p itself (the
    // pinned buffer is device-mapped under UVA); ST_CG_ZC=0 copies it instead
    ST_TRY(cg_beta_p(&c, par, part, thr, zero_copy ? c.pinned + par : nullptr, z, p, nv, s));
    if (!zero_copy)
      ST_CUDA(cudaMemcpyAsync(c.pinned + par, s + 3, sizeof(double), cudaMemcpyDeviceToHost,
                              c.stream));
    return ST_OK;
  };
  // iterations 2.. replay a captured graph of the iteration (one per
  // parity of the pinned slot): the ~10 small launches of an iteration
  // dominate at cool-down mesh sizes.  ST_CG_GRAPH=0 launches directly.
  static const bool use_graph = !(getenv("ST_CG_GRAPH") && getenv("ST_CG_GRAPH")[0] == '0');
  int64_t graph_kernels = 0;
  auto capture = [&](int par) -> int {
    cudaGraph_t g = nullptr;
    const int64_t l0 = c.launches;
    ST_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    const int brc = body(par);
    const cudaError_t e = cudaStreamEndCapture(c.stream, &g);
    graph_kernels = c.launches - l0;
    c.launches = l0;
    if (brc != ST_OK || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      if (brc != ST_OK) return brc;
      ST_CUDA(e);
    }
    cudaGraphExec_t& ex = c.cg_exec[par];
    if (ex) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(ex, g, &info) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphExecDestroy(ex);
        ex = nullptr;
      }
    }
    cudaError_t ie = ex ? cudaSuccess : cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    ST_CUDA(ie);
    return ST_OK;
  };
  auto enqueue = [&](int it) -> int {
    if (use_graph && it > 1) {
      ST_CUDA(cudaGraphLaunch(c.cg_exec[it & 1], c.stream));
      c.launches += graph_kernels;
    } else {
      ST_TRY(body(it & 1));
    }
    ST_CUDA(cudaEventRecord(c.cg_ev[it & 1], c.stream));
    return ST_OK;
  };
  ST_TRY(enqueue(1));
  if (use_graph && max_iter > 1) {
    ST_TRY(capture(0));
    ST_TRY(capture(1));
  }
  for (int it = 1; it <= max_iter; it++) {
    if (it < max_iter) ST_TRY(enqueue(it + 1));
    ST_CUDA(cudaEventSynchronize(c.cg_ev[it & 1]));
    if (std::sqrt(c.pinned[it & 1]) <= thr) {
      *iters = it;
      ST_CUDA(cudaStreamSynchronize(c.stream));  // the queued no-op iteration
      return ST_OK;
    }
  }
  ST_CUDA(cudaStreamSynchronize(c.stream));
  *iters = max_iter;
  *converged = 0;
  return ST_OK;
}

extern "C" {

int st_set_field(st_ctx* ctx, int field, const double* host, int64_t n) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (field == ST_FIELD_T) {
    if (n != c.nv) {
      set_error("T has the wrong length");
      return ST_EINVAL;
    }
    if ((int64_t)c.T.n < n) ST_TRY(c.T.alloc(n));
    ST_TRY(c.h2d(c.T.p, host, n));
    ST_TRY(c.sync());
    c.have_T = 1;
    c.history_pending = 0;
    return ST_OK;
  }
  if (field == ST_FIELD_RC) {
    if (n != c.n_cells * c.qpc) {
      set_error("r_c has the wrong length");
      return ST_EINVAL;
    }
    if ((int64_t)c.rc.n < n) ST_TRY(c.rc.alloc(n));
    ST_TRY(c.h2d(c.rc.p, host, n));
    ST_TRY(c.sync());
    c.have_rc = 1;
    c.rc_uniform = 0;
    c.history_pending = 0;
    return ST_OK;
  }
  set_error("unknown field");
  return ST_EINVAL;
}

int st_get_uniform_rc(st_ctx* ctx, double* value) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!c.rc_uniform) return 0;
  if (value) *value = c.rc_value;
  return 1;
}

int st_set_uniform_rc(st_ctx* ctx, double value) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  c.history_pending = 0;
  if (value >= 1.0) {
    // max(r_c, g) == r_c for r_c >= 1 >= g: the history never changes
    c.rc_uniform = 1;
    c.rc_value = value;
    c.have_rc = 1;
    return ST_OK;
  }
  int64_t n = c.n_cells * c.qpc;
  std::vector<double> h(n, value);
  return st_set_field(ctx, ST_FIELD_RC, h.data(), n);
}

int st_get_field(st_ctx* ctx, int field, double* host, int64_t n) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  ST_TRY(flush_history(c));
  if (field == ST_FIELD_T) {
    if (n != c.nv) {
      set_error("T has the wrong length");
      return ST_EINVAL;
    }
    return c.d2h(host, c.T.p, n);
  }
  if (field == ST_FIELD_RC) {
    if (n != c.n_cells * c.qpc) {
      set_error("r_c has the wrong length");
      return ST_EINVAL;
    }
    if (c.rc_uniform) {
      for (int64_t i = 0; i < n; i++) host[i] = c.rc_value;
      return ST_OK;
    }
    return c.d2h(host, c.rc.p, n);
  }
  set_error("unknown field");
  return ST_EINVAL;
}

// Asynchronous snapshot of the resident state (the output / checkpoint
// phase of run_build, driver.py:275-337, without stalling the step loop): a
// device-to-device copy of T (and of a stored r_c, after the owed history
// update) on the context stream, then the device-to-host drain on a separate
// copy stream that overlaps the steps queued after it.  host_T / host_rc
// should be pinned for the drain to be asynchronous; host_rc may be NULL; a
// uniform r_c is written on the host directly.
int st_snapshot_begin(st_ctx* ctx, double* host_T, double* host_rc) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  if (!host_T) {
    set_error("st_snapshot_begin: host_T is NULL");
    return ST_EINVAL;
  }
  if (!c.copy_stream) {
    ST_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    ST_CUDA(cudaEventCreateWithFlags(&c.ev_snap_src, cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&c.ev_snap_done, cudaEventDisableTiming));
  }
  if (c.snap_busy) ST_CUDA(cudaEventSynchronize(c.ev_snap_done));  // one in flight
  c.snap_busy = 0;
  const bool want_rc = host_rc != nullptr;
  const int64_t nrc = c.n_cells * c.qpc;
  if (want_rc) ST_TRY(flush_history(c));
  if ((int64_t)c.snap_T.n < c.nv) ST_TRY(c.snap_T.alloc(c.nv));
  ST_CUDA(cudaMemcpyAsync(c.snap_T.p, c.T.p, c.nv * sizeof(double), cudaMemcpyDeviceToDevice,
                          c.stream));
  const bool rc_dev = want_rc && !c.rc_uniform;
  if (rc_dev) {
    if ((int64_t)c.snap_rc.n < nrc) ST_TRY(c.snap_rc.alloc(nrc));
    ST_CUDA(cudaMemcpyAsync(c.snap_rc.p, c.rc.p, nrc * sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
  }
  ST_CUDA(cudaEventRecord(c.ev_snap_src, c.stream));
  ST_CUDA(cudaStreamWaitEvent(c.copy_stream, c.ev_snap_src, 0));
  ST_CUDA(cudaMemcpyAsync(host_T, c.snap_T.p, c.nv * sizeof(double), cudaMemcpyDeviceToHost,
                          c.copy_stream));
  if (rc_dev)
    ST_CUDA(cudaMemcpyAsync(host_rc, c.snap_rc.p, nrc * sizeof(double), cudaMemcpyDeviceToHost,
                            c.copy_stream));
  if (want_rc && c.rc_uniform)
    for (int64_t i = 0; i < nrc; i++) host_rc[i] = c.rc_value;
  ST_CUDA(cudaEventRecord(c.ev_snap_done, c.copy_stream));
  c.snap_busy = 1;
  return ST_OK;
}

// 1 when the last snapshot has reached the host (wait != 0: block until it
// has), 0 while it is in flight
int st_snapshot_wait(st_ctx* ctx, int wait) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!c.snap_busy) return 1;
  if (wait) {
    ST_CUDA(cudaEventSynchronize(c.ev_snap_done));
  } else {
    const cudaError_t e = cudaEventQuery(c.ev_snap_done);
    if (e == cudaErrorNotReady) return 0;
    ST_CUDA(e);
  }
  c.snap_busy = 0;
  return 1;
}

double* st_field_device_ptr(st_ctx* ctx, int field) {
  if (!ctx) return nullptr;
  Ctx& c = ctx->impl;
  if (flush_history(c) != ST_OK) return nullptr;
  if (field == ST_FIELD_T) return c.T.p;
  if (field == ST_FIELD_RC) return c.rc_uniform ? nullptr : c.rc.p;
  return nullptr;
}

int st_evaluate_rhs(st_ctx* ctx, const double* T, const double* rc, int flags, double frozen_k,
                    const st_beam* beams, int n_beams, double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if ((flags & ST_RHS_DIFFUSION) && !(flags & ST_RHS_FROZEN_K) && !rc && !c.be->uniform_rc_ok()) {
    set_error("evaluate_rhs needs r_c unless the conductivity is frozen");
    return ST_EINVAL;
  }
  double *Td, *fd, *rcd;
  ST_TRY(c.vec(0, &Td));
  ST_TRY(c.vec(1, &fd));
  ST_TRY(c.h2d(Td, T, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  int nb = (beams && (flags & ST_RHS_SOURCE)) ? n_beams : 0;
  ST_TRY(c.upload_beams(beams, nb));
  ST_TRY(c.be->rhs(Td, rcd, flags, frozen_k, nb, c.beams.p, fd, 0));
  return c.d2h(out, fd, c.nv);
}

int st_lumped_capacity(st_ctx* ctx, const double* T, double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *Td = nullptr, *od;
  if (T && c.dp.latent) {
    ST_TRY(c.vec(0, &Td));
    ST_TRY(c.h2d(Td, T, c.nv));
  }
  ST_TRY(c.vec(1, &od));
  ST_TRY(c.be->capacity(Td, od));
  return c.d2h(out, od, c.nv);
}

int st_apply_mass(st_ctx* ctx, const double* v, double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *vd, *od;
  ST_TRY(c.vec(0, &vd));
  ST_TRY(c.vec(1, &od));
  ST_TRY(c.h2d(vd, v, c.nv));
  ST_TRY(c.be->mass(vd, od));
  return c.d2h(out, od, c.nv);
}

int st_explicit_step(st_ctx* ctx, const double* T, double dt, const double* rc,
                     const st_beam* beams, int n_beams, double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!rc && !c.be->uniform_rc_ok()) {
    set_error("explicit step needs r_c");
    return ST_EINVAL;
  }
  double *Td, *od, *rcd;
  ST_TRY(c.vec(0, &Td));
  ST_TRY(c.vec(1, &od));
  ST_TRY(c.h2d(Td, T, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  int nb = beams ? n_beams : 0;
  ST_TRY(c.upload_beams(beams, nb));
  ST_CUDA(cudaMemsetAsync(c.red.p + kRedBlocks + 64, 0, 2 * sizeof(double), c.stream));
  ST_TRY(c.be->explicit_step(Td, rcd, dt, nb, c.beams.p, od, 0, c.red.p + kRedBlocks + 64));
  return c.d2h(out, od, c.nv);
}

int st_update_history(st_ctx* ctx, const double* T, double* rc) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *Td, *rcd;
  ST_TRY(c.vec(0, &Td));
  ST_TRY(c.h2d(Td, T, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  ST_TRY(c.be->history(Td, rcd));
  return c.d2h(rc, rcd, c.n_cells * c.qpc);
}

int st_apply_jacobian(st_ctx* ctx, const double* v, const double* T_lin, const double* rc,
                      double dt, double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *vd, *Td, *od, *rcd;
  ST_TRY(c.vec(0, &Td));
  ST_TRY(c.vec(6, &vd));
  ST_TRY(c.vec(7, &od));
  ST_TRY(c.h2d(Td, T_lin, c.nv));
  ST_TRY(c.h2d(vd, v, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  ST_TRY(c.be->jacobian(vd, Td, rcd, dt, od));
  return c.d2h(out, od, c.nv);
}

int st_jacobian_diagonal(st_ctx* ctx, const double* T_lin, const double* rc, double dt,
                         double* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *Td, *od, *rcd;
  ST_TRY(c.vec(0, &Td));
  ST_TRY(c.vec(1, &od));
  ST_TRY(c.h2d(Td, T_lin, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  ST_TRY(c.be->jac_diag(Td, rcd, dt, od));
  return c.d2h(out, od, c.nv);
}

int st_pcg(st_ctx* ctx, const double* T_lin, const double* rc, double dt, const double* b,
           double tol, int max_iter, int precond, const double* diag_inv, double* x, int* iters,
           int* converged) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  double *Td, *bd, *xd, *di = nullptr, *rcd;
  ST_TRY(c.vec(0, &Td));
  // b has a slot of its own (the Jacobian apply uses slot 5 for its input)
  ST_TRY(c.vec(8, &bd));
  ST_TRY(c.vec(6, &xd));
  ST_TRY(c.h2d(Td, T_lin, c.nv));
  ST_TRY(c.h2d(bd, b, c.nv));
  ST_TRY(stage_rc(c, rc, &rcd));
  if (precond) {
    ST_TRY(c.vec(7, &di));
    if (diag_inv) {  // the caller's preconditioner, as krylov_solve applies it
      ST_TRY(c.h2d(di, diag_inv, c.nv));
    } else {  // the exact Jacobian diagonal, inverted
      ST_TRY(c.be->jac_diag(Td, rcd, dt, di));
      ST_TRY(vec_recip(&c, di, di, c.nv));
    }
  }
  ST_TRY(pcg_dev(c, Td, rcd, dt, bd, tol, max_iter, di, xd, iters, converged));
  return c.d2h(x, xd, c.nv);
}

// estimate_spectral_radius over the step-criteria apply (timestepping.py:49-99),
// all vectors and scalars on the device.  The iterations run in batches
// without a host round-trip: each records its (w.w, v.w) pair in a device
// history and normalises v by the device ||w||; the host then applies the
// reference's stopping rule to the history in order.  Iterations queued
// past the stopping one only touch scratch vectors, so the result is the
// one-iteration-at-a-time result (same kernels, same sqrt and division).
// Iterations 2.. replay a captured graph of one iteration (ST_PW_GRAPH=0
// launches directly).
int st_spectral_radius(st_ctx* ctx, double k_frozen, const double* v0, double tol, int max_iter,
                       double* rho, int* iters) {
  NvtxScope nvtx_scope("st_spectral_radius");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!v0 || !rho || !iters || max_iter < 0) {
    set_error("spectral_radius: null argument or negative max_iter");
    return ST_EINVAL;
  }
  const int64_t nv = c.nv;
  double *v, *vd, *f, *w, *cinv;
  ST_TRY(c.vec(0, &v));
  ST_TRY(c.vec(1, &vd));
  ST_TRY(c.vec(2, &f));
  ST_TRY(c.vec(3, &w));
  ST_TRY(c.vec(4, &cinv));
  ST_TRY(c.h2d(v, v0, nv));
  ST_TRY(c.be->capacity(nullptr, cinv));
  ST_TRY(vec_recip(&c, cinv, cinv, nv));
  *rho = 0.0;
  *iters = 0;
  if (max_iter == 0) return c.sync();
  constexpr int kMaxBatch = 64;
  if ((int64_t)c.cgs.n < kCgsSize) ST_TRY(c.cgs.alloc(kCgsSize));
  if ((int64_t)c.pws.n < 4 + 2 * kMaxBatch) ST_TRY(c.pws.alloc(4 + 2 * kMaxBatch));
  double* part = c.cgs.p;
  double* pws = c.pws.p;
  auto body = [&]() -> int {
    // vd = v by a kernel (1.0 * x is exact), not a copy node: the
    // iteration's kernels are chained with programmatic dependent launch
    ST_TRY(vec_scal_copy(&c, 1.0, v, vd, nv));
    ST_TRY(c.be->distribute(vd));
    ST_TRY(c.be->pin_dirichlet(vd, 0.0));
    ST_TRY(c.be->rhs(vd, nullptr, ST_RHS_DIFFUSION | ST_RHS_FROZEN_K, k_frozen, 0, nullptr, f,
                     0));
    ST_TRY(vec_neg_mul(&c, f, cinv, w, nv));
    ST_TRY(c.be->mask_rows(w));
    ST_TRY(dot_to_device(&c, w, w, nv, part, pws + 1));
    ST_TRY(dot_to_device(&c, v, w, nv, part, pws + 2));
    ST_TRY(pw_record(&c, pws));
    ST_TRY(pw_div(&c, w, pws, v, nv));
    return ST_OK;
  };
  static const bool use_graph = !(getenv("ST_PW_GRAPH") && getenv("ST_PW_GRAPH")[0] == '0');
  bool graph = false;
  int64_t graph_kernels = 0;
  std::vector<double> hist(2 * kMaxBatch);
  double lam_prev = 0.0, lam = 0.0;
  int done = 0, batch = 4;
  while (done < max_iter) {
    const int nb_ = std::min(batch, max_iter - done);
    ST_CUDA(cudaMemsetAsync(pws, 0, sizeof(double), c.stream));
    for (int i = 0; i < nb_; i++) {
      if (graph) {
        ST_CUDA(cudaGraphLaunch(c.pw_exec, c.stream));
        c.launches += graph_kernels;
      } else {
        ST_TRY(body());
      }
    }
    if (use_graph && !graph && nb_ < max_iter - done) {
      // the first batch ran directly (lazy allocations are done); capture
      cudaGraph_t g = nullptr;
      const int64_t l0 = c.launches;
      ST_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      const int brc = body();
      const cudaError_t e = cudaStreamEndCapture(c.stream, &g);
      graph_kernels = c.launches - l0;
      c.launches = l0;
      if (brc != ST_OK || e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        if (brc != ST_OK) return brc;
        ST_CUDA(e);
      }
      if (c.pw_exec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(c.pw_exec, g, &info) != cudaSuccess) {
          cudaGetLastError();
          cudaGraphExecDestroy(c.pw_exec);
          c.pw_exec = nullptr;
        }
      }
      const cudaError_t ie = c.pw_exec ? cudaSuccess : cudaGraphInstantiate(&c.pw_exec, g, 0);
      cudaGraphDestroy(g);
      ST_CUDA(ie);
      graph = true;
    }
    ST_CUDA(cudaMemcpyAsync(hist.data(), pws + 4, 2 * nb_ * sizeof(double),
                            cudaMemcpyDeviceToHost, c.stream));
    ST_CUDA(cudaStreamSynchronize(c.stream));
    for (int i = 0; i < nb_; i++) {
      *iters = done + i + 1;
      const double nw = std::sqrt(hist[2 * i]);
      if (nw == 0.0) return ST_OK;
      lam_prev = lam;
      lam = hist[2 * i + 1];
      if (std::fabs(lam - lam_prev) <= tol * std::fabs(lam)) {
        *rho = std::max(std::fabs(lam), std::fabs(lam_prev));
        return ST_OK;
      }
    }
    done += nb_;
    batch = std::min(2 * batch, kMaxBatch);
  }
  *rho = std::max(std::fabs(lam), std::fabs(lam_prev));
  return ST_OK;
}

// ---------------------------------------------------------------------------
// device-resident explicit loop (run_scan_phase, timestepping.py:195-226)
// ---------------------------------------------------------------------------
static const double kDiverged = 1.0e7;  // timestepping.py:183

static int explicit_steps_resident(Ctx& c, int n_steps, const double* dts, int nb,
                                   int* fail_step, double* t_extreme, double* t_max);

int st_explicit_steps(st_ctx* ctx, int n_steps, const double* dts, const st_beam* beams,
                      int n_beams, int* fail_step, double* t_extreme, double* t_max) {
  NvtxScope nvtx_scope("st_explicit_steps");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  if (fail_step) *fail_step = 0;
  if (n_steps <= 0) return ST_OK;
  const int nb = beams ? n_beams : 0;
  ST_TRY(c.upload_beams(beams, (int64_t)n_steps * nb));
  return explicit_steps_resident(c, n_steps, dts, nb, fail_step, t_extreme, t_max);
}

// ---------------------------------------------------------------------------
// device beam schedule (physics.py:135-151 layer_beam_state at tau = (step-1)
// dt for every step of a scan phase, several concurrently scanned paths):
// one thread per (step, path); closed segment windows, first match, the
// reference's float expressions with explicit roundings (no FMA), so the
// records equal the host expansion (flatten_schedule) bit for bit.
// ---------------------------------------------------------------------------
struct SegDev {
  double x0, y0, x1, y1, v, power, length, duration, t_start;
};

__global__ void k_beam_schedule(const SegDev* __restrict__ segs, const int* __restrict__ seg_off,
                                const double* __restrict__ z_top, int n_paths, int step0,
                                int n_steps, double dt, double denom, st_beam* recs,
                                DevBeam* dev) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_steps * n_paths) return;
  const int i = (int)(t / n_paths), k = (int)(t - (int64_t)i * n_paths);
  const double tau = __dmul_rn((double)(step0 + i - 1), dt);
  st_beam r;
  r.x = 0.0;
  r.y = 0.0;
  r.z_top = z_top[k];
  r.power = 0.0;
  r.active = 0;
  r._pad = 0;
  for (int sg = seg_off[k]; sg < seg_off[k + 1]; sg++) {
    const SegDev g = segs[sg];
    if (g.t_start <= tau && tau <= __dadd_rn(g.t_start, g.duration)) {
      const double sv = __dmul_rn(__dsub_rn(tau, g.t_start), g.v);
      const double frac = g.length > 0.0 ? __ddiv_rn(sv, g.length) : 0.0;
      r.x = __dadd_rn(g.x0, __dmul_rn(frac, __dsub_rn(g.x1, g.x0)));
      r.y = __dadd_rn(g.y0, __dmul_rn(frac, __dsub_rn(g.y1, g.y0)));
      r.power = g.power;
      r.active = g.power > 0.0 ? 1 : 0;
      break;
    }
  }
  if (recs) recs[t] = r;
  if (dev) {
    DevBeam b;
    b.x = r.x;
    b.y = r.y;
    b.z_top = r.z_top;
    b.peak = r.active ? __ddiv_rn(__dmul_rn(2.0, r.power), denom) : 0.0;
    dev[t] = b;
  }
}

static int beam_schedule(Ctx& c, int n_steps, int step0, double dt, int n_paths,
                         const int32_t* seg_count, const st_segment* segs, const double* z_top,
                         st_beam* recs_dev) {
  if (n_paths < 0 || (n_paths > 0 && (!seg_count || !z_top))) {
    set_error("beam schedule: invalid paths");
    return ST_EINVAL;
  }
  std::vector<int> off(n_paths + 1, 0);
  for (int k = 0; k < n_paths; k++) off[k + 1] = off[k] + seg_count[k];
  std::vector<SegDev> hs(std::max(off[n_paths], 1));
  for (int q = 0; q < off[n_paths]; q++) {
    const st_segment& g = segs[q];
    hs[q] = SegDev{g.x0, g.y0, g.x1, g.y1, g.v, g.power, g.length, g.duration, g.t_start};
  }
  DevBuf<SegDev> dsegs;
  DevBuf<int> doff;
  DevBuf<double> dz;
  ST_TRY(dsegs.upload(hs.data(), hs.size(), c.stream));
  ST_TRY(doff.upload(off.data(), off.size(), c.stream));
  ST_TRY(dz.upload(z_top, std::max(n_paths, 1), c.stream));
  const int64_t n = (int64_t)n_steps * n_paths;
  if (!recs_dev && (int64_t)c.beams.n < n) ST_TRY(c.beams.alloc(n));
  const double R = c.params.las.radius, hp = c.params.las.h_powder;
  const double denom = M_PI * R * R * hp;
  if (n > 0) {
    k_beam_schedule<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(
        dsegs.p, doff.p, dz.p, n_paths, step0, n_steps, dt, denom, recs_dev,
        recs_dev ? nullptr : c.beams.p);
    ST_LAUNCHED();
    c.launches++;
  }
  // the staging buffers die here
  ST_CUDA(cudaStreamSynchronize(c.stream));
  return ST_OK;
}

int st_beam_schedule(st_ctx* ctx, int n_steps, int step0, double dt, int n_paths,
                     const int32_t* seg_count, const st_segment* segs, const double* z_top,
                     st_beam* out) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!out || n_steps < 0) {
    set_error("st_beam_schedule: invalid arguments");
    return ST_EINVAL;
  }
  const int64_t n = (int64_t)n_steps * n_paths;
  DevBuf<st_beam> recs;
  ST_TRY(recs.alloc(std::max<int64_t>(n, 1)));
  ST_TRY(beam_schedule(c, n_steps, step0, dt, n_paths, seg_count, segs, z_top, recs.p));
  if (n) ST_CUDA(cudaMemcpyAsync(out, recs.p, n * sizeof(st_beam), cudaMemcpyDeviceToHost, c.stream));
  ST_CUDA(cudaStreamSynchronize(c.stream));
  return ST_OK;
}

int st_scan_layer(st_ctx* ctx, int n_steps, int step0, double dt, double duration, int n_paths,
                  const int32_t* seg_count, const st_segment* segs, const double* z_top,
                  int* fail_step, double* t_extreme, double* t_max) {
  NvtxScope nvtx_scope("st_scan_layer");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  if (fail_step) *fail_step = 0;
  if (n_steps <= 0) return ST_OK;
  // the step sizes on the host (the last step is clipped to the scan end,
  // timestepping.py:210-213): dt = min(dt, duration - tau)
  std::vector<double> dts(n_steps);
  for (int i = 0; i < n_steps; i++) {
    const double tau = (double)(step0 + i - 1) * dt;
    dts[i] = std::min(dt, duration - tau);
  }
  ST_TRY(beam_schedule(c, n_steps, step0, dt, n_paths, seg_count, segs, z_top, nullptr));
  return explicit_steps_resident(c, n_steps, dts.data(), n_paths, fail_step, t_extreme, t_max);
}

// the step loop over beams already resident in c.beams (nb per step)
static int explicit_steps_resident(Ctx& c, int n_steps, const double* dts, int nb,
                                   int* fail_step, double* t_extreme, double* t_max) {
  if (fail_step) *fail_step = 0;
  if ((int64_t)c.T_alt.n < c.nv) ST_TRY(c.T_alt.alloc(c.nv));
  const int64_t nrc = c.rc_uniform ? 0 : c.n_cells * c.qpc;
  const int kBatch = 512;
  double tmax_all = -INFINITY;
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(c.red.p + kRedBlocks + 64);
  std::vector<unsigned long long> hs(2 * kBatch);
  for (int b0 = 0; b0 < n_steps; b0 += kBatch) {
    const int nbatch = std::min(kBatch, n_steps - b0);
    // snapshot so that a divergence leaves the state at the failing step
    if ((int64_t)c.T_snap.n < c.nv) ST_TRY(c.T_snap.alloc(c.nv));
    ST_CUDA(cudaMemcpyAsync(c.T_snap.p, c.T.p, c.nv * sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
    if (nrc) {
      if ((int64_t)c.rc_snap.n < nrc) ST_TRY(c.rc_snap.alloc(nrc));
      ST_CUDA(cudaMemcpyAsync(c.rc_snap.p, c.rc.p, nrc * sizeof(double),
                              cudaMemcpyDeviceToDevice, c.stream));
    }
    const int pending0 = c.history_pending;
    ST_CUDA(cudaMemsetAsync(slots, 0, 2 * nbatch * sizeof(unsigned long long), c.stream));
    // the whole batch as one persistent launch where the backend has one
    // (unstructured; ST_SCAN_PERSISTENT=0 turns it off), else step by step
    const int prc = c.be->explicit_steps_persistent(c.T.p, c.T_alt.p, rc_ptr(c), dts + b0,
                                                    nbatch, nb, c.beams.p + (int64_t)b0 * nb,
                                                    c.history_pending, slots);
    if (prc == ST_OK) {
      if (nbatch & 1) {
        std::swap(c.T.p, c.T_alt.p);
        std::swap(c.T.n, c.T_alt.n);
      }
      c.history_pending = 1;
    } else if (prc != ST_EUNSUPPORTED) {
      return prc;
    } else {
      for (int i = 0; i < nbatch; i++) {
        const int s = b0 + i;
        ST_TRY(c.be->explicit_step(c.T.p, rc_ptr(c), dts[s], nb, c.beams.p + (int64_t)s * nb,
                                   c.T_alt.p, c.history_pending,
                                   reinterpret_cast<double*>(slots + 2 * i)));
        std::swap(c.T.p, c.T_alt.p);
        std::swap(c.T.n, c.T_alt.n);
        c.history_pending = 1;
      }
    }
    ST_CUDA(cudaMemcpyAsync(hs.data(), slots, 2 * nbatch * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c.stream));
    ST_CUDA(cudaStreamSynchronize(c.stream));
    for (int i = 0; i < nbatch; i++) {
      double am;
      std::memcpy(&am, &hs[2 * i], 8);
      double sm = key_to_double(hs[2 * i + 1]);
      if (!std::isfinite(am) || am > kDiverged) {
        // replay the batch up to the failing step; its history update is
        // never applied (the reference raises before update_history)
        ST_CUDA(cudaMemcpyAsync(c.T.p, c.T_snap.p, c.nv * sizeof(double),
                                cudaMemcpyDeviceToDevice, c.stream));
        if (nrc)
          ST_CUDA(cudaMemcpyAsync(c.rc.p, c.rc_snap.p, nrc * sizeof(double),
                                  cudaMemcpyDeviceToDevice, c.stream));
        c.history_pending = pending0;
        for (int j = 0; j <= i; j++) {
          const int s = b0 + j;
          ST_TRY(c.be->explicit_step(c.T.p, rc_ptr(c), dts[s], nb, c.beams.p + (int64_t)s * nb,
                                     c.T_alt.p, c.history_pending,
                                     reinterpret_cast<double*>(slots)));
          std::swap(c.T.p, c.T_alt.p);
          std::swap(c.T.n, c.T_alt.n);
          c.history_pending = 1;
        }
        c.history_pending = 0;
        ST_TRY(c.sync());
        if (fail_step) *fail_step = b0 + i + 1;
        if (t_extreme) *t_extreme = am;
        if (t_max) *t_max = tmax_all;
        return ST_OK;
      }
      tmax_all = std::max(tmax_all, sm);
    }
  }
  if (t_max) *t_max = tmax_all;
  return ST_OK;
}

// ---------------------------------------------------------------------------
// backward Euler (timestepping.py:229-283, 355-362)
// ---------------------------------------------------------------------------
int st_implicit_step(st_ctx* ctx, double dt, double newton_tol, double newton_abs_tol,
                     int newton_max_iter, double krylov_tol, int krylov_max_iter, int precond,
                     int* newton_iters, int* krylov_iters, int* converged) {
  NvtxScope nvtx_scope("st_implicit_step");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  ST_TRY(flush_history(c));
  const int64_t nv = c.nv;
  static_assert(sizeof(DevBuf<double>) > 0, "");
  // the step's vectors live in the context (allocated once: a cudaMalloc /
  // cudaFree pair per vector and step cost more than the step itself at
  // cool-down mesh sizes)
  for (auto& v : c.imp)
    if ((int64_t)v.n < nv) ST_TRY(v.alloc(nv));
  DevBuf<double>&Tn = c.imp[0], &Ti = c.imp[1], &fre = c.imp[2], &f = c.imp[3], &r = c.imp[4],
                 &tmp = c.imp[5], &di = c.imp[6], &delta = c.imp[7];
  double* rc = rc_ptr(c);
  ST_CUDA(cudaMemcpyAsync(Tn.p, c.T.p, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ST_CUDA(cudaMemcpyAsync(Ti.p, c.T.p, nv * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  // boundary flux frozen at the step start
  ST_TRY(c.be->rhs(Tn.p, rc, ST_RHS_FACES, 0.0, 0, nullptr, fre.p, 0));
  double norm0 = -1.0;
  int nn = 0, nk = 0;
  *converged = 0;
  for (int k = 0; k < newton_max_iter; k++) {
    ST_TRY(c.be->rhs(Ti.p, rc, ST_RHS_DIFFUSION, 0.0, 0, nullptr, f.p, 0));
    ST_TRY(vec_sub(&c, Ti.p, Tn.p, tmp.p, nv));
    double* Md;
    ST_TRY(c.vec(0, &Md));
    ST_TRY(c.be->mass(tmp.p, Md));
    ST_TRY(vec_sub_scale(&c, Md, f.p, dt, fre.p, r.p, nv));
    ST_TRY(c.be->mask_rows(r.p));
    double rr;
    ST_TRY(c.dot(r.p, r.p, nv, &rr));
    double norm = std::sqrt(rr);
    if (norm0 < 0) norm0 = norm;
    if (norm <= newton_abs_tol || norm <= newton_tol * norm0) {
      ST_CUDA(cudaMemcpyAsync(c.T.p, Ti.p, nv * sizeof(double), cudaMemcpyDeviceToDevice,
                              c.stream));
      ST_TRY(c.sync());
      *newton_iters = nn;
      *krylov_iters = nk;
      *converged = 1;
      return ST_OK;
    }
    double* dip = nullptr;
    if (precond) {
      ST_TRY(c.be->jac_diag(Ti.p, rc, dt, di.p));
      ST_TRY(vec_recip(&c, di.p, di.p, nv));
      dip = di.p;
    }
    ST_TRY(vec_scal_copy(&c, -1.0, r.p, r.p, nv));
    int it = 0, ok = 0;
    ST_TRY(pcg_dev(c, Ti.p, rc, dt, r.p, krylov_tol, krylov_max_iter, dip, delta.p, &it, &ok));
    nk += it;
    if (!ok) break;
    ST_TRY(vec_axpy(&c, 1.0, delta.p, Ti.p, nv));
    ST_TRY(c.be->distribute(Ti.p));
    nn++;
  }
  ST_TRY(c.sync());
  *newton_iters = nn;
  *krylov_iters = nk;
  *converged = 0;
  return ST_OK;
}

int st_finish_implicit_step(st_ctx* ctx) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(c.be->pin_dirichlet(c.T.p, c.dp.T_inf));
  ST_TRY(c.be->history(c.T.p, rc_ptr(c)));
  c.history_pending = 0;
  return c.sync();
}

// ---------------------------------------------------------------------------
// measurement
// ---------------------------------------------------------------------------
int st_profile_enable(st_ctx* ctx, int enable) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  c.prof = enable ? 1 : 0;
  c.prof_ms = 0.0;
  c.prof_launches = 0;
  return ST_OK;
}

int st_profile_read(st_ctx* ctx, double* main_ms, int64_t* main_launches, char* main_name,
                    int name_len) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(c.sync());
  if (main_ms) *main_ms = c.prof_ms;
  if (main_launches) *main_launches = c.prof_launches;
  if (main_name && name_len > 0) {
    std::strncpy(main_name, c.be->main_kernel(), name_len - 1);
    main_name[name_len - 1] = 0;
  }
  return ST_OK;
}

double st_algorithmic_bytes_per_dof(const st_ctx* ctx) {
  if (!ctx || !ctx->impl.be) return 0.0;
  return ctx->impl.be->bytes_per_dof();
}

// ---------------------------------------------------------------------------
// multi-GPU slab step
// ---------------------------------------------------------------------------
// per-step stability maxima of split steps: a ring of kSplitRing slot pairs
static int split_slot(Ctx& c, unsigned long long** out) {
  if (!c.split_ring.p) {
    ST_TRY(c.split_ring.alloc(2 * kSplitRing));
    ST_CUDA(cudaMemsetAsync(c.split_ring.p, 0, 2 * kSplitRing * sizeof(double), c.stream));
  }
  *out = reinterpret_cast<unsigned long long*>(c.split_ring.p) + 2 * (c.split_count % kSplitRing);
  return ST_OK;
}

int st_explicit_step_begin(st_ctx* ctx, double dt, const st_beam* beams, int n_beams) {
  NvtxScope nvtx_scope("st_explicit_step_begin");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  if (c.split_count - c.split_read >= kSplitRing) {
    set_error("st_step_maxima / st_step_maxima_history must be read at least every " +
              std::to_string(kSplitRing) + " split steps");
    return ST_EINVAL;
  }
  const int nb = beams ? n_beams : 0;
  ST_TRY(c.upload_beams(beams, nb));
  if ((int64_t)c.T_alt.n < c.nv) ST_TRY(c.T_alt.alloc(c.nv));
  unsigned long long* slot;
  ST_TRY(split_slot(c, &slot));
  ST_CUDA(cudaMemsetAsync(slot, 0, 2 * sizeof(unsigned long long), c.stream));
  return c.be->step_begin(c.T.p, rc_ptr(c), dt, nb, c.beams.p, c.T_alt.p, c.history_pending,
                          reinterpret_cast<double*>(slot));
}

int st_iface_partials(st_ctx* ctx, int side, double** f_plane, double** c_plane, int64_t* n) {
  ST_TRY(check_ctx(ctx));
  return ctx->impl.be->iface_ptrs(side, f_plane, c_plane, n);
}

int st_iface_wait(st_ctx* ctx, void* stream) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  if (!c.ev_iface) {
    set_error("st_iface_wait before st_explicit_step_begin");
    return ST_EINVAL;
  }
  ST_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, c.ev_iface, 0));
  return ST_OK;
}

int st_explicit_step_end(st_ctx* ctx, const double* recv_lo_f, const double* recv_lo_c,
                         const double* recv_hi_f, const double* recv_hi_c) {
  NvtxScope nvtx_scope("st_explicit_step_end");
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(c.be->step_end(recv_lo_f, recv_lo_c, recv_hi_f, recv_hi_c));
  std::swap(c.T.p, c.T_alt.p);
  std::swap(c.T.n, c.T_alt.n);
  c.history_pending = 1;
  c.split_count++;
  return ST_OK;
}

int st_step_maxima_history(st_ctx* ctx, int n, double* absmax, double* tmax) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  const int64_t avail = c.split_count - c.split_read;
  if (n < 0 || n > avail) {
    set_error("st_step_maxima_history: " + std::to_string(avail) + " unread steps");
    return ST_EINVAL;
  }
  if (n == 0 || !c.split_ring.p) return ST_OK;
  std::vector<unsigned long long> h(2 * kSplitRing);
  ST_CUDA(cudaMemcpyAsync(h.data(), c.split_ring.p, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
  ST_CUDA(cudaStreamSynchronize(c.stream));
  // the oldest n unread steps, in step order
  for (int i = 0; i < n; i++) {
    const int64_t s = c.split_read + i;
    const unsigned long long* e = h.data() + 2 * (s % kSplitRing);
    double am;
    std::memcpy(&am, &e[0], 8);
    if (absmax) absmax[i] = am;
    if (tmax) tmax[i] = key_to_double(e[1]);
  }
  c.split_read += n;
  return ST_OK;
}

int st_step_maxima(st_ctx* ctx, double* absmax, double* tmax) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  const int n = (int)(c.split_count - c.split_read);
  std::vector<double> a(n), t(n);
  ST_TRY(st_step_maxima_history(ctx, n, a.data(), t.data()));
  double am = 0.0, tm = -INFINITY;
  bool bad = false;
  for (int i = 0; i < n; i++) {
    bad |= !(a[i] == a[i]);
    am = std::max(am, a[i]);
    tm = std::max(tm, t[i]);
  }
  if (absmax) *absmax = bad ? NAN : am;
  if (tmax) *tmax = tm;
  return ST_OK;
}

// reads n bytes (16-byte vectors); the store is never taken but keeps the
// loads alive.  Used after the flush write so the flush's dirty lines are
// written back before the timed step, not during it.
__global__ void k_read_sweep(const double2* __restrict__ p, int64_t n2, double2* sink) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = p[i];
    acc += v.x + v.y;
  }
  if (acc == -1.0) sink[0] = make_double2(acc, acc);
}

int st_bench_explicit(st_ctx* ctx, int n_steps, const double* dts, const st_beam* beams,
                      int n_beams, int64_t flush_bytes, float* step_ms, float* main_ms) {
  ST_TRY(check_ctx(ctx));
  Ctx& c = ctx->impl;
  ST_TRY(need_state(c));
  if (n_steps <= 0) return ST_OK;
  const int nb = beams ? n_beams : 0;
  ST_TRY(c.upload_beams(beams, (int64_t)n_steps * nb));
  if ((int64_t)c.T_alt.n < c.nv) ST_TRY(c.T_alt.alloc(c.nv));
  DevBuf<char> flush, sweep;
  if (flush_bytes > 0) {
    ST_TRY(flush.alloc(flush_bytes));
    ST_TRY(sweep.alloc(flush_bytes));
    ST_CUDA(cudaMemsetAsync(sweep.p, 0, flush_bytes, c.stream));
  }
  std::vector<cudaEvent_t> ev(4 * (size_t)n_steps);
  for (auto& e : ev) ST_CUDA(cudaEventCreate(&e));
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(c.red.p + kRedBlocks + 64);
  int rc = ST_OK;
  for (int s = 0; s < n_steps && rc == ST_OK; s++) {
    if (flush_bytes > 0) {
      // alternate the fill byte so the writes cannot be elided
      if (cudaMemsetAsync(flush.p, s & 0xff, flush_bytes, c.stream) != cudaSuccess) {
        set_error("flush memset failed");
        rc = ST_ECUDA;
        break;
      }
      // then read another buffer of the same size: L2 holds only clean
      // lines of it when the timed step starts
      k_read_sweep<<<148 * 8, 256, 0, c.stream>>>(reinterpret_cast<const double2*>(sweep.p),
                                                  flush_bytes / 16,
                                                  reinterpret_cast<double2*>(flush.p));
    }
    cudaMemsetAsync(slots, 0, 2 * sizeof(unsigned long long), c.stream);
    cudaEventRecord(ev[4 * s], c.stream);
    c.bench_ev0 = &ev[4 * s + 1];
    c.bench_ev1 = &ev[4 * s + 2];
    rc = c.be->explicit_step(c.T.p, rc_ptr(c), dts[s], nb, c.beams.p + (int64_t)s * nb,
                             c.T_alt.p, c.history_pending, reinterpret_cast<double*>(slots));
    c.bench_ev0 = c.bench_ev1 = nullptr;
    cudaEventRecord(ev[4 * s + 3], c.stream);
    std::swap(c.T.p, c.T_alt.p);
    std::swap(c.T.n, c.T_alt.n);
    c.history_pending = 1;
  }
  if (rc == ST_OK) {
    ST_CUDA(cudaStreamSynchronize(c.stream));
    for (int s = 0; s < n_steps; s++) {
      float ms = 0.f;
      ST_CUDA(cudaEventElapsedTime(&ms, ev[4 * s], ev[4 * s + 3]));
      step_ms[s] = ms;
      if (main_ms) {
        ST_CUDA(cudaEventElapsedTime(&ms, ev[4 * s + 1], ev[4 * s + 2]));
        main_ms[s] = ms;
      }
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

}  // extern "C"
