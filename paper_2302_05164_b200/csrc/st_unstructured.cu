// Q1 operator on arbitrary (adaptive, hanging-node) meshes.
//
// Restates reference operators.py for general DofMap tables:
//   cell kernels  : one thread per active cell, 2x2x2 sum factorisation
//                   in registers (operators.py:44-55, 247-316, 341-424)
//   node kernels  : one thread per vertex; deterministic gather of the
//                   per-cell element vectors through a vertex incidence
//                   CSR in canonical cell order (= np.bincount order,
//                   operators.py:229-237), hanging-node condensation in
//                   np.add.at order (mesh.py:663-670), then the fused
//                   forward-Euler update + Dirichlet pin (operators.py:
//                   352-369); slaves are re-interpolated afterwards
//                   (mesh.py:652-661).
// An atomic-scatter variant (SolverSettings.deterministic = False, the
// analogue of the reference's colored scatter) skips the element buffer.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <vector>

#include <cooperative_groups.h>

#include "st_common.cuh"

namespace cg = cooperative_groups;

namespace st {


__constant__ double cV[2][2];   // V1[i][q] (operators.py:33-34)
__constant__ double cD[2][2];   // D1
__constant__ double cU[2];      // (GAUSS_1D + 1) / 2
__constant__ double cPhi[8][8];      // PHI_REF[c][q]
__constant__ double cG[3][8][8];     // GRAD_REF[d][c][q]
__constant__ double cPhi2[8];        // sum_q PHI^2
__constant__ double cGG[8][8];       // sum_d GRAD[d][c][q]^2

template <int D>
__device__ __forceinline__ double M1(int i, int q) {
  return D ? cD[i][q] : cV[i][q];
}

// out[a,b,c] = sum_ijk A[i][a] B[j][b] C[k][c] in[i,j,k]; flat index x*4+y*2+z
template <int DX, int DY, int DZ>
__device__ __forceinline__ void interp(const double* t, double* o) {
  double s[8], r[8];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int jk = 0; jk < 4; jk++)
      s[a * 4 + jk] = fma(M1<DX>(1, a), t[4 + jk], M1<DX>(0, a) * t[jk]);
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++)
#pragma unroll
      for (int k = 0; k < 2; k++)
        r[a * 4 + b * 2 + k] = fma(M1<DY>(1, b), s[a * 4 + 2 + k], M1<DY>(0, b) * s[a * 4 + k]);
#pragma unroll
  for (int ab = 0; ab < 4; ab++)
#pragma unroll
    for (int c = 0; c < 2; c++)
      o[ab * 2 + c] = fma(M1<DZ>(1, c), r[ab * 2 + 1], M1<DZ>(0, c) * r[ab * 2]);
}

// transpose: out[i,j,k] = sum_abc A[i][a] B[j][b] C[k][c] in[a,b,c]
template <int DX, int DY, int DZ>
__device__ __forceinline__ void project(const double* t, double* o) {
  double s[8], r[8];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int bc = 0; bc < 4; bc++)
      s[i * 4 + bc] = fma(M1<DX>(i, 1), t[4 + bc], M1<DX>(i, 0) * t[bc]);
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int c = 0; c < 2; c++)
        r[i * 4 + j * 2 + c] = fma(M1<DY>(j, 1), s[i * 4 + 2 + c], M1<DY>(j, 0) * s[i * 4 + c]);
#pragma unroll
  for (int ij = 0; ij < 4; ij++)
#pragma unroll
    for (int k = 0; k < 2; k++)
      o[ij * 2 + k] = fma(M1<DZ>(k, 1), r[ij * 2 + 1], M1<DZ>(k, 0) * r[ij * 2]);
}

struct CellGeo {
  const int* cv;
  const double* h;
  const double* anc;
  const double* detw;
};

struct FaceTab {
  const int* ptr;  // per cell CSR (n+1)
  const double* vx;
  const double* vy;
  const double* area;
};

__device__ __forceinline__ void gather8(const int* cv, int64_t c, const double* X, double* t) {
#pragma unroll
  for (int i = 0; i < 8; i++) t[i] = X[cv[c * 8 + i]];
}

// dev hook (-DST_SCAN_TIMING): thread 0 of block 0 of the three scan kernels
// logs (kernel, entry, wait returned, exit) globaltimer stamps into a ring;
// the backend prints the mean phase and gap times when it is destroyed
#ifdef ST_SCAN_TIMING
__device__ unsigned long long st_scan_ring[4 * 8192];
__device__ unsigned st_scan_cnt;
__device__ __forceinline__ unsigned long long st_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ST_SCAN_T0() const unsigned long long ts_in_ = st_gtime();
#define ST_SCAN_T1() const unsigned long long ts_w_ = st_gtime();
#define ST_SCAN_T2(k)                                               \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                        \
    const unsigned s_ = atomicAdd(&st_scan_cnt, 1u) % 8192u;        \
    st_scan_ring[4 * s_] = (k);                                     \
    st_scan_ring[4 * s_ + 1] = ts_in_;                              \
    st_scan_ring[4 * s_ + 2] = ts_w_;                               \
    st_scan_ring[4 * s_ + 3] = st_gtime();                          \
  }
#else
#define ST_SCAN_T0()
#define ST_SCAN_T1()
#define ST_SCAN_T2(k)
#endif

// A/B hook (-DST_PDL_EARLY=1): the scan kernels release their successor
// before their own wait instead of after it, so that it is staged and
// prefetches its tables a kernel earlier.  Measured slower (20.97 against
// 16.76 us per step on the config-3 layer-0 mesh: kernels running ahead hold
// SM resources the running one's successor needs), so off.
#ifndef ST_PDL_EARLY
#define ST_PDL_EARLY 0
#endif
#if ST_PDL_EARLY
#define ST_PDL_EARLY_RELEASE() pdl_release()
#define ST_PDL_WAIT() pdl_wait()
#else
#define ST_PDL_EARLY_RELEASE()
#define ST_PDL_WAIT() pdl_wait_release()
#endif

// liquid_fraction (st_common.cuh) with the ramp's division only where a lane
// is inside the melting interval -- the same value for every input (NaN
// included); cold and fully molten cells skip the division's dependent
// instruction sequence (15 % of k_rhs_cells's stall samples after the
// prefetches)
__device__ __forceinline__ double liquid_fraction_br(const DevParams& P, double T) {
  double g = T > P.T_l ? 1.0 : 0.0;
  if (!(T < P.T_s) && !(T > P.T_l)) g = liquid_fraction(P, T);
  return g;
}

// What rhs_cell reads from the static tables (and the step's beam records,
// which are in place before the chain starts): k_rhs_cells loads it before
// the programmatic-launch wait, so that only the gather of T, the history
// and the arithmetic are left on the step's chain of dependent launches.
constexpr int kPreBeams = 4;
struct CellPre {
  int cv[8];
  int f0, f1;
  double h, detw, ax, ay, az;
  double vx[4], vy[4], area;  // the first facet of the cell
  // the cell's history (written by the previous step's cell kernel, which
  // has completed before this kernel can start; ncu had a third of this
  // kernel's stall samples on the wait for these loads, issued after the
  // gather of T had come back)
  double r[8];
  bool have_r;
};

__device__ __forceinline__ void cell_prefetch(int64_t c, const CellGeo& g, const FaceTab& ft,
                                              int flags, int nb, const DevBeam* beams,
                                              const double* rc, CellPre& p, DevBeam* bm) {
  p.have_r = rc && (flags & ST_RHS_DIFFUSION) && !(flags & ST_RHS_FROZEN_K);
  if (p.have_r) {
#pragma unroll
    for (int q = 0; q < 8; q++) p.r[q] = rc[c * 8 + q];
  }
#pragma unroll
  for (int i = 0; i < 8; i++) p.cv[i] = g.cv[c * 8 + i];
  p.h = g.h[c];
  p.detw = g.detw[c];
  p.ax = g.anc[c * 3];
  p.ay = g.anc[c * 3 + 1];
  p.az = g.anc[c * 3 + 2];
  p.f0 = p.f1 = 0;
  if ((flags & ST_RHS_FACES) && ft.ptr) {
    p.f0 = ft.ptr[c];
    p.f1 = ft.ptr[c + 1];
  }
#pragma unroll
  for (int b = 0; b < kPreBeams; b++)
    if ((flags & ST_RHS_SOURCE) && b < nb) bm[b] = beams[b];
  if (p.f1 > p.f0) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      p.vx[k] = ft.vx[p.f0 * 4 + k];
      p.vy[k] = ft.vy[p.f0 * 4 + k];
    }
    p.area = ft.area[p.f0];
  }
}

// ---------------------------------------------------------------------------
// rhs element vectors: -diffusion + faces + sources   (operators.py:247-316)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rhs_cell(int64_t c, const CellGeo& g, const FaceTab& ft,
                                         const DevParams& P, const double* __restrict__ T,
                                         double* rc, double rc_value, int flags, double frozen_k,
                                         int pending, int nb, const DevBeam* beams, double* E,
                                         double* Ec, double* f_atomic, double* c_atomic,
                                         const CellPre* pre = nullptr,
                                         const DevBeam* pbm = nullptr) {
  double t[8], e[8];
  if (pre) {  // vertex ids already loaded (k_rhs_cells)
#pragma unroll
    for (int i = 0; i < 8; i++) t[i] = T[pre->cv[i]];
  } else {
    gather8(g.cv, c, T, t);
  }
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] = 0.0;
  const double h = pre ? pre->h : g.h[c];
  double tq[8];
  bool need_tq = ((flags & ST_RHS_DIFFUSION) && !(flags & ST_RHS_FROZEN_K)) || Ec || c_atomic;
  if (need_tq) interp<0, 0, 0>(t, tq);
  if (flags & ST_RHS_DIFFUSION) {
    double k[8];
    if (flags & ST_RHS_FROZEN_K) {
#pragma unroll
      for (int q = 0; q < 8; q++) k[q] = frozen_k;
    } else {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        double r = rc ? ((pre && pre->have_r) ? pre->r[q] : rc[c * 8 + q]) : rc_value;
        double gq = liquid_fraction_br(P, tq[q]);
        if (pending && rc) {
          r = fmax(r, gq);
          rc[c * 8 + q] = r;
        }
        k[q] = conductivity(P, gq, r);
      }
    }
    const double hh = h / 2.0;
    double gd[8], pr[8];
    interp<1, 0, 0>(t, gd);
#pragma unroll
    for (int q = 0; q < 8; q++) gd[q] = (hh * k[q]) * gd[q];
    project<1, 0, 0>(gd, pr);
#pragma unroll
    for (int i = 0; i < 8; i++) e[i] -= pr[i];
    interp<0, 1, 0>(t, gd);
#pragma unroll
    for (int q = 0; q < 8; q++) gd[q] = (hh * k[q]) * gd[q];
    project<0, 1, 0>(gd, pr);
#pragma unroll
    for (int i = 0; i < 8; i++) e[i] -= pr[i];
    interp<0, 0, 1>(t, gd);
#pragma unroll
    for (int q = 0; q < 8; q++) gd[q] = (hh * k[q]) * gd[q];
    project<0, 0, 1>(gd, pr);
#pragma unroll
    for (int i = 0; i < 8; i++) e[i] -= pr[i];
  }
  if ((flags & ST_RHS_FACES) && ft.ptr) {
    const int f0 = pre ? pre->f0 : ft.ptr[c], f1 = pre ? pre->f1 : ft.ptr[c + 1];
    for (int fi = f0; fi < f1; fi++) {
      double vx[4], vy[4];  // [i][q]
      const bool have = pre && fi == f0;
#pragma unroll
      for (int k = 0; k < 4; k++) {
        vx[k] = have ? pre->vx[k] : ft.vx[fi * 4 + k];
        vy[k] = have ? pre->vy[k] : ft.vy[fi * 4 + k];
      }
      double tf[2][2], s[2][2], q[2][2];
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) tf[i][j] = t[i * 4 + j * 2 + 1];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int j = 0; j < 2; j++) s[a][j] = fma(vx[2 + a], tf[1][j], vx[a] * tf[0][j]);
      const double ar = -(have ? pre->area : ft.area[fi]);
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
          double tqf = fma(vy[2 + b], s[a][1], vy[b] * s[a][0]);
          q[a][b] = surface_flux(P, tqf) * ar;
        }
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int b = 0; b < 2; b++) s[i][b] = fma(vx[i * 2 + 1], q[1][b], vx[i * 2] * q[0][b]);
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) e[i * 4 + j * 2 + 1] += fma(vy[j * 2 + 1], s[i][1], vy[j * 2] * s[i][0]);
    }
  }
  if ((flags & ST_RHS_SOURCE) && nb > 0) {
    const double ax = pre ? pre->ax : g.anc[c * 3], ay = pre ? pre->ay : g.anc[c * 3 + 1],
                 az = pre ? pre->az : g.anc[c * 3 + 2];
    for (int b = 0; b < nb; b++) {
      DevBeam bm;
      if (pbm && b < kPreBeams) {
        bm = pbm[b];  // (a thread-local array: the runtime index keeps only it out of registers)
      } else {
        bm = beams[b];
      }
      if (!beam_hits_cell(P, bm, ax, ay, az, h)) continue;
      double qv[8], pr[8];
      const double dw = pre ? pre->detw : g.detw[c];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int bb = 0; bb < 2; bb++)
#pragma unroll
          for (int cc = 0; cc < 2; cc++)
            qv[a * 4 + bb * 2 + cc] =
                beam_source(P, bm, ax + cU[a] * h, ay + cU[bb] * h, az + cU[cc] * h) * dw;
      project<0, 0, 0>(qv, pr);
#pragma unroll
      for (int i = 0; i < 8; i++) e[i] += pr[i];
    }
  }
  double ec[8];
  if (Ec || c_atomic) {
    const double dw = pre ? pre->detw : g.detw[c];
#pragma unroll
    for (int q = 0; q < 8; q++) tq[q] = heat_capacity(P, tq[q]) * dw;
    project<0, 0, 0>(tq, ec);
  }
  if (E) {
#pragma unroll
    for (int i = 0; i < 8; i++) E[c * 8 + i] = e[i];
    if (Ec)
#pragma unroll
      for (int i = 0; i < 8; i++) Ec[c * 8 + i] = ec[i];
  } else {
#pragma unroll
    for (int i = 0; i < 8; i++) atomicAdd(f_atomic + g.cv[c * 8 + i], e[i]);
    if (c_atomic)
#pragma unroll
      for (int i = 0; i < 8; i++) atomicAdd(c_atomic + g.cv[c * 8 + i], ec[i]);
  }
}

__global__ void k_rhs_cells(int64_t n, CellGeo g, FaceTab ft, DevParams P,
                            const double* __restrict__ T, double* rc,
                            double rc_value, int flags, double frozen_k,
                            int pending, int nb, const DevBeam* beams,
                            double* E, double* Ec, double* f_atomic,
                            double* c_atomic) {
  // programmatic dependent launch (explicit scan loop): wait for the
  // previous kernel of the stream in every CTA, then release the next one
  ST_SCAN_T0()
  ST_PDL_EARLY_RELEASE();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // the cell's static data and the beam records before the wait (CellPre)
  CellPre pre;
  DevBeam bm[kPreBeams];
  if (c < n) cell_prefetch(c, g, ft, flags, nb, beams, rc, pre, bm);
  ST_PDL_WAIT();
  ST_SCAN_T1()
  if (c >= n) return;
  rhs_cell(c, g, ft, P, T, rc, rc_value, flags, frozen_k, pending, nb, beams, E, Ec, f_atomic,
           c_atomic, &pre, bm);
  ST_SCAN_T2(0)
}

// consistent capacity apply / lumped capacity (operators.py:325-348):
// v == nullptr => ones; T != nullptr => rho c_app(T_q)
__global__ void k_mass_cells(int64_t n, CellGeo g, DevParams P, const double* v,
                             const double* T, double scale, double* E) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double t[8], q[8], o[8];
  if (v) {
    gather8(g.cv, c, v, t);
    interp<0, 0, 0>(t, q);
  } else {
#pragma unroll
    for (int i = 0; i < 8; i++) t[i] = 1.0;
    interp<0, 0, 0>(t, q);
  }
  const double dw = g.detw[c];
  if (T) {
    double tt[8], tq[8];
    gather8(g.cv, c, T, tt);
    interp<0, 0, 0>(tt, tq);
#pragma unroll
    for (int i = 0; i < 8; i++) q[i] = q[i] * (heat_capacity(P, tq[i]) * dw);
  } else {
#pragma unroll
    for (int i = 0; i < 8; i++) q[i] = q[i] * (P.rhoc * dw);
  }
  project<0, 0, 0>(q, o);
#pragma unroll
  for (int i = 0; i < 8; i++) E[c * 8 + i] = o[i] * scale;
}

// r_c <- max(r_c, g(T_q))  (operators.py:219-225)
__global__ void k_history(int64_t n, const int* cv, DevParams P, const double* T, double* rc) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double t[8], tq[8];
  gather8(cv, c, T, t);
  interp<0, 0, 0>(t, tq);
#pragma unroll
  for (int q = 0; q < 8; q++) rc[c * 8 + q] = fmax(rc[c * 8 + q], liquid_fraction(P, tq[q]));
}

// tangent fields at qps (operators.py:373-378)
__device__ __forceinline__ void tangent(const DevParams& P, const double* tl, const double* rc,
                                        double rc_value, int64_t c, double gscale, double* k,
                                        double* dk, double* gx, double* gy, double* gz) {
  double tq[8];
  interp<0, 0, 0>(tl, tq);
#pragma unroll
  for (int q = 0; q < 8; q++) {
    double r = rc ? rc[c * 8 + q] : rc_value;
    k[q] = conductivity(P, liquid_fraction(P, tq[q]), r);
    dk[q] = conductivity_derivative(P, tq[q]);
  }
  interp<1, 0, 0>(tl, gx);
  interp<0, 1, 0>(tl, gy);
  interp<0, 0, 1>(tl, gz);
#pragma unroll
  for (int q = 0; q < 8; q++) {
    gx[q] *= gscale;
    gy[q] *= gscale;
    gz[q] *= gscale;
  }
}

// J v element vectors: D + L + C/dt (operators.py:380-410) of cell c from
// its tangent fields (k, dk, grad T_lin at the Gauss points)
__device__ __forceinline__ void jac_apply(int64_t c, const CellGeo& g, const DevParams& P,
                                          const double* vd, const double* k, const double* dk,
                                          const double* gx, const double* gy, const double* gz,
                                          double dt, double* E) {
  double v[8], e[8], tmp[8], pr[8];
  gather8(g.cv, c, vd, v);
  const double h = g.h[c];
  const double gscale = 2.0 / h;
  const double hh = h / 2.0;
  interp<1, 0, 0>(v, tmp);
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = (hh * k[q]) * tmp[q];
  project<1, 0, 0>(tmp, e);
  interp<0, 1, 0>(v, tmp);
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = (hh * k[q]) * tmp[q];
  project<0, 1, 0>(tmp, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] += pr[i];
  interp<0, 0, 1>(v, tmp);
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = (hh * k[q]) * tmp[q];
  project<0, 0, 1>(tmp, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] += pr[i];
  double vq[8], w[8];
  interp<0, 0, 0>(v, vq);
  const double dw = g.detw[c];
  const double dwg = dw * gscale;
#pragma unroll
  for (int q = 0; q < 8; q++) w[q] = dwg * dk[q] * vq[q];
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = w[q] * gx[q];
  project<1, 0, 0>(tmp, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] += pr[i];
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = w[q] * gy[q];
  project<0, 1, 0>(tmp, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] += pr[i];
#pragma unroll
  for (int q = 0; q < 8; q++) tmp[q] = w[q] * gz[q];
  project<0, 0, 1>(tmp, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) e[i] += pr[i];
  // + apply_mass(v) / dt
#pragma unroll
  for (int q = 0; q < 8; q++) vq[q] = vq[q] * (P.rhoc * dw);
  project<0, 0, 0>(vq, pr);
#pragma unroll
  for (int i = 0; i < 8; i++) E[c * 8 + i] = e[i] + pr[i] / dt;
}

__device__ __forceinline__ void jac_cell(int64_t c, const CellGeo& g, const DevParams& P,
                                         const double* vd, const double* Tl, const double* rc,
                                         double rc_value, double dt, double* E) {
  double tl[8], k[8], dk[8], gx[8], gy[8], gz[8];
  gather8(g.cv, c, Tl, tl);
  tangent(P, tl, rc, rc_value, c, 2.0 / g.h[c], k, dk, gx, gy, gz);
  jac_apply(c, g, P, vd, k, dk, gx, gy, gz, dt, E);
}

// the tangent fields of every cell, structure of arrays: TG[(f * 8 + q) * n + c]
// for f = k, dk, gx, gy, gz (the reference's _tangent_fields, operators.py:373)
__device__ __forceinline__ void tangent_store(int64_t c, int64_t n, const CellGeo& g,
                                              const DevParams& P, const double* Tl,
                                              const double* rc, double rc_value, double* TG) {
  double tl[8], f[5][8];
  gather8(g.cv, c, Tl, tl);
  tangent(P, tl, rc, rc_value, c, 2.0 / g.h[c], f[0], f[1], f[2], f[3], f[4]);
#pragma unroll
  for (int j = 0; j < 5; j++)
#pragma unroll
    for (int q = 0; q < 8; q++) TG[(j * 8 + q) * n + c] = f[j][q];
}

__device__ __forceinline__ void jac_cell_tg(int64_t c, int64_t n, const CellGeo& g,
                                            const DevParams& P, const double* vd,
                                            const double* TG, double dt, double* E) {
  double f[5][8];
#pragma unroll
  for (int j = 0; j < 5; j++)
#pragma unroll
    for (int q = 0; q < 8; q++) f[j][q] = TG[(j * 8 + q) * n + c];
  jac_apply(c, g, P, vd, f[0], f[1], f[2], f[3], f[4], dt, E);
}

__global__ void k_jac_cells(int64_t n, CellGeo g, DevParams P, const double* vd,
                            const double* Tl, const double* rc, double rc_value,
                            double dt, double* E) {
  pdl_wait_release();  // see st_common.cuh
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  jac_cell(c, g, P, vd, Tl, rc, rc_value, dt, E);
}

// element Jacobian entry A[a][b] (operators.py:412-424)
__device__ __forceinline__ double elem_entry(int a, int b, double rcdt_dw, double hh,
                                             double dwg, const double* k, const double* dk,
                                             const double* gx, const double* gy,
                                             const double* gz) {
  double m = 0.0, d = 0.0, l = 0.0;
#pragma unroll
  for (int q = 0; q < 8; q++) {
    m += cPhi[a][q] * cPhi[b][q];
    d += k[q] * (cG[0][a][q] * cG[0][b][q] + cG[1][a][q] * cG[1][b][q] + cG[2][a][q] * cG[2][b][q]);
    l += dk[q] * cPhi[b][q] *
         (cG[0][a][q] * gx[q] + cG[1][a][q] * gy[q] + cG[2][a][q] * gz[q]);
  }
  return rcdt_dw * m + hh * d + dwg * l;
}

// element diagonals (plain cells) / full matrices (cells touching a
// hanging vertex; fold tables operators.py:158-195)
__global__ void k_jdiag_cells(int64_t n, CellGeo g, DevParams P, const double* Tl,
                              const double* rc, double rc_value, double dt,
                              const int* touched_pos, double* E, double* Ae) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double tl[8], k[8], dk[8], gx[8], gy[8], gz[8];
  gather8(g.cv, c, Tl, tl);
  const double h = g.h[c];
  const double gscale = 2.0 / h;
  tangent(P, tl, rc, rc_value, c, gscale, k, dk, gx, gy, gz);
  const double dw = g.detw[c];
  const double rcdt_dw = (P.rhoc / dt) * dw;
  const double hh = h / 2.0;
  const double dwg = dw * gscale;
  int tp = touched_pos ? touched_pos[c] : -1;
  if (tp < 0) {
#pragma unroll
    for (int a = 0; a < 8; a++) {
      double d = 0.0, l = 0.0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        d += k[q] * cGG[a][q];
        l += dk[q] * cPhi[a][q] *
             (cG[0][a][q] * gx[q] + cG[1][a][q] * gy[q] + cG[2][a][q] * gz[q]);
      }
      E[c * 8 + a] = (P.rhoc / dt) * (dw * cPhi2[a]) + hh * d + dwg * l;
    }
  } else {
#pragma unroll
    for (int a = 0; a < 8; a++) E[c * 8 + a] = 0.0;
    for (int a = 0; a < 8; a++)
      for (int b = 0; b < 8; b++)
        Ae[(int64_t)tp * 64 + a * 8 + b] = elem_entry(a, b, rcdt_dw, hh, dwg, k, dk, gx, gy, gz);
  }
}

// ---------------------------------------------------------------------------
// node kernels
// ---------------------------------------------------------------------------
struct NodeTab {
  const int* inc_ptr;  // (nv+1)
  const int* inc_ent;  // cell*8+corner, ascending per vertex
  const int* cond_ptr;  // (nv+1) per master: slaves folding into it
  const int* cond_s;
  const double* cond_w;
  const uint8_t* is_slave;
  const uint8_t* is_dir;
  // the condensation flattened per master: the incident entries of its
  // slaves in cond order (cfe_ptr / cfe) and each slave's entry count (cgl)
  const int* cfe_ptr;
  const int* cfe;
  const int* cgl;
};

// sum of the element entries incident to vertex v, in incidence order
// (np.bincount's order).  A vertex is a corner of at most 8 leaves (one per
// octant), so the entry indices and then the entries are loaded up front
// (two dependent round trips instead of two per entry) and summed in order.
__device__ __forceinline__ double gather_v(const NodeTab& nt, const double* E, int64_t v) {
  const int a = nt.inc_ptr[v], b = nt.inc_ptr[v + 1];
  int ix[8];
  double e[8];
#pragma unroll
  for (int k = 0; k < 8; k++) ix[k] = a + k < b ? nt.inc_ent[a + k] : -1;
#pragma unroll
  for (int k = 0; k < 8; k++) e[k] = ix[k] >= 0 ? E[ix[k]] : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; k++)
    if (ix[k] >= 0) acc += e[k];
  for (int i = a + 8; i < b; i++) acc += E[nt.inc_ent[i]];
  return acc;
}

// condensed sum at a non-slave vertex (bincount then np.add.at order):
// f = own entries, then f + w * (the slave's entries) per folded slave, one
// thread per vertex (the opt-in persistent scan; the kernels below use the
// warp version)
__device__ __forceinline__ double gather_condensed(const NodeTab& nt, const double* E, int64_t v) {
  double f = gather_v(nt, E, v);
  for (int i = nt.cond_ptr[v]; i < nt.cond_ptr[v + 1]; i++)
    f = f + nt.cond_w[i] * gather_v(nt, E, nt.cond_s[i]);
  return f;
}

// The same sum with the condensation done by the whole warp.  Every warp of a
// 2:1 mesh holds about one vertex with slaves folding into it (config 3,
// layer 0: 616 of 691 warps have one or two), and a thread doing that
// vertex's up to 32 extra entries alone makes its 31 neighbours wait (the
// node kernels ran ~1000 warp instructions per vertex that way).  Here each
// thread gathers its own entries, then the warp takes the vertices with
// slaves one at a time: lane q loads entry q of the flattened table (cfe),
// lane j the entry count and weight of slave j; lane j sums slave j's entries
// in order (shuffles from the lanes that hold them), and the weighted slave
// sums are added in slave order -- the same additions in the same order as
// the plain loops.  All 32 lanes call this together; ``live`` marks the lanes
// with a (non-slave) vertex.
// (the part that only reads the static tables -- CSR pointers and the own
// entry indices -- is split off as gather_prep, so that a kernel of the
// programmatic-dependent-launch chain can run it before it waits for its
// predecessor)
struct GatherPrep {
  int a, b, ga, gb, e0, ne;
  int ix[8];
  // the warp's first vertex with slaves, spread over the lanes: lane q holds
  // the id of its flattened entry q, lane j the count and weight of slave j
  int first, jx, len;
  double w;
};

// PF: also the flattened entries of the warp's first vertex with slaves
// (k_step_nodes: 15.85 -> 15.15 us per step of the config-3 scan; the
// backward-Euler kernels measured slower with it, 0.44 against 0.40 ms per
// step, and go without)
template <bool PF = false>
__device__ __forceinline__ GatherPrep gather_prep(const NodeTab& nt, int64_t v, bool live) {
  GatherPrep g;
  g.a = g.b = g.ga = g.gb = g.e0 = g.ne = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) g.ix[k] = -1;
  if (live) {
    g.a = nt.inc_ptr[v];
    g.b = nt.inc_ptr[v + 1];
    g.ga = nt.cond_ptr[v];
    g.gb = nt.cond_ptr[v + 1];
    g.e0 = nt.cfe_ptr[v];
    g.ne = nt.cfe_ptr[v + 1] - g.e0;
#pragma unroll
    for (int k = 0; k < 8; k++) g.ix[k] = g.a + k < g.b ? nt.inc_ent[g.a + k] : -1;
  }
  const int lane = threadIdx.x & 31;
  const unsigned todo = PF ? __ballot_sync(0xffffffffu, g.gb > g.ga) : 0u;
  g.first = todo ? __ffs(todo) - 1 : -1;
  g.jx = -1;
  g.len = 0;
  g.w = 0.0;
  if (todo) {
    const int gas = __shfl_sync(0xffffffffu, g.ga, g.first);
    const int ng = __shfl_sync(0xffffffffu, g.gb, g.first) - gas;
    const int e0s = __shfl_sync(0xffffffffu, g.e0, g.first);
    const int nes = __shfl_sync(0xffffffffu, g.ne, g.first);
    if (nes <= 32 && ng <= 32) {
      if (lane < nes) g.jx = nt.cfe[e0s + lane];
      if (lane < ng) {
        g.len = nt.cgl[gas + lane];
        g.w = nt.cond_w[gas + lane];
      }
    } else {
      g.first = -1;
    }
  }
  return g;
}

__device__ __forceinline__ double gather_condensed_warp(const NodeTab& nt, const double* E,
                                                        const GatherPrep& g, bool live) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double f = 0.0;
  if (live) {
    // own entries in incidence order (gather_v)
    double e[8];
#pragma unroll
    for (int k = 0; k < 8; k++) e[k] = g.ix[k] >= 0 ? E[g.ix[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++)
      if (g.ix[k] >= 0) f += e[k];
    for (int i = g.a + 8; i < g.b; i++) f += E[nt.inc_ent[i]];
  }
  // the entry of the first vertex with slaves goes out with the own entries
  const double e_first = g.jx >= 0 ? E[g.jx] : 0.0;
  unsigned todo = __ballot_sync(kFull, g.gb > g.ga);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int gas = __shfl_sync(kFull, g.ga, src), ng = __shfl_sync(kFull, g.gb, src) - gas;
    const int e0s = __shfl_sync(kFull, g.e0, src), nes = __shfl_sync(kFull, g.ne, src);
    double fs = __shfl_sync(kFull, f, src);
    if (nes <= 32 && ng <= 32) {
      const bool pf = src == g.first;  // warp-uniform
      const double e = pf ? e_first : (lane < nes ? E[nt.cfe[e0s + lane]] : 0.0);
      const int len = pf ? g.len : (lane < ng ? nt.cgl[gas + lane] : 0);
      const double w = pf ? g.w : (lane < ng ? nt.cond_w[gas + lane] : 0.0);
      int start = len;  // inclusive scan of the entry counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, start, o);
        if (lane >= o) start += t;
      }
      start -= len;
      const int maxlen = __reduce_max_sync(kFull, len);
      double sv = 0.0;
      for (int t = 0; t < maxlen; t++) {
        const double x = __shfl_sync(kFull, e, (start + t) & 31);
        if (t < len) sv += x;
      }
      for (int j = 0; j < ng; j++) {
        const double wj = __shfl_sync(kFull, w, j), sj = __shfl_sync(kFull, sv, j);
        fs = fs + wj * sj;
      }
    } else {
      // more than a warp's worth of entries: one slave after the other
      // (every lane computes the same sum)
      for (int i = gas; i < gas + ng; i++) fs = fs + nt.cond_w[i] * gather_v(nt, E, nt.cond_s[i]);
    }
    if (lane == src) f = fs;
  }
  return f;
}

__device__ __forceinline__ double gather_condensed_warp(const NodeTab& nt, const double* E,
                                                        int64_t v, bool live) {
  return gather_condensed_warp(nt, E, gather_prep(nt, v, live), live);
}

// condensed(E) at v; slave rows 0 (or slave_val); Dirichlet rows <- dir_src.
// Called by all lanes of a warp (in: lanes with a vertex).
__device__ __forceinline__ double gather_row_warp(int64_t v, bool in, const NodeTab& nt,
                                                  const double* E, const double* dir_src,
                                                  int set_slave, double slave_val) {
  const bool slave = in && nt.is_slave[v];
  // (the Dirichlet flag and its value with the other loads, not a round trip
  // after the gather)
  const bool dir = in && dir_src && nt.is_dir[v];
  const double dv = dir ? dir_src[v] : 0.0;
  double r = gather_condensed_warp(nt, E, v, in && !slave);
  if (slave) r = set_slave ? slave_val : 0.0;
  if (dir && !slave) r = dv;
  return r;
}

// out = condensed(E); slave rows 0; optional: dirichlet rows <- dir_src, slave rows <- slave_val
__global__ void k_gather(int64_t nv, NodeTab nt, const double* E, double* out,
                         const double* dir_src, int set_slave, double slave_val) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // the static tables before the wait for the predecessor (st_common.cuh)
  const bool in = v < nv;
  const bool slave = in && nt.is_slave[v];
  const bool dir = in && !slave && dir_src && nt.is_dir[v];
  const GatherPrep g = gather_prep(nt, v, in && !slave);
  pdl_wait_release();
  double r = gather_condensed_warp(nt, E, g, in && !slave);
  if (slave) r = set_slave ? slave_val : 0.0;
  if (dir) r = dir_src[v];
  if (in) out[v] = r;
}

// ---------------------------------------------------------------------------
// persistent PCG (krylov_solve, timestepping.py:102-131) for the Newton
// step of the cool-down: one cooperative launch runs the whole solve with
// grid-wide barriers instead of kernel boundaries.  Per iteration:
//   1. p = z + beta p (beta = 0 on the first iteration) and the Jacobian
//      input vd (Dirichlet rows zeroed, slaves interpolated from the same
//      z + beta p of their masters, operators.py:380-410),
//   2. element vectors J vd (cells),
//   3. Ap = condensed gather (Dirichlet rows identity, slave rows 0) and
//      the p.Ap block partials,
//   4. alpha = rz / p.Ap, x += alpha p, r -= alpha Ap, z = D^-1 r and the
//      r.r / r.z block partials; every block sums the partials in the same
//      fixed order, so all blocks take the same stopping decision
//      (||r|| <= tol ||b||, x0 = 0) and the same beta.
// The result (iterations, converged) is written to the device; the host
// reads it once after the solve.
// ---------------------------------------------------------------------------
constexpr int kPcgThreads = 256;

struct PcgArgs {
  int64_t n, nv, ns;
  CellGeo g;
  NodeTab nt;
  DevParams P;
  const double* Tl;
  const double* rc;
  double rc_value, dt;
  const int64_t* slaves;
  const int64_t* sptr;
  const int64_t* smast;
  const double* sw;
  const double* b;
  const double* dinv;  // nullable: no preconditioner
  double *x, *r, *z, *p0, *p1, *Ap, *vd, *E;
  double* TG;          // tangent fields (40 per cell, structure of arrays)
  double* part;        // 4 x gridDim.x block partials
  double thr;          // tol * ||b||
  int max_iter;
  int* out;            // [iterations, converged]
};

// deterministic block sums of (a, b): an xor butterfly inside each warp
// (every lane ends with the same bits: a + b == b + a), then the same over
// the warp totals; the totals are returned to every thread
__device__ __forceinline__ double2 block_sum2(double a, double b, double2* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int nw = kPcgThreads / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();  // red is free (previous use finished)
  if (lane == 0) red[w] = make_double2(a, b);
  __syncthreads();
  double2 v = lane < nw ? red[lane] : make_double2(0.0, 0.0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// sums of the nb block partials pa[0..nb) and pb[0..nb), the same order in
// every block
__device__ __forceinline__ double2 sum_partials2(const double* pa, const double* pb, int nb,
                                                 double2* red) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += kPcgThreads) {
    a += pa[i];
    b += pb ? pb[i] : 0.0;
  }
  return block_sum2(a, b, red);
}

#ifndef ST_PCG_MINB
// resident blocks per SM the register allocation aims at.  1 (no register
// cap, one block per SM): the cells and the staged gather keep their state
// in registers and the grid barriers synchronise half as many blocks --
// measured on the config-3-sized box 18.9 against 23.7 us per iteration
// inside the kernel (phase clocks of -DST_PCG_TIMING), 36.4 against 41.6 us
// per iteration of a whole solve, 0.48 against 0.54 ms per BE step
#define ST_PCG_MINB 1
#endif
// dev hook (-DST_PCG_TIMING, tools/time_implicit.py): block 0 accumulates the
// time of every phase and barrier of the iteration loop (globaltimer, ns)
// behind the block partials
#ifdef ST_PCG_TIMING
#define ST_PCG_TS(k)                                                      \
  if (tid == 0) {                                                         \
    unsigned long long t_;                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
    a.part[4 * nb + (k)] += (double)(t_ - ts_last);                       \
    ts_last = t_;                                                         \
  }
#else
#define ST_PCG_TS(k)
#endif
__global__ void __launch_bounds__(kPcgThreads, ST_PCG_MINB) k_pcg_persistent(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 red[32];
  const int nb = gridDim.x;
  const int64_t tid = blockIdx.x * (int64_t)kPcgThreads + threadIdx.x;
#ifdef ST_PCG_TIMING
  unsigned long long ts_last;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_last));
#endif
  const int64_t nth = (int64_t)nb * kPcgThreads;
  double* pa = a.part;
  // the tangent at T_lin once per solve (it is fixed over the iterations)
  for (int64_t c = tid; c < a.n; c += nth) tangent_store(c, a.n, a.g, a.P, a.Tl, a.rc, a.rc_value, a.TG);
  // x = 0, r = b, z = D^-1 r, p = z, rz = r.z
  double l = 0.0;
  for (int64_t i = tid; i < a.nv; i += nth) {
    const double ri = a.b[i];
    const double zi = a.dinv ? ri * a.dinv[i] : ri;
    a.x[i] = 0.0;
    a.r[i] = ri;
    a.z[i] = zi;
    a.p0[i] = zi;
    l += ri * zi;
  }
  double2 t2 = block_sum2(l, 0.0, red);
  if (threadIdx.x == 0) pa[blockIdx.x] = t2.x;
  grid.sync();
  double rz = sum_partials2(pa, nullptr, nb, red).x;
  double beta = 0.0;
  double* p = a.p0;
  double* pn = a.p1;
  ST_PCG_TS(0)
  for (int it = 1; it <= a.max_iter; it++) {
    // 1. p_new = z + beta p and the Jacobian input
    for (int64_t i = tid; i < a.nv + a.ns; i += nth) {
      if (i < a.nv) {
        // (both flags up front: behind the branch the second load waits for
        // the first, a round trip more in every iteration)
        const bool sl = a.nt.is_slave[i] != 0, dr = a.nt.is_dir[i] != 0;
        const double q = fma(beta, p[i], a.z[i]);
        pn[i] = q;
        if (!sl) a.vd[i] = dr ? 0.0 : q;
      } else {
        const int64_t s = i - a.nv;
        double acc = 0.0;
        for (int64_t k = a.sptr[s]; k < a.sptr[s + 1]; k++) {
          const int64_t m = a.smast[k];
          acc += a.sw[k] * fma(beta, p[m], a.z[m]);
        }
        a.vd[a.slaves[s]] = acc;
      }
    }
    {
      double* t = p;
      p = pn;
      pn = t;
    }
    ST_PCG_TS(1)
    grid.sync();
    ST_PCG_TS(2)
    // 2. element vectors of J vd
    for (int64_t c = tid; c < a.n; c += nth) jac_cell_tg(c, a.n, a.g, a.P, a.vd, a.TG, a.dt, a.E);
    ST_PCG_TS(3)
    grid.sync();
    ST_PCG_TS(4)
    // 3. Ap and p.Ap
    l = 0.0;
    for (int64_t v0 = tid - (threadIdx.x & 31); v0 < a.nv; v0 += nth) {  // whole warps
      const int64_t v = v0 + (threadIdx.x & 31);
      const double ap = gather_row_warp(v, v < a.nv, a.nt, a.E, p, 0, 0.0);
      if (v < a.nv) {
        a.Ap[v] = ap;
        l += p[v] * ap;
      }
    }
    ST_PCG_TS(11)
    t2 = block_sum2(l, 0.0, red);
    if (threadIdx.x == 0) pa[nb + blockIdx.x] = t2.x;
    ST_PCG_TS(5)
    grid.sync();
    ST_PCG_TS(6)
    const double alpha = rz / sum_partials2(pa + nb, nullptr, nb, red).x;
    ST_PCG_TS(7)
    // 4. x, r, z and r.r / r.z
    double lrr = 0.0, lrz = 0.0;
    for (int64_t i = tid; i < a.nv; i += nth) {
      a.x[i] += alpha * p[i];
      const double ri = a.r[i] - alpha * a.Ap[i];
      const double zi = a.dinv ? ri * a.dinv[i] : ri;
      a.r[i] = ri;
      a.z[i] = zi;
      lrr += ri * ri;
      lrz += ri * zi;
    }
    t2 = block_sum2(lrr, lrz, red);
    if (threadIdx.x == 0) {
      pa[2 * nb + blockIdx.x] = t2.x;
      pa[3 * nb + blockIdx.x] = t2.y;
    }
    ST_PCG_TS(8)
    grid.sync();
    ST_PCG_TS(9)
    t2 = sum_partials2(pa + 2 * nb, pa + 3 * nb, nb, red);
    const double rr = t2.x, rzn = t2.y;
    ST_PCG_TS(10)
    if (sqrt(rr) <= a.thr) {
      if (tid == 0) {
        a.out[0] = it;
        a.out[1] = 1;
      }
      return;
    }
    beta = rzn / rz;
    rz = rzn;
  }
  if (tid == 0) {
    a.out[0] = a.max_iter;
    a.out[1] = 0;
  }
}

// the update of a non-slave vertex from its gathered f and inverse capacity
__device__ __forceinline__ double step_node_with(int64_t v, const NodeTab& nt, double f, double ci,
                                                 const double* T, double dt, double T_inf,
                                                 double* Tout) {
  // T + dt (C^-1 f) with the reference's three roundings (no FMA), so a
  // step equals the host composition of the same pieces bit for bit
  double out = __dadd_rn(T[v], __dmul_rn(dt, __dmul_rn(ci, f)));
  if (nt.is_dir[v]) out = T_inf;
  Tout[v] = out;
  return out;
}

// forward Euler with the lumped capacity (operators.py:352-369) at a
// non-slave vertex v; returns T'(v)
__device__ __forceinline__ double step_node(int64_t v, const NodeTab& nt, const double* E,
                                            const double* Ec, const double* f_atomic,
                                            const double* c_atomic, const double* cinv,
                                            const double* T, double dt, double T_inf,
                                            double* Tout) {
  double f = E ? gather_condensed(nt, E, v) : f_atomic[v];
  double ci;
  if (Ec)
    ci = 1.0 / gather_condensed(nt, Ec, v);
  else if (c_atomic)
    ci = 1.0 / c_atomic[v];
  else
    ci = cinv[v];
  return step_node_with(v, nt, f, ci, T, dt, T_inf, Tout);
}

// block_max2 (st_common.cuh) with both running maxima read before the first
// atomic: its second volatile read waits for the first atomic otherwise, a
// round trip at the end of a kernel that is nothing but round trips.  (Kept
// here: the shared one is part of the structured hot kernels' translation
// units.)
__device__ __forceinline__ void block_max2_both(double absval, double val,
                                                unsigned long long* slot) {
  __shared__ unsigned long long s_a[32], s_s[32];
  unsigned long long ka = __double_as_longlong(fabs(absval));  // >= 0: bits monotone
  unsigned long long ks = order_key(val);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a2 = __shfl_xor_sync(0xffffffffu, ka, o);
    unsigned long long s2 = __shfl_xor_sync(0xffffffffu, ks, o);
    ka = a2 > ka ? a2 : ka;
    ks = s2 > ks ? s2 : ks;
  }
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_a[w] = ka;
    s_s[w] = ks;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const volatile unsigned long long* vs = slot;
    const unsigned long long m0 = vs[0], m1 = vs[1];
    for (int i = 1; i < nw; i++) {
      ka = s_a[i] > ka ? s_a[i] : ka;
      ks = s_s[i] > ks ? s_s[i] : ks;
    }
    if (ka > m0) atomicMax(slot, ka);
    if (ks > m1) atomicMax(slot + 1, ks);
  }
}

__global__ void k_step_nodes(int64_t nv, NodeTab nt, const double* E, const double* Ec,
                             const double* f_atomic, const double* c_atomic,
                             const double* cinv, const double* T, double dt, double T_inf,
                             double* Tout, unsigned long long* red) {
  // programmatic dependent launch (explicit scan loop): wait for the
  // previous kernel of the stream in every CTA, then release the next one
  ST_SCAN_T0()
  ST_PDL_EARLY_RELEASE();
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double out = 0.0;
  bool live = v < nv && !nt.is_slave[v];
  // the static gather tables before the wait: two dependent round trips off
  // the step's chain of three launches
  const GatherPrep g = gather_prep<true>(nt, v, live && (E || Ec));
  // T(v) (this step's input: its writers completed before the cell kernel
  // started), the constant inverse capacity and the Dirichlet flag too (ncu
  // had them issued after the gather had come back: a second round trip)
  const double Tv = live ? T[v] : 0.0;
  const double civ = (live && !Ec && !c_atomic) ? cinv[v] : 0.0;
  const bool dirv = live && nt.is_dir[v];
  ST_PDL_WAIT();
  ST_SCAN_T1()
  // the condensed gathers by the whole warp, then step_node's update
  const double fg = E ? gather_condensed_warp(nt, E, g, live) : 0.0;
  const double cg_ = Ec ? gather_condensed_warp(nt, Ec, g, live) : 0.0;
  if (live) {
    const double f = E ? fg : f_atomic[v];
    const double ci = Ec ? 1.0 / cg_ : (c_atomic ? 1.0 / c_atomic[v] : civ);
    // step_node_with's update (the reference's three roundings, no FMA)
    out = __dadd_rn(Tv, __dmul_rn(dt, __dmul_rn(ci, f)));
    if (dirv) out = T_inf;
    Tout[v] = out;
  }
  block_max2_both(live ? out : 0.0, live ? out : -INFINITY, red);
  ST_SCAN_T2(1)
}

// hanging-vertex closure (mesh.py:652-661)
__device__ __forceinline__ void distribute_slave(int64_t i, const int64_t* slaves,
                                                 const int64_t* ptr, const int64_t* masters,
                                                 const double* w, double* v) {
  // the rounding of the reference's segmented sum (numpy add.reduceat:
  // first product, plus the rest summed from zero, 8-lane pairwise blocks
  // beyond 8 terms), every product rounded on its own
  const int64_t b = ptr[i], e = ptr[i + 1];
  if (e <= b) return;
  const int64_t n = e - b - 1;
  double rest = 0.0;
  if (n < 8) {
    for (int64_t p = b + 1; p < e; p++) rest = __dadd_rn(rest, __dmul_rn(w[p], v[masters[p]]));
  } else {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = __dmul_rn(w[b + 1 + j], v[masters[b + 1 + j]]);
    int64_t k = 8;
    for (; k < n - (n % 8); k += 8)
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], __dmul_rn(w[b + 1 + k + j], v[masters[b + 1 + k + j]]));
    rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                     __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; k < n; k++) rest = __dadd_rn(rest, __dmul_rn(w[b + 1 + k], v[masters[b + 1 + k]]));
  }
  v[slaves[i]] = __dadd_rn(__dmul_rn(w[b], v[masters[b]]), rest);
}

__global__ void k_distribute(int64_t ns, const int64_t* slaves, const int64_t* ptr,
                             const int64_t* masters, const double* w, double* v) {
  // programmatic dependent launch (explicit scan loop): wait for the
  // previous kernel of the stream in every CTA, then release the next one
  // This kernel alone releases its successor before its own wait: its body is
  // a fraction of a launch latency, so the next step's cell kernel, released
  // only after the wait, would arrive (and prefetch its tables) after this
  // kernel is done.  Released first, it is staged while the node kernel still
  // runs; it reads nothing but static tables until its own wait, which
  // returns when this kernel -- and with it the node kernel -- has completed.
  // It releases its own successor after its wait, so nothing runs further
  // ahead (releasing early in all three kernels measured slower, see above).
#ifndef ST_DIST_EARLY
#define ST_DIST_EARLY 1
#endif
  ST_SCAN_T0()
  if (ST_DIST_EARLY) pdl_release();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // the constraint row (static) before the wait; rows of up to four masters
  // (edge and face midpoints) are finished from registers
  int64_t sl = 0, b = 0, e = 0, m[4] = {0, 0, 0, 0};
  double ww[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < ns) {
    sl = slaves[i];
    b = ptr[i];
    e = ptr[i + 1];
    if (e - b <= 4) {
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (b + k < e) {
          m[k] = masters[b + k];
          ww[k] = w[b + k];
        }
    }
  }
  if (ST_DIST_EARLY) {
    pdl_wait();
  } else {
    ST_PDL_WAIT();
  }
  ST_SCAN_T1()
  if (i >= ns) return;
  if (e > b && e - b <= 4) {
    // distribute_slave's order: the first product plus the rest summed from zero
    double x[4];
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = b + k < e ? v[m[k]] : 0.0;
    double rest = 0.0;
#pragma unroll
    for (int k = 1; k < 4; k++)
      if (b + k < e) rest = __dadd_rn(rest, __dmul_rn(ww[k], x[k]));
    v[sl] = __dadd_rn(__dmul_rn(ww[0], x[0]), rest);
    ST_SCAN_T2(2)
    return;
  }
  distribute_slave(i, slaves, ptr, masters, w, v);
  ST_SCAN_T2(2)
}

// ---------------------------------------------------------------------------
// persistent explicit scan (run_scan_phase's step loop, timestepping.py:211-
// 221) for the unstructured backend: one cooperative launch integrates a
// batch of steps; per step the cell phase (element vectors, the owed history
// update first), a grid barrier, the node phase (condensed gather, forward
// Euler with the lumped capacity, Dirichlet pin, the step's |T| / T maxima
// into its own slot pair), a grid barrier, the slave closure and a barrier.
// The same device functions as the per-kernel path, so a step is bitwise the
// one k_rhs_cells -> k_step_nodes -> k_distribute computes.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 128;

struct ScanArgs {
  int64_t n, nv, ns;
  CellGeo g;
  FaceTab ft;
  NodeTab nt;
  DevParams P;
  double* Ta;  // step s reads Ta when s is even, Tb when odd, writes the other
  double* Tb;
  double* rc;
  double rc_value;
  int pending0, nsteps, nb, latent;
  const double* dts;
  const DevBeam* beams;  // nb per step
  double* E;
  double* Ec;
  const double* cinv;
  const int64_t* slaves;
  const int64_t* sptr;
  const int64_t* smast;
  const double* sw;
  unsigned long long* slots;  // 2 per step
};

__global__ void __launch_bounds__(kScanThreads) k_scan_persistent(ScanArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * kScanThreads;
  const int flags = ST_RHS_DIFFUSION | ST_RHS_FACES | ST_RHS_SOURCE;
  for (int s = 0; s < a.nsteps; s++) {
    const double* T = (s & 1) ? a.Tb : a.Ta;
    double* Tout = (s & 1) ? a.Ta : a.Tb;
    for (int64_t c = tid; c < a.n; c += nth)
      rhs_cell(c, a.g, a.ft, a.P, T, a.rc, a.rc_value, flags, 0.0, s ? 1 : a.pending0, a.nb,
               a.beams + (int64_t)s * a.nb, a.E, a.latent ? a.Ec : nullptr, nullptr, nullptr);
    grid.sync();
    unsigned long long ka = 0ull;
    double tm = -INFINITY;
    const double dt = a.dts[s];
    for (int64_t v = tid; v < a.nv; v += nth) {
      if (a.nt.is_slave[v]) continue;
      const double o = step_node(v, a.nt, a.E, a.latent ? a.Ec : nullptr, nullptr, nullptr,
                                 a.cinv, T, dt, a.P.T_inf, Tout);
      const unsigned long long b = (unsigned long long)__double_as_longlong(o) & 0x7fffffffffffffffull;
      ka = b > ka ? b : ka;
      tm = o > tm ? o : tm;
    }
    block_max2(__longlong_as_double((long long)ka), tm, a.slots + 2 * s);
    grid.sync();
    if (a.ns) {
      for (int64_t i = tid; i < a.ns; i += nth)
        distribute_slave(i, a.slaves, a.sptr, a.smast, a.sw, Tout);
      grid.sync();
    }
  }
}

// atomic-mode condensation (fold slave rows into masters, zero slaves)
__global__ void k_condense_atomic(int64_t ns, const int64_t* slaves, const int64_t* ptr,
                                  const int64_t* masters, const double* w, double* v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  double x = v[slaves[i]];
  for (int64_t p = ptr[i]; p < ptr[i + 1]; p++) atomicAdd(v + masters[p], w[p] * x);
  v[slaves[i]] = 0.0;
}

__global__ void k_fold(int64_t nv, const int* fptr, const int* fent, const double* fw,
                       const double* Ae, double* diag) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int a = fptr[v], b = fptr[v + 1];
  if (a == b) return;
  double d = diag[v];
  for (int i = a; i < b; i++) d = d + fw[i] * Ae[fent[i]];
  diag[v] = d;
}


// Jacobian input in one launch: threads < nv copy v with Dirichlet rows
// zeroed (non-slave nodes), threads nv .. nv+ns-1 interpolate the slaves
// from v (the same values the copy -> distribute -> zero sequence gives:
// slaves and Dirichlet nodes are disjoint, masters are read before zeroing)
__global__ void k_prep_jac(int64_t nv, int64_t ns, const uint8_t* is_dir, const uint8_t* is_slave,
                           const double* v, const int64_t* slaves, const int64_t* ptr,
                           const int64_t* masters, const double* w, double* vd) {
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nv) {
    if (!is_slave[i]) vd[i] = is_dir[i] ? 0.0 : v[i];
    return;
  }
  i -= nv;
  if (i >= ns) return;
  double acc = 0.0;
  for (int64_t p = ptr[i]; p < ptr[i + 1]; p++) acc += w[p] * v[masters[p]];
  vd[slaves[i]] = acc;
}

__global__ void k_mask_rows(int64_t nv, const uint8_t* is_dir, const uint8_t* is_slave, double* v) {
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nv) return;
  if (is_dir[i] || is_slave[i]) v[i] = 0.0;
}

__global__ void k_pin(int64_t nv, const uint8_t* is_dir, double* v, double val) {
  pdl_wait_release();  // see st_common.cuh
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nv) return;
  if (is_dir[i]) v[i] = val;
}

__global__ void k_diag_fix(int64_t nv, const uint8_t* is_dir, const uint8_t* is_slave, double* d) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nv) return;
  if (is_dir[i] || is_slave[i]) d[i] = 1.0;
}

// ---------------------------------------------------------------------------
// backend
// ---------------------------------------------------------------------------
static inline unsigned nblk(int64_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }
// per-cell kernels at cool-down mesh sizes (~2e4 cells) are latency bound:
// small blocks spread them over every SM.  Config-3-sized explicit step with
// the PDL chain: 32 -> 10.6, 64 -> 10.7, 128 -> 10.3, 256 -> 10.95 us (before
// PDL, 64 was 8 % faster than 256)
#ifndef ST_CELL_THREADS
#define ST_CELL_THREADS 128  // A/B hook (ST_VARIANT builds)
#endif
constexpr int kCellThreads = ST_CELL_THREADS;
// block size of the scan's node kernel (A/B hook, ST_VARIANT builds)
#ifndef ST_NODE_THREADS
#define ST_NODE_THREADS 128  // 14.95 -> 14.69 us per step of the config-3 scan against 256; 64 the same
#endif
constexpr int kNodeThreads = ST_NODE_THREADS;
static inline unsigned nblk_cells(int64_t n) {
  return (unsigned)((n + kCellThreads - 1) / kCellThreads);
}

struct Unstructured : Backend {
#ifdef ST_SCAN_TIMING
  ~Unstructured() override {
    cudaDeviceSynchronize();
    unsigned cnt = 0;
    std::vector<unsigned long long> r(4 * 8192);
    cudaMemcpyFromSymbol(&cnt, st_scan_cnt, sizeof(cnt));
    cudaMemcpyFromSymbol(r.data(), st_scan_ring, r.size() * 8);
    if (cnt < 64) return;
    // records in launch order: the ring is filled in completion order of
    // block 0, which is the launch order of the chain
    const unsigned m = std::min(cnt, 8192u), first = cnt > 8192u ? cnt % 8192u : 0u;
    double pre[3] = {}, body[3] = {}, gap[3] = {};
    int nk[3] = {};
    unsigned long long prev_exit = 0;
    for (unsigned q = 0; q < m; q++) {
      const unsigned long long* e = &r[4 * ((first + q) % 8192u)];
      const int k = (int)e[0];
      if (k < 0 || k > 2) continue;
      if (prev_exit && e[2] >= prev_exit && e[2] - prev_exit < 1000000ull) {
        pre[k] += (double)(e[2] - e[1]);
        body[k] += (double)(e[3] - e[2]);
        gap[k] += (double)(e[2] - prev_exit);  // predecessor's block 0 exit -> this wait returned
        nk[k]++;
      }
      prev_exit = e[3];
    }
    static const char* nm[3] = {"cells", "nodes", "slaves"};
    for (int k = 0; k < 3; k++)
      if (nk[k])
        fprintf(stderr, "scan timing %s: n %d, entry->wait %.0f ns, prev exit->wait returned %.0f ns, "
                "wait->exit (block 0) %.0f ns\n", nm[k], nk[k], pre[k] / nk[k], gap[k] / nk[k],
                body[k] / nk[k]);
  }
#endif
  int64_t n = 0, nv = 0, ns = 0, nf = 0;
  DevBuf<int> cv, inc_ptr, inc_ent, cond_ptr, cond_s, face_ptr, touched_pos, fold_ptr, fold_ent;
  DevBuf<int> cfe_ptr, cfe, cgl;
  DevBuf<double> h, anc, detw, cond_w, fvx, fvy, farea, cinv, E, Ec, Ae, fold_w;
  DevBuf<uint8_t> is_slave, is_dir;
  DevBuf<int64_t> slaves, sptr, smast;
  DevBuf<double> sw;
  int64_t n_touched = 0;

  CellGeo geo() const { return CellGeo{cv.p, h.p, anc.p, detw.p}; }
  FaceTab faces() const { return FaceTab{nf ? face_ptr.p : nullptr, fvx.p, fvy.p, farea.p}; }
  NodeTab nodes() const {
    return NodeTab{inc_ptr.p, inc_ent.p, cond_ptr.p, cond_s.p, cond_w.p, is_slave.p, is_dir.p,
                   cfe_ptr.p, cfe.p, cgl.p};
  }

  int launched() {
    c->launches++;
    ST_LAUNCHED();
    return ST_OK;
  }

  int distribute(double* v) override { return distribute_pdl(v, use_pdl() && !c->prof); }

  int distribute_pdl(double* v, bool pdl) {
    if (!ns) return ST_OK;
    ST_CUDA(launch_pdl(pdl, k_distribute, dim3(nblk(ns)), dim3(kThreads), c->stream, ns,
                       (const int64_t*)slaves.p, (const int64_t*)sptr.p, (const int64_t*)smast.p,
                       (const double*)sw.p, v));
    return launched();
  }

  int mask_rows(double* v) override {
    ST_CUDA(launch_pdl(use_pdl(), k_mask_rows, dim3(nblk(nv)), dim3(kThreads), c->stream, nv,
                       (const uint8_t*)is_dir.p, (const uint8_t*)is_slave.p, v));
    return launched();
  }

  int pin_dirichlet(double* v, double value) override {
    ST_CUDA(launch_pdl(use_pdl(), k_pin, dim3(nblk(nv)), dim3(kThreads), c->stream, nv,
                       (const uint8_t*)is_dir.p, v, value));
    return launched();
  }

  int cells_rhs(const double* T, double* rc, int flags, double frozen_k, int nb,
                const DevBeam* beams, int pending, bool want_cap, double* f_atomic,
                double* c_atomic, bool pdl = false) {
    double* rcp = rc;
    bool det = c->deterministic || f_atomic == nullptr;
    ST_CUDA(launch_pdl(pdl, k_rhs_cells, dim3(nblk_cells(n)), dim3(kCellThreads), c->stream, n,
                       geo(), faces(), c->dp, T, rcp, c->rc_value, flags, frozen_k, pending, nb,
                       beams, det ? E.p : nullptr, (det && want_cap) ? Ec.p : nullptr,
                       det ? nullptr : f_atomic, (!det && want_cap) ? c_atomic : nullptr));
    return launched();
  }

  int rhs(const double* T, double* rc, int flags, double frozen_k, int nb,
          const DevBeam* beams, double* f, int pending) override {
    if (c->deterministic) {
      const bool pdl = use_pdl() && !c->prof;
      ST_TRY(cells_rhs(T, rc, flags, frozen_k, nb, beams, pending, false, nullptr, nullptr, pdl));
      ST_CUDA(launch_pdl(pdl, k_gather, dim3(nblk(nv)), dim3(kThreads), c->stream, nv, nodes(),
                         (const double*)E.p, f, (const double*)nullptr, 0, 0.0));
      return launched();
    }
    ST_CUDA(cudaMemsetAsync(f, 0, nv * sizeof(double), c->stream));
    ST_TRY(cells_rhs(T, rc, flags, frozen_k, nb, beams, pending, false, f, nullptr));
    if (ns) {
      k_condense_atomic<<<nblk(ns), kThreads, 0, c->stream>>>(ns, slaves.p, sptr.p, smast.p, sw.p, f);
      ST_TRY(launched());
    }
    return ST_OK;
  }

  int explicit_step(const double* T, double* rc, double dt, int nb, const DevBeam* beams,
                    double* Tout, int pending, double* red) override {
    const bool latent = c->dp.latent != 0;
    const int flags = ST_RHS_DIFFUSION | ST_RHS_FACES | ST_RHS_SOURCE;
    double* fa = nullptr;
    double* ca = nullptr;
    if (!c->deterministic) {
      ST_TRY(c->vec(6, &fa));
      ST_CUDA(cudaMemsetAsync(fa, 0, nv * sizeof(double), c->stream));
      if (latent) {
        ST_TRY(c->vec(7, &ca));
        ST_CUDA(cudaMemsetAsync(ca, 0, nv * sizeof(double), c->stream));
      }
    }
    // the scan loop chains its kernels with programmatic dependent launch
    // (ST_NO_PDL=1 turns it off); every kernel waits for its predecessor
    // before touching memory, so the order is the plain stream order
    const bool pdl = use_pdl() && c->deterministic && !c->prof;
    c->prof_begin();
    ST_TRY(cells_rhs(T, rc, flags, 0.0, nb, beams, pending, latent, fa, ca, pdl));
    c->prof_end();
    if (!c->deterministic && ns) {
      k_condense_atomic<<<nblk(ns), kThreads, 0, c->stream>>>(ns, slaves.p, sptr.p, smast.p, sw.p, fa);
      ST_TRY(launched());
      if (latent) {
        k_condense_atomic<<<nblk(ns), kThreads, 0, c->stream>>>(ns, slaves.p, sptr.p, smast.p, sw.p, ca);
        ST_TRY(launched());
      }
    }
    const bool det = c->deterministic != 0;
    ST_CUDA(launch_pdl(pdl, k_step_nodes, dim3((unsigned)((nv + kNodeThreads - 1) / kNodeThreads)),
                       dim3(kNodeThreads), c->stream, nv,
                       nodes(), (const double*)(det ? E.p : nullptr),
                       (const double*)((det && latent) ? Ec.p : nullptr),
                       (const double*)(det ? nullptr : fa),
                       (const double*)((!det && latent) ? ca : nullptr), (const double*)cinv.p, T,
                       dt, c->dp.T_inf, Tout, reinterpret_cast<unsigned long long*>(red)));
    ST_TRY(launched());
    return distribute_pdl(Tout, pdl);
  }

  DevBuf<double> scan_dts;
  int scan_blocks = 0;

  int explicit_steps_persistent(double* Ta, double* Tb, double* rc, const double* dts,
                                int nsteps, int nb, const DevBeam* beams, int pending0,
                                unsigned long long* slots) override {
    // measured slower than the PDL kernel chain at config-3 sizes (14.6 vs
    // 10.4 us per step: three grid barriers per step at low occupancy), so
    // opt-in: ST_SCAN_PERSISTENT=1
    static const bool on = getenv("ST_SCAN_PERSISTENT") && getenv("ST_SCAN_PERSISTENT")[0] == '1';
    if (!on || !c->deterministic) return ST_EUNSUPPORTED;
    if (!scan_blocks) {
      int per_sm = 0, sms = 0;
      ST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan_persistent,
                                                            kScanThreads, 0));
      ST_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      scan_blocks = std::max(1, std::min(per_sm, 4) * sms);
    }
    if ((int64_t)scan_dts.n < nsteps) ST_TRY(scan_dts.alloc(std::max(nsteps, 512)));
    ST_CUDA(cudaMemcpyAsync(scan_dts.p, dts, nsteps * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
    ScanArgs a{};
    a.n = n;
    a.nv = nv;
    a.ns = ns;
    a.g = geo();
    a.ft = faces();
    a.nt = nodes();
    a.P = c->dp;
    a.Ta = Ta;
    a.Tb = Tb;
    a.rc = rc;
    a.rc_value = c->rc_value;
    a.pending0 = pending0;
    a.nsteps = nsteps;
    a.nb = nb;
    a.latent = c->dp.latent != 0;
    a.dts = scan_dts.p;
    a.beams = beams;
    a.E = E.p;
    a.Ec = Ec.p;
    a.cinv = cinv.p;
    a.slaves = slaves.p;
    a.sptr = sptr.p;
    a.smast = smast.p;
    a.sw = sw.p;
    a.slots = slots;
    void* args[] = {&a};
    c->prof_begin();
    ST_CUDA(cudaLaunchCooperativeKernel((const void*)k_scan_persistent, dim3(scan_blocks),
                                        dim3(kScanThreads), args, 0, c->stream));
    c->prof_end();
    // the host copy of dts must outlive the async upload
    ST_CUDA(cudaStreamSynchronize(c->stream));
    return launched();
  }

  int history(const double* T, double* rc) override {
    if (!rc) return ST_OK;  // uniform r_c (== 1) is a fixed point
    k_history<<<nblk(n), kThreads, 0, c->stream>>>(n, cv.p, c->dp, T, rc);
    return launched();
  }

  int capacity(const double* T, double* out) override {
    k_mass_cells<<<nblk(n), kThreads, 0, c->stream>>>(n, geo(), c->dp, nullptr, T, 1.0, E.p);
    ST_TRY(launched());
    k_gather<<<nblk(nv), kThreads, 0, c->stream>>>(nv, nodes(), E.p, out, nullptr, 1, 1.0);
    return launched();
  }

  int mass(const double* v, double* out) override {
    k_mass_cells<<<nblk(n), kThreads, 0, c->stream>>>(n, geo(), c->dp, v, nullptr, 1.0, E.p);
    ST_TRY(launched());
    k_gather<<<nblk(nv), kThreads, 0, c->stream>>>(nv, nodes(), E.p, out, nullptr, 0, 0.0);
    return launched();
  }

  int jacobian(const double* v, const double* Tl, const double* rc, double dt,
               double* out) override {
    double* vd;
    ST_TRY(c->vec(5, &vd));
    // chained with programmatic dependent launch (the PCG iteration)
    const bool pdl = use_pdl() && !c->prof;
    ST_CUDA(launch_pdl(pdl, k_prep_jac, dim3(nblk(nv + ns)), dim3(kThreads), c->stream, nv, ns,
                       (const uint8_t*)is_dir.p, (const uint8_t*)is_slave.p, v,
                       (const int64_t*)slaves.p, (const int64_t*)sptr.p, (const int64_t*)smast.p,
                       (const double*)sw.p, vd));
    ST_TRY(launched());
    c->prof_begin();
    ST_CUDA(launch_pdl(pdl, k_jac_cells, dim3(nblk_cells(n)), dim3(kCellThreads), c->stream, n,
                       geo(), c->dp, (const double*)vd, Tl, rc, c->rc_value, dt, E.p));
    ST_TRY(launched());
    c->prof_end();
    ST_CUDA(launch_pdl(pdl, k_gather, dim3(nblk(nv)), dim3(kThreads), c->stream, nv, nodes(),
                       (const double*)E.p, out, v, 0, 0.0));
    return launched();
  }

  DevBuf<double> pcg_part, pcg_tg;
  DevBuf<int> pcg_out;
  int pcg_blocks = 0;

  int pcg_persistent(const double* Tl, const double* rc, double dt, const double* b, double thr,
                     int max_iter, const double* dinv, double* x, int* iters,
                     int* converged) override {
    static const bool off = getenv("ST_CG_PERSISTENT") && getenv("ST_CG_PERSISTENT")[0] == '0';
    if (off) return ST_EUNSUPPORTED;
    if (!pcg_blocks) {
      int per_sm = 0, sms = 0;
      ST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persistent,
                                                            kPcgThreads, 0));
      ST_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      pcg_blocks = std::max(1, std::min(per_sm, 2) * sms);
      ST_TRY(pcg_part.alloc(4 * (size_t)pcg_blocks + 16));
      ST_TRY(pcg_out.alloc(2));
#ifdef ST_PCG_TIMING
      ST_CUDA(cudaMemsetAsync(pcg_part.p + 4 * (size_t)pcg_blocks, 0, 16 * sizeof(double),
                              c->stream));
#endif
    }
    PcgArgs a{};
    a.n = n;
    a.nv = nv;
    a.ns = ns;
    a.g = geo();
    a.nt = nodes();
    a.P = c->dp;
    a.Tl = Tl;
    a.rc = rc;
    a.rc_value = c->rc_value;
    a.dt = dt;
    a.slaves = slaves.p;
    a.sptr = sptr.p;
    a.smast = smast.p;
    a.sw = sw.p;
    a.b = b;
    a.dinv = dinv;
    a.x = x;
    ST_TRY(c->vec(1, &a.r));
    ST_TRY(c->vec(2, &a.z));
    ST_TRY(c->vec(3, &a.p0));
    ST_TRY(c->vec(9, &a.p1));
    ST_TRY(c->vec(4, &a.Ap));
    ST_TRY(c->vec(5, &a.vd));
    a.E = E.p;
    if ((int64_t)pcg_tg.n < 40 * n) ST_TRY(pcg_tg.alloc(40 * n));
    a.TG = pcg_tg.p;
    a.part = pcg_part.p;
    a.thr = thr;
    a.max_iter = max_iter;
    a.out = pcg_out.p;
    void* args[] = {&a};
    c->prof_begin();
    ST_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_persistent, dim3(pcg_blocks),
                                        dim3(kPcgThreads), args, 0, c->stream));
    c->prof_end();
    ST_TRY(launched());
    int h[2];
    ST_CUDA(cudaMemcpyAsync(h, pcg_out.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    ST_CUDA(cudaStreamSynchronize(c->stream));
    *iters = h[0];
    *converged = h[1];
#ifdef ST_PCG_TIMING
    {
      static long long total_it = 0;
      total_it += h[0];
      double ph[16];
      ST_CUDA(cudaMemcpy(ph, pcg_part.p + 4 * (size_t)pcg_blocks, sizeof(ph),
                         cudaMemcpyDeviceToHost));
      static const char* nm[12] = {"setup", "p/vd", "sync1", "cells", "sync2", "blocksum(pAp)",
                                   "sync3", "sum1", "update", "sync4", "sum2", "gather(thread 0)"};
      fprintf(stderr, "pcg phases, ns per iteration over %lld iterations:", total_it);
      for (int k = 0; k < 12; k++) fprintf(stderr, " %s %.0f", nm[k], ph[k] / (double)total_it);
      fprintf(stderr, "\n");
    }
#endif
    return ST_OK;
  }

  int jac_diag(const double* Tl, const double* rc, double dt, double* out) override {
    k_jdiag_cells<<<nblk(n), kThreads, 0, c->stream>>>(
        n, geo(), c->dp, Tl, rc, c->rc_value, dt,
        n_touched ? touched_pos.p : nullptr, E.p, Ae.p);
    ST_TRY(launched());
    k_gather<<<nblk(nv), kThreads, 0, c->stream>>>(nv, nodes(), E.p, out, nullptr, 0, 0.0);
    ST_TRY(launched());
    if (n_touched) {
      k_fold<<<nblk(nv), kThreads, 0, c->stream>>>(nv, fold_ptr.p, fold_ent.p, fold_w.p, Ae.p, out);
      ST_TRY(launched());
    }
    k_diag_fix<<<nblk(nv), kThreads, 0, c->stream>>>(nv, is_dir.p, is_slave.p, out);
    return launched();
  }

  double bytes_per_dof() const override {
    // T read + T' write + C^-1 read (8+8+8) + r_c read/write (2*64 per
    // cell) + cell_verts (32 per cell), SURVEY §8d config 3 accounting
    double cells_per_dof = (double)n / (double)(nv - ns);
    double b = 24.0 + cells_per_dof * 32.0;
    if (!c->rc_uniform) b += cells_per_dof * 128.0;
    return b;
  }
  const char* main_kernel() const override { return "k_rhs_cells"; }
};

int init_q1_constants() {
  static bool done = false;
  if (done) return ST_OK;
  // reference operators.py:30-36 (same expressions, same rounding)
  const double sq3 = std::sqrt(3.0);
  const double g[2] = {-1.0 / sq3, 1.0 / sq3};
  double V[2][2], D[2][2], U[2];
  for (int q = 0; q < 2; q++) {
    V[0][q] = (1.0 - g[q]) / 2.0;
    V[1][q] = (1.0 + g[q]) / 2.0;
    D[0][q] = -0.5;
    D[1][q] = 0.5;
    U[q] = (g[q] + 1.0) / 2.0;
  }
  double Phi[8][8], G[3][8][8], Phi2[8], GG[8][8];
  for (int c = 0; c < 8; c++) {
    int ix = (c >> 2) & 1, iy = (c >> 1) & 1, iz = c & 1;
    Phi2[c] = 0.0;
    for (int q = 0; q < 8; q++) {
      int qx = (q >> 2) & 1, qy = (q >> 1) & 1, qz = q & 1;
      Phi[c][q] = V[ix][qx] * V[iy][qy] * V[iz][qz];
      G[0][c][q] = D[ix][qx] * V[iy][qy] * V[iz][qz];
      G[1][c][q] = V[ix][qx] * D[iy][qy] * V[iz][qz];
      G[2][c][q] = V[ix][qx] * V[iy][qy] * D[iz][qz];
      Phi2[c] += Phi[c][q] * Phi[c][q];
      GG[c][q] = G[0][c][q] * G[0][c][q] + G[1][c][q] * G[1][c][q] + G[2][c][q] * G[2][c][q];
    }
  }
  ST_CUDA(cudaMemcpyToSymbol(cV, V, sizeof(V)));
  ST_CUDA(cudaMemcpyToSymbol(cD, D, sizeof(D)));
  ST_CUDA(cudaMemcpyToSymbol(cU, U, sizeof(U)));
  ST_CUDA(cudaMemcpyToSymbol(cPhi, Phi, sizeof(Phi)));
  ST_CUDA(cudaMemcpyToSymbol(cG, G, sizeof(G)));
  ST_CUDA(cudaMemcpyToSymbol(cPhi2, Phi2, sizeof(Phi2)));
  ST_CUDA(cudaMemcpyToSymbol(cGG, GG, sizeof(GG)));
  done = true;
  return ST_OK;
}

static int build_unstructured(Unstructured* u, Ctx* c, const st_unstructured_mesh* m) {
  const int64_t n = m->n_cells, nv = m->n_vertices, ns = m->n_slaves, nf = m->n_faces;
  if (n < 0 || nv <= 0 || ns < 0 || nf < 0 || (n > 0 && !m->cell_verts)) {
    set_error("invalid unstructured mesh description");
    return ST_EINVAL;
  }
  if (8 * n >= (int64_t)1 << 31) {
    set_error("unstructured backend limited to 2^28 cells");
    return ST_EUNSUPPORTED;
  }
  u->n = n;
  u->nv = nv;
  u->ns = ns;
  u->nf = nf;
  cudaStream_t s = c->stream;
  ST_TRY(init_q1_constants());
  for (int64_t i = 0; i < 8 * n; i++)
    if (m->cell_verts[i] < 0 || m->cell_verts[i] >= nv) {
      set_error("cell_verts out of range");
      return ST_EINVAL;
    }
  // vertex incidence CSR in canonical (cell, corner) order
  std::vector<int> ip(nv + 1, 0), ie(8 * n);
  for (int64_t i = 0; i < 8 * n; i++) ip[m->cell_verts[i] + 1]++;
  for (int64_t v = 0; v < nv; v++) ip[v + 1] += ip[v];
  {
    std::vector<int> fill(ip.begin(), ip.end() - 1);
    for (int64_t i = 0; i < 8 * n; i++) ie[fill[m->cell_verts[i]]++] = (int)i;
  }
  // condensation CSR per master, in np.add.at order of the (slave, master) pairs
  std::vector<int> cp(nv + 1, 0), cs;
  std::vector<double> cw;
  if (ns) {
    int64_t np_ = m->slave_ptr[ns];
    std::vector<int64_t> owner(np_);
    for (int64_t i = 0; i < ns; i++)
      for (int64_t p = m->slave_ptr[i]; p < m->slave_ptr[i + 1]; p++) owner[p] = i;
    for (int64_t p = 0; p < np_; p++) cp[m->slave_masters[p] + 1]++;
    for (int64_t v = 0; v < nv; v++) cp[v + 1] += cp[v];
    cs.resize(np_);
    cw.resize(np_);
    std::vector<int> fill(cp.begin(), cp.end() - 1);
    for (int64_t p = 0; p < np_; p++) {
      int64_t mm = m->slave_masters[p];
      cs[fill[mm]] = (int)m->slaves[owner[p]];
      cw[fill[mm]++] = m->slave_weights[p];
    }
  } else {
    cs.push_back(0);
    cw.push_back(0.0);
  }
  // the condensation flattened per master (gather_condensed): each folded
  // slave's incident entries in cond order, and the entry count per slave
  std::vector<int> cfp(nv + 1, 0), cfe, cgl(cs.size(), 0);
  for (int64_t v = 0; v < nv; v++) {
    cfp[v + 1] = cfp[v];
    if (!ns) continue;
    for (int i = cp[v]; i < cp[v + 1]; i++) {
      const int sl = cs[i];
      cgl[i] = ip[sl + 1] - ip[sl];
      for (int q = ip[sl]; q < ip[sl + 1]; q++) cfe.push_back(ie[q]);
      cfp[v + 1] += cgl[i];
    }
  }
  if (cfe.empty()) cfe.push_back(0);
  // per-cell face CSR (faces sorted by cell)
  std::vector<int> fp(n + 1, 0);
  for (int64_t f = 0; f < nf; f++) {
    int64_t cc = m->face_cell[f];
    if (cc < 0 || cc >= n || (f && m->face_cell[f - 1] > cc)) {
      set_error("face_cell must be sorted cell positions");
      return ST_EINVAL;
    }
    fp[cc + 1]++;
  }
  for (int64_t i = 0; i < n; i++) fp[i + 1] += fp[i];
  // det_w = (h/2)^3 with libm pow as numpy's ** (operators.py:106)
  std::vector<double> dw(n);
  for (int64_t i = 0; i < n; i++) dw[i] = std::pow(m->cell_h[i] / 2.0, 3.0);
  // fold tables for cells touching hanging vertices (operators.py:158-195)
  std::vector<int> tpos(n, -1);
  std::vector<int> fptr(nv + 1, 0), fent;
  std::vector<double> fw;
  int64_t nt = 0;
  if (ns) {
    std::map<int64_t, std::pair<std::vector<int64_t>, std::vector<double>>> expand;
    std::vector<uint8_t> sl(nv, 0);
    for (int64_t i = 0; i < ns; i++) {
      sl[m->slaves[i]] = 1;
      auto& e = expand[m->slaves[i]];
      for (int64_t p = m->slave_ptr[i]; p < m->slave_ptr[i + 1]; p++) {
        e.first.push_back(m->slave_masters[p]);
        e.second.push_back(m->slave_weights[p]);
      }
    }
    struct FE { int64_t m; int ent; double w; };
    std::vector<FE> ents;
    for (int64_t cc = 0; cc < n; cc++) {
      bool t = false;
      for (int a = 0; a < 8; a++) t |= sl[m->cell_verts[cc * 8 + a]] != 0;
      if (!t) continue;
      tpos[cc] = (int)nt;
      std::vector<int64_t> ms[8];
      std::vector<double> ws[8];
      for (int a = 0; a < 8; a++) {
        int64_t gv = m->cell_verts[cc * 8 + a];
        auto it = expand.find(gv);
        if (it == expand.end()) {
          ms[a] = {gv};
          ws[a] = {1.0};
        } else {
          // intersect1d works on sorted unique masters
          std::vector<std::pair<int64_t, double>> pr;
          for (size_t k = 0; k < it->second.first.size(); k++)
            pr.push_back({it->second.first[k], it->second.second[k]});
          std::sort(pr.begin(), pr.end(),
                    [](const std::pair<int64_t, double>& x, const std::pair<int64_t, double>& y) {
                      return x.first < y.first;
                    });
          for (auto& q : pr) {
            ms[a].push_back(q.first);
            ws[a].push_back(q.second);
          }
        }
      }
      for (int a = 0; a < 8; a++)
        for (int b = 0; b < 8; b++) {
          size_t i = 0, j = 0;
          while (i < ms[a].size() && j < ms[b].size()) {
            if (ms[a][i] == ms[b][j]) {
              ents.push_back({ms[a][i], (int)(nt * 64 + a * 8 + b), ws[a][i] * ws[b][j]});
              i++;
              j++;
            } else if (ms[a][i] < ms[b][j]) {
              i++;
            } else {
              j++;
            }
          }
        }
      nt++;
    }
    for (auto& e : ents) fptr[e.m + 1]++;
    for (int64_t v = 0; v < nv; v++) fptr[v + 1] += fptr[v];
    fent.resize(ents.size());
    fw.resize(ents.size());
    std::vector<int> fill(fptr.begin(), fptr.end() - 1);
    for (auto& e : ents) {
      fent[fill[e.m]] = e.ent;
      fw[fill[e.m]++] = e.w;
    }
  }
  if (fent.empty()) {
    fent.push_back(0);
    fw.push_back(0.0);
  }
  u->n_touched = nt;
  ST_TRY(u->cv.upload(m->cell_verts, 8 * n, s));
  ST_TRY(u->h.upload(m->cell_h, n, s));
  ST_TRY(u->anc.upload(m->cell_anchor, 3 * n, s));
  ST_TRY(u->detw.upload(dw.data(), n, s));
  ST_TRY(u->inc_ptr.upload(ip.data(), nv + 1, s));
  ST_TRY(u->inc_ent.upload(ie.data(), 8 * n, s));
  ST_TRY(u->cond_ptr.upload(cp.data(), nv + 1, s));
  ST_TRY(u->cond_s.upload(cs.data(), cs.size(), s));
  ST_TRY(u->cond_w.upload(cw.data(), cw.size(), s));
  ST_TRY(u->cfe_ptr.upload(cfp.data(), nv + 1, s));
  ST_TRY(u->cfe.upload(cfe.data(), cfe.size(), s));
  ST_TRY(u->cgl.upload(cgl.data(), cgl.size(), s));
  ST_TRY(u->face_ptr.upload(fp.data(), n + 1, s));
  if (nf) {
    ST_TRY(u->fvx.upload(m->face_vx, 4 * nf, s));
    ST_TRY(u->fvy.upload(m->face_vy, 4 * nf, s));
    ST_TRY(u->farea.upload(m->face_area, nf, s));
  }
  ST_TRY(u->is_slave.upload(m->is_slave, nv, s));
  ST_TRY(u->is_dir.upload(m->is_dirichlet, nv, s));
  if (ns) {
    ST_TRY(u->slaves.upload(m->slaves, ns, s));
    ST_TRY(u->sptr.upload(m->slave_ptr, ns + 1, s));
    ST_TRY(u->smast.upload(m->slave_masters, m->slave_ptr[ns], s));
    ST_TRY(u->sw.upload(m->slave_weights, m->slave_ptr[ns], s));
  }
  ST_TRY(u->touched_pos.upload(tpos.data(), n, s));
  ST_TRY(u->fold_ptr.upload(fptr.data(), nv + 1, s));
  ST_TRY(u->fold_ent.upload(fent.data(), fent.size(), s));
  ST_TRY(u->fold_w.upload(fw.data(), fw.size(), s));
  ST_TRY(u->E.alloc(8 * std::max<int64_t>(n, 1)));
  if (c->dp.latent) ST_TRY(u->Ec.alloc(8 * std::max<int64_t>(n, 1)));
  ST_TRY(u->Ae.alloc(64 * std::max<int64_t>(nt, 1)));
  ST_TRY(u->cinv.alloc(nv));
  // C^-1 cached per operator (operators.py:336-339)
  ST_TRY(u->capacity(nullptr, u->cinv.p));
  ST_TRY(vec_recip(c, u->cinv.p, u->cinv.p, nv));
  ST_CUDA(cudaStreamSynchronize(s));
  return ST_OK;
}

Backend* make_unstructured(Ctx* c, const st_unstructured_mesh* m, int* err) {
  Unstructured* u = new Unstructured();
  u->c = c;
  int rc = build_unstructured(u, c, m);
  if (rc != ST_OK) {
    delete u;
    *err = rc;
    return nullptr;
  }
  c->nv = m->n_vertices;
  c->n_cells = m->n_cells;
  c->qpc = 8;
  *err = ST_OK;
  return u;
}

}  // namespace st
