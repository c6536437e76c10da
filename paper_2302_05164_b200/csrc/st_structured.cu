// Structured backend: a uniform box of degree-p hexahedra (p = 1..4),
// nodes numbered x-major / z-fastest (reference rule mesh.py:712-715 on
// the p-refined lattice), GLL nodes, (p+1)^3 Gauss points.
//
// Hot kernel (k_xmarch): one CTA owns a (y, z) tile of CY x CZ cells and
// marches along x over a chunk of Lx cell layers; one thread per cell.
// Per cell layer the CTA
//   1. stages the p new node planes of T in shared memory (coalesced
//      along z, the contiguous axis),
//   2. evaluates every cell fully in registers with sum factorisation in
//      collocation form: T at the Gauss points (3 sweeps), grad T by the
//      Gauss-point differentiation matrix, k(T, r_c) per point
//      (material.py:46-85), fluxes accumulated back with the transposed
//      differentiation matrix, the Gaussian source added at the same
//      points (physics.py:154-171), one transposed interpolation (3
//      sweeps) to the element vector, plus the top-face radiation /
//      evaporation / convection term (operators.py:275-290),
//   3. sums the element vectors into shared node-plane accumulators in 4
//      conflict-free phases (deterministic within the CTA),
//   4. finalises the completed planes in the same pass: T' = T + dt C^-1 f
//      with the Dirichlet pin (operators.py:359-368), writes T', and folds
//      |T'| / max T' into the stability slots (timestepping.py:186-192).
// Nodes on tile seams (shared with another CTA) are sent with fp64
// atomics to a seam buffer and finalised by k_seams.
#include <cmath>
#include <vector>

#include "st_common.cuh"

namespace st {

constexpr int kMQ = 5;
__constant__ double sV[4][kMQ][kMQ];   // V[a][q]   nodal basis a at Gauss point q
__constant__ double sDq[4][kMQ][kMQ];  // Dq[m][q]: dT/dxi(q) = sum_m Dq[m][q] T(m)
__constant__ double sW[4][kMQ];        // Gauss weights
__constant__ double sU[4][kMQ];        // (x_q + 1) / 2
__constant__ double sM[4][kMQ];        // 1D lumped mass of node a: sum_q W_q V[a][q]

struct SArgs {
  int nx, ny, nz, NX, NY, NZ;
  int Lx;
  double h, hh, detw0;  // h, h/2, (h/2)^3
  double ox, oy, oz;    // origin (m)
  long long lx, ly, lz; // lattice origin (cells) when exact
  int use_lat;
  int dir_bottom, top_faces;
  int mode;  // 0: explicit step (out = T'), 1: rhs (out = f)
  int flags;
  double frozen_k;
  const double* T;
  double* out;
  const double* cinv;
  double* rc;
  double rc_value;
  int pending;
  double* fseam;
  double* cseam;
  int nb;
  const DevBeam* beams;
  double dt;
  DevParams P;
  unsigned long long* red;
};

template <int P>
__device__ __forceinline__ double coord(const SArgs& A, int axis, int cell, int q) {
  // qp coordinate = anchor + u_q h with anchor = lattice * h when the box
  // origin is on the lattice (one rounding, like the reference's
  // anchor * h_fine, operators.py:105-112)
  double anc;
  if (A.use_lat) {
    long long l = axis == 0 ? A.lx : (axis == 1 ? A.ly : A.lz);
    anc = (double)(cell + l) * A.h;
  } else {
    anc = (axis == 0 ? A.ox : (axis == 1 ? A.oy : A.oz)) + (double)cell * A.h;
  }
  return q < 0 ? anc : anc + sU[P - 1][q] * A.h;
}

// in-place 1D sweep along one axis of a Q^3 register tensor:
// out[.., q, ..] = sum_m M[m][q] in[.., m, ..]   (TR: M[q][m])
template <int P, int AX, bool TR>
__device__ __forceinline__ void sweep_v(double* t) {
  constexpr int Q = P + 1;
  constexpr int S = AX == 0 ? Q * Q : (AX == 1 ? Q : 1);
#pragma unroll
  for (int o1 = 0; o1 < Q; o1++)
#pragma unroll
    for (int o2 = 0; o2 < Q; o2++) {
      int base = AX == 0 ? (o1 * Q + o2) : (AX == 1 ? (o1 * Q * Q + o2) : (o1 * Q * Q + o2 * Q));
      double in[Q];
#pragma unroll
      for (int m = 0; m < Q; m++) in[m] = t[base + m * S];
#pragma unroll
      for (int q = 0; q < Q; q++) {
        double acc = (TR ? sV[P - 1][q][0] : sV[P - 1][0][q]) * in[0];
#pragma unroll
        for (int m = 1; m < Q; m++) acc = fma(TR ? sV[P - 1][q][m] : sV[P - 1][m][q], in[m], acc);
        t[base + q * S] = acc;
      }
    }
}

template <int P>
__device__ __forceinline__ void interp3(double* t) {
  sweep_v<P, 2, false>(t);
  sweep_v<P, 1, false>(t);
  sweep_v<P, 0, false>(t);
}
template <int P>
__device__ __forceinline__ void project3(double* t) {
  sweep_v<P, 0, true>(t);
  sweep_v<P, 1, true>(t);
  sweep_v<P, 2, true>(t);
}

struct CellFlags {
  bool diffusion, faces, source, frozen;
};

// Element vector of one cell (operators.py:247-316 generalised to degree
// P).  t: node values in, element vector out.  With LATENT, ec receives
// the apparent-capacity increment rho L/(dT) projected onto the nodes
// (zero unless a Gauss point lies in the latent interval).
template <int P, bool RCF, bool LATENT>
__device__ __forceinline__ void cell_element(const SArgs& A, const CellFlags& F, int i, int j,
                                             int k, int64_t cell, double* t, double* ec,
                                             bool& has_lat) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  const DevParams& PP = A.P;
  const bool top = F.faces && A.top_faces && (k == A.nz - 1);
  double tf[Q * Q];
  if (top) {
#pragma unroll
    for (int a = 0; a < Q; a++)
#pragma unroll
      for (int b = 0; b < Q; b++) tf[a * Q + b] = t[(a * Q + b) * Q + P];
  }
  interp3<P>(t);  // t now holds T at the Gauss points
  double G[Q3];
#pragma unroll
  for (int q = 0; q < Q3; q++) G[q] = 0.0;

  // beams hitting this cell (operators.py:295-307)
  unsigned hits = 0;
  if (F.source) {
    const double ax = coord<P>(A, 0, i, -1), ay = coord<P>(A, 1, j, -1), az = coord<P>(A, 2, k, -1);
    for (int b = 0; b < A.nb && b < 32; b++)
      if (beam_hits_cell(PP, A.beams[b], ax, ay, az, A.h)) hits |= 1u << b;
  }
  has_lat = false;
#pragma unroll
  for (int qa = 0; qa < Q; qa++)
#pragma unroll
    for (int qb = 0; qb < Q; qb++)
#pragma unroll
      for (int qc = 0; qc < Q; qc++) {
        const int q = (qa * Q + qb) * Q + qc;
        const double Tq = t[q];
        const double w3 = sW[P - 1][qa] * sW[P - 1][qb] * sW[P - 1][qc];
        if (F.diffusion) {
          double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
          for (int m = 0; m < Q; m++) {
            gx = fma(sDq[P - 1][m][qa], t[(m * Q + qb) * Q + qc], gx);
            gy = fma(sDq[P - 1][m][qb], t[(qa * Q + m) * Q + qc], gy);
            gz = fma(sDq[P - 1][m][qc], t[(qa * Q + qb) * Q + m], gz);
          }
          double kq;
          if (F.frozen) {
            kq = A.frozen_k;
          } else {
            const double g = liquid_fraction_fast(PP, Tq);
            double r;
            if (RCF) {
              r = A.rc[cell * Q3 + q];
              if (A.pending) {
                r = fmax(r, g);
                A.rc[cell * Q3 + q] = r;
              }
            } else {
              r = A.rc_value;
            }
            kq = conductivity(PP, g, r);
          }
          // w detJ (2/h)^2 = (h/2) w;  f_diff = - sum_d D_d^T (c D_d T)
          const double c = (A.hh * w3) * kq;
          const double fx = c * gx, fy = c * gy, fz = c * gz;
#pragma unroll
          for (int m = 0; m < Q; m++) {
            G[(m * Q + qb) * Q + qc] = fma(-sDq[P - 1][m][qa], fx, G[(m * Q + qb) * Q + qc]);
            G[(qa * Q + m) * Q + qc] = fma(-sDq[P - 1][m][qb], fy, G[(qa * Q + m) * Q + qc]);
            G[(qa * Q + qb) * Q + m] = fma(-sDq[P - 1][m][qc], fz, G[(qa * Q + qb) * Q + m]);
          }
        }
        if (hits) {
          const double x = coord<P>(A, 0, i, qa), y = coord<P>(A, 1, j, qb),
                       z = coord<P>(A, 2, k, qc);
          double s = 0.0;
          for (int b = 0; b < A.nb && b < 32; b++)
            if (hits & (1u << b)) s += beam_source(PP, A.beams[b], x, y, z);
          G[q] = fma(s, A.detw0 * w3, G[q]);
        }
      }
  project3<P>(G);
  if (LATENT) {
    // apparent-capacity increment at the Gauss points in the latent
    // interval (t still holds T_q; it is free afterwards)
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
#pragma unroll
        for (int qc = 0; qc < Q; qc++) {
          const int q = (qa * Q + qb) * Q + qc;
          const bool in = t[q] > PP.T_lat_s && t[q] < PP.T_lat_l;
          has_lat |= in;
          t[q] = in ? PP.lat_bump * (A.detw0 * (sW[P - 1][qa] * sW[P - 1][qb] * sW[P - 1][qc]))
                    : 0.0;
        }
    if (has_lat) {
      project3<P>(t);
#pragma unroll
      for (int q = 0; q < Q3; q++) ec[q] = t[q];
    }
  }
#pragma unroll
  for (int q = 0; q < Q3; q++) t[q] = G[q];
  if (top) {
    // facet quadrature on the +z face (operators.py:275-290), full facets
    double fq[Q * Q];
#pragma unroll
    for (int a = 0; a < Q * Q; a++) fq[a] = tf[a];
    // interpolate to face Gauss points: y then x
#pragma unroll
    for (int a = 0; a < Q; a++) {
      double in[Q];
#pragma unroll
      for (int b = 0; b < Q; b++) in[b] = fq[a * Q + b];
#pragma unroll
      for (int qb = 0; qb < Q; qb++) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < Q; b++) acc = fma(sV[P - 1][b][qb], in[b], acc);
        fq[a * Q + qb] = acc;
      }
    }
#pragma unroll
    for (int qb = 0; qb < Q; qb++) {
      double in[Q];
#pragma unroll
      for (int a = 0; a < Q; a++) in[a] = fq[a * Q + qb];
#pragma unroll
      for (int qa = 0; qa < Q; qa++) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < Q; a++) acc = fma(sV[P - 1][a][qa], in[a], acc);
        fq[qa * Q + qb] = acc;
      }
    }
    const double area0 = A.hh * A.hh;
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
        fq[qa * Q + qb] = surface_flux(PP, fq[qa * Q + qb]) *
                          (-(area0 * (sW[P - 1][qa] * sW[P - 1][qb])));
    // project back: x then y
#pragma unroll
    for (int qb = 0; qb < Q; qb++) {
      double in[Q];
#pragma unroll
      for (int qa = 0; qa < Q; qa++) in[qa] = fq[qa * Q + qb];
#pragma unroll
      for (int a = 0; a < Q; a++) {
        double acc = 0.0;
#pragma unroll
        for (int qa = 0; qa < Q; qa++) acc = fma(sV[P - 1][a][qa], in[qa], acc);
        fq[a * Q + qb] = acc;
      }
    }
#pragma unroll
    for (int a = 0; a < Q; a++) {
      double in[Q];
#pragma unroll
      for (int qb = 0; qb < Q; qb++) in[qb] = fq[a * Q + qb];
#pragma unroll
      for (int b = 0; b < Q; b++) {
        double acc = 0.0;
#pragma unroll
        for (int qb = 0; qb < Q; qb++) acc = fma(sV[P - 1][b][qb], in[qb], acc);
        t[(a * Q + b) * Q + P] += acc;
      }
    }
  }
}

// seam membership of node (I, J, K): shared with another CTA
__device__ __forceinline__ bool on_seam(const SArgs& A, int P, int CY, int CZ, int I, int J, int K) {
  const bool xs = I > 0 && I < A.NX - 1 && (I % (P * A.Lx)) == 0;
  const bool ys = J > 0 && J < A.NY - 1 && (J % (P * CY)) == 0;
  const bool zs = K > 0 && K < A.NZ - 1 && (K % (P * CZ)) == 0;
  return xs || ys || zs;
}

// finalise one node with its complete f (and latent capacity increment)
__device__ __forceinline__ double finalize_node(const SArgs& A, int64_t idx, int K, double T,
                                                double f, double dc, bool latent) {
  if (A.mode == 1) return f;
  double ci = A.cinv[idx];
  if (latent && dc != 0.0) ci = 1.0 / (1.0 / ci + dc);
  double o = T + A.dt * (ci * f);
  if (A.dir_bottom && K == 0) o = A.P.T_inf;
  return o;
}

template <int P, int CY, int CZ, bool LATENT, bool RCF>
__global__ void __launch_bounds__(CY* CZ) k_xmarch(SArgs A) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  constexpr int NYT = P * CY + 1, NZT = P * CZ + 1, PL = NYT * NZT;
  constexpr int NACC = LATENT ? 2 : 1;
  extern __shared__ double sm[];
  double* ring = sm;                // Q planes of T
  double* acc = sm + Q * PL;        // P planes of f (+ P of dC)
  const int tid = threadIdx.x;
  const int jl = tid / CZ, kl = tid % CZ;
  const int j0 = blockIdx.x * CY, k0 = blockIdx.y * CZ, i0 = blockIdx.z * A.Lx;
  if (i0 >= A.nx) return;
  const int i1 = min(i0 + A.Lx, A.nx);
  const int j = j0 + jl, k = k0 + kl;
  const bool live = j < A.ny && k < A.nz;
  const int Jn = min(P * CY, P * (A.ny - j0)) + 1;
  const int Kn = min(P * CZ, P * (A.nz - k0)) + 1;
  const CellFlags F{(A.flags & ST_RHS_DIFFUSION) != 0, (A.flags & ST_RHS_FACES) != 0,
                    (A.flags & ST_RHS_SOURCE) != 0 && A.nb > 0, (A.flags & ST_RHS_FROZEN_K) != 0};

  for (int t = tid; t < NACC * P * PL; t += CY * CZ) acc[t] = 0.0;
  auto load_plane = [&](int I) {
    double* dst = ring + (I % Q) * PL;
    const double* src = A.T + ((int64_t)I * A.NY + (int64_t)P * j0) * A.NZ + (int64_t)P * k0;
    for (int t = tid; t < Jn * Kn; t += CY * CZ) {
      int jj = t / Kn, kk = t - jj * Kn;
      dst[jj * NZT + kk] = src[(int64_t)jj * A.NZ + kk];
    }
  };
  double carry[Q * Q], carryC[LATENT ? Q * Q : 1];
#pragma unroll
  for (int q = 0; q < Q * Q; q++) carry[q] = 0.0;
  if (LATENT)
#pragma unroll
    for (int q = 0; q < Q * Q; q++) carryC[q] = 0.0;
  double amax = 0.0, smax = -INFINITY;
  bool bad = false;

  // finalise node plane I from accumulator plane a
  auto finalize_plane = [&](int I, int a) {
    const double* tp = ring + (I % Q) * PL;
    double* ap = acc + a * PL;
    double* cp = acc + (P + a) * PL;
    for (int t = tid; t < Jn * Kn; t += CY * CZ) {
      int jj = t / Kn, kk = t - jj * Kn;
      const int J = P * j0 + jj, K = P * k0 + kk;
      const int64_t idx = ((int64_t)I * A.NY + J) * A.NZ + K;
      const double f = ap[jj * NZT + kk];
      ap[jj * NZT + kk] = 0.0;
      double dc = 0.0;
      if (LATENT) {
        dc = cp[jj * NZT + kk];
        cp[jj * NZT + kk] = 0.0;
      }
      if (on_seam(A, P, CY, CZ, I, J, K)) {
        atomicAdd(A.fseam + idx, f);
        if (LATENT && dc != 0.0) atomicAdd(A.cseam + idx, dc);
      } else {
        const double o = finalize_node(A, idx, K, tp[jj * NZT + kk], f, dc, LATENT);
        A.out[idx] = o;
        amax = fmax(amax, fabs(o));
        smax = fmax(smax, o);
        bad |= (o != o);
      }
    }
  };

  // accumulate this thread's element planes a = 0..P-1 (e) into acc in 4
  // conflict-free phases; nodes of cells in the same phase never coincide
  auto accumulate = [&](const double* e, const double* ec, bool lat, int planes) {
#pragma unroll
    for (int ph = 0; ph < 4; ph++) {
      if (live && ((jl & 1) == (ph >> 1)) && ((kl & 1) == (ph & 1))) {
        for (int a = 0; a < planes; a++) {
#pragma unroll
          for (int b = 0; b < Q; b++)
#pragma unroll
            for (int c = 0; c < Q; c++) {
              const int s = a * PL + (P * jl + b) * NZT + (P * kl + c);
              acc[s] += e[(a * Q + b) * Q + c];
              if (LATENT && lat) acc[P * PL + s] += ec[(a * Q + b) * Q + c];
            }
        }
      }
      __syncthreads();
    }
  };

  load_plane(P * i0);
  for (int i = i0; i < i1; i++) {
#pragma unroll
    for (int a = 1; a <= P; a++) load_plane(P * i + a);
    __syncthreads();
    double t[Q3], ec[LATENT ? Q3 : 1];
    bool lat = false;
    if (live) {
#pragma unroll
      for (int a = 0; a < Q; a++) {
        const double* tp = ring + ((P * i + a) % Q) * PL;
#pragma unroll
        for (int b = 0; b < Q; b++)
#pragma unroll
          for (int c = 0; c < Q; c++) t[(a * Q + b) * Q + c] = tp[(P * jl + b) * NZT + P * kl + c];
      }
      const int64_t cell = ((int64_t)i * A.ny + j) * A.nz + k;
      if (LATENT)
#pragma unroll
        for (int q = 0; q < Q3; q++) ec[q] = 0.0;
      cell_element<P, RCF, LATENT>(A, F, i, j, k, cell, t, ec, lat);
      // x-face shared with the previous layer: add carry, keep the new one
#pragma unroll
      for (int q = 0; q < Q * Q; q++) {
        t[q] += carry[q];
        carry[q] = t[P * Q * Q + q];
      }
      if (LATENT) {
        if (lat) {
#pragma unroll
          for (int q = 0; q < Q * Q; q++) {
            ec[q] += carryC[q];
            carryC[q] = ec[P * Q * Q + q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < Q * Q; q++) {
            ec[q] = carryC[q];
            carryC[q] = 0.0;
          }
          lat = true;
#pragma unroll
          for (int q = Q * Q; q < Q3; q++) ec[q] = 0.0;
        }
      }
    }
    accumulate(t, ec, lat, P);
    for (int a = 0; a < P; a++) finalize_plane(P * i + a, a);
    __syncthreads();
  }
  // last node plane of the chunk: the carried x-face
  {
    double e[Q3];
#pragma unroll
    for (int q = 0; q < Q * Q; q++) e[q] = carry[q];
    double ecc[LATENT ? Q3 : 1];
    if (LATENT)
#pragma unroll
      for (int q = 0; q < Q * Q; q++) ecc[q] = carryC[q];
    accumulate(e, ecc, LATENT, 1);
    finalize_plane(P * i1, 0);
  }
  block_max2(bad ? (double)NAN : amax, smax, A.red);
}

// finalise the seam nodes (x planes, then y planes not on an x seam, then
// z planes on neither)
__global__ void k_seams(SArgs A, int P, int CY, int CZ, int nxs, int nys, int nzs, int latent) {
  const int64_t nxp = (int64_t)A.NY * A.NZ, nyp = (int64_t)A.NX * A.NZ, nzp = (int64_t)A.NX * A.NY;
  const int64_t tot = nxs * nxp + nys * nyp + nzs * nzp;
  double amax = 0.0, smax = -INFINITY;
  bool bad = false;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < tot;
       g += (int64_t)gridDim.x * blockDim.x) {
    int I, J, K;
    bool mine = true;
    if (g < nxs * nxp) {
      int s = (int)(g / nxp);
      int64_t r = g - s * nxp;
      I = P * A.Lx * (s + 1);
      J = (int)(r / A.NZ);
      K = (int)(r - (int64_t)J * A.NZ);
    } else if (g < nxs * nxp + nys * nyp) {
      int64_t h = g - nxs * nxp;
      int s = (int)(h / nyp);
      int64_t r = h - s * nyp;
      J = P * CY * (s + 1);
      I = (int)(r / A.NZ);
      K = (int)(r - (int64_t)I * A.NZ);
      mine = !(I > 0 && I < A.NX - 1 && (I % (P * A.Lx)) == 0);
    } else {
      int64_t h = g - nxs * nxp - nys * nyp;
      int s = (int)(h / nzp);
      int64_t r = h - s * nzp;
      K = P * CZ * (s + 1);
      I = (int)(r / A.NY);
      J = (int)(r - (int64_t)I * A.NY);
      mine = !(I > 0 && I < A.NX - 1 && (I % (P * A.Lx)) == 0) &&
             !(J > 0 && J < A.NY - 1 && (J % (P * CY)) == 0);
    }
    if (!mine) continue;
    const int64_t idx = ((int64_t)I * A.NY + J) * A.NZ + K;
    const double f = A.fseam[idx];
    A.fseam[idx] = 0.0;
    double dc = 0.0;
    if (latent) {
      dc = A.cseam[idx];
      A.cseam[idx] = 0.0;
    }
    const double o = finalize_node(A, idx, K, A.T[idx], f, dc, latent != 0);
    A.out[idx] = o;
    amax = fmax(amax, fabs(o));
    smax = fmax(smax, o);
    bad |= (o != o);
  }
  block_max2(bad ? (double)NAN : amax, smax, A.red);
}

// ---------------------------------------------------------------------------
// generic one-thread-per-cell kernels with fp64 atomics (per-call API and
// the implicit path on structured meshes; not the explicit hot loop)
// ---------------------------------------------------------------------------
__constant__ double sD[4][kMQ][kMQ];  // D[a][q] = l_a'(x_q) (reference-coordinate slope)

struct GArgs {
  int nx, ny, nz, NX, NY, NZ;
  double h, hh, detw0;
  const double* T;   // linearisation / state temperature
  const double* v;   // input vector (nullable)
  double* rc;
  double rc_value;
  double dt;
  double* out;
  DevParams P;
};

template <int P>
__device__ __forceinline__ void cell_nodes(const GArgs& A, int64_t cell, int64_t* ids) {
  constexpr int Q = P + 1;
  const int i = (int)(cell / ((int64_t)A.ny * A.nz));
  const int r = (int)(cell - (int64_t)i * A.ny * A.nz);
  const int j = r / A.nz, k = r - (r / A.nz) * A.nz;
#pragma unroll
  for (int a = 0; a < Q; a++)
#pragma unroll
    for (int b = 0; b < Q; b++)
#pragma unroll
      for (int c = 0; c < Q; c++)
        ids[(a * Q + b) * Q + c] = ((int64_t)(P * i + a) * A.NY + (P * j + b)) * A.NZ + (P * k + c);
}

// mode 0: history  r_c <- max(r_c, g(T_q))                (operators.py:219)
// mode 1: capacity  (v == null: ones) rho c_app(T_q) detJ   (operators.py:325)
// mode 2: mass      rho c detJ (V v)                         (operators.py:341)
// mode 3: J v       D + L + C/dt                             (operators.py:380)
// mode 4: diag J                                             (operators.py:426)
template <int P>
__global__ void k_sgeneric(GArgs A, int mode) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  const int64_t ncell = (int64_t)A.nx * A.ny * A.nz;
  const int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (cell >= ncell) return;
  int64_t ids[Q3];
  cell_nodes<P>(A, cell, ids);
  const DevParams& PP = A.P;
  double tq[Q3];
  if (A.T) {
#pragma unroll
    for (int q = 0; q < Q3; q++) tq[q] = A.T[ids[q]];
    interp3<P>(tq);
  }
  if (mode == 0) {
    if (!A.rc) return;
#pragma unroll
    for (int q = 0; q < Q3; q++)
      A.rc[cell * Q3 + q] = fmax(A.rc[cell * Q3 + q], liquid_fraction_fast(PP, tq[q]));
    return;
  }
  double G[Q3];
  if (mode == 1 || mode == 2) {
    double vq[Q3];
#pragma unroll
    for (int q = 0; q < Q3; q++) vq[q] = A.v ? A.v[ids[q]] : 1.0;
    interp3<P>(vq);
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
#pragma unroll
        for (int qc = 0; qc < Q; qc++) {
          const int q = (qa * Q + qb) * Q + qc;
          const double dw = A.detw0 * (sW[P - 1][qa] * sW[P - 1][qb] * sW[P - 1][qc]);
          const double rc = (mode == 1 && A.T) ? heat_capacity(PP, tq[q]) : PP.rhoc;
          G[q] = vq[q] * (rc * dw);
        }
    project3<P>(G);
#pragma unroll
    for (int q = 0; q < Q3; q++) atomicAdd(A.out + ids[q], G[q]);
    return;
  }
  // tangent at the Gauss points
  double kq[Q3], dkq[Q3];
#pragma unroll
  for (int q = 0; q < Q3; q++) {
    const double r = A.rc ? A.rc[cell * Q3 + q] : A.rc_value;
    kq[q] = conductivity(PP, liquid_fraction_fast(PP, tq[q]), r);
    dkq[q] = conductivity_derivative(PP, tq[q]);
  }
  const double gs = 2.0 / A.h;
  if (mode == 3) {
    double vq[Q3];
#pragma unroll
    for (int q = 0; q < Q3; q++) vq[q] = A.v[ids[q]];
    interp3<P>(vq);
#pragma unroll
    for (int q = 0; q < Q3; q++) G[q] = 0.0;
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
#pragma unroll
        for (int qc = 0; qc < Q; qc++) {
          const int q = (qa * Q + qb) * Q + qc;
          const double w3 = sW[P - 1][qa] * sW[P - 1][qb] * sW[P - 1][qc];
          double gv[3] = {0, 0, 0}, gt[3] = {0, 0, 0};
#pragma unroll
          for (int m = 0; m < Q; m++) {
            gv[0] = fma(sDq[P - 1][m][qa], vq[(m * Q + qb) * Q + qc], gv[0]);
            gv[1] = fma(sDq[P - 1][m][qb], vq[(qa * Q + m) * Q + qc], gv[1]);
            gv[2] = fma(sDq[P - 1][m][qc], vq[(qa * Q + qb) * Q + m], gv[2]);
            gt[0] = fma(sDq[P - 1][m][qa], tq[(m * Q + qb) * Q + qc], gt[0]);
            gt[1] = fma(sDq[P - 1][m][qb], tq[(qa * Q + m) * Q + qc], gt[1]);
            gt[2] = fma(sDq[P - 1][m][qc], tq[(qa * Q + qb) * Q + m], gt[2]);
          }
          const double c = (A.hh * w3) * kq[q];
          const double wl = (A.detw0 * w3) * gs * dkq[q] * vq[q] * gs;
          double fl[3];
#pragma unroll
          for (int d = 0; d < 3; d++) fl[d] = c * gv[d] + wl * gt[d];
#pragma unroll
          for (int m = 0; m < Q; m++) {
            G[(m * Q + qb) * Q + qc] = fma(sDq[P - 1][m][qa], fl[0], G[(m * Q + qb) * Q + qc]);
            G[(qa * Q + m) * Q + qc] = fma(sDq[P - 1][m][qb], fl[1], G[(qa * Q + m) * Q + qc]);
            G[(qa * Q + qb) * Q + m] = fma(sDq[P - 1][m][qc], fl[2], G[(qa * Q + qb) * Q + m]);
          }
          G[q] = fma(PP.rhoc * (A.detw0 * w3) / A.dt, vq[q], G[q]);
        }
    project3<P>(G);
#pragma unroll
    for (int q = 0; q < Q3; q++) atomicAdd(A.out + ids[q], G[q]);
    return;
  }
  // mode 4: element diagonal
  double gt[3][Q3];
#pragma unroll
  for (int q = 0; q < Q3; q++) {
    const int qa = q / (Q * Q), qb = (q / Q) % Q, qc = q % Q;
    gt[0][q] = gt[1][q] = gt[2][q] = 0.0;
#pragma unroll
    for (int m = 0; m < Q; m++) {
      gt[0][q] = fma(sDq[P - 1][m][qa], tq[(m * Q + qb) * Q + qc], gt[0][q]);
      gt[1][q] = fma(sDq[P - 1][m][qb], tq[(qa * Q + m) * Q + qc], gt[1][q]);
      gt[2][q] = fma(sDq[P - 1][m][qc], tq[(qa * Q + qb) * Q + m], gt[2][q]);
    }
  }
  for (int nd = 0; nd < Q3; nd++) {
    const int a = nd / (Q * Q), b = (nd / Q) % Q, c = nd % Q;
    double m_ = 0.0, d_ = 0.0, l_ = 0.0;
    for (int q = 0; q < Q3; q++) {
      const int qa = q / (Q * Q), qb = (q / Q) % Q, qc = q % Q;
      const double w3 = sW[P - 1][qa] * sW[P - 1][qb] * sW[P - 1][qc];
      const double phi = sV[P - 1][a][qa] * sV[P - 1][b][qb] * sV[P - 1][c][qc];
      const double g0 = sD[P - 1][a][qa] * sV[P - 1][b][qb] * sV[P - 1][c][qc];
      const double g1 = sV[P - 1][a][qa] * sD[P - 1][b][qb] * sV[P - 1][c][qc];
      const double g2 = sV[P - 1][a][qa] * sV[P - 1][b][qb] * sD[P - 1][c][qc];
      m_ += w3 * phi * phi;
      d_ += w3 * kq[q] * (g0 * g0 + g1 * g1 + g2 * g2);
      l_ += w3 * dkq[q] * phi * (g0 * gt[0][q] + g1 * gt[1][q] + g2 * gt[2][q]);
    }
    const double val = (PP.rhoc / A.dt) * A.detw0 * m_ + A.hh * d_ + A.detw0 * gs * gs * l_;
    atomicAdd(A.out + ids[nd], val);
  }
}

// C^-1 of the constant lumped capacity as a tensor product of 1D lumped
// masses (row sums of the consistent capacity, operators.py:325-334)
template <int P>
__global__ void k_cinv(int NX, int NY, int NZ, double rc_detw, double* out) {
  const int64_t n = (int64_t)NX * NY * NZ;
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= n) return;
  const int I = (int)(id / ((int64_t)NY * NZ));
  const int r = (int)(id - (int64_t)I * NY * NZ);
  const int J = r / NZ, K = r - (r / NZ) * NZ;
  auto m1 = [](int L, int N) {
    const int a = L % P;
    if (a != 0) return sM[P - 1][a];
    double s = 0.0;
    if (L > 0) s += sM[P - 1][P];
    if (L < N - 1) s += sM[P - 1][0];
    return s;
  };
  out[id] = 1.0 / (rc_detw * (m1(I, NX) * m1(J, NY) * m1(K, NZ)));
}

__global__ void k_pin_bottom(int64_t nplane, int NZ, double* v, double val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nplane) v[t * NZ] = val;
}

__global__ void k_jac_fix(int64_t nplane, int NZ, const double* v, double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nplane) out[t * NZ] = v[t * NZ];
}

// ---------------------------------------------------------------------------
// backend
// ---------------------------------------------------------------------------
static int init_struct_constants() {
  static bool done = false;
  if (done) return ST_OK;
  double V[4][kMQ][kMQ] = {}, D[4][kMQ][kMQ] = {}, Dq[4][kMQ][kMQ] = {}, W[4][kMQ] = {},
         U[4][kMQ] = {}, M[4][kMQ] = {};
  for (int p = 1; p <= 4; p++) {
    const int n = p + 1;
    long double xq[kMQ], wq[kMQ], xn[kMQ];
    if (p == 1) {
      // reference operators.py:30-36, same expressions
      const double s3 = std::sqrt(3.0);
      const double g[2] = {-1.0 / s3, 1.0 / s3};
      for (int q = 0; q < 2; q++) {
        V[0][0][q] = (1.0 - g[q]) / 2.0;
        V[0][1][q] = (1.0 + g[q]) / 2.0;
        D[0][0][q] = -0.5;
        D[0][1][q] = 0.5;
        W[0][q] = 1.0;
        U[0][q] = (g[q] + 1.0) / 2.0;
        xq[q] = g[q];
      }
      xn[0] = -1.0L;
      xn[1] = 1.0L;
    } else {
      // Gauss-Legendre by Newton on P_{n}; GLL nodes: +-1 and roots of P_p'
      for (int q = 0; q < n; q++) {
        long double x = cosl(M_PI * (q + 0.75L) / (n + 0.5L));
        for (int it = 0; it < 100; it++) {
          long double p0 = 1.0L, p1 = x;
          for (int l = 2; l <= n; l++) {
            long double p2 = ((2 * l - 1) * x * p1 - (l - 1) * p0) / l;
            p0 = p1;
            p1 = p2;
          }
          long double dp = n * (x * p1 - p0) / (x * x - 1.0L);
          long double dx = p1 / dp;
          x -= dx;
          if (fabsl(dx) < 1e-19L) break;
        }
        long double p0 = 1.0L, p1 = x;
        for (int l = 2; l <= n; l++) {
          long double p2 = ((2 * l - 1) * x * p1 - (l - 1) * p0) / l;
          p0 = p1;
          p1 = p2;
        }
        long double dp = n * (x * p1 - p0) / (x * x - 1.0L);
        xq[n - 1 - q] = x;
        wq[n - 1 - q] = 2.0L / ((1.0L - x * x) * dp * dp);
      }
      const long double gll[4][5] = {{-1, 1},
                                      {-1, 0, 1},
                                      {-1, -0.447213595499957939281834733746255247L,
                                       0.447213595499957939281834733746255247L, 1},
                                      {-1, -0.654653670707977143798292456246858356L, 0,
                                       0.654653670707977143798292456246858356L, 1}};
      for (int a = 0; a < n; a++) xn[a] = gll[p - 1][a];
      for (int q = 0; q < n; q++) {
        W[p - 1][q] = (double)wq[q];
        U[p - 1][q] = (double)((xq[q] + 1.0L) / 2.0L);
      }
      for (int a = 0; a < n; a++)
        for (int q = 0; q < n; q++) {
          long double val = 1.0L, der = 0.0L;
          for (int m = 0; m < n; m++)
            if (m != a) val *= (xq[q] - xn[m]) / (xn[a] - xn[m]);
          for (int l = 0; l < n; l++) {
            if (l == a) continue;
            long double term = 1.0L / (xn[a] - xn[l]);
            for (int m = 0; m < n; m++)
              if (m != a && m != l) term *= (xq[q] - xn[m]) / (xn[a] - xn[m]);
            der += term;
          }
          V[p - 1][a][q] = (double)val;
          D[p - 1][a][q] = (double)der;
        }
    }
    // Dq = V^-1 D (long double Gauss-Jordan)
    long double A[kMQ][2 * kMQ];
    for (int r = 0; r < n; r++)
      for (int c = 0; c < n; c++) {
        A[r][c] = V[p - 1][r][c];
        A[r][n + c] = (r == c) ? 1.0L : 0.0L;
      }
    for (int c = 0; c < n; c++) {
      int piv = c;
      for (int r = c + 1; r < n; r++)
        if (fabsl(A[r][c]) > fabsl(A[piv][c])) piv = r;
      for (int cc = 0; cc < 2 * n; cc++) std::swap(A[c][cc], A[piv][cc]);
      long double d = A[c][c];
      for (int cc = 0; cc < 2 * n; cc++) A[c][cc] /= d;
      for (int r = 0; r < n; r++)
        if (r != c) {
          long double f = A[r][c];
          for (int cc = 0; cc < 2 * n; cc++) A[r][cc] -= f * A[c][cc];
        }
    }
    for (int m = 0; m < n; m++)
      for (int q = 0; q < n; q++) {
        long double s = 0.0L;
        for (int a = 0; a < n; a++) s += A[m][n + a] * (long double)D[p - 1][a][q];
        Dq[p - 1][m][q] = (double)s;
      }
    for (int a = 0; a < n; a++) {
      long double s = 0.0L;
      for (int q = 0; q < n; q++) s += (long double)W[p - 1][q] * V[p - 1][a][q];
      M[p - 1][a] = (double)s;
    }
  }
  ST_CUDA(cudaMemcpyToSymbol(sV, V, sizeof(V)));
  ST_CUDA(cudaMemcpyToSymbol(sD, D, sizeof(D)));
  ST_CUDA(cudaMemcpyToSymbol(sDq, Dq, sizeof(Dq)));
  ST_CUDA(cudaMemcpyToSymbol(sW, W, sizeof(W)));
  ST_CUDA(cudaMemcpyToSymbol(sU, U, sizeof(U)));
  ST_CUDA(cudaMemcpyToSymbol(sM, M, sizeof(M)));
  done = true;
  return ST_OK;
}

template <int P>
struct Tile;
template <>
struct Tile<1> {
  static constexpr int CY = 8, CZ = 32;
};
template <>
struct Tile<2> {
  static constexpr int CY = 8, CZ = 16;
};
template <>
struct Tile<3> {
  static constexpr int CY = 8, CZ = 8;
};
template <>
struct Tile<4> {
  static constexpr int CY = 4, CZ = 8;
};

struct Structured : Backend {
  st_structured_mesh m{};
  int p = 1;
  int NX = 0, NY = 0, NZ = 0;
  int Lx = 1, cy = 8, cz = 8;
  int use_lat = 0;
  long long lx = 0, ly = 0, lz = 0;
  DevBuf<double> cinv, fseam, cseam;
  int64_t nv = 0;

  int launched() {
    c->launches++;
    ST_LAUNCHED();
    return ST_OK;
  }

  SArgs sargs() const {
    SArgs A{};
    A.nx = m.nx;
    A.ny = m.ny;
    A.nz = m.nz;
    A.NX = NX;
    A.NY = NY;
    A.NZ = NZ;
    A.Lx = Lx;
    A.h = m.h;
    A.hh = m.h / 2.0;
    A.detw0 = std::pow(m.h / 2.0, 3.0);
    A.ox = m.x0;
    A.oy = m.y0;
    A.oz = m.z0;
    A.lx = lx;
    A.ly = ly;
    A.lz = lz;
    A.use_lat = use_lat;
    A.dir_bottom = m.dirichlet_bottom;
    A.top_faces = m.top_faces;
    A.cinv = cinv.p;
    A.rc_value = c->rc_value;
    A.fseam = fseam.p;
    A.cseam = cseam.p;
    A.P = c->dp;
    return A;
  }

  GArgs gargs() const {
    GArgs A{};
    A.nx = m.nx;
    A.ny = m.ny;
    A.nz = m.nz;
    A.NX = NX;
    A.NY = NY;
    A.NZ = NZ;
    A.h = m.h;
    A.hh = m.h / 2.0;
    A.detw0 = std::pow(m.h / 2.0, 3.0);
    A.rc_value = c->rc_value;
    A.P = c->dp;
    return A;
  }

  template <int P, bool LAT, bool RCF>
  int launch_xmarch_t(const SArgs& A) {
    constexpr int CY = Tile<P>::CY, CZ = Tile<P>::CZ;
    constexpr int PL = (P * CY + 1) * (P * CZ + 1);
    const size_t smem = (size_t)((P + 1) * PL + (LAT ? 2 : 1) * P * PL) * sizeof(double);
    auto kern = k_xmarch<P, CY, CZ, LAT, RCF>;
    static bool attr = false;
    if (!attr) {
      ST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    dim3 grid((m.ny + CY - 1) / CY, (m.nz + CZ - 1) / CZ, (m.nx + Lx - 1) / Lx);
    kern<<<grid, CY * CZ, smem, c->stream>>>(A);
    return launched();
  }

  template <int P>
  int launch_xmarch_p(const SArgs& A, bool lat, bool rcf) {
    if (lat) return rcf ? launch_xmarch_t<P, true, true>(A) : launch_xmarch_t<P, true, false>(A);
    return rcf ? launch_xmarch_t<P, false, true>(A) : launch_xmarch_t<P, false, false>(A);
  }

  int xmarch(SArgs& A, bool rcf) {
    const bool lat = c->dp.latent != 0 && A.mode == 0;
    c->prof_begin();
    int rc;
    switch (p) {
      case 1: rc = launch_xmarch_p<1>(A, lat, rcf); break;
      case 2: rc = launch_xmarch_p<2>(A, lat, rcf); break;
      case 3: rc = launch_xmarch_p<3>(A, lat, rcf); break;
      default: rc = launch_xmarch_p<4>(A, lat, rcf); break;
    }
    c->prof_end();
    ST_TRY(rc);
    const int nxs = (m.nx + Lx - 1) / Lx - 1, nys = (m.ny + cy - 1) / cy - 1,
              nzs = (m.nz + cz - 1) / cz - 1;
    const int64_t tot = (int64_t)nxs * NY * NZ + (int64_t)nys * NX * NZ + (int64_t)nzs * NX * NY;
    if (tot > 0) {
      int blocks = (int)std::min<int64_t>((tot + kThreads - 1) / kThreads, 148 * 16);
      k_seams<<<blocks, kThreads, 0, c->stream>>>(A, p, cy, cz, nxs, nys, nzs, lat ? 1 : 0);
      ST_TRY(launched());
    }
    return ST_OK;
  }

  int rhs(const double* T, double* rc, int flags, double frozen_k, int nb,
          const DevBeam* beams, double* f, int pending) override {
    SArgs A = sargs();
    A.mode = 1;
    A.flags = flags;
    A.frozen_k = frozen_k;
    A.T = T;
    A.out = f;
    A.rc = rc;
    A.pending = pending;
    A.nb = (flags & ST_RHS_SOURCE) ? nb : 0;
    A.beams = beams;
    A.red = reinterpret_cast<unsigned long long*>(c->red.p + kRedBlocks + 64 + 2 * 1000);
    return xmarch(A, rc != nullptr && !(flags & ST_RHS_FROZEN_K));
  }

  int explicit_step(const double* T, double* rc, double dt, int nb, const DevBeam* beams,
                    double* Tout, int pending, double* red) override {
    SArgs A = sargs();
    A.mode = 0;
    A.flags = ST_RHS_DIFFUSION | ST_RHS_FACES | ST_RHS_SOURCE;
    A.T = T;
    A.out = Tout;
    A.rc = rc;
    A.pending = pending;
    A.nb = nb;
    A.beams = beams;
    A.dt = dt;
    A.red = reinterpret_cast<unsigned long long*>(red);
    return xmarch(A, rc != nullptr);
  }

  int generic(int mode, const double* T, const double* v, double* rc, double dt, double* out) {
    GArgs A = gargs();
    A.T = T;
    A.v = v;
    A.rc = rc;
    A.dt = dt;
    A.out = out;
    const int64_t n = (int64_t)m.nx * m.ny * m.nz;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (p) {
      case 1: k_sgeneric<1><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      case 2: k_sgeneric<2><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      case 3: k_sgeneric<3><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      default: k_sgeneric<4><<<blocks, 128, 0, c->stream>>>(A, mode); break;
    }
    return launched();
  }

  int history(const double* T, double* rc) override {
    if (!rc) return ST_OK;
    return generic(0, T, nullptr, rc, 0.0, nullptr);
  }

  int capacity(const double* T, double* out) override {
    if (!T || !c->dp.latent) {
      ST_TRY(vec_recip(c, cinv.p, out, nv));
      return ST_OK;
    }
    ST_CUDA(cudaMemsetAsync(out, 0, nv * sizeof(double), c->stream));
    return generic(1, T, nullptr, nullptr, 0.0, out);
  }

  int mass(const double* v, double* out) override {
    ST_CUDA(cudaMemsetAsync(out, 0, nv * sizeof(double), c->stream));
    return generic(2, nullptr, v, nullptr, 0.0, out);
  }

  int jacobian(const double* v, const double* Tl, const double* rc, double dt,
               double* out) override {
    double* vd;
    ST_TRY(c->vec(5, &vd));
    ST_CUDA(cudaMemcpyAsync(vd, v, nv * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    if (m.dirichlet_bottom) ST_TRY(pin_dirichlet(vd, 0.0));
    ST_CUDA(cudaMemsetAsync(out, 0, nv * sizeof(double), c->stream));
    c->prof_begin();
    ST_TRY(generic(3, Tl, vd, const_cast<double*>(rc), dt, out));
    c->prof_end();
    if (m.dirichlet_bottom) {
      const int64_t np_ = (int64_t)NX * NY;
      k_jac_fix<<<(unsigned)((np_ + 255) / 256), 256, 0, c->stream>>>(np_, NZ, v, out);
      ST_TRY(launched());
    }
    return ST_OK;
  }

  int jac_diag(const double* Tl, const double* rc, double dt, double* out) override {
    ST_CUDA(cudaMemsetAsync(out, 0, nv * sizeof(double), c->stream));
    ST_TRY(generic(4, Tl, nullptr, const_cast<double*>(rc), dt, out));
    if (m.dirichlet_bottom) ST_TRY(pin_dirichlet(out, 1.0));
    return ST_OK;
  }

  int distribute(double*) override { return ST_OK; }

  int mask_rows(double* v) override {
    if (m.dirichlet_bottom) return pin_dirichlet(v, 0.0);
    return ST_OK;
  }

  int pin_dirichlet(double* v, double value) override {
    if (!m.dirichlet_bottom) return ST_OK;
    const int64_t np_ = (int64_t)NX * NY;
    k_pin_bottom<<<(unsigned)((np_ + 255) / 256), 256, 0, c->stream>>>(np_, NZ, v, value);
    return launched();
  }

  double bytes_per_dof() const override {
    // T_n read + T_{n+1} write + C^-1 read, + r_c traffic
    // when the history is a stored field
    double b = 24.0;
    if (!c->rc_uniform) {
      const double q = (double)(p + 1) * (p + 1) * (p + 1);
      b += 16.0 * q * ((double)m.nx * m.ny * m.nz) / (double)nv;
    }
    return b;
  }
  const char* main_kernel() const override { return "k_xmarch"; }
};

static bool lattice_origin(double o, double h, long long* l) {
  double r = std::nearbyint(o / h);
  if (std::fabs(r * h - o) <= 1e-12 * std::max(h, std::fabs(o))) {
    *l = (long long)r;
    return true;
  }
  return false;
}

Backend* make_structured(Ctx* c, const st_structured_mesh* m, int* err) {
  if (!m || m->nx <= 0 || m->ny <= 0 || m->nz <= 0 || m->degree < 1 || m->degree > 4 ||
      !(m->h > 0)) {
    set_error("invalid structured mesh description");
    *err = ST_EINVAL;
    return nullptr;
  }
  if ((int64_t)m->degree * m->ny + 1 > (1 << 30) || (int64_t)m->degree * m->nz + 1 > (1 << 30)) {
    set_error("structured mesh too large");
    *err = ST_EUNSUPPORTED;
    return nullptr;
  }
  int rc = init_struct_constants();
  if (rc != ST_OK) {
    *err = rc;
    return nullptr;
  }
  Structured* s = new Structured();
  s->c = c;
  s->m = *m;
  s->p = m->degree;
  s->NX = m->degree * m->nx + 1;
  s->NY = m->degree * m->ny + 1;
  s->NZ = m->degree * m->nz + 1;
  s->nv = (int64_t)s->NX * s->NY * s->NZ;
  switch (s->p) {
    case 1: s->cy = Tile<1>::CY; s->cz = Tile<1>::CZ; break;
    case 2: s->cy = Tile<2>::CY; s->cz = Tile<2>::CZ; break;
    case 3: s->cy = Tile<3>::CY; s->cz = Tile<3>::CZ; break;
    default: s->cy = Tile<4>::CY; s->cz = Tile<4>::CZ; break;
  }
  // x chunk: enough CTAs for ~4 per SM on 148 SMs
  const int64_t nyz = (int64_t)((m->ny + s->cy - 1) / s->cy) * ((m->nz + s->cz - 1) / s->cz);
  const int64_t want = 4 * 148;
  int64_t chunks = std::max<int64_t>(1, (want + nyz - 1) / nyz);
  s->Lx = (int)std::max<int64_t>(4, (m->nx + chunks - 1) / chunks);
  s->Lx = std::min(s->Lx, m->nx);
  s->use_lat = lattice_origin(m->x0, m->h, &s->lx) && lattice_origin(m->y0, m->h, &s->ly) &&
               lattice_origin(m->z0, m->h, &s->lz);
  c->nv = s->nv;
  c->n_cells = (int64_t)m->nx * m->ny * m->nz;
  c->qpc = (s->p + 1) * (s->p + 1) * (s->p + 1);
  rc = s->cinv.alloc(s->nv);
  if (rc == ST_OK) rc = s->fseam.alloc(s->nv);
  if (rc == ST_OK && c->dp.latent) rc = s->cseam.alloc(s->nv);
  if (rc == ST_OK && cudaMemsetAsync(s->fseam.p, 0, s->nv * sizeof(double), c->stream) != cudaSuccess)
    rc = ST_ECUDA;
  if (rc == ST_OK && c->dp.latent &&
      cudaMemsetAsync(s->cseam.p, 0, s->nv * sizeof(double), c->stream) != cudaSuccess)
    rc = ST_ECUDA;
  if (rc == ST_OK) {
    const double rc_detw = c->dp.rhoc * std::pow(m->h / 2.0, 3.0);
    const unsigned blocks = (unsigned)((s->nv + 255) / 256);
    switch (s->p) {
      case 1: k_cinv<1><<<blocks, 256, 0, c->stream>>>(s->NX, s->NY, s->NZ, rc_detw, s->cinv.p); break;
      case 2: k_cinv<2><<<blocks, 256, 0, c->stream>>>(s->NX, s->NY, s->NZ, rc_detw, s->cinv.p); break;
      case 3: k_cinv<3><<<blocks, 256, 0, c->stream>>>(s->NX, s->NY, s->NZ, rc_detw, s->cinv.p); break;
      default: k_cinv<4><<<blocks, 256, 0, c->stream>>>(s->NX, s->NY, s->NZ, rc_detw, s->cinv.p); break;
    }
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) {
      set_error("structured setup kernels failed");
      rc = ST_ECUDA;
    }
  }
  if (rc != ST_OK) {
    delete s;
    *err = rc;
    return nullptr;
  }
  *err = ST_OK;
  return s;
}

}  // namespace st
