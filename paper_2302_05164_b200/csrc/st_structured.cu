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
//   3. stores the element planes entry-major in shared memory and each
//      thread gathers the <= 4 contributions of the nodes its cell owns in
//      a fixed order (deterministic),
//   4. finalises the completed planes in the same pass: T' = T + dt C^-1 f
//      with the Dirichlet pin (operators.py:359-368), writes T', and folds
//      |T'| / max T' into the stability slots (timestepping.py:186-192).
// Nodes on tile / chunk seams (shared with another CTA) store this CTA's
// partial with a plain store to its own slot of the seam buffer (slot =
// side of the CTA per seam axis); k_seam_list then sums the slots of every
// seam node in a fixed order and finalises it, so a step is bitwise
// reproducible.
// Explicit steps at p = 2 with a uniform history run k_xmarch2
// (st_xmarch2_kernel.cuh), the same scheme and arithmetic with the work
// around the cell evaluation rebuilt for instruction count (bitwise the same
// fields); Structured::xmarch picks the kernel per launch.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "st_structured.cuh"

namespace st {

__constant__ double sV[4][kMQ][kMQ];   // V[a][q]   nodal basis a at Gauss point q
__constant__ double sD[4][kMQ][kMQ];  // D[a][q] = l_a'(x_q) (reference-coordinate slope)
__constant__ double sDq[4][kMQ][kMQ];  // Dq[m][q]: dT/dxi(q) = sum_m Dq[m][q] T(m)
__constant__ double sW[4][kMQ];        // Gauss weights
__constant__ double sU[4][kMQ];        // (x_q + 1) / 2
__constant__ double sM[4][kMQ];        // 1D lumped mass of node a: sum_q W_q V[a][q]




// inverse 1D lumped mass, runtime degree (seam kernel)
__device__ __forceinline__ double inv_mass1_rt(const SArgs& A, int P, int L, int N) {
  const int a = L % P;
  if (a != 0) return A.imr[a];
  return (L == 0 || L == N - 1) ? A.imv_end : A.imv_int;
}

// Seam nodes as a static list (built once per context, st_structured.cu
// build_seam_list): entry e is node sidx[e] with a 16-bit code
//   bits 0-7  the slots (x side + 2 y side + 4 z side of the writing CTA)
//             this node has partials in,
//   bits 8-9  rank-interface side + 1 (0: none),
//   bit 10    bottom plane (Dirichlet),
// and its inverse lumped capacity sci[e] (host-computed with the hot
// kernel's expression).  The partials are summed in the fixed order of
// k_seams: x side outermost, then z side, then y side; a remote x side
// reads the neighbour rank's pre-summed plane.
// Seam pass over the static list: for each entry the (up to 8) slot
// partials are all loaded up front (predicated, 0 for slots the node does
// not have), then summed in the fixed order of the old per-plane pass: x
// side outermost, then z side, then y side (adding the exact zeros of
// absent slots does not change the sum).  A remote x side (rank interface)
// reads the neighbour rank's pre-summed plane instead of its slots.
template <bool LAT>
__global__ void __launch_bounds__(256) k_seam_list(SArgs A, int64_t n,
                                                   const int64_t* __restrict__ sidx,
                                                   const unsigned short* __restrict__ scode,
                                                   const double* __restrict__ sci) {
  // one entry per thread (measured: maximal parallelism beats batching
  // entries per thread); the loop form keeps U > 1 available
  constexpr int U = 1;
  double amax = 0.0, smax = -INFINITY;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool pair = LAT && A.seam_pair;
  for (int64_t eb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; eb < n; eb += U * stride) {
    int64_t idx[U];
    unsigned code[U];
    double ci[U], T[U], fv[U][8], cv[U][8];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t e = eb + u * stride;
      idx[u] = e < n ? sidx[e] : -1;
      code[u] = e < n ? scode[e] : 0u;
      ci[u] = e < n ? sci[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool in = idx[u] >= 0;
      T[u] = in ? A.T[idx[u]] : 0.0;
      const int side = (int)((code[u] >> 8) & 3u) - 1;
#pragma unroll
      for (int s = 0; s < 8; s++) {
        const int xb = s & 1;
        const bool use = in && ((code[u] >> s) & 1u) && xb != side;
        const int64_t so = (int64_t)s * A.snv + idx[u];
        fv[u][s] = 0.0;
        cv[u][s] = 0.0;
        if (use) {
          if (pair) {
            const double2 v = reinterpret_cast<const double2*>(A.fseam)[so];
            fv[u][s] = v.x;
            cv[u][s] = v.y;
          } else {
            fv[u][s] = A.fseam[so];
            if (LAT) cv[u][s] = A.cseam[so];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (idx[u] < 0) continue;
      const int side = (int)((code[u] >> 8) & 3u) - 1;
      double rf[2] = {0.0, 0.0}, rc[2] = {0.0, 0.0};
      if (side >= 0) {
        const int64_t o = side == 0 ? idx[u] : idx[u] - A.ioff_hi;
        rf[side] = A.irf[side][o];
        if (LAT) rc[side] = A.irc[side][o];
      }
      double f = 0.0, dc = 0.0;
#pragma unroll
      for (int xb = 0; xb < 2; xb++) {
        double sf_, sc_;
        if (xb == side) {
          sf_ = rf[xb];
          sc_ = rc[xb];
        } else {
          sf_ = ((fv[u][xb] + fv[u][xb + 2]) + fv[u][xb + 4]) + fv[u][xb + 6];
          sc_ = ((cv[u][xb] + cv[u][xb + 2]) + cv[u][xb + 4]) + cv[u][xb + 6];
        }
        f += sf_;
        dc += sc_;
      }
      const double o = finalize_node(A, ci[u], (code[u] & 1024u) != 0, T[u], f, dc, LAT);
      A.out[idx[u]] = o;
      amax = dmax(amax, fabs(o));
      smax = dmax(smax, o);
      bad |= (o != o);
    }
  }
  block_max2(bad ? (double)NAN : amax, smax, A.red);
}

// rank interface: this rank's pre-summed seam partials on local plane 0
// (it is the high x side there) or NX-1 (low side), in the same z-then-y
// slot order k_seams uses, so both ranks add bitwise the same numbers
__global__ void k_iface_pack(SArgs A, int P, int CY, int CZ, int side, int latent) {
  const int I = side == 0 ? 0 : A.NX - 1, xb = side == 0 ? 1 : 0;
  const int kmI = A.pkmin ? A.pkmin[I] : 0;
  const int sI = A.NZ - kmI;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)A.NY * sI) return;
  const int J = (int)(t / sI), K = kmI + (int)(t - (int64_t)(t / sI) * sI);
  const bool ys = J > 0 && J < A.NY - 1 && (J % (P * CY)) == 0;
  const bool zs = K > kmI && K < A.NZ - 1 && (K % (P * CZ)) == 0;
  const int64_t idx = (A.pbase ? A.pbase[I] : (int64_t)I * A.NY * A.NZ) + (int64_t)J * sI + K;
  double sf_ = 0.0, sc_ = 0.0;
  for (int zb = 0; zb <= (zs ? 1 : 0); zb++)
    for (int yb = 0; yb <= (ys ? 1 : 0); yb++) {
      seam_add(A, idx, xb + 2 * yb + 4 * zb, sf_, sc_, latent != 0);
    }
  A.ipf[side][t] = sf_;
  if (latent) A.ipc[side][t] = sc_;
}

// fitted part: inverse constant lumped capacity of every node (row sums
// over the active cells around it; operators.py:325-339), plane I =
// blockIdx.y
template <int P>
__global__ void k_fit_cinv(SArgs A, const int* xext, double rc_detw, double* out) {
  const int I = blockIdx.y;
  const int kmI = A.pkmin[I];
  const int sI = A.NZ - kmI;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)A.NY * sI) return;
  const int J = (int)(t / sI), K = kmI + (int)(t - (int64_t)(t / sI) * sI);
  auto m1y = [&](int L, int N) {
    const int a = L % P;
    if (a != 0) return sM[P - 1][a];
    double s = 0.0;
    if (L > 0) s += sM[P - 1][P];
    if (L < N - 1) s += sM[P - 1][0];
    return s;
  };
  // (x, z) cells around the node, each with the node's 1D masses in it
  double mxz = 0.0;
  const int ax = I % P, az = K % P;
  for (int dx = 0; dx < (ax != 0 ? 1 : 2); dx++) {
    const int i = ax != 0 ? I / P : I / P - 1 + dx;
    const double wx = ax != 0 ? sM[P - 1][ax] : sM[P - 1][dx == 0 ? P : 0];
    for (int dz = 0; dz < (az != 0 ? 1 : 2); dz++) {
      const int k = az != 0 ? K / P : K / P - 1 + dz;
      const double wz = az != 0 ? sM[P - 1][az] : sM[P - 1][dz == 0 ? P : 0];
      if (i >= 0 && k >= 0 && k < A.nz && i < xext[k]) mxz += wx * wz;
    }
  }
  out[A.pbase[I] + (int64_t)J * sI + K] = 1.0 / (rc_detw * (m1y(J, A.NY) * mxz));
}

// fitted part: bottom node plane (rows K = 0 of the planes that reach it);
// mode 0: out = val there, mode 1: out = v there
__global__ void k_fit_pin(SArgs A, int mode, const double* v, double* out, double val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)A.NX * A.NY) return;
  const int I = (int)(t / A.NY), J = (int)(t - (int64_t)I * A.NY);
  if (A.pkmin[I] != 0) return;
  const int64_t idx = A.pbase[I] + (int64_t)J * A.NZ;
  out[idx] = mode == 0 ? val : v[idx];
}

// ---------------------------------------------------------------------------
// generic one-thread-per-cell kernels (per-call API and the implicit path
// on structured meshes; not the explicit hot loop): element vectors to a
// buffer, then a fixed-order node gather (k_sgather) -- deterministic
// ---------------------------------------------------------------------------

struct GArgs {
  int nx, ny, nz, NX, NY, NZ;
  double h, hh, detw0;
  const double* T;   // linearisation / state temperature
  const double* v;   // input vector (nullable)
  double* rc;
  double rc_value;
  double dt;
  double* out;
  double* E;  // element vectors (n_cells x (p+1)^3), gathered per node by k_sgather
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
    for (int q = 0; q < Q3; q++) A.E[cell * Q3 + q] = G[q];
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
    for (int q = 0; q < Q3; q++) A.E[cell * Q3 + q] = G[q];
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
    A.E[cell * Q3 + nd] = val;
  }
}

// node sums of the element vectors of k_sgeneric in a fixed order (cells
// low before high in x, then y, then z): deterministic, no atomics
template <int P>
__global__ void k_sgather(GArgs A, const double* __restrict__ E, double* out) {
  constexpr int Q = P + 1;
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= (int64_t)A.NX * A.NY * A.NZ) return;
  const int I = (int)(id / ((int64_t)A.NY * A.NZ));
  const int r = (int)(id - (int64_t)I * A.NY * A.NZ);
  const int J = r / A.NZ, K = r - (r / A.NZ) * A.NZ;
  double acc = 0.0;
#pragma unroll
  for (int dx = 0; dx < 2; dx++) {
    const int i = (I % P) ? I / P : I / P - 1 + dx;
    if ((I % P && dx) || i < 0 || i >= A.nx) continue;
#pragma unroll
    for (int dy = 0; dy < 2; dy++) {
      const int j = (J % P) ? J / P : J / P - 1 + dy;
      if ((J % P && dy) || j < 0 || j >= A.ny) continue;
#pragma unroll
      for (int dz = 0; dz < 2; dz++) {
        const int k = (K % P) ? K / P : K / P - 1 + dz;
        if ((K % P && dz) || k < 0 || k >= A.nz) continue;
        const int64_t cell = ((int64_t)i * A.ny + j) * A.nz + k;
        acc += E[cell * (Q * Q * Q) + ((I - P * i) * Q + (J - P * j)) * Q + (K - P * k)];
      }
    }
  }
  out[id] = acc;
}

// C^-1 of the constant lumped capacity as a tensor product of 1D lumped
// masses (row sums of the consistent capacity, operators.py:325-334)
// lumped apparent capacity floored at the constant one (finalize_node)
__global__ void k_cap_floor(int64_t n, const double* cinv, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double c0 = 1.0 / cinv[i];
    out[i] = out[i] > c0 ? out[i] : c0;
  }
}

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

// 1D lumped mass of local node a at degree p (host)
static double host_m1(int p, int a) {
  switch (p) {
    case 1: return Basis<1>::M(a);
    case 2: return Basis<2>::M(a);
    case 3: return Basis<3>::M(a);
    default: return Basis<4>::M(a);
  }
}

struct Structured : Backend {
  ~Structured() override {
    if (latstat_h) cudaFreeHost(latstat_h);
    if (lat_ev) cudaEventDestroy(lat_ev);
    for (auto& e : ev_hot)
      if (e) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_seams) cudaEventDestroy(ev_seams);
    if (hot_s) cudaStreamDestroy(hot_s);
    if (seam_s) cudaStreamDestroy(seam_s);
  }
  st_structured_mesh m{};
  // fitted part (m.xext != NULL): per cell row x extent, per node plane
  // lowest row and first-node base, per tile row x extent
  bool fitted = false;
  std::vector<int> xext_h, kmin_h, text_h;
  std::vector<int64_t> base_h;
  DevBuf<int64_t> pbase_d;
  DevBuf<int> pkmin_d, text_d, xext_d;
  int p = 1;
  int NX = 0, NY = 0, NZ = 0;
  int Lx = 1, cy = 8, cz = 8;
  bool slab = false;  // k_xslab (p+1 threads per cell) instead of k_xmarch
  int use_lat = 0;
  long long lx = 0, ly = 0, lz = 0;
  DevBuf<double> cinv, fseam, cseam, lcarry, ecg, packf[2], packc[2];
  DevBuf<double> Eg;  // element vectors of the generic (implicit-path) kernels
  // seam lists (k_seam_list): [0] every seam node (the general kernels;
  // built when first needed), [1] only the nodes k_xmarch2 leaves to the
  // pass when it completes the ordinary planes' seams itself (x-seam planes
  // and rank interfaces)
  struct SeamList {
    DevBuf<int64_t> sidx;
    DevBuf<unsigned short> scode;
    DevBuf<double> sci;
    int64_t n = 0;
    bool built = false;
    // entries on node planes <= I (the list is in node order, so the seam
    // nodes of a range of planes are a contiguous range of entries)
    std::vector<int64_t> plane_end;
  } slist[2];
  // pipelined seam pass (xmarch_piped): the x chunks go out as groups of
  // launches alternating between the library stream and hot_s, and the seam
  // entries of a group's planes run on the high-priority seam_s as soon as
  // the groups that write them are done, under the later groups' cells
  static constexpr int kMaxPipe = 16;
  cudaStream_t hot_s = nullptr, seam_s = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_seams = nullptr, ev_hot[kMaxPipe] = {};
  int pipe_groups = 0;  // 0: off
  double pipe_min_waves = 2.0;  // least waves of CTAs per group (ST_SEAM_PIPE_MINWAVES)
  int64_t hot_slots = 444;  // resident CTAs of the hot kernel on the device
  // latent-dense fields (every tile gathers latent increments in most
  // layers, e.g. config 2's random field): k_xmarch2 keeps the increments in
  // an L2 scratch and loses to the general kernel's shared-memory copy there,
  // so the kernels count their latent CTA-layers and the host, reading the
  // counter asynchronously every few steps, picks the kernel (both give
  // bitwise the same field)
  DevBuf<unsigned long long> latstat;
  unsigned long long* latstat_h = nullptr;  // pinned
  cudaEvent_t lat_ev = nullptr;
  bool lat_pending = false, prefer_general = false;
  bool last_x2 = false;  // the last hot launch was k_xmarch2 (main_kernel)
  unsigned long long lat_seen = 0;
  double lat_launched = 0.0, lat_launched_rec = 0.0, lat_launched_seen = 0.0;
  int lat_calls = 0;
  DevBuf<int> seamcnt;  // arrival counters of k_xmarch2's in-kernel seam completion
  int GY = 0, GZ = 0;
  bool inseam = false;  // k_xmarch2 completes ordinary-plane seams in the kernel
  int64_t nv = 0;

  // nodes of node plane I
  int64_t plane_n(int I) const { return (int64_t)NY * (NZ - (fitted ? kmin_h[I] : 0)); }

  int unsupported_fitted(const char* what) const {
    set_error(std::string(what) + " is not available on a fitted part (explicit steps and "
              "evaluate_rhs with a uniform history are)");
    return ST_EUNSUPPORTED;
  }

  // (f, dc) pairs in fseam (one 16-byte access per slot entry): k_xslab and
  // the k_xmarch / k_xmarch2 contexts (p <= 2) with latent heat (config 4:
  // step 16.4 -> 15.2 ms, config 2 at p = 1: 2.54 -> 2.47 ms);
  // ST_SEAM_PAIR=0: split arrays
  bool seam_pairs() const {
    if (!c->dp.latent) return false;
    if (slab) return true;
    const char* e = getenv("ST_SEAM_PAIR");
    return p <= 2 && !(e && e[0] == '0');
  }

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
    A.seam_pair = seam_pairs() ? 1 : 0;
    A.lcarry = lcarry.p;
    A.ecg = ecg.p;
    A.latstat = latstat.p;
    A.seamcnt = inseam ? seamcnt.p : nullptr;
    A.GY = GY;
    A.GZ = GZ;
    A.m1_0 = host_m1(p, 0);
    A.m1_p = host_m1(p, p);
    A.snv = nv;
    for (int sd = 0; sd < 2; sd++) {
      A.ipf[sd] = packf[sd].p;
      A.ipc[sd] = packc[sd].p;
      A.irf[sd] = nullptr;
      A.irc[sd] = nullptr;
    }
    A.P = c->dp;
    const DevParams& d = c->dp;
    A.kA = (1.0 - c->rc_value) * d.k_p + c->rc_value * d.k_s;
    A.kB = d.k_m - d.k_s;
    A.mhh = -(m.h / 2.0);
    A.kAh = A.mhh * A.kA;
    A.kBh = A.mhh * A.kB;
    A.glo = -d.T_s * d.inv_dT_l;
    A.lat_mid = 0.5 * (d.T_lat_s + d.T_lat_l);
    A.lat_half = 0.5 * (d.T_lat_l - d.T_lat_s);
    {
      // high words of the interval ends, widened by one (k_xmarch2's
      // candidate window; positive temperatures)
      auto hiword = [](double x) {
        long long b;
        memcpy(&b, &x, 8);
        return (int)(b >> 32);
      };
      A.lat_hi0 = hiword(A.lat_mid - A.lat_half) - 1;
      A.lat_hiw = hiword(A.lat_mid + A.lat_half) + 1 - A.lat_hi0;
    }
    const int q = p + 1;
    std::vector<double> w(q), m1(q);
    switch (p) {
      case 1: for (int i = 0; i < q; i++) { w[i] = Basis<1>::W(i); m1[i] = Basis<1>::M(i); } break;
      case 2: for (int i = 0; i < q; i++) { w[i] = Basis<2>::W(i); m1[i] = Basis<2>::M(i); } break;
      case 3: for (int i = 0; i < q; i++) { w[i] = Basis<3>::W(i); m1[i] = Basis<3>::M(i); } break;
      default: for (int i = 0; i < q; i++) { w[i] = Basis<4>::W(i); m1[i] = Basis<4>::M(i); } break;
    }
    A.inv_rcdw = 1.0 / (d.rhoc * A.detw0);
    for (int a = 0; a < 5; a++) A.imr[a] = (a > 0 && a < p) ? 1.0 / m1[a] : 0.0;
    A.imv_int = 1.0 / (m1[0] + m1[p]);
    A.imv_end = 1.0 / m1[0];
    A.gI0 = m.gNX > 0 ? m.gx0 : 0;
    A.gNX = m.gNX > 0 ? m.gNX : NX;
    A.iface_lo = m.iface_lo ? 1 : 0;
    A.iface_hi = m.iface_hi ? 1 : 0;
    A.pbase = fitted ? pbase_d.p : nullptr;
    A.pkmin = fitted ? pkmin_d.p : nullptr;
    A.text = fitted ? text_d.p : nullptr;
    A.ioff_hi = fitted ? base_h[NX - 1] + kmin_h[NX - 1] : (int64_t)(NX - 1) * NY * NZ;
    for (int a = 0; a < q; a++)
      for (int b = 0; b < q; b++)
        for (int cc = 0; cc < q; cc++) {
          const double w3 = w[a] * w[b] * w[cc];
          A.hw3[(a * q + b) * q + cc] = A.hh * w3;
          A.lw3[(a * q + b) * q + cc] = d.lat_bump * (A.detw0 * w3);
        }
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

  // resident CTAs per SM of the hot kernel this context launches
  int resident(bool lat) const {
    switch (p) {
      case 1: return hot_resident<1>(slab, lat);
      case 2: return hot_resident<2>(slab, lat);
      case 3: return hot_resident<3>(slab, lat);
      default: return hot_resident<4>(slab, lat);
    }
  }

  // seam pass over the entries [e0, e1) of the context's list (e1 < 0: all)
  int seams(SArgs& A, int64_t e0 = 0, int64_t e1 = -1, cudaStream_t stream = nullptr) {
    const bool lat = c->dp.latent != 0 && A.mode == 0;
    const int which = (A.x2 && A.seamcnt) ? 1 : 0;
    if (!slist[which].built) ST_TRY(build_seam_list(which));
    const SeamList& L = slist[which];
    if (e1 < 0) e1 = L.n;
    if (!stream) stream = c->stream;
    const int64_t n = e1 - e0;
    if (n > 0) {
      // one thread per seam node: the pass is latency bound
      constexpr int kSB = 128;  // measured a hair faster than 256
      const unsigned grid = (unsigned)((n + kSB - 1) / kSB);
      if (lat)
        k_seam_list<true><<<grid, kSB, 0, stream>>>(A, n, L.sidx.p + e0, L.scode.p + e0,
                                                    L.sci.p + e0);
      else
        k_seam_list<false><<<grid, kSB, 0, stream>>>(A, n, L.sidx.p + e0, L.scode.p + e0,
                                                     L.sci.p + e0);
      ST_TRY(launched());
    }
    return ST_OK;
  }

  // static seam-node list (see k_seam_list), in node order.  A node is a
  // seam when two or more CTAs (tile row t, tile column u, x chunk c)
  // write it: each CTA owns the closed node box of its cells and stores
  // its partial of a shared node to slot (first plane of a chunk c > 0
  // or a low rank interface) + 2 (first column of a tile u > 0) + 4
  // (first row of a tile row t > 0 with material below), exactly the
  // hot kernel's rule; the list records which slots each node has.
  // which = 1: only the nodes with an x seam among their contributors (a
  // tile row with two x chunks at the node's plane) or on a rank interface
  int build_seam_list(int which) {
    const bool xonly = which == 1;
    const int sx = p * Lx, sy = p * cy, sz = p * cz;
    const int nty = (m.ny + cy - 1) / cy, ntz = (m.nz + cz - 1) / cz;
    auto ext_t = [&](int t) { return fitted ? text_h[t] : m.nx; };
    auto kmin_of = [&](int I) { return fitted ? kmin_h[I] : 0; };
    auto base_of = [&](int I) { return fitted ? base_h[I] : (int64_t)I * NY * NZ; };
    auto ext_row = [&](int k) { return fitted ? xext_h[k] : m.nx; };
    const SArgs A = sargs();
    double M1[5] = {};
    for (int a = 0; a <= p; a++) M1[a] = host_m1(p, a);
    auto im1 = [&](int L, int N) {  // inverse 1D lumped mass on a full line
      const int a = L % p;
      if (a != 0) return A.imr[a];
      return (L == 0 || L == N - 1) ? A.imv_end : A.imv_int;
    };
    std::vector<char> xcand(NX, 0);
    for (int I = 0; I < NX; I++)
      for (int t = 0; t < ntz; t++)
        if (I > 0 && I % sx == 0 && I < p * ext_t(t)) xcand[I] = 1;
    if (m.iface_lo) xcand[0] = 1;
    if (m.iface_hi) xcand[NX - 1] = 1;
    std::vector<int64_t> idx;
    std::vector<unsigned short> code;
    std::vector<double> ci;
    auto visit = [&](int I, int J, int K, int kmI) {
      int tl[2], nt = 0, ul[2], nu = 0;
      for (int t : {K / sz - ((K % sz == 0 && K > 0) ? 1 : 0), K / sz}) {
        if (t < 0 || t >= ntz || (nt && tl[nt - 1] == t)) continue;
        if (t * sz <= K && K <= p * std::min((t + 1) * cz, m.nz) && I <= p * ext_t(t)) tl[nt++] = t;
      }
      for (int u : {J / sy - ((J % sy == 0 && J > 0) ? 1 : 0), J / sy}) {
        if (u < 0 || u >= nty || (nu && ul[nu - 1] == u)) continue;
        if (u * sy <= J && J <= p * std::min((u + 1) * cy, m.ny)) ul[nu++] = u;
      }
      unsigned mask = 0;
      int count = 0;
      bool xany = false;
      for (int a = 0; a < nt; a++) {
        const int t = tl[a], ext = ext_t(t);
        int cl[2], nc = 0;
        for (int cc : {I / sx - ((I % sx == 0 && I > 0) ? 1 : 0), I / sx}) {
          if (cc < 0 || (nc && cl[nc - 1] == cc)) continue;
          if (cc * Lx < ext && cc * sx <= I && I <= p * std::min((cc + 1) * Lx, ext)) cl[nc++] = cc;
        }
        xany |= nc == 2;
        for (int b = 0; b < nu; b++)
          for (int e = 0; e < nc; e++) {
            const int bit = ((I == cl[e] * sx && (cl[e] > 0 || m.iface_lo)) ? 1 : 0) +
                            ((J == ul[b] * sy && ul[b] > 0) ? 2 : 0) +
                            ((K == t * sz && t > 0 && kmI < K) ? 4 : 0);
            mask |= 1u << bit;
            count++;
          }
      }
      const int side = (I == 0 && m.iface_lo) ? 0 : ((I == NX - 1 && m.iface_hi) ? 1 : -1);
      if (count < 2 && side < 0) return;
      if (xonly && !xany && side < 0) return;
      idx.push_back(base_of(I) + (int64_t)J * (NZ - kmI) + K);
      code.push_back((unsigned short)(mask | ((side + 1) << 8) | (K == 0 ? 1024 : 0)));
      // inverse lumped capacity: the hot kernel's tensor product where the
      // active (x, z) cells around the node form a rectangle, else the row
      // sum over the cells present (re-entrant edge of a fitted part)
      const int ax = I % p, az = K % p;
      bool pres[2][2] = {};
      int npres = 0;
      for (int dx = 0; dx < (ax ? 1 : 2); dx++)
        for (int dz = 0; dz < (az ? 1 : 2); dz++) {
          const int i = ax ? I / p : I / p - 1 + dx, k = az ? K / p : K / p - 1 + dz;
          bool on = k >= 0 && k < m.nz && i >= 0 && i < ext_row(k);
          if (k >= 0 && k < m.nz && i < 0 && m.iface_lo) on = true;
          if (k >= 0 && k < m.nz && i >= m.nx && m.iface_hi && ext_row(k) == m.nx) on = true;
          pres[dx][dz] = on;
          npres += on;
        }
      const int nxs = ax ? 1 : 2, nzs = az ? 1 : 2;
      bool rect = true;
      for (int dx = 0; dx < nxs; dx++)
        for (int dz = 0; dz < nzs; dz++) {
          bool anyx = false, anyz = false;
          for (int e = 0; e < nzs; e++) anyx |= pres[dx][e];
          for (int e = 0; e < nxs; e++) anyz |= pres[e][dz];
          if (anyx && anyz && !pres[dx][dz]) rect = false;
        }
      const double my = im1(J, NY);
      if (rect) {
        auto side_inv = [&](int a, bool lo, bool hi) {
          if (a) return A.imr[a];
          return (lo && hi) ? A.imv_int : A.imv_end;
        };
        bool xlo = false, xhi = false, zlo = false, zhi = false;
        for (int dz = 0; dz < nzs; dz++) {
          xlo |= pres[0][dz];
          if (nxs == 2) xhi |= pres[1][dz];
        }
        for (int dx = 0; dx < nxs; dx++) {
          zlo |= pres[dx][0];
          if (nzs == 2) zhi |= pres[dx][1];
        }
        const double mx = ax ? A.imr[ax] : side_inv(0, xlo, xhi);
        const double mz = az ? A.imr[az] : side_inv(0, zlo, zhi);
        ci.push_back(mz * (my * (mx * A.inv_rcdw)));
      } else {
        double mxz = 0.0;
        for (int dx = 0; dx < nxs; dx++)
          for (int dz = 0; dz < nzs; dz++)
            if (pres[dx][dz]) mxz += M1[ax ? ax : (dx ? 0 : p)] * M1[az ? az : (dz ? 0 : p)];
        ci.push_back((1.0 / mxz) * (my * A.inv_rcdw));
      }
      (void)npres;
    };
    std::vector<int64_t> plane_end(NX, 0);
    for (int I = 0; I < NX; I++) {
      if (I > 0) plane_end[I] = plane_end[I - 1];
      if (xonly && !xcand[I]) continue;
      const int kmI = kmin_of(I);
      for (int J = 0; J < NY; J++) {
        const bool yc = J > 0 && J < NY - 1 && J % sy == 0;
        if (xcand[I] || yc) {
          for (int K = kmI; K < NZ; K++) visit(I, J, K, kmI);
        } else {
          for (int K = (kmI / sz + 1) * sz; K < NZ - 1; K += sz) visit(I, J, K, kmI);
        }
      }
      plane_end[I] = (int64_t)idx.size();
    }
    SeamList& L = slist[which];
    L.built = true;
    L.plane_end = std::move(plane_end);
    L.n = (int64_t)idx.size();
    if (L.n == 0) return ST_OK;
    ST_TRY(L.sidx.upload(idx.data(), idx.size(), c->stream));
    ST_TRY(L.scode.upload(code.data(), code.size(), c->stream));
    ST_TRY(L.sci.upload(ci.data(), ci.size(), c->stream));
    // the host vectors die here: finish the uploads first
    ST_CUDA(cudaStreamSynchronize(c->stream));
    return ST_OK;
  }

  int n_chunks() const { return (m.nx + Lx - 1) / Lx; }

  int xmarch(SArgs& A, bool rcf, bool with_seams = true, int z0 = 0, int z1 = -1) {
    const bool lat = c->dp.latent != 0 && A.mode == 0;
    if (fitted && rcf) return unsupported_fitted("a stored per-point history");
    if (!slab && p >= 2 && (A.flags & ST_RHS_SOURCE) && A.nb > kMaxTabBeams) {
      set_error("the structured p >= 2 kernel tables at most " + std::to_string(kMaxTabBeams) +
                " beams per step");
      return ST_EUNSUPPORTED;
    }
    if (lat && latstat_h) poll_latent();
    // (k_xmarch2 packs node coordinates in 16 bits and indexes a plane with
    // 32-bit offsets)
    const bool x2_fits = 2 * m.ny < 32768 && 2 * m.nz < 32768 &&
                         (int64_t)(2 * m.ny + 1) * (2 * m.nz + 1) < (1ll << 31);
    A.x2 = (p == 2 && !slab && !rcf && A.mode == 0 && x2_fits &&
            A.flags == (ST_RHS_DIFFUSION | ST_RHS_FACES | ST_RHS_SOURCE) && use_xmarch2() &&
            !(lat && prefer_general))
               ? 1
               : 0;
    last_x2 = A.x2 != 0;
    const bool whole = z0 == 0 && (z1 < 0 || z1 == n_chunks());
    if (z1 < 0) z1 = n_chunks();
    if (z1 <= z0) return with_seams ? seams(A) : ST_OK;
    if (with_seams && whole && A.x2 && !A.seamcnt && pipe_groups >= 2) {
      int nb = 0, bounds[kMaxPipe + 1];
      pipe_bounds(bounds, &nb);
      if (nb >= 2) return xmarch_piped(A, lat, bounds, nb);
    }
    c->prof_begin();
    int rc = hot(A, lat, rcf, z0, z1, c->stream);
    c->prof_end();
    ST_TRY(rc);
    if (lat && latstat_h) record_latent(z0, z1);
    return with_seams ? seams(A) : ST_OK;
  }

  // the hot kernel over the x chunks [z0, z1)
  int hot(SArgs& A, bool lat, bool rcf, int z0, int z1, cudaStream_t stream) {
    const dim3 grid((m.ny + cy - 1) / cy, (m.nz + cz - 1) / cz, z1 - z0);
    A.zoff = z0;
    cudaError_t e;
    switch (p) {
      case 1: e = hot_launch<1>(A, slab, lat, rcf, grid, stream); break;
      case 2: e = hot_launch<2>(A, slab, lat, rcf, grid, stream); break;
      case 3: e = hot_launch<3>(A, slab, lat, rcf, grid, stream); break;
      default: e = hot_launch<4>(A, slab, lat, rcf, grid, stream); break;
    }
    if (e != cudaSuccess) {
      set_error(std::string("hot kernel launch: ") + cudaGetErrorString(e));
      return ST_ECUDA;
    }
    return launched();
  }

  // chunk groups of the pipelined step, balanced by CTA-layers; a part with
  // less than pipe_min_waves waves of CTAs per group stays on the single launch
  void pipe_bounds(int* bounds, int* nb) const {
    const int nch = n_chunks();
    const double total = launch_layers(0, nch);
    int G = std::min(std::min(pipe_groups, (int)kMaxPipe), nch);
    // live CTAs (a CTA marches Lx layers) against the resident ones
    const double waves = total / Lx / (double)hot_slots;
    G = std::min(G, pipe_min_waves > 0.0 ? (int)(waves / pipe_min_waves) : G);
    *nb = 0;
    if (G < 2) return;
    bounds[0] = 0;
    int g = 1;
    for (int z = 1; z < nch && g < G; z++)
      if (launch_layers(0, z) >= total * g / G) bounds[g++] = z;
    bounds[g] = nch;
    *nb = g;
  }

  // One explicit step of k_xmarch2 with the seam pass under the cells: the
  // chunk groups alternate between the library stream and hot_s (a group's
  // CTAs fill the SMs the previous group's tail leaves idle), and the seam
  // entries of the node planes (first plane of group g, first plane of group
  // g + 1] (plane 0 with group 0) run on seam_s once groups g and g + 1 are
  // done.  The pass is bandwidth bound and the cells fp64 bound, so only the
  // last group's entries stay exposed.  Same kernels, same partials, same
  // summation order as the single launch: bitwise the same field.
  int xmarch_piped(SArgs& A, bool lat, const int* bounds, int nb) {
    const int which = 0;
    if (!slist[which].built) ST_TRY(build_seam_list(which));
    const SeamList& L = slist[which];
    const int sx = p * Lx;
    auto entries_to = [&](int g) {  // entries on the planes <= first plane of group g
      if (g >= nb) return L.n;
      return L.plane_end[std::min(bounds[g] * sx, NX - 1)];
    };
    ST_CUDA(cudaEventRecord(ev_fork, c->stream));
    ST_CUDA(cudaStreamWaitEvent(hot_s, ev_fork, 0));
    ST_CUDA(cudaStreamWaitEvent(seam_s, ev_fork, 0));
    c->prof_begin();
    for (int g = 0; g < nb; g++) {
      cudaStream_t hs = (g & 1) ? hot_s : c->stream;
      ST_TRY(hot(A, lat, false, bounds[g], bounds[g + 1], hs));
      ST_CUDA(cudaEventRecord(ev_hot[g], hs));
      ST_CUDA(cudaStreamWaitEvent(seam_s, ev_hot[g], 0));
      if (g >= 1)
        ST_TRY(seams(A, g == 1 ? 0 : entries_to(g - 1), entries_to(g), seam_s));
    }
    // the hot kernel's time for the bench: until the last group of either
    // stream is done
    ST_CUDA(cudaStreamWaitEvent(c->stream, ev_hot[nb - 1], 0));
    if (nb >= 2) ST_CUDA(cudaStreamWaitEvent(c->stream, ev_hot[nb - 2], 0));
    c->prof_end();
    ST_TRY(seams(A, entries_to(nb - 1), L.n, seam_s));
    ST_CUDA(cudaEventRecord(ev_seams, seam_s));
    ST_CUDA(cudaStreamWaitEvent(c->stream, ev_seams, 0));
    if (lat && latstat_h) record_latent(0, n_chunks());
    return ST_OK;
  }

  // CTA-layers of a launch over the x chunks [z0, z1)
  double launch_layers(int z0, int z1) const {
    const int nty = (m.ny + cy - 1) / cy, ntz = (m.nz + cz - 1) / cz;
    double n = 0.0;
    for (int t = 0; t < ntz; t++) {
      const int e = fitted ? text_h[t] : m.nx;
      n += (double)nty * (std::min(e, z1 * Lx) - std::min(e, z0 * Lx));
    }
    return n;
  }
  void poll_latent() {
    if (!lat_pending || cudaEventQuery(lat_ev) != cudaSuccess) return;
    lat_pending = false;
    const double d = (double)(*latstat_h - lat_seen), n = lat_launched_rec - lat_launched_seen;
    lat_seen = *latstat_h;
    lat_launched_seen = lat_launched_rec;
    if (n <= 0.0) return;
    const double frac = d / n;
    // hysteresis: dense above one half, sparse again below a quarter
    if (frac > 0.5) prefer_general = true;
    if (frac < 0.25) prefer_general = false;
  }
  void record_latent(int z0, int z1) {
    lat_launched += launch_layers(z0, z1);
    // the first launch and every fourth after it
    if (lat_pending || (lat_calls++ & 3) != 0) return;
    if (cudaMemcpyAsync(latstat_h, latstat.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c->stream) != cudaSuccess ||
        cudaEventRecord(lat_ev, c->stream) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    lat_launched_rec = lat_launched;
    lat_pending = true;
  }

  // --- multi-GPU slab step (rank interfaces exchanged between the halves)
  SArgs split{};
  bool split_open = false;

  int step_begin(const double* T, double* rc, double dt, int nb, const DevBeam* beams,
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
    // the chunks that touch a rank interface first, then the packed
    // interface planes (event ev_iface: the exchange may start), then the
    // interior chunks, which the exchange overlaps (ST_NO_OVERLAP=1: one
    // launch for all chunks, then the pack)
    const int nch = n_chunks();
    const int a = m.iface_lo ? 1 : 0, b = m.iface_hi ? nch - 1 : nch;
    static const bool no_overlap = getenv("ST_NO_OVERLAP") && atoi(getenv("ST_NO_OVERLAP"));
    const bool overlap = !no_overlap && a < b && (m.iface_lo || m.iface_hi);
    if (overlap) {
      if (m.iface_lo) ST_TRY(xmarch(A, rc != nullptr, false, 0, 1));
      if (m.iface_hi) ST_TRY(xmarch(A, rc != nullptr, false, nch - 1, nch));
    } else {
      ST_TRY(xmarch(A, rc != nullptr, false));
    }
    const bool lat = c->dp.latent != 0;
    for (int sd = 0; sd < 2; sd++) {
      if (!(sd == 0 ? m.iface_lo : m.iface_hi)) continue;
      const int64_t plane = plane_n(sd == 0 ? 0 : NX - 1);
      k_iface_pack<<<(unsigned)((plane + kThreads - 1) / kThreads), kThreads, 0, c->stream>>>(
          A, p, cy, cz, sd, lat ? 1 : 0);
      ST_TRY(launched());
    }
    ST_TRY(c->iface_event_record());
    if (overlap) ST_TRY(xmarch(A, rc != nullptr, false, a, b));
    split = A;
    split_open = true;
    return ST_OK;
  }

  int iface_ptrs(int side, double** f, double** cp, int64_t* n) override {
    *f = packf[side].p;
    *cp = c->dp.latent ? packc[side].p : nullptr;
    *n = plane_n(side == 0 ? 0 : NX - 1);
    return ST_OK;
  }

  int step_end(const double* lo_f, const double* lo_c, const double* hi_f,
               const double* hi_c) override {
    if (!split_open) {
      set_error("st_explicit_step_end without st_explicit_step_begin");
      return ST_EINVAL;
    }
    split.irf[0] = lo_f;
    split.irc[0] = lo_c;
    split.irf[1] = hi_f;
    split.irc[1] = hi_c;
    if ((m.iface_lo && !lo_f) || (m.iface_hi && !hi_f)) {
      set_error("missing neighbour partials for a rank interface");
      return ST_EINVAL;
    }
    split_open = false;
    return seams(split);
  }

  int rhs(const double* T, double* rc, int flags, double frozen_k, int nb,
          const DevBeam* beams, double* f, int pending) override {
    SArgs A = sargs();
    A.mode = 1;
    A.flags = flags;
    A.frozen_k = frozen_k;
    if (flags & ST_RHS_FROZEN_K) {  // k_xmarch: the frozen value through the uniform law
      A.kAh = A.mhh * frozen_k;
      A.kBh = 0.0;
    }
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
    const int64_t q3 = (int64_t)(p + 1) * (p + 1) * (p + 1);
    if (mode != 0 && (int64_t)Eg.n < n * q3) ST_TRY(Eg.alloc(n * q3));
    A.E = Eg.p;
    switch (p) {
      case 1: k_sgeneric<1><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      case 2: k_sgeneric<2><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      case 3: k_sgeneric<3><<<blocks, 128, 0, c->stream>>>(A, mode); break;
      default: k_sgeneric<4><<<blocks, 128, 0, c->stream>>>(A, mode); break;
    }
    ST_TRY(launched());
    if (mode == 0) return ST_OK;
    const unsigned nb = (unsigned)((nv + 255) / 256);
    switch (p) {
      case 1: k_sgather<1><<<nb, 256, 0, c->stream>>>(A, Eg.p, out); break;
      case 2: k_sgather<2><<<nb, 256, 0, c->stream>>>(A, Eg.p, out); break;
      case 3: k_sgather<3><<<nb, 256, 0, c->stream>>>(A, Eg.p, out); break;
      default: k_sgather<4><<<nb, 256, 0, c->stream>>>(A, Eg.p, out); break;
    }
    return launched();
  }

  int history(const double* T, double* rc) override {
    if (!rc) return ST_OK;
    if (fitted) return unsupported_fitted("a stored per-point history");
    return generic(0, T, nullptr, rc, 0.0, nullptr);
  }

  int capacity(const double* T, double* out) override {
    if (!T || !c->dp.latent) {
      ST_TRY(vec_recip(c, cinv.p, out, nv));
      return ST_OK;
    }
    if (fitted) return unsupported_fitted("the apparent lumped capacity");
    ST_TRY(generic(1, T, nullptr, nullptr, 0.0, out));
    k_cap_floor<<<(unsigned)((nv + 255) / 256), 256, 0, c->stream>>>(nv, cinv.p, out);
    return launched();
  }

  int mass(const double* v, double* out) override {
    if (fitted) return unsupported_fitted("apply_mass");
    return generic(2, nullptr, v, nullptr, 0.0, out);
  }

  int jacobian(const double* v, const double* Tl, const double* rc, double dt,
               double* out) override {
    if (fitted) return unsupported_fitted("apply_jacobian");
    double* vd;
    ST_TRY(c->vec(5, &vd));
    ST_CUDA(cudaMemcpyAsync(vd, v, nv * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    if (m.dirichlet_bottom) ST_TRY(pin_dirichlet(vd, 0.0));
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
    if (fitted) return unsupported_fitted("jacobian_diagonal");
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
    if (fitted) {
      const int64_t n = (int64_t)NX * NY;
      k_fit_pin<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(sargs(), 0, nullptr, v, value);
      return launched();
    }
    const int64_t np_ = (int64_t)NX * NY;
    k_pin_bottom<<<(unsigned)((np_ + 255) / 256), 256, 0, c->stream>>>(np_, NZ, v, value);
    return launched();
  }

  double bytes_per_dof() const override {
    // T_n read + T_{n+1} write.  SURVEY §8d counts 24 B with a C^-1 read;
    // this kernel evaluates C^-1 from the tensor-product lumped mass and
    // reads no per-DoF diagonal, so 16 B is what it must move.  Plus the
    // r_c traffic when the history is a stored field.
    double b = 16.0;
    if (!c->rc_uniform) {
      const double q = (double)(p + 1) * (p + 1) * (p + 1);
      b += 16.0 * q * ((double)m.nx * m.ny * m.nz) / (double)nv;
    }
    return b;
  }
  const char* main_kernel() const override {
    return slab ? "k_xslab" : (last_x2 ? "k_xmarch2" : "k_xmarch");
  }
  bool uniform_rc_ok() const override { return true; }
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
  // kernel per degree (measured); ST_KERNEL=march|slab overrides
  s->slab = s->p >= 3;
  if (const char* e = getenv("ST_KERNEL")) {
    if (!strcmp(e, "slab")) s->slab = true;
    if (!strcmp(e, "march")) s->slab = false;
  }
  if (m->xext) {
    // fitted part: node plane I holds rows K >= kmin(I) (the first cell row
    // whose extent reaches the plane), numbered plane by plane (the
    // reference's sorted-key rule on the active nodes); k_xmarch only
    s->fitted = true;
    s->slab = false;
    s->xext_h.assign(m->xext, m->xext + m->nz);
    for (int k = 0; k < m->nz; k++)
      if (s->xext_h[k] < 1 || s->xext_h[k] > m->nx || (k && s->xext_h[k] < s->xext_h[k - 1])) {
        set_error("fitted part: xext must be non-decreasing extents in [1, nx]");
        delete s;
        *err = ST_EINVAL;
        return nullptr;
      }
    s->kmin_h.resize(s->NX);
    s->base_h.resize(s->NX);
    int64_t off = 0;
    for (int I = 0; I < s->NX; I++) {
      const int need = std::max((I + s->p - 1) / s->p, 1);
      const int k = (int)(std::lower_bound(s->xext_h.begin(), s->xext_h.end(), need) - s->xext_h.begin());
      s->kmin_h[I] = s->p * k;
      s->base_h[I] = off - s->kmin_h[I];
      off += (int64_t)s->NY * (s->NZ - s->kmin_h[I]);
    }
    s->nv = off;
  }
  if (s->slab) {
    switch (s->p) {
      case 1: s->cy = SlabTile<1>::CY; s->cz = SlabTile<1>::CZ; break;
      case 2: s->cy = SlabTile<2>::CY; s->cz = SlabTile<2>::CZ; break;
      case 3: s->cy = SlabTile<3>::CY; s->cz = SlabTile<3>::CZ; break;
      default: s->cy = SlabTile<4>::CY; s->cz = SlabTile<4>::CZ; break;
    }
  } else {
    switch (s->p) {
      case 1: s->cy = Tile<1>::CY; s->cz = Tile<1>::CZ; break;
      case 2: s->cy = Tile<2>::CY; s->cz = Tile<2>::CZ; break;
      case 3: s->cy = Tile<3>::CY; s->cz = Tile<3>::CZ; break;
      default: s->cy = Tile<4>::CY; s->cz = Tile<4>::CZ; break;
    }
  }
  // x chunk length: the CTAs (yz tiles x chunks) run in waves of
  // (resident per SM) x (SMs); pick the chunking with the smallest
  // waves x (layers per CTA + overhead) (ties: fewer chunks, fewer x seams)
  const int64_t nty = (m->ny + s->cy - 1) / s->cy, ntz = (m->nz + s->cz - 1) / s->cz;
  const int64_t nyz = nty * ntz;
  if (s->fitted) {
    // a tile row must not straddle an extent change
    s->text_h.resize(ntz);
    for (int t = 0; t < ntz; t++) {
      s->text_h[t] = s->xext_h[t * s->cz];
      for (int k = t * s->cz; k < std::min((t + 1) * s->cz, m->nz); k++)
        if (s->xext_h[k] != s->text_h[t]) {
          set_error("fitted part: the x extent may change only at multiples of " +
                    std::to_string(s->cz) + " cell rows (tile rows of the degree-" +
                    std::to_string(s->p) + " kernel)");
          delete s;
          *err = ST_EUNSUPPORTED;
          return nullptr;
        }
    }
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int64_t slots = (int64_t)s->resident(c->dp.latent != 0) * std::max(sms, 1);
  s->hot_slots = std::max<int64_t>(slots, 1);
  int64_t best = -1;
  s->Lx = m->nx;
  for (int L = m->nx; L >= std::min(2, m->nx); L--) {
    const int64_t ch = (m->nx + L - 1) / L;
    if ((m->nx + ch - 1) / ch != L) continue;  // same chunking as a longer L
    // work items: tiles x chunks (a fitted part's short rows have fewer)
    int64_t items = nyz * ch;
    if (s->fitted) {
      items = 0;
      for (int t = 0; t < ntz; t++) items += nty * ((s->text_h[t] + L - 1) / L);
    }
    // + 2 layers per CTA for its prologue planes, tail plane and x seam
    const int64_t cost = ((items + slots - 1) / slots) * (int64_t)(L + 2);
    if (best < 0 || cost < best) {
      best = cost;
      s->Lx = L;
    }
  }
  if (const char* e = getenv("ST_LX")) s->Lx = std::max(1, std::min(atoi(e), m->nx));
  s->use_lat = lattice_origin(m->x0, m->h, &s->lx) && lattice_origin(m->y0, m->h, &s->ly) &&
               lattice_origin(m->z0, m->h, &s->lz);
  c->nv = s->nv;
  c->n_cells = (int64_t)m->nx * m->ny * m->nz;
  if (s->fitted) {
    int64_t cells = 0;
    for (int k = 0; k < m->nz; k++) cells += s->xext_h[k];
    c->n_cells = cells * m->ny;
  }
  c->qpc = (s->p + 1) * (s->p + 1) * (s->p + 1);
  rc = s->cinv.alloc(s->nv);
  if (rc == ST_OK && s->fitted) {
    rc = s->pbase_d.upload(s->base_h.data(), s->base_h.size(), c->stream);
    if (rc == ST_OK) rc = s->pkmin_d.upload(s->kmin_h.data(), s->kmin_h.size(), c->stream);
    if (rc == ST_OK) rc = s->text_d.upload(s->text_h.data(), s->text_h.size(), c->stream);
    if (rc == ST_OK) rc = s->xext_d.upload(s->xext_h.data(), s->xext_h.size(), c->stream);
  }
  // seam slots (see SArgs::fseam / seam_pair)
  const bool pair = s->seam_pairs();
  const size_t nseam = (size_t)(pair ? 16 : 8) * s->nv;
  if (rc == ST_OK) rc = s->fseam.alloc(nseam);
  if (rc == ST_OK && c->dp.latent && !pair) rc = s->cseam.alloc(nseam);
  if (rc == ST_OK && c->dp.latent && !s->slab) {
    const size_t ctas = (size_t)((m->ny + s->cy - 1) / s->cy) * ((m->nz + s->cz - 1) / s->cz) *
                        ((m->nx + s->Lx - 1) / s->Lx);
    rc = s->lcarry.alloc(ctas * s->cy * s->cz * (s->p + 1) * (s->p + 1));
    if (rc == ST_OK && s->p == 2)
      rc = s->ecg.alloc(ctas * s->cy * s->cz * s->p * (s->p + 1) * (s->p + 1));
  }
  if (rc == ST_OK &&
      cudaMemsetAsync(s->fseam.p, 0, nseam * sizeof(double), c->stream) != cudaSuccess)
    rc = ST_ECUDA;
  if (rc == ST_OK && s->cseam.p &&
      cudaMemsetAsync(s->cseam.p, 0, nseam * sizeof(double), c->stream) != cudaSuccess)
    rc = ST_ECUDA;
  for (int sd = 0; sd < 2 && rc == ST_OK; sd++) {
    if (!(sd == 0 ? m->iface_lo : m->iface_hi)) continue;
    rc = s->packf[sd].alloc((size_t)s->plane_n(sd == 0 ? 0 : s->NX - 1));
    if (rc == ST_OK && c->dp.latent) rc = s->packc[sd].alloc((size_t)s->plane_n(sd == 0 ? 0 : s->NX - 1));
  }
  if (rc == ST_OK) {
    const double rc_detw = c->dp.rhoc * std::pow(m->h / 2.0, 3.0);
    const unsigned blocks = (unsigned)((s->nv + 255) / 256);
    if (s->fitted) {
      const SArgs A = s->sargs();
      const dim3 g((unsigned)(((int64_t)s->NY * s->NZ + 255) / 256), (unsigned)s->NX);
      switch (s->p) {
        case 1: k_fit_cinv<1><<<g, 256, 0, c->stream>>>(A, s->xext_d.p, rc_detw, s->cinv.p); break;
        case 2: k_fit_cinv<2><<<g, 256, 0, c->stream>>>(A, s->xext_d.p, rc_detw, s->cinv.p); break;
        case 3: k_fit_cinv<3><<<g, 256, 0, c->stream>>>(A, s->xext_d.p, rc_detw, s->cinv.p); break;
        default: k_fit_cinv<4><<<g, 256, 0, c->stream>>>(A, s->xext_d.p, rc_detw, s->cinv.p); break;
      }
    } else
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
  if (rc == ST_OK && !s->slab && s->p == 2 && c->dp.latent && use_xmarch2()) {
    const char* e = getenv("ST_X2_ADAPT");  // ST_X2_ADAPT=0: never leave k_xmarch2
    if (!(e && e[0] == '0')) {
      rc = s->latstat.alloc(1);
      if (rc == ST_OK &&
          (cudaMemsetAsync(s->latstat.p, 0, sizeof(unsigned long long), c->stream) != cudaSuccess ||
           cudaMallocHost(&s->latstat_h, sizeof(unsigned long long)) != cudaSuccess ||
           cudaEventCreateWithFlags(&s->lat_ev, cudaEventDisableTiming) != cudaSuccess))
        rc = ST_ECUDA;
      if (rc == ST_OK) *s->latstat_h = 0;
    }
  }
  // opt-in (ST_INSEAM=1): k_xmarch2 completes the seams of ordinary planes
  // itself (arrival counters per chunk and seam group).  Measured slower than
  // the seam pass on config 4 (21.1 ms against 12.8 + 3.6 ms): the completion
  // is a latency-bound gather that a CTA runs with far fewer loads in flight
  // than the pass's one thread per node.
  if (rc == ST_OK && !s->slab && s->p == 2) {
    const char* e = getenv("ST_INSEAM");
    s->GY = 2 * (int)nty + 1;
    s->GZ = 2 * (int)ntz + 1;
    const int64_t ncnt = (int64_t)s->NX * s->GY * s->GZ;
    if (e && e[0] == '1' && ncnt < (1ll << 31)) {
      rc = s->seamcnt.alloc((size_t)ncnt);
      if (rc == ST_OK &&
          cudaMemsetAsync(s->seamcnt.p, 0, (size_t)ncnt * sizeof(int), c->stream) != cudaSuccess)
        rc = ST_ECUDA;
      s->inseam = rc == ST_OK;
    }
  }
  // pipelined seam pass of the k_xmarch2 step (xmarch_piped): ST_SEAM_PIPE=n
  // chunk groups (0 / 1: the single launch followed by the whole pass)
  if (rc == ST_OK && !s->slab && s->p == 2 && !s->inseam && !m->iface_lo && !m->iface_hi) {
    // off by default: measured slower on config 4 (15.9 ms per step with 4
    // groups, 16.2 with 12, against 15.2): both kernels are bound by resident
    // threads (the cells by registers, the pass by loads in flight), so the
    // pass under the cells takes from them what it gains
    int G = 0;
    if (const char* e = getenv("ST_SEAM_PIPE")) G = atoi(e);
    G = std::max(0, std::min(G, (int)Structured::kMaxPipe));
    if (G >= 2) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      bool ok = cudaStreamCreateWithFlags(&s->hot_s, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithPriority(&s->seam_s, cudaStreamNonBlocking, hi) ==
                    cudaSuccess &&
                cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&s->ev_seams, cudaEventDisableTiming) == cudaSuccess;
      for (int g = 0; ok && g < G; g++)
        ok = cudaEventCreateWithFlags(&s->ev_hot[g], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) {
        set_error("structured context: streams / events of the pipelined seam pass");
        rc = ST_ECUDA;
      } else {
        s->pipe_groups = G;
        if (const char* e = getenv("ST_SEAM_PIPE_MINWAVES")) s->pipe_min_waves = atof(e);
      }
    }
  }
  // the list the context's explicit steps use; the other one is built when a
  // launch first needs it
  if (rc == ST_OK) rc = s->build_seam_list(s->inseam ? 1 : 0);
  if (rc != ST_OK) {
    delete s;
    *err = rc;
    return nullptr;
  }
  *err = ST_OK;
  return s;
}

}  // namespace st
