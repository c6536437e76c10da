// k_xmarch: the explicit-step / rhs hot kernel of the structured backend
// (included by st_structured.cu after the basis tables).  See the header
// of st_structured.cu for the overall scheme.
#pragma once
#include <type_traits>
#include <utility>

namespace st {

struct CellFlags {
  bool diffusion, faces, source, frozen;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int P>
__device__ __forceinline__ double anchor(const SArgs& A, int axis, int cell) {
  // anchor = lattice * h when the box origin is on the lattice (one
  // rounding, like the reference's anchor * h_fine, operators.py:105-112)
  if (A.use_lat) {
    const long long l = axis == 0 ? A.lx : (axis == 1 ? A.ly : A.lz);
    return (double)(cell + l) * A.h;
  }
  return (axis == 0 ? A.ox : (axis == 1 ? A.oy : A.oz)) + (double)cell * A.h;
}

// 1D projection of the separable Gaussian slab source of one beam
// (physics.py:154-171): exp(-2 r^2/R^2) = exp(-2 dx^2/R^2) exp(-2 dy^2/R^2),
// so V^T (x) V^T (x) V^T of the point values is an outer product of three
// 1D projections s_d[a] = sum_q V[a][q] W[q] f_d(q).
template <int P>
__device__ __forceinline__ void source_factors(const SArgs& A, const DevBeam& b, double ax,
                                               double ay, double az, double* sx, double* sy,
                                               double* sz) {
  constexpr int Q = P + 1;
  const DevParams& PP = A.P;
  double fx[Q], fy[Q], fz[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const double dx = (ax + kTab.U[q] * A.h) - b.x;
    const double dy = (ay + kTab.U[q] * A.h) - b.y;
    const double z = az + kTab.U[q] * A.h;
    fx[q] = exp((-2.0 * (dx * dx)) / PP.R2) * kTab.W[q];
    fy[q] = exp((-2.0 * (dy * dy)) / PP.R2) * kTab.W[q];
    fz[q] = (z >= b.z_top - PP.h_powder && z <= b.z_top) ? kTab.W[q] : 0.0;
  }
#pragma unroll
  for (int a = 0; a < Q; a++) {
    double x = 0.0, y = 0.0, zz = 0.0;
#pragma unroll
    for (int q = 0; q < Q; q++) {
      x = fma(Basis<P>::V(a, q), fx[q], x);
      y = fma(Basis<P>::V(a, q), fy[q], y);
      zz = fma(Basis<P>::V(a, q), fz[q], zz);
    }
    sx[a] = x;
    sy[a] = y;
    sz[a] = zz;
  }
}

// Which update of the diffusion loop touches G[(A, B, C)] first (0: the
// x-term at q = (0, B, C), m = A; 1: the y-term at (A, 0, C), m = B; 2: the
// z-term at (A, B, 0), m = C), in the loop's order: q lexicographic, then m,
// then x, y, z
template <int Q>
__host__ __device__ constexpr int first_touch(int A, int B, int C) {
  const int kx = ((0 * Q + B) * Q + C) * 3 * Q + A * 3 + 0;
  const int ky = ((A * Q + 0) * Q + C) * 3 * Q + B * 3 + 1;
  const int kz = ((A * Q + B) * Q + 0) * 3 * Q + C * 3 + 2;
  return kx <= ky ? (kx <= kz ? 0 : 2) : (ky <= kz ? 1 : 2);
}

// Beams whose cell-level hit test (beam_hits_cell) can pass for some cell
// of the (y, z) column (j, k): the y box distance and the slab overlap are
// fixed over the x march, and dy^2 <= cut^2 is necessary for
// dx^2 + dy^2 <= cut^2.  The exact test still runs per cell.
template <int P>
__device__ __forceinline__ unsigned beam_column_mask(const SArgs& A, int j, int k) {
  unsigned mask = 0;
  const double ay = anchor<P>(A, 1, j), az = anchor<P>(A, 2, k);
  const int nb = A.nb < 32 ? A.nb : 32;
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const DevBeam bm = A.beams[b];
    if (bm.peak == 0.0) continue;
    const double dy = fmax(fmax(ay - bm.y, bm.y - ay - A.h), 0.0);
    if (dy * dy <= A.P.cut2 && az <= bm.z_top && az + A.h >= bm.z_top - A.P.h_powder)
      mask |= 1u << b;
  }
  return mask;
}

// Separable source tables of a k_xmarch CTA (COOP): per beam, the y factor
// of each tile row jl and the z factor of each tile column kl are fixed over
// the x march (Sy[(jl * kMaxTabBeams + b) * Q + a], Sz likewise); the x
// factor Sx[b * Q + a] changes per cell layer (kMaxTabBeams beams).

// 1D projected factor s[a] = sum_q V(a, q) f(q) of one axis of the
// separable slab source (the expressions of source_factors)
template <int P>
__device__ __forceinline__ void src_factor_xy(const SArgs& A, double anc, double bc, double* s) {
  constexpr int Q = P + 1;
  double f[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const double d = (anc + kTab.U[q] * A.h) - bc;
    f[q] = exp((-2.0 * (d * d)) / A.P.R2) * kTab.W[q];
  }
#pragma unroll
  for (int a = 0; a < Q; a++) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < Q; q++) x = fma(Basis<P>::V(a, q), f[q], x);
    s[a] = x;
  }
}
template <int P>
__device__ __forceinline__ void src_factor_z(const SArgs& A, double az, const DevBeam& b,
                                             double* s) {
  constexpr int Q = P + 1;
  double f[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const double z = az + kTab.U[q] * A.h;
    f[q] = (z >= b.z_top - A.P.h_powder && z <= b.z_top) ? kTab.W[q] : 0.0;
  }
#pragma unroll
  for (int a = 0; a < Q; a++) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < Q; q++) x = fma(Basis<P>::V(a, q), f[q], x);
    s[a] = x;
  }
}

// +z facet term of top cells r0 .. r1-1 of a tile row, by the 32 lanes of
// one warp (COOP): Gauss-point temperatures and fluxes, then the
// projection to the facet nodes, each item in the summation order of the
// per-cell code (operators.py:275-290); fo[r][a * Q + b]
template <int P, class NodeF>
__device__ __forceinline__ void face_phase(const SArgs& A, int lane, int r0, int r1, double* fq,
                                           double* fo, const NodeF& node) {
  constexpr int Q = P + 1, Q2 = Q * Q;
  const double area0 = A.hh * A.hh;
  const int n = (r1 - r0) * Q2;
#pragma unroll 1
  for (int it = lane; it < n; it += 32) {
    const int r = r0 + it / Q2, s = it - (it / Q2) * Q2, qa = s / Q, qb = s - (s / Q) * Q;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < Q; a++) {
      double v = kTab.V[0][qb] * node(r, a, 0);
#pragma unroll
      for (int b = 1; b < Q; b++) v = fma(kTab.V[b][qb], node(r, a, b), v);
      acc = a == 0 ? kTab.V[0][qa] * v : fma(kTab.V[a][qa], v, acc);
    }
    fq[r * Q2 + s] = surface_flux(A.P, acc) * (-(area0 * (kTab.W[qa] * kTab.W[qb])));
  }
  __syncwarp();
#pragma unroll 1
  for (int it = lane; it < n; it += 32) {
    const int r = r0 + it / Q2, s = it - (it / Q2) * Q2, a = s / Q, b = s - (s / Q) * Q;
    const double* f = fq + r * Q2;
    double acc = 0.0;
#pragma unroll
    for (int qb = 0; qb < Q; qb++) {
      double v = kTab.V[a][0] * f[qb];
#pragma unroll
      for (int qa = 1; qa < Q; qa++) v = fma(kTab.V[a][qa], f[qa * Q + qb], v);
      acc = qb == 0 ? kTab.V[b][0] * v : fma(kTab.V[b][qb], v, acc);
    }
    fo[r * Q2 + s] = acc;
  }
}

// Element vector of one cell, degree P (operators.py:247-316 generalised):
//   t in : T at the Gauss points (a x b x c, z fastest; kept for the
//          latent capacity pass of the caller)
//   G out: element vector
//   node(a, b, c): re-reads a node value (top facet; keeps t's copy out of
//          the register budget)
// COOP (p >= 2, z-major cells): the source uses the CTA's separable factor
// tables (sxl: Sx of this layer, syj / szk: this cell's [beam][Q] rows of
// Sy / Sz, see kMaxTabBeams) and the +z facet term of a
// top cell comes precomputed from the top warp (fo: [a * Q + b], face_phase);
// both give the same values in the same summation order as the per-cell code.
template <int P, bool RCF, bool COOP, class NodeF>
__device__ __forceinline__ void cell_element(const SArgs& A, const CellFlags& F, int i, int j,
                                             int k, int64_t cell, const double* t, double* G,
                                             unsigned ymask, const NodeF& node, const double* sxl,
                                             const double* syj, const double* szk,
                                             const double* fo) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  using B = Basis<P>;
  const DevParams& PP = A.P;
  const bool top = F.faces && A.top_faces && (k == A.nz - 1);
  // p >= 2: the first update of each flux-accumulator entry is a product,
  // so no zero initialisation (measured: config 1 -1.5 %, p = 1 +3 %)
  constexpr bool FT = P >= 2;
  if (!FT || !F.diffusion)
#pragma unroll
    for (int q = 0; q < Q3; q++) G[q] = 0.0;
  if (F.diffusion) {
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
#pragma unroll
        for (int qc = 0; qc < Q; qc++) {
          const int q = (qa * Q + qb) * Q + qc;
          // reference-coordinate gradient by Gauss-point collocation (exact
          // zeros of Dq skipped at compile time, see sweep_v)
          double gx = 0.0, gy = 0.0, gz = 0.0;
          bool ix = false, iy = false, iz = false;
#pragma unroll
          for (int mm = 0; mm < Q; mm++) {
            if (B::Dq(mm, qa) != 0.0) {
              gx = ix ? fma(B::Dq(mm, qa), t[(mm * Q + qb) * Q + qc], gx)
                      : B::Dq(mm, qa) * t[(mm * Q + qb) * Q + qc];
              ix = true;
            }
            if (B::Dq(mm, qb) != 0.0) {
              gy = iy ? fma(B::Dq(mm, qb), t[(qa * Q + mm) * Q + qc], gy)
                      : B::Dq(mm, qb) * t[(qa * Q + mm) * Q + qc];
              iy = true;
            }
            if (B::Dq(mm, qc) != 0.0) {
              gz = iz ? fma(B::Dq(mm, qc), t[(qa * Q + qb) * Q + mm], gz)
                      : B::Dq(mm, qc) * t[(qa * Q + qb) * Q + mm];
              iz = true;
            }
          }
          // -(h/2) k(T, r_c) at the Gauss point: g(T) (material.py:46-57) as
          // a clamped ramp; with a uniform consolidated history the law is
          // one FMA with -(h/2) folded into its constants (kAh, kBh; a
          // frozen conductivity is kAh = -(h/2) k_frozen, kBh = 0), so
          // c = W3 (-(h/2) k) takes a compile-time weight
          const double g = clamp01_hi(fma(t[q], PP.inv_dT_l, A.glo));
          double kh;
          if (RCF) {
            double r = A.rc[cell * Q3 + q];
            if (A.pending && !F.frozen) {
              r = dmax(r, g);
              A.rc[cell * Q3 + q] = r;
            }
            kh = A.mhh * conductivity(PP, g, r);
          } else {
            kh = fma(g, A.kBh, A.kAh);
          }
          // -(w detJ (2/h)^2) k = -(h/2) W3 k ;  f_diff = sum_d Dq_d^T (c grad_d):
          // the quadrature weight W3 rides in the compile-time coefficients
          // Dq W3 of the transposed differentiation (27 multiplies less per
          // cell than scaling the conductivity)
          // (p = 1 keeps the reference's operation order: c = W3 k first)
          const double W3 = B::W(qa) * B::W(qb) * B::W(qc);  // folded after unrolling
          const double c = FT ? kh : W3 * kh;
          const double fx = c * gx, fy = c * gy, fz = c * gz;
#pragma unroll
          for (int m = 0; m < Q; m++) {
            // first touches (a product, or 0 for a zero coefficient) and
            // exact-zero coefficients are folded at compile time after
            // unrolling
            const double wd = FT ? W3 : 1.0;
            const double dxa = B::Dq(m, qa) * wd, dyb = B::Dq(m, qb) * wd, dzc = B::Dq(m, qc) * wd;
            if (FT && qa == 0 && first_touch<Q>(m, qb, qc) == 0)
              G[(m * Q + qb) * Q + qc] = B::Dq(m, qa) == 0.0 ? 0.0 : dxa * fx;
            else if (B::Dq(m, qa) != 0.0)
              G[(m * Q + qb) * Q + qc] = fma(dxa, fx, G[(m * Q + qb) * Q + qc]);
            if (FT && qb == 0 && first_touch<Q>(qa, m, qc) == 1)
              G[(qa * Q + m) * Q + qc] = B::Dq(m, qb) == 0.0 ? 0.0 : dyb * fy;
            else if (B::Dq(m, qb) != 0.0)
              G[(qa * Q + m) * Q + qc] = fma(dyb, fy, G[(qa * Q + m) * Q + qc]);
            if (FT && qc == 0 && first_touch<Q>(qa, qb, m) == 2)
              G[(qa * Q + qb) * Q + m] = B::Dq(m, qc) == 0.0 ? 0.0 : dzc * fz;
            else if (B::Dq(m, qc) != 0.0)
              G[(qa * Q + qb) * Q + m] = fma(dzc, fz, G[(qa * Q + qb) * Q + m]);
          }
        }
  }
  project3<P>(G);
  if (F.source && __builtin_expect(ymask != 0u || A.nb > 32, 0)) {
    const double ax = anchor<P>(A, 0, i), ay = anchor<P>(A, 1, j), az = anchor<P>(A, 2, k);
#pragma unroll 1
    for (int b = 0; b < A.nb; b++) {
      if (b < 32 && !((ymask >> b) & 1u)) continue;  // column prefilter
      const DevBeam bm = A.beams[b];
      if (!beam_hits_cell(PP, bm, ax, ay, az, A.h)) continue;
      double sx[Q], sy[Q], sz[Q];
      if (COOP) {
#pragma unroll
        for (int a = 0; a < Q; a++) {
          sx[a] = sxl[b * Q + a];
          sy[a] = syj[b * Q + a];
          sz[a] = szk[b * Q + a];
        }
      } else {
        source_factors<P>(A, bm, ax, ay, az, sx, sy, sz);
      }
      const double coef = bm.peak * A.detw0;
#pragma unroll
      for (int a = 0; a < Q; a++)
#pragma unroll
        for (int bb = 0; bb < Q; bb++) {
          const double sab = coef * sx[a] * sy[bb];
#pragma unroll
          for (int c = 0; c < Q; c++) G[(a * Q + bb) * Q + c] = fma(sab, sz[c], G[(a * Q + bb) * Q + c]);
        }
    }
  }
  if (COOP && top) {
#pragma unroll
    for (int a = 0; a < Q; a++)
#pragma unroll
      for (int b = 0; b < Q; b++) G[(a * Q + b) * Q + P] += fo[a * Q + b];
  }
  if (!COOP && top) {
    // +z facet quadrature (operators.py:275-290), full facets
    double tf[Q * Q];
#pragma unroll
    for (int a = 0; a < Q; a++)
#pragma unroll
      for (int b = 0; b < Q; b++) tf[a * Q + b] = node(a, b, P);
#pragma unroll
    for (int a = 0; a < Q; a++) {
      double in[Q];
#pragma unroll
      for (int b = 0; b < Q; b++) in[b] = tf[a * Q + b];
#pragma unroll
      for (int qb = 0; qb < Q; qb++) {
        double acc = B::V(0, qb) * in[0];
#pragma unroll
        for (int b = 1; b < Q; b++) acc = fma(B::V(b, qb), in[b], acc);
        tf[a * Q + qb] = acc;
      }
    }
    double fq[Q * Q];
#pragma unroll
    for (int qb = 0; qb < Q; qb++) {
      double in[Q];
#pragma unroll
      for (int a = 0; a < Q; a++) in[a] = tf[a * Q + qb];
#pragma unroll
      for (int qa = 0; qa < Q; qa++) {
        double acc = B::V(0, qa) * in[0];
#pragma unroll
        for (int a = 1; a < Q; a++) acc = fma(B::V(a, qa), in[a], acc);
        fq[qa * Q + qb] = acc;
      }
    }
    const double area0 = A.hh * A.hh;
#pragma unroll
    for (int qa = 0; qa < Q; qa++)
#pragma unroll
      for (int qb = 0; qb < Q; qb++)
        fq[qa * Q + qb] = surface_flux(PP, fq[qa * Q + qb]) * (-(area0 * (B::W(qa) * B::W(qb))));
#pragma unroll
    for (int qb = 0; qb < Q; qb++) {
      double in[Q];
#pragma unroll
      for (int qa = 0; qa < Q; qa++) in[qa] = fq[qa * Q + qb];
#pragma unroll
      for (int a = 0; a < Q; a++) {
        double acc = B::V(a, 0) * in[0];
#pragma unroll
        for (int qa = 1; qa < Q; qa++) acc = fma(B::V(a, qa), in[qa], acc);
        tf[a * Q + qb] = acc;
      }
    }
#pragma unroll
    for (int a = 0; a < Q; a++)
#pragma unroll
      for (int b = 0; b < Q; b++) {
        double acc = B::V(b, 0) * tf[a * Q + 0];
#pragma unroll
        for (int qb = 1; qb < Q; qb++) acc = fma(B::V(b, qb), tf[a * Q + qb], acc);
        G[(a * Q + b) * Q + P] += acc;
      }
  }
}

// compile-time loops (node offsets inside a cell become immediates)
template <int N>
using IC = std::integral_constant<int, N>;
template <class F, int... I>
__device__ __forceinline__ void static_for_(F&& f, std::integer_sequence<int, I...>) {
  (f(IC<I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_(f, std::make_integer_sequence<int, N>{});
}
#include "st_xmarch_kernel.cuh"
#if ST_HOT_P == 2
#include "st_xmarch2_kernel.cuh"
#endif
#include "st_xslab_kernel.cuh"

}  // namespace st
