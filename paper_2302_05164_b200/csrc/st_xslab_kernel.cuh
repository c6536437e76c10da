// k_xslab: the x-marching explicit-step / rhs kernel with (p+1) threads per
// cell (included from st_xmarch.cuh).
//
// k_xmarch keeps a whole cell (2 (p+1)^3 doubles) in one thread's
// registers, which stops fitting at p >= 3.  Here thread s of a cell owns
// the x-slab s of its Gauss-point tensor ((p+1)^2 values): the y and z
// sweeps stay in registers, and the three x-direction contractions go
// through conflict-free shared-memory exchanges among the p+1 slab threads
// of the cell (entry-major X[(b, c, s)][cell], a warp = 32 cells of one s).
// Per cell layer:
//   B1  the layer's node planes are in the ring (cp.async, prefetched
//       from B3 of the previous layer)
//   1.  T and dT/dx at Gauss point s of x in one pass over the ring (V and
//       D columns s), y/z interpolation sweeps of both; top facet term
//   2.  grad_y / grad_z by Gauss-point collocation, k(T, r_c), fluxes; y/z
//       flux terms accumulated in registers, x fluxes written to Y      B3
//   3.  x flux term from Y (Dq row s); y/z transposed sweeps; Gaussian
//       source (x factor at Gauss point s) and top facet (x-interpolated
//       at s) added before the x projection; write to X              B4
//   4.  thread s = node plane a: x projection from X (V row a); plane 0
//       adds the carried face of the previous layer, plane p becomes the
//       carry, planes a < p go to Y as element planes                 B5
//   5.  node finalisation of planes a < p (same fixed-order gather and
//       seam slots as k_xmarch)
// The latent capacity increments follow the same projections through X
// (three extra barriers) in layers where some cell of the CTA has a Gauss
// point in the latent interval (__syncthreads_or at B4); their element
// planes stay in X for the finalisation and their x face is carried in CL.
#pragma once

// shared memory of k_xslab in doubles
template <int P, int CY, int CZ, bool LATENT>
constexpr int slab_smem_doubles() {
  constexpr int Q = P + 1, Q2 = Q * Q, Q3 = Q2 * Q, NC = CY * CZ;
  constexpr int PL = (P * CY + 1) * (P * CZ + 1);
  return (SlabTile<P>::SHORT ? P + 1 : 2 * P + 1) * PL + 2 * Q3 * NC + 2 * Q2 * NC +
         (LATENT ? 2 * Q2 * NC : 0);
}

// in-place 1D sweep of a Q x Q register slab t[b * Q + c] along b (AX 0)
// or c (AX 1): out[q] = sum_m M[m][q] in[m]   (TR: M[q][m])
template <int P, int AX, bool TR, bool DER>
__device__ __forceinline__ void sweep2(double* t) {
  constexpr int Q = P + 1;
  using B = Basis<P>;
#pragma unroll
  for (int o = 0; o < Q; o++) {
    double in[Q];
#pragma unroll
    for (int m = 0; m < Q; m++) in[m] = t[AX == 0 ? m * Q + o : o * Q + m];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      auto M = [](int r, int cidx) { return DER ? B::Dq(r, cidx) : B::V(r, cidx); };
      // exact zeros skipped, a leading 1.0 copied (see sweep_v)
      double acc = 0.0;
      bool init = false;
#pragma unroll
      for (int m = 0; m < Q; m++) {
        const double cf = TR ? M(q, m) : M(m, q);
        if (cf == 0.0) continue;
        acc = init ? fma(cf, in[m], acc) : (cf == 1.0 ? in[m] : cf * in[m]);
        init = true;
      }
      t[AX == 0 ? q * Q + o : o * Q + q] = acc;
    }
  }
}

template <int P, int CY, int CZ, bool LATENT, bool RCF>
__global__ void __launch_bounds__((P + 1) * CY * CZ, SlabTile<P>::MINB) k_xslab(SArgs A) {
  constexpr int Q = P + 1, Q2 = Q * Q, Q3 = Q2 * Q;
  constexpr int NC = CY * CZ, NT = Q * NC;
  constexpr int NYT = P * CY + 1, NZT = P * CZ + 1, PL = NYT * NZT;
  // ring: the layer's P+1 node planes; the next layer's P new planes are
  // prefetched into the first P slots once step 1 is done with them (B3)
  constexpr bool SHORT = SlabTile<P>::SHORT;
  constexpr int NR = SHORT ? P + 1 : 2 * P + 1;
  using B = Basis<P>;
  extern __shared__ double sm[];
  double* Tr = sm;                 // NR planes of T
  double* X = Tr + NR * PL;        // exchange: Gauss-point T, then y/z-projected G
  double* Y = X + Q3 * NC;         // exchange: x fluxes, then element planes a < P
  double* Cx = Y + Q3 * NC;        // carried x face [layer parity][Q2][NC]
  double* CL = Cx + 2 * Q2 * NC;   // LATENT: carried face of the increments
  const int tid = threadIdx.x;
  const int s = tid / NC, cl = tid - (tid / NC) * NC;
  const int jl = cl / CZ, kl = cl - (cl / CZ) * CZ;
  const int chunk = blockIdx.z + A.zoff;  // x chunk (launches may cover a chunk range)
  const int j0 = blockIdx.x * CY, k0 = blockIdx.y * CZ, i0 = chunk * A.Lx;
  if (i0 >= A.nx) return;
  const int i1 = min(i0 + A.Lx, A.nx);
  const int j = j0 + jl, k = k0 + kl;
  const bool live = j < A.ny && k < A.nz;
  const bool hiY = live && (jl == CY - 1 || j == A.ny - 1);
  const bool hiZ = live && (kl == CZ - 1 || k == A.nz - 1);
  const int Jn = min(P * CY, P * (A.ny - j0)) + 1;
  const int Kn = min(P * CZ, P * (A.nz - k0)) + 1;
  const bool sy_lo = jl == 0 && j0 > 0, sy_hi = jl == CY - 1 && j0 + CY < A.ny;
  const bool sz_lo = kl == 0 && k0 > 0, sz_hi = kl == CZ - 1 && k0 + CZ < A.nz;
  const CellFlags F{(A.flags & ST_RHS_DIFFUSION) != 0, (A.flags & ST_RHS_FACES) != 0,
                    (A.flags & ST_RHS_SOURCE) != 0 && A.nb > 0, (A.flags & ST_RHS_FROZEN_K) != 0};
  const bool top = F.faces && A.top_faces && (k == A.nz - 1);
  const DevParams& PP = A.P;
  const int64_t plane_stride = (int64_t)A.NY * A.NZ;
  const int64_t tile0 = (int64_t)P * j0 * A.NZ + (int64_t)P * k0;
  const int64_t my0 = (int64_t)P * j * A.NZ + (int64_t)P * k;
  const int ms0 = P * jl * NZT + P * kl;

  auto load_planes = [&](int Ib, int n) {
#pragma unroll 1
    for (int pa = 0; pa < n; pa++) {
      const double* srcT = A.T + (int64_t)(Ib + pa) * plane_stride + tile0;
      double* dT = Tr + ((Ib + pa) % NR) * PL;
#pragma unroll
      for (int e0 = 0; e0 < PL; e0 += NT) {
        const int e = e0 + tid;
        const int r = e / NZT, cc = e - (e / NZT) * NZT;
        if ((e0 + NT <= PL || e < PL) && r < Jn && cc < Kn)
          cp_async8(dT + e, srcT + r * A.NZ + cc);
      }
    }
  };

  const double my_0 = inv_mass1<P>(A, P * j, A.NY), my_P = inv_mass1<P>(A, P * j + P, A.NY);
  const double mz_0 = inv_mass1<P>(A, P * k, A.NZ), mz_P = inv_mass1<P>(A, P * k + P, A.NZ);
  double amax = 0.0, smax = -INFINITY;
  bool bad = false;

  auto finalize_node3 = [&](auto bb, auto cc, const double* pe, const double* pc,
                            const double* tpl, int64_t g0, int xc, bool latn, double imIs) {
    constexpr int b = decltype(bb)::value, c = decltype(cc)::value;
    double f = pe[(b * Q + c) * NC];
    if (b == 0 && jl > 0) f += pe[(P * Q + c) * NC - CZ];
    if (c == 0 && kl > 0) f += pe[(b * Q + P) * NC - 1];
    if (b == 0 && c == 0 && jl > 0 && kl > 0) f += pe[(P * Q + P) * NC - CZ - 1];
    const int64_t idx = g0 + b * A.NZ + c;
    const bool ys_lo = b == 0 && sy_lo, zs_lo = c == 0 && sz_lo;
    const bool seam = xc || ys_lo || (b == P && sy_hi) || zs_lo || (c == P && sz_hi);
    double dc = 0.0;
    if (LATENT && latn) {
      dc = pc[(b * Q + c) * NC];
      if (b == 0 && jl > 0) dc += pc[(P * Q + c) * NC - CZ];
      if (c == 0 && kl > 0) dc += pc[(b * Q + P) * NC - 1];
      if (b == 0 && c == 0 && jl > 0 && kl > 0) dc += pc[(P * Q + P) * NC - CZ - 1];
    }
    if (seam) {
      const int slot = (xc == 2 ? 1 : 0) + (ys_lo ? 2 : 0) + (zs_lo ? 4 : 0);
      seam_store(A, idx, slot, f, dc, LATENT);
    } else {
      const double mzc = c == 0 ? mz_0 : (c == P ? mz_P : A.imr[c]);
      const double myb = b == 0 ? my_0 : (b == P ? my_P : A.imr[b]);
      const double ci = mzc * (myb * imIs);
      const double Tn = SHORT ? A.T[idx] : tpl[b * NZT + c];
      const double o = finalize_node(A, ci, c == 0 && k == 0, Tn, f, dc, LATENT);
      A.out[idx] = o;
      amax = dmax(amax, fabs(o));
      smax = dmax(smax, o);
      bad |= (o != o);
    }
  };

  // nodes of plane I owned by this cell, element plane at pe (stride NC)
  auto finalize_owned = [&](int I, const double* pe, const double* pc, int xc, bool latn) {
    const double imIs = inv_mass1<P>(A, I + A.gI0, A.gNX) * A.inv_rcdw;
    const int64_t g0 = (int64_t)I * plane_stride + my0;
    const double* tpl = Tr + (I % NR) * PL + ms0;
    static_for<P>([&](auto bb) {
      static_for<P>([&](auto cc) { finalize_node3(bb, cc, pe, pc, tpl, g0, xc, latn, imIs); });
    });
    if (hiZ)
      static_for<P>([&](auto bb) { finalize_node3(bb, IC<P>{}, pe, pc, tpl, g0, xc, latn, imIs); });
    if (hiY) {
      static_for<P>([&](auto cc) { finalize_node3(IC<P>{}, cc, pe, pc, tpl, g0, xc, latn, imIs); });
      if (hiZ) finalize_node3(IC<P>{}, IC<P>{}, pe, pc, tpl, g0, xc, latn, imIs);
    }
  };

  // zero carries for the first layer
  for (int e = tid; e < 2 * Q2 * NC; e += NT) {
    Cx[e] = 0.0;
    if (LATENT) CL[e] = 0.0;
  }
  load_planes(P * i0, P + 1);
  cp_commit();
  bool lat_prev = false;

#pragma unroll 1
  for (int i = i0; i < i1; i++) {
    cp_wait<0>();
    __syncthreads();  // B1: ring holds layer i; last layer's X / Y reads are done
    if (!SHORT && i + 1 < i1) {
      load_planes(P * (i + 1) + 1, P);
      cp_commit();
    }
    const int ib = P * i;
    const int64_t cell = ((int64_t)i * A.ny + j) * A.nz + k;
    double T[Q2], G[Q2], ftop[Q];
    unsigned lmask = 0;
    if (live) {
      // 1. T and dT/dx at Gauss point s of x from the ring (one pass over
      //    the layer's nodes), then the y and z interpolation sweeps
      double Tx[Q2];
#pragma unroll
      for (int a = 0; a < Q; a++) {
        const double va = kTab.V[a][s], da = kTab.D[a][s];
        const double* tp = Tr + ((ib + a) % NR) * PL + ms0;
#pragma unroll
        for (int b = 0; b < Q; b++)
#pragma unroll
          for (int c = 0; c < Q; c++) {
            const double v = tp[b * NZT + c];
            // first plane: a product (no zero initialisation)
            T[b * Q + c] = a == 0 ? va * v : fma(va, v, T[b * Q + c]);
            Tx[b * Q + c] = a == 0 ? da * v : fma(da, v, Tx[b * Q + c]);
          }
      }
      if (top) {
        // +z facet (operators.py:275-290): the c = P face values are
        // x-interpolated at Gauss point s already; y-interpolate, flux,
        // y-project onto the nodes (b, P)
        const double area0 = A.hh * A.hh;
        const double ws = kTab.W[s];
        double fq[Q];
#pragma unroll
        for (int qb = 0; qb < Q; qb++) {
          double acc = B::V(0, qb) * T[0 * Q + P];
#pragma unroll
          for (int b = 1; b < Q; b++) acc = fma(B::V(b, qb), T[b * Q + P], acc);
          fq[qb] = surface_flux(PP, acc) * (-(area0 * (ws * B::W(qb))));
        }
#pragma unroll
        for (int b = 0; b < Q; b++) {
          double acc = B::V(b, 0) * fq[0];
#pragma unroll
          for (int qb = 1; qb < Q; qb++) acc = fma(B::V(b, qb), fq[qb], acc);
          ftop[b] = acc;
        }
      }
      sweep2<P, 1, false, false>(T);
      sweep2<P, 0, false, false>(T);
#pragma unroll
      for (int q = 0; q < Q2; q++) G[q] = 0.0;
      if (F.diffusion) {
        sweep2<P, 1, false, false>(Tx);
        sweep2<P, 0, false, false>(Tx);
        // 2. fluxes at the Gauss points of slab s
#pragma unroll
        for (int qb = 0; qb < Q; qb++)
#pragma unroll
          for (int qc = 0; qc < Q; qc++) {
            const int q = qb * Q + qc;
            const double gx = Tx[q];
            double gy = B::Dq(0, qb) * T[0 * Q + qc];
            double gz = B::Dq(0, qc) * T[qb * Q + 0];
#pragma unroll
            for (int m = 1; m < Q; m++) {
              gy = fma(B::Dq(m, qb), T[m * Q + qc], gy);
              gz = fma(B::Dq(m, qc), T[qb * Q + m], gz);
            }
            const int q3 = s * Q2 + q;
            double kq;
            if (P >= 4) {
              // branch-free: the law always, the frozen value selected
              // (measured: p = 4 faster, p = 3 slower)
              const double g = clamp01(fma(T[q], PP.inv_dT_l, A.glo));
              if (RCF) {
                double r = A.rc[cell * Q3 + q3];
                if (A.pending && !F.frozen) {
                  r = dmax(r, g);
                  A.rc[cell * Q3 + q3] = r;
                }
                kq = conductivity(PP, g, r);
              } else {
                kq = fma(g, A.kB, A.kA);
              }
              kq = F.frozen ? A.frozen_k : kq;
            } else if (F.frozen) {
              kq = A.frozen_k;
            } else {
              const double g = clamp01(fma(T[q], PP.inv_dT_l, A.glo));
              if (RCF) {
                double r = A.rc[cell * Q3 + q3];
                if (A.pending) {
                  r = dmax(r, g);
                  A.rc[cell * Q3 + q3] = r;
                }
                kq = conductivity(PP, g, r);
              } else {
                kq = fma(g, A.kB, A.kA);
              }
            }
            const double cq = -A.hw3[q3] * kq;
            Y[(q * Q + s) * NC + cl] = cq * gx;
            const double fy = cq * gy, fz = cq * gz;
#pragma unroll
            for (int m = 0; m < Q; m++) {
              G[m * Q + qc] = fma(B::Dq(m, qb), fy, G[m * Q + qc]);
              G[qb * Q + m] = fma(B::Dq(m, qc), fz, G[qb * Q + m]);
            }
          }
      }
      if (LATENT) {
#pragma unroll
        for (int q = 0; q < Q2; q++)
          if (fabs(T[q] - A.lat_mid) < A.lat_half) lmask |= 1u << q;
      }
    }
    __syncthreads();  // B3: (SHORT) the ring's first P slots are free
    if (SHORT && i + 1 < i1) {
      load_planes(P * (i + 1) + 1, P);
      cp_commit();
    }
    if (live) {
      if (F.diffusion) {
        double dqt[Q];
#pragma unroll
        for (int m = 0; m < Q; m++) dqt[m] = kTab.Dq[s][m];
#pragma unroll
        for (int q = 0; q < Q2; q++) {
          const double* yp = Y + q * Q * NC + cl;
          double acc = G[q];
#pragma unroll
          for (int m = 0; m < Q; m++) acc = fma(dqt[m], yp[m * NC], acc);
          G[q] = acc;
        }
      }
      // 3. y and z projections of slab s
      sweep2<P, 0, true, false>(G);
      sweep2<P, 1, true, false>(G);
      if (F.source) {
        const double ax = anchor<P>(A, 0, i), ay = anchor<P>(A, 1, j), az = anchor<P>(A, 2, k);
#pragma unroll 1
        for (int bi = 0; bi < A.nb; bi++) {
          const DevBeam bm = A.beams[bi];
          if (!beam_hits_cell(PP, bm, ax, ay, az, A.h)) continue;
          double sy[Q], sz[Q], fyq[Q], fzq[Q];
#pragma unroll
          for (int q = 0; q < Q; q++) {
            const double dy = (ay + B::U(q) * A.h) - bm.y;
            const double z = az + B::U(q) * A.h;
            fyq[q] = exp((-2.0 * (dy * dy)) / PP.R2) * B::W(q);
            fzq[q] = (z >= bm.z_top - PP.h_powder && z <= bm.z_top) ? B::W(q) : 0.0;
          }
#pragma unroll
          for (int a = 0; a < Q; a++) {
            double y = 0.0, zz = 0.0;
#pragma unroll
            for (int q = 0; q < Q; q++) {
              y = fma(B::V(a, q), fyq[q], y);
              zz = fma(B::V(a, q), fzq[q], zz);
            }
            sy[a] = y;
            sz[a] = zz;
          }
          const double dx = (ax + kTab.U[s] * A.h) - bm.x;
          const double fxs = exp((-2.0 * (dx * dx)) / PP.R2) * kTab.W[s];
          const double coef = (bm.peak * A.detw0) * fxs;
#pragma unroll
          for (int b = 0; b < Q; b++) {
            const double sab = coef * sy[b];
#pragma unroll
            for (int c = 0; c < Q; c++) G[b * Q + c] = fma(sab, sz[c], G[b * Q + c]);
          }
        }
      }
      if (top) {
#pragma unroll
        for (int b = 0; b < Q; b++) G[b * Q + P] += ftop[b];
      }
#pragma unroll
      for (int q = 0; q < Q2; q++) X[(q * Q + s) * NC + cl] = G[q];
      if (LATENT) {
        // y/z-projected capacity increments of slab s, kept in T
#pragma unroll
        for (int q = 0; q < Q2; q++) T[q] = (lmask >> q) & 1u ? A.lw3[s * Q2 + q] : 0.0;
        if (lmask) {
          sweep2<P, 0, true, false>(T);
          sweep2<P, 1, true, false>(T);
        }
      }
    }
    // B4 (+ does any cell of the tile have latent increments in this layer)
    const bool lat_now = LATENT ? __syncthreads_or(lmask != 0u) != 0 : (__syncthreads(), false);
    const bool latn = LATENT && (lat_now || lat_prev);
    const int par = i & 1;
    double vt[Q];
#pragma unroll
    for (int m = 0; m < Q; m++) vt[m] = kTab.V[s][m];
    if (live) {
      // 4. x projection onto node plane a = s
#pragma unroll
      for (int q = 0; q < Q2; q++) {
        const double* xp = X + q * Q * NC + cl;
        double acc = vt[0] * xp[0];
#pragma unroll
        for (int m = 1; m < Q; m++) acc = fma(vt[m], xp[m * NC], acc);
        G[q] = acc;
      }
      if (s == 0) {
#pragma unroll
        for (int q = 0; q < Q2; q++) G[q] += Cx[((par ^ 1) * Q2 + q) * NC + cl];
      }
      double* dst = s == P ? Cx + par * Q2 * NC : Y + s * Q2 * NC;
#pragma unroll
      for (int q = 0; q < Q2; q++) dst[q * NC + cl] = G[q];
    }
    if (LATENT && latn) {
      // latent layers only: the same x projection through X (three extra
      // barriers), element planes of the increments back into X
      if (lat_now) {
        __syncthreads();
        if (live) {
#pragma unroll
          for (int q = 0; q < Q2; q++) X[(q * Q + s) * NC + cl] = T[q];
        }
        __syncthreads();
        if (live) {
#pragma unroll
          for (int q = 0; q < Q2; q++) {
            const double* xp = X + q * Q * NC + cl;
            double acc = vt[0] * xp[0];
#pragma unroll
            for (int m = 1; m < Q; m++) acc = fma(vt[m], xp[m * NC], acc);
            T[q] = acc;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < Q2; q++) T[q] = 0.0;
      }
      if (live && s == 0 && lat_prev) {
#pragma unroll
        for (int q = 0; q < Q2; q++) T[q] += CL[((par ^ 1) * Q2 + q) * NC + cl];
      }
      __syncthreads();
      if (live) {
        double* dl = s == P ? CL + par * Q2 * NC : X + s * Q2 * NC;
#pragma unroll
        for (int q = 0; q < Q2; q++) dl[q * NC + cl] = T[q];
      }
    }
    __syncthreads();  // B5
    if (live && s < P)
      finalize_owned(ib + s, Y + s * Q2 * NC + cl, X + s * Q2 * NC + cl,
                     (s == 0 && i == i0 && (i0 > 0 || A.iface_lo)) ? 2 : 0, latn);
    lat_prev = lat_now;
  }
  // last node plane of the chunk: the carried x face
  if (live && s == 0) {
    const int par = (i1 - 1) & 1;
    finalize_owned(P * i1, Cx + par * Q2 * NC + cl, CL + par * Q2 * NC + cl,
                   (i1 < A.nx || A.iface_hi) ? 1 : 0, LATENT && lat_prev);
  }
  block_max2(bad ? (double)NAN : amax, smax, A.red);
}
