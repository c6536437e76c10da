// k_xmarch kernel body (included from st_xmarch.cuh).
//
// One CTA = CY x CZ cells of a (y, z) tile, marching over Lx cell layers
// in x; one thread per cell.  Per layer:
//   prefetch (cp.async) the next layer's P node planes of T,
//   evaluate the cell (cell_element, all in registers),
//   store the element planes a < P in an entry-major buffer E[q][cell]
//   (conflict-free), one barrier, then every thread finalises the nodes
//   its cell owns (local b, c < P; plus the b = P / c = P faces on the
//   tile's high edges): the <= 4 contributions of the (y, z) neighbour
//   cells are summed in a fixed order (deterministic), the update is
//   applied and T' written, or the partial sum of a tile-seam node is
//   sent to the seam buffer.
// C^-1 is the tensor-product lumped mass (inv_mass1), so the only HBM
// streams are T (read once) and T' (written once).  The apparent-capacity
// increments of the latent extension use a second element buffer Ec,
// gathered only when some cell of the CTA had a Gauss point in the latent
// interval in this or the previous layer.
#pragma once

#ifndef ST_LAT_NOINLINE
#define ST_LAT_NOINLINE 0  // A/B hook: the rare latent projection out of line (measured: the call saves
                           // ~170 live registers, 2.7 KB of stack, and the code grows 6.2k -> 7.2k)
#endif

// apparent-capacity increments rho L/dT_lat of one cell, projected from its
// Gauss points inside the latent interval (the rare path of k_xmarch, kept
// out of line so the hot loop's code stays small): the Gauss-point
// temperatures are recomputed from the staged node planes, the x face is
// carried in lcar, the element planes a < P go to ec[q * NT]
template <int P, int NT, int NZT, int PL, int NR>
__device__ __noinline__ void latent_cell(const SArgs& A, const double* Tr, int ib, int ms0,
                                         double* lcar, bool lat_had, double* ec) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  constexpr int EW = P * Q * Q;
  double t[Q3];
#pragma unroll
  for (int a = 0; a < Q; a++) {
    const double* tp = Tr + ((ib + a) % NR) * PL + ms0;
#pragma unroll
    for (int b = 0; b < Q; b++)
#pragma unroll
      for (int c = 0; c < Q; c++) t[(a * Q + b) * Q + c] = tp[b * NZT + c];
  }
  interp3<P>(t);
#pragma unroll
  for (int q = 0; q < Q3; q++) t[q] = fabs(t[q] - A.lat_mid) < A.lat_half ? A.lw3[q] : 0.0;
  project3<P>(t);
#pragma unroll
  for (int q = 0; q < Q * Q; q++) {
    if (lat_had) t[q] += lcar[q * NT];
    lcar[q * NT] = t[P * Q * Q + q];
  }
#pragma unroll
  for (int q = 0; q < EW; q++) ec[q * NT] = t[q];
}

#ifndef ST_ROWSTORE
#define ST_ROWSTORE 0  // A/B hook: T' staged in the ring and written out as whole rows
#endif

template <int P>
struct MinBlocks {
  static constexpr int v = P == 1 ? 2 : (P == 2 ? 3 : 1);
};

template <int P, int CY, int CZ, bool LATENT, bool RCF>
__global__ void __launch_bounds__(CY* CZ, MinBlocks<P>::v) k_xmarch(SArgs A) {
  constexpr int Q = P + 1;
  constexpr int Q3 = Q * Q * Q;
  constexpr int NT = CY * CZ;
  constexpr int NW = NT / 32;
  constexpr int NYT = P * CY + 1, NZT = P * CZ + 1, PL = NYT * NZT;
  constexpr int NR = 2 * P + 1;  // ring: current layer (P+1 planes) + next layer (P)
  constexpr int EW = P * Q * Q;  // stored element entries per cell (planes a < P)
  static_assert(NT % 32 == 0, "tile must be whole warps");
  extern __shared__ double sm[];
  double* Tr = sm;            // NR planes of T
  double* E = sm + NR * PL;   // E[q * NT + cell]
  double* Ec = E + EW * NT;   // latent increments (LATENT)
  // x face carried to the next layer (thread-private slots; smem keeps it
  // out of the register budget of the cell evaluation)
  double* Cx = Ec + (LATENT ? EW * NT : 0);
  // COOP (p >= 2): separable source tables and the top row's facet term
  constexpr bool COOP = P >= 2;
  constexpr int MB = kMaxTabBeams;
  double* Sy = Cx + Q * Q * NT;          // [CY][MB][Q]
  double* Sz = Sy + (COOP ? CY * MB * Q : 0);  // [CZ][MB][Q]
  double* Sx = Sz + (COOP ? CZ * MB * Q : 0);  // [MB][Q], current layer
  double* Fq = Sx + (COOP ? MB * Q : 0);       // [CY][Q * Q] facet fluxes
  double* Fo = Fq + (COOP ? CY * Q * Q : 0);   // [CY][Q * Q] facet node terms
  __shared__ int lat_any[3];  // latent increments per layer (slot i % 3)
  __shared__ long long pinfo_b[NR];  // ring: first node id (- lowest row) of a staged plane
  __shared__ int pinfo_k[NR];        // ring: lowest node row of a staged plane
  __shared__ long long pf_b[2][P];   // fitted layout of the next layer's planes (prefetch)
  __shared__ int pf_k[2][P];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // P >= 2: z-major cell order inside the CTA (tid = kl * CY + jl), so the
  // top cell row of a tile (facet term) falls in one warp instead of every
  // warp.  P = 1 keeps z-fastest lanes (unit-stride ring reads and T'
  // stores; its facet term is cheap)
  constexpr bool ZMAJ = P >= 2;
  const int kl = ZMAJ ? tid / CY : tid % CZ, jl = ZMAJ ? tid % CY : tid / CZ;
  constexpr int SY = ZMAJ ? 1 : CZ, SZ = ZMAJ ? CY : 1;  // tid stride of the y / z neighbour
  const int chunk = blockIdx.z + A.zoff;  // x chunk (launches may cover a chunk range)
  const int j0 = blockIdx.x * CY, k0 = blockIdx.y * CZ, i0 = chunk * A.Lx;
  // x extent of this tile row (a fitted part's base rows end early)
  const int ext = A.text ? A.text[blockIdx.y] : A.nx;
  if (i0 >= ext) return;
  const int i1 = min(i0 + A.Lx, ext);
  const int j = j0 + jl, k = k0 + kl;
  const bool live = j < A.ny && k < A.nz;
  const bool hiY = live && (jl == CY - 1 || j == A.ny - 1);
  const bool hiZ = live && (kl == CZ - 1 || k == A.nz - 1);
  const int Jn = min(P * CY, P * (A.ny - j0)) + 1;
  const int Kn = min(P * CZ, P * (A.nz - k0)) + 1;
  // tile-edge node planes are seams unless they are the domain boundary
  const bool sy_lo = jl == 0 && j0 > 0, sy_hi = jl == CY - 1 && j0 + CY < A.ny;
  const bool sz_lo = kl == 0 && k0 > 0, sz_hi = kl == CZ - 1 && k0 + CZ < A.nz;
  const CellFlags F{(A.flags & ST_RHS_DIFFUSION) != 0, (A.flags & ST_RHS_FACES) != 0,
                    (A.flags & ST_RHS_SOURCE) != 0 && A.nb > 0, (A.flags & ST_RHS_FROZEN_K) != 0};
  const int64_t plane_stride = (int64_t)A.NY * A.NZ;
  // node plane I: first node id (minus its lowest row) and lowest row
  auto pl_base = [&](int I) -> int64_t { return A.pbase ? A.pbase[I] : (int64_t)I * plane_stride; };
  auto pl_kmin = [&](int I) -> int { return A.pkmin ? A.pkmin[I] : 0; };
  // this thread's node origin within a plane (smem slot)
  const int ms0 = P * jl * NZT + P * kl;
  if (tid < 3) lat_any[tid] = 0;

  // stage planes Ib .. Ib+n-1: warp w copies tile rows w, w + NW, ...;
  // lane l the row entries l and l + 32 (rows run along z, contiguous)
  static_assert(NZT <= 64, "tile row wider than two warp passes");
  const bool c_lo = lane < Kn, c_hi = NZT > 32 && lane + 32 < Kn;
  // a fitted part's plane layout is read from global one layer ahead of the
  // staging that needs it (pf[layer parity]), so the table loads do not sit
  // in front of the cp.async issue
  auto prefetch_layout = [&](int Ib, int buf) {
    if (A.pbase && tid < P) {
      pf_b[buf][tid] = A.pbase[Ib + tid];
      pf_k[buf][tid] = A.pkmin[Ib + tid];
    }
  };
  auto load_planes = [&](int Ib, int n, int buf) {
#pragma unroll 1
    for (int pa = 0; pa < n; pa++) {
      const int I = Ib + pa;
      const bool pre = buf >= 0 && A.pbase;
      const int kmI = pre ? pf_k[buf][pa] : pl_kmin(I);
      const int64_t bI = pre ? pf_b[buf][pa] : pl_base(I);
      const int64_t sI = A.NZ - kmI;  // row stride of plane I
      // the plane's layout rides along in the ring for its finalisation
      if (tid == 0) {
        pinfo_b[I % NR] = bI;
        pinfo_k[I % NR] = kmI;
      }
      const double* srcT = A.T + bI + (int64_t)P * j0 * sI + P * k0 + lane;
      double* dT = Tr + (I % NR) * PL + lane;
#pragma unroll
      for (int it = 0; it < (NYT + NW - 1) / NW; it++) {
        const int r = warp + it * NW;
        if (r < Jn) {
          if (c_lo) cp_async8(dT + r * NZT, srcT + (int64_t)r * sI);
          if (c_hi) cp_async8(dT + r * NZT + 32, srcT + (int64_t)r * sI + 32);
        }
      }
    }
  };

  // 1D lumped inverse-mass factors of this thread's cell corners in y and
  // z (fixed over the march); interior residues are A.imr[b]
  const double my_0 = inv_mass1<P>(A, P * j, A.NY), my_P = inv_mass1<P>(A, P * j + P, A.NY);
  const double mz_0 = inv_mass1<P>(A, P * k, A.NZ), mz_P = inv_mass1<P>(A, P * k + P, A.NZ);

#pragma unroll
  for (int q = 0; q < Q * Q; q++) Cx[q * NT + tid] = 0.0;
  // latent x-face carry of this thread (global scratch, valid when lat_had)
  double* lcar = LATENT ? A.lcarry + (((int64_t)chunk * gridDim.y + blockIdx.y) * gridDim.x +
                                      blockIdx.x) * (Q * Q * NT) + tid
                        : nullptr;
  bool lat_had = false;
  const unsigned ymask = F.source && live ? beam_column_mask<P>(A, j, k) : 0u;
  // tabled beams (host: nb <= MB); none when no cell of the tile is within
  // a beam's y / z reach (the x factors are then never read)
  const int nbt = (F.source && __syncthreads_or(ymask != 0u)) ? min(A.nb, MB) : 0;
  if (COOP) {
    for (int e = tid; e < nbt * CY; e += NT) {
      const int b = e / CY, r = e - (e / CY) * CY;
      src_factor_xy<P>(A, anchor<P>(A, 1, j0 + r), A.beams[b].y, Sy + (r * MB + b) * Q);
    }
    for (int e = tid; e < nbt * CZ; e += NT) {
      const int b = e / CZ, r = e - (e / CZ) * CZ;
      src_factor_z<P>(A, anchor<P>(A, 2, k0 + r), A.beams[b], Sz + (r * MB + b) * Q);
    }
  }
  // the tile row of top cells (facet term) and its warp
  const int kl_top = A.nz - 1 - k0;
  const bool has_top = COOP && F.faces && A.top_faces && kl_top < CZ;
  // per-layer side work of COOP, spread over all warps: the facet terms of
  // the top row (cells split between the warps) and the source x factors
  constexpr int CPW = (CY + NW - 1) / NW;  // top-row cells per warp
  auto side_work = [&](int il) {
    if (has_top) {
      const int ib = P * il;
      face_phase<P>(A, lane, min(warp * CPW, CY), min(warp * CPW + CPW, CY), Fq, Fo,
                    [&](int r, int a, int b) {
                      return Tr[((ib + a) % NR) * PL + P * r * NZT + P * kl_top + b * NZT + P];
                    });
    }
    if (COOP && tid < nbt) src_factor_xy<P>(A, anchor<P>(A, 0, il), A.beams[tid].x, Sx + tid * Q);
  };
  // max |T'| as the bit pattern of |T'| (monotone for non-negative doubles;
  // a NaN is above +inf, so it sticks without a separate flag)
  unsigned long long amaxb = 0ull;
  double smax = -INFINITY;

  // node (b, c) of plane I owned by this thread (element plane a at pe);
  // b, c are compile-time.  xc: 0 = not an x seam, 1 = x seam with this CTA
  // on the low side (the chunk's last plane), 2 = on the high side (the
  // chunk's first plane)
  auto finalize_node3 = [&](auto bb, auto cc, const double* pe, const double* pc,
                            const double* tpl, int64_t g0, int64_t sI, bool zlo, double mz0,
                            int xc, bool latn, double imIs) {
    constexpr int b = decltype(bb)::value, c = decltype(cc)::value;
    // own cell, then the y-, z- and yz-neighbour below (fixed order)
    double f = pe[(b * Q + c) * NT];
    if (b == 0 && jl > 0) f += pe[(P * Q + c) * NT - SY];
    if (c == 0 && kl > 0) f += pe[(b * Q + P) * NT - SZ];
    if (b == 0 && c == 0 && jl > 0 && kl > 0) f += pe[(P * Q + P) * NT - SY - SZ];
    const int64_t idx = g0 + b * sI + c;
    const bool ys_lo = b == 0 && sy_lo, zs_lo = c == 0 && zlo;
    const bool seam = xc || ys_lo || (b == P && sy_hi) || zs_lo || (c == P && sz_hi);
    double dc = 0.0;
    if (LATENT && latn) {
      dc = pc[(b * Q + c) * NT];
      if (b == 0 && jl > 0) dc += pc[(P * Q + c) * NT - SY];
      if (c == 0 && kl > 0) dc += pc[(b * Q + P) * NT - SZ];
      if (b == 0 && c == 0 && jl > 0 && kl > 0) dc += pc[(P * Q + P) * NT - SY - SZ];
    }
    // branch-free: a seam node stores its partial to this CTA's slot (side
    // code per seam axis), any other node its update
    const double mzc = c == 0 ? mz0 : (c == P ? mz_P : A.imr[c]);
    const double myb = b == 0 ? my_0 : (b == P ? my_P : A.imr[b]);
    const double ci = mzc * (myb * imIs);
    const double o = finalize_node(A, ci, c == 0 && k == 0, tpl[b * NZT + c], f, dc, LATENT);
    const int slot = (xc == 2 ? 1 : 0) + (ys_lo ? 2 : 0) + (zs_lo ? 4 : 0);
    const int64_t so = (int64_t)slot * A.snv + idx;
    if (LATENT && A.seam_pair) {
      // the context keeps (f, dc) pairs (SArgs::seam_pair): one 16-byte store
      if (seam)
        reinterpret_cast<double2*>(A.fseam)[so] = make_double2(f, dc);
      else
        A.out[idx] = o;
    } else if (ST_ROWSTORE) {
      // the update goes back into the staged plane (T of this node is no
      // longer needed); the plane leaves as whole coalesced rows
      // (store_planes) -- a seam node's row entry is then a stale T that the
      // seam pass overwrites
      if (seam) {
        A.fseam[so] = f;
        if (LATENT) A.cseam[so] = dc;
      } else {
        const_cast<double*>(tpl)[b * NZT + c] = o;
      }
    } else {
      *(seam ? A.fseam + so : A.out + idx) = seam ? f : o;
      if (LATENT && seam) A.cseam[so] = dc;
    }
    if (!seam) {
      const unsigned long long ab = (unsigned long long)__double_as_longlong(o) & 0x7fffffffffffffffull;
      amaxb = ab > amaxb ? ab : amaxb;
      smax = dmax(smax, o);
    }
  };

  // a finished plane from the ring to T' as whole rows, the
  // staging's own row / lane mapping (so the prefetch that reuses a slot
  // next is ordered after these reads in every thread, no barrier needed);
  // cb / ck: the planes' layout, read from the ring before it is rewritten
  auto store_plane = [&](int I, long long base, int km) {
    const int64_t sI = A.NZ - km;
    double* dst = A.out + base + (int64_t)P * j0 * sI + P * k0 + lane;
    const double* src = Tr + (I % NR) * PL + lane;
#pragma unroll
    for (int it = 0; it < (NYT + NW - 1) / NW; it++) {
      const int r = warp + it * NW;
      if (r < Jn) {
        if (c_lo) dst[(int64_t)r * sI] = src[r * NZT];
        if (c_hi) dst[(int64_t)r * sI + 32] = src[r * NZT + 32];
      }
    }
  };
  long long cb[P];  // layout of the planes finalised in the previous layer
  int ck[P];

  // every node of plane I owned by this thread (element plane a)
  auto finalize_owned = [&](int I, int a, int xc, bool latn) {
    if (!live) return;
    // x factor of the inverse lumped mass: a line end at the box ends and
    // where this tile row's extent stops inside the box
    const int G = I + A.gI0;
    const bool xend = G == 0 || G == A.gNX - 1 || (ext < A.nx && I == P * ext);
    const double imx = (I % P) != 0 ? A.imr[I % P] : (xend ? A.imv_end : A.imv_int);
    const double imIs = imx * A.inv_rcdw;
    const double* pe = E + a * Q * Q * NT + tid;
    const double* pc = Ec + a * Q * Q * NT + tid;
    const double* tpl = Tr + (I % NR) * PL + ms0;
    // plane I's row layout (staged with its T plane); its lowest node row
    // is a z line end, and the tile's bottom nodes are a seam only where
    // material lies below
    const int kmI = pinfo_k[I % NR];
    const int64_t sI = A.NZ - kmI;
    const int64_t g0 = pinfo_b[I % NR] + (int64_t)P * j * sI + P * k;
    const bool zlo = sz_lo && kmI < P * k0;
    const double mz0 = P * k == kmI ? A.imv_end : mz_0;
    static_for<P>([&](auto bb) {
      static_for<P>([&](auto cc) { finalize_node3(bb, cc, pe, pc, tpl, g0, sI, zlo, mz0, xc, latn, imIs); });
    });
    if (hiZ)
      static_for<P>([&](auto bb) { finalize_node3(bb, IC<P>{}, pe, pc, tpl, g0, sI, zlo, mz0, xc, latn, imIs); });
    if (hiY) {
      static_for<P>([&](auto cc) { finalize_node3(IC<P>{}, cc, pe, pc, tpl, g0, sI, zlo, mz0, xc, latn, imIs); });
      if (hiZ) finalize_node3(IC<P>{}, IC<P>{}, pe, pc, tpl, g0, sI, zlo, mz0, xc, latn, imIs);
    }
  };

  // prologue: the first layer's P+1 planes (and its COOP side work)
  load_planes(P * i0, P + 1, -1);
  if (i0 + 1 < i1) prefetch_layout(P * (i0 + 1) + 1, (i0 + 1) & 1);
  cp_commit();
  if (COOP) {
    cp_wait<0>();
    __syncthreads();
    side_work(i0);
  }

  int nlat = 0;  // layers that gathered latent increments (SArgs::latstat)
  // two barriers per layer: the top one publishes the layer's staged planes
  // and retires the previous layer's finalisation (E, its ring slots and its
  // latent flag slot are free), so the next layer's prefetch goes out right
  // after it and has a whole layer to land
#pragma unroll 1
  for (int i = i0; i < i1; i++) {
    // the layer's planes landed before the previous mid barrier (or in the
    // prologue); this barrier retires the previous finalisation and
    // publishes the facet terms / x factors made during it
    cp_wait<0>();
    __syncthreads();
    if (ST_ROWSTORE && i > i0)
#pragma unroll
      for (int a = 0; a < P; a++) store_plane(P * (i - 1) + a, cb[a], ck[a]);
    if (i + 1 < i1) load_planes(P * (i + 1) + 1, P, (i + 1) & 1);
    if (i + 2 < i1) prefetch_layout(P * (i + 2) + 1, i & 1);
    cp_commit();
    if (LATENT && tid == 0) lat_any[(i + 1) % 3] = 0;  // last read by layer i-1
    if (live) {
      double t[Q3], G[Q3];
#pragma unroll
      for (int a = 0; a < Q; a++) {
        const double* tp = Tr + ((P * i + a) % NR) * PL + ms0;
#pragma unroll
        for (int b = 0; b < Q; b++)
#pragma unroll
          for (int c = 0; c < Q; c++) t[(a * Q + b) * Q + c] = tp[b * NZT + c];
      }
      interp3<P>(t);  // T at the Gauss points
      const int64_t cell = ((int64_t)i * A.ny + j) * A.nz + k;
      const int ib = P * i;
      cell_element<P, RCF, COOP>(
          A, F, i, j, k, cell, t, G, ymask,
          [&](int a, int b, int c) { return Tr[((ib + a) % NR) * PL + ms0 + b * NZT + c]; }, Sx,
          Sy + jl * MB * Q, Sz + kl * MB * Q, Fo + jl * Q * Q);
      // x face shared with the previous layer: add the carry, keep the new one
#pragma unroll
      for (int q = 0; q < Q * Q; q++) {
        G[q] += Cx[q * NT + tid];
        Cx[q * NT + tid] = G[P * Q * Q + q];
      }
#pragma unroll
      for (int q = 0; q < EW; q++) E[q * NT + tid] = G[q];
      if (LATENT) {
        // apparent-capacity increments rho L/dT_lat projected from the Gauss
        // points inside the latent interval (G is dead here, so t can be
        // reused); a predicate pass first, most cells have none
        const bool lat = any_abs_lt<Q3>(t, A.lat_mid, A.lat_half);
        if (ST_LAT_NOINLINE && lat) {
          lat_any[i % 3] = 1;
          latent_cell<P, NT, NZT, PL, NR>(A, Tr, P * i, ms0, lcar, lat_had, Ec + tid);
        } else if (lat) {
          lat_any[i % 3] = 1;
#pragma unroll
          for (int q = 0; q < Q3; q++) t[q] = fabs(t[q] - A.lat_mid) < A.lat_half ? A.lw3[q] : 0.0;
          project3<P>(t);
#pragma unroll
          for (int q = 0; q < Q * Q; q++) {
            if (lat_had) t[q] += lcar[q * NT];
            lcar[q * NT] = t[P * Q * Q + q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < Q * Q; q++) t[q] = lat_had ? lcar[q * NT] : 0.0;
#pragma unroll
          for (int q = Q * Q; q < EW; q++) t[q] = 0.0;
        }
        if (!(ST_LAT_NOINLINE && lat)) {  // (the out-of-line path stored its own)
#pragma unroll
          for (int q = 0; q < EW; q++) Ec[q * NT + tid] = t[q];
        }
        lat_had = lat;
      }
    }
    cp_wait<0>();  // the next layer's planes (prefetched at the top) have landed
    __syncthreads();
    if (COOP && i + 1 < i1) side_work(i + 1);
    // latent increments of this layer or carried from the previous one
    const bool latn = LATENT && (lat_any[i % 3] | lat_any[(i + 2) % 3]);
    if (LATENT && latn) nlat++;
#pragma unroll
    for (int a = 0; a < P; a++) {
      cb[a] = pinfo_b[(P * i + a) % NR];
      ck[a] = pinfo_k[(P * i + a) % NR];
    }
#pragma unroll 1
    for (int a = 0; a < P; a++)
      finalize_owned(P * i + a, a, (a == 0 && i == i0 && (i0 > 0 || A.iface_lo)) ? 2 : 0, latn);
  }
  cp_wait<0>();
  __syncthreads();  // the last layer's finalisation is done with E
  const long long cbl = pinfo_b[(P * i1) % NR];
  const int ckl = pinfo_k[(P * i1) % NR];
  if (ST_ROWSTORE)
#pragma unroll
    for (int a = 0; a < P; a++) store_plane(P * (i1 - 1) + a, cb[a], ck[a]);
  // last node plane of the chunk: the carried x face (as element plane 0)
  if (live) {
#pragma unroll
    for (int q = 0; q < Q * Q; q++) E[q * NT + tid] = Cx[q * NT + tid];
    if (LATENT)
#pragma unroll
      for (int q = 0; q < Q * Q; q++) Ec[q * NT + tid] = lat_had ? lcar[q * NT] : 0.0;
  }
  __syncthreads();
  finalize_owned(P * i1, 0, (i1 < ext || (A.iface_hi && ext == A.nx)) ? 1 : 0,
                 LATENT && lat_any[(i1 - 1) % 3] != 0);
  if (ST_ROWSTORE) {
    __syncthreads();
    store_plane(P * i1, cbl, ckl);
  }
  if (LATENT && tid == 0 && nlat > 0 && A.latstat) atomicAdd(A.latstat, (unsigned long long)nlat);
  block_max2(__longlong_as_double((long long)amaxb), smax, A.red);
}
