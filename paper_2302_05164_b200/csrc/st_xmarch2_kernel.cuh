// k_xmarch2: the lean Q2 explicit-step kernel (included from st_xmarch.cuh).
//
// Same scheme and the same arithmetic as k_xmarch<2, 8, 16, LATENT, false> in
// explicit-step mode (one CTA = an 8 x 16 cell (y, z) tile marching over an x
// chunk, one thread per cell, cell_element in registers, element planes in
// shared memory, fixed-order gathers, seam partials to the CTA's slots), with
// the per-layer work around the cell evaluation rebuilt for instruction
// count and stalls (ncu of k_xmarch: 28 % of all warp instructions in the
// node finalisation, 11 % in the plane staging, 5 % re-deriving per-thread
// constants the cell evaluation had pushed out of the registers):
//   * element entries are stored with a ring of zero ghost cells around the
//     tile, so the <= 4 contributions of a node are summed without
//     neighbour tests;
//   * every thread finalises the four nodes (b, c < 2) of its cell with no
//     seam logic: T' is stored unconditionally (a seam node's value there
//     is overwritten by the seam pass, which runs after this kernel) and
//     only the stability maxima skip seam nodes;
//   * the tile's perimeter nodes (high edges; low edges where they are
//     seams) are a dense second pass, one node per lane, from a per-CTA
//     table of gather offsets (absent contributions point at a zero ghost
//     entry), instead of divergent per-thread branches in every warp;
//   * per-thread constants (shared-memory offsets, node coordinates, flags)
//     and per-plane constants (layout, x factor of the lumped mass) are
//     records in shared memory, loaded where a phase starts;
//   * the staging keeps one running row pointer per plane and copies the
//     33rd column with one instruction of one warp; the fitted layout of
//     the next planes arrives by cp.async in the same group;
//   * the stability maxima live in shared memory and are only updated by
//     nodes whose high word reaches the running maximum's;
//   * the latent check is an integer window test on the high words (exact
//     test only for candidates); the rare latent increments live in an
//     L2-resident global scratch instead of 18 KB of shared memory;
//   * one loop body serves the layers and the chunk's last plane, so the
//     finalisation code exists once (instruction cache).
// Opt-in in-kernel seam completion (ST_INSEAM=1, A.seamcnt != 0; bitwise the
// seam pass but measured slower than it): the seams of
// ordinary planes (y / z tile seams; everything but the x-seam planes at chunk boundaries and
// rank interfaces, which stay with the seam pass) are finished by the last
// CTA to arrive.  Every CTA stores its partials to its slots as before; when
// its chunk is done, one lane per seam group (the tile's 4 faces and 4 corner
// lines over the chunk) bumps the group's arrival counter (after a barrier,
// fence + atomicInc that wraps back to zero), and the CTA that sees the last
// arrival sums the slots of the group's nodes in the seam pass's fixed order
// and finalises them (a dense loop with several loads in flight per thread).
// No CTA ever waits for another, and the sums do not depend on the arrival
// order.
// Results are bitwise those of k_xmarch (except the sign of exact zeros).
#pragma once

// rare paths (latent cells, x-seam planes) off the hot loop's fall-through
// code (instruction cache)
#define ST_UNLIKELY(x) __builtin_expect(!!(x), 0)

#ifndef ST_X2_MINB
#define ST_X2_MINB 3  // A/B hook: resident CTAs per SM the register allocation aims at
#endif

#ifdef ST_X2_MAXREG  // A/B hook: an explicit register cap instead of the occupancy target
#define ST_X2_BOUNDS __maxnreg__(ST_X2_MAXREG)
#else
#define ST_X2_BOUNDS __launch_bounds__(128, ST_X2_MINB)
#endif
#ifndef ST_X2_FIN_UNROLL
#define ST_X2_FIN_UNROLL 1  // A/B hook: unroll factor of the per-plane finalisation loop
#endif
#define ST_PRAGMA_(x) _Pragma(#x)
#define ST_UNROLL_N(n) ST_PRAGMA_(unroll n)

template <bool LATENT>
__global__ void ST_X2_BOUNDS k_xmarch2(SArgs A) {
  constexpr int P = 2, Q = 3, Q3 = 27, CY = 8, CZ = 16, NT = 128, NW = 4;
  constexpr int NYT = P * CY + 1, NZT = P * CZ + 1;
  constexpr bool BULK = ST_X2_BULK != 0;
  constexpr int NZP = 33;            // row pitch of the cp.async staging
  constexpr int PL = kX2Plane;       // staged plane (doubles), rows at x2_rowoff(J)
  constexpr int R1 = x2_rowoff(1) - x2_rowoff(0), R2 = x2_rowoff(2) - x2_rowoff(0);
  constexpr int NR = 2 * P + 1;
  constexpr int EW = P * Q * Q;
  // padded cell index of the element arrays: (kl + 1) * ES + jl + 1, ghost
  // cells at jl = -1, CY and kl = -1, CZ stay zero
  constexpr int ES = CY + 2, EN = ES * (CZ + 2);
  constexpr int MB = kMaxTabBeams;
  constexpr int NPER = 2 * NZT + 2 * (NYT - 2);
  extern __shared__ double sm[];
  double* Tr = sm;              // NR planes of T
  double* E = Tr + NR * PL;     // E[q * EN + cp]
  double* Cx = E + EW * EN;     // x face carried to the next layer, Cx[q * NT + tid]
  double* Sy = Cx + Q * Q * NT;          // [CY][MB][Q]
  double* Sz = Sy + CY * MB * Q;         // [CZ][MB][Q]
  double* Sx = Sz + CZ * MB * Q;         // [MB][Q], current layer
  double* Fq = Sx + MB * Q;              // [CY][Q * Q] facet fluxes
  double* Fo = Fq + CY * Q * Q;          // [CY][Q * Q] facet node terms
  // ring: per staged plane, first node id (- lowest row), lowest node row,
  // x factor of the inverse lumped mass times 1 / (rho c detw)
  __shared__ long long pinfo_b[NR];
  __shared__ int pinfo_k[NR];
  __shared__ double pinfo_im[NR];
  // bulk staging: a row lands at its 16-byte aligned position, so its first
  // node sits 0 or 1 doubles into the slot row; the shift alternates with the
  // row parity (odd row pitch): bit 0 = even rows, bit 1 = odd rows
  __shared__ int pinfo_sh[NR];
  __shared__ unsigned long long mbar[2];  // staging completion, by layer parity
  __shared__ long long pf_b[2][P];   // fitted layout of the next layer's planes (prefetch)
  __shared__ int pf_k[2][P];
  // perimeter nodes of the tile (high edges first): x = gather offsets 0, 1
  // (u16 each, into an element plane), y = offsets 2, 3, z = J | K << 8 |
  // flags << 16, w = x2_rowoff(J) + K
  __shared__ int4 peri[NPER];
  // per-thread record: x = ms0 (plane offset of the cell's low corner), y =
  // cp (padded cell index), z = flags, w = 2 j | 2 k << 16
  __shared__ int4 rec4[NT];
  // inverse 1D masses of the cell's low corner, running max |T'| (bit
  // pattern) and max T'
  __shared__ double rec_my[NT], rec_mz[NT], rec_smax[NT];
  __shared__ unsigned long long rec_amax[NT];
  __shared__ unsigned rec_ym[NT];  // beams that can reach the cell's (y, z) column
  __shared__ unsigned char latf[LATENT ? EN : 1];  // cell has latent increments this layer
  __shared__ double beam_x[MB];  // x of the tabled beams (read per layer for the x factors)
  // record flags
  constexpr int RF_LIVE = 1, RF_SY = 2, RF_SZ = 4, RF_DIR = 8;
  // perimeter flags
  constexpr int PF_LOJ = 1, PF_LOK = 2, PF_HI = 4, PF_SEAM = 8, PF_SLOT2 = 16;

  const int tid = threadIdx.x;
  const int chunk = blockIdx.z + A.zoff;
  const int j0 = blockIdx.x * CY, k0 = blockIdx.y * CZ, i0 = chunk * A.Lx;
  const int ext = A.text ? A.text[blockIdx.y] : A.nx;
  if (i0 >= ext) return;
  const int i1 = min(i0 + A.Lx, ext);
  const int Jn = min(P * CY, P * (A.ny - j0)) + 1;
  const int Kn = min(P * CZ, P * (A.nz - k0)) + 1;
#define nhi (Kn + Jn - 1)
#define nper (2 * Kn + 2 * (Jn - 2))
  // tile-edge node lines are seams unless they are the domain boundary
  const bool ty_lo = j0 > 0, ty_hi = j0 + CY < A.ny;
  const bool tz_lo = k0 > 0, tz_hi = k0 + CZ < A.nz;
  const CellFlags F{true, true, A.nb > 0, false};
  const int64_t plane_stride = (int64_t)A.NY * A.NZ;
  const double imr1 = A.imr[1];

  {
    const int kl = tid / CY, jl = tid % CY;  // z-major cell order
    const int j = j0 + jl, k = k0 + kl;
    const bool live = j < A.ny && k < A.nz;
    rec4[tid] = make_int4(x2_rowoff(P * jl) + P * kl, (kl + 1) * ES + jl + 1,
                          (live ? RF_LIVE : 0) | ((jl == 0 && ty_lo) ? RF_SY : 0) |
                              ((kl == 0 && tz_lo) ? RF_SZ : 0) |
                              ((k == 0 && A.dir_bottom) ? RF_DIR : 0),
                          (P * j) | ((P * k) << 16));
    rec_my[tid] = inv_mass1<P>(A, P * j, A.NY);
    rec_mz[tid] = inv_mass1<P>(A, P * k, A.NZ);
    rec_amax[tid] = 0ull;
    rec_smax[tid] = -INFINITY;
  }
  // zero the element arrays once (ghost and dead cells are never written)
  for (int e = tid; e < EW * EN; e += NT) E[e] = 0.0;
  if (LATENT)
    for (int e = tid; e < EN; e += NT) latf[e] = 0;
  // perimeter table: row J = Jn-1, column K = Kn-1 (high edges), then row
  // J = 0 and column K = 0 (low edges)
  for (int e = tid; e < nper; e += NT) {
    int J, K;
    if (e < Kn) {
      J = Jn - 1, K = e;
    } else if (e < nhi) {
      J = e - Kn, K = Kn - 1;
    } else if (e < nhi + Kn - 1) {
      J = 0, K = e - nhi;
    } else {
      J = e - (nhi + Kn - 1) + 1, K = 0;
    }
    const int bj = J >> 1, b = J & 1, bk = K >> 1, c = K & 1;
    const int cpn = (bk + 1) * ES + bj + 1;
    // own cell, y-, z-, yz-neighbour below (the gather's order); entry 0 of
    // the ghost corner cell is always zero
    const int o0 = (b * 3 + c) * EN + cpn;
    const int o1 = b == 0 ? (6 + c) * EN + cpn - 1 : 0;
    const int o2 = c == 0 ? (b * 3 + 2) * EN + cpn - ES : 0;
    const int o3 = (b == 0 && c == 0) ? 8 * EN + cpn - ES - 1 : 0;
    const bool loJ = J == 0, loK = K == 0, hiJ = J == Jn - 1, hiK = K == Kn - 1;
    // seams fixed over the march (the z-low seam depends on the plane)
    const bool seam = (loJ && ty_lo) || (hiJ && ty_hi) || (hiK && tz_hi);
    const int fl = (loJ ? PF_LOJ : 0) | (loK ? PF_LOK : 0) | ((hiJ || hiK) ? PF_HI : 0) |
                   (seam ? PF_SEAM : 0) | ((loJ && ty_lo) ? PF_SLOT2 : 0);
    peri[e] = make_int4(o0 | (o1 << 16), o2 | (o3 << 16), J | (K << 8) | (fl << 16), x2_rowoff(J) + K);
  }

  // x factor of the inverse lumped mass of plane I (times 1 / (rho c detw))
  auto plane_imx = [&](int I) {
    const int G = I + A.gI0;
    const bool xend = G == 0 || G == A.gNX - 1 || (ext < A.nx && I == P * ext);
    const double imx = (I & 1) ? imr1 : (xend ? A.imv_end : A.imv_int);
    return imx * A.inv_rcdw;
  };
  // (asynchronous copies in the staging's commit group: no load sits in
  // front of the barrier)
  auto prefetch_layout = [&](int Ib, int buf) {
    if (A.pbase && tid < P) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&pf_b[buf][tid])),
                   "l"(A.pbase + Ib + tid)
                   : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&pf_k[buf][tid])),
                   "l"(A.pkmin + Ib + tid)
                   : "memory");
    }
  };
  // stage plane I into ring slot rs: warp w copies tile rows w, w + 4, ...
  // (lane l the row entry l), one running row pointer; the 33rd column goes
  // with one instruction of warp 1 (lane l the row l)
  const unsigned tr_s = (unsigned)__cvta_generic_to_shared(Tr);
  const bool full = Jn == NYT && Kn == NZT;
  // bulk variant: lane r of warp pw copies tile row r with one
  // cp.async.bulk of (Kn + 1) doubles from the row's 16-byte aligned start
  // (one double before the row or one after it rides along), completing on
  // mbar[mslot]
  auto load_plane = [&](int I, int rs, long long bI, int kmI, int pw, int mslot) {
    const int lane = tid & 31, warp = tid >> 5;
    const int sI = A.NZ - kmI;
    if (tid == 0) {
      pinfo_b[rs] = bI;
      pinfo_k[rs] = kmI;
      pinfo_im[rs] = plane_imx(I);
      if (BULK) pinfo_sh[rs] = (int)(bI & 1) | ((int)((bI + sI) & 1) << 1);
    }
    if (BULK) {
      if (warp == pw && lane < Jn) {
        const long long g = bI + ((P * j0 + lane) * sI + P * k0);  // first node of the row
        const double* src = A.T + (g - (g & 1));
        const unsigned dst = tr_s + (unsigned)((rs * PL + x2_rowoff(lane)) * 8);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
            "l"(src), "r"((Kn + 1) * 8), "r"((unsigned)__cvta_generic_to_shared(&mbar[mslot]))
            : "memory");
      }
      return;
    }
    const double* src = A.T + (bI + ((P * j0 + warp) * sI + P * k0 + lane));
    const unsigned dst = tr_s + (unsigned)((rs * PL + warp * NZP + lane) * 8);
    const int64_t step = (int64_t)(NW * sI) * 8;
    if (full) {
#pragma unroll
      for (int it = 0; it < NYT / NW; it++) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + it * NW * NZP * 8),
                     "l"(src)
                     : "memory");
        src = (const double*)((const char*)src + step);
      }
      if (warp == 0)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + (NYT - 1) * NZP * 8),
                     "l"(src)
                     : "memory");
    } else {
      const bool c_lo = lane < Kn;
#pragma unroll
      for (int it = 0; it < (NYT + NW - 1) / NW; it++) {
        if (c_lo && warp + it * NW < Jn)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + it * NW * NZP * 8),
                       "l"(src)
                       : "memory");
        src = (const double*)((const char*)src + step);
      }
    }
    if (warp == 1 && Kn == NZT && lane < Jn) {
      const double* s2 = A.T + (bI + ((P * j0 + lane) * sI + P * k0 + (NZT - 1)));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                       tr_s + (unsigned)((rs * PL + lane * NZP + NZT - 1) * 8)),
                   "l"(s2)
                   : "memory");
    }
  };

  // one thread arms the layer's barrier with the bytes of its np planes;
  // every thread waits for the phase (a bounded spin: a miscount traps
  // instead of hanging the GPU)
  auto stage_arm = [&](int mslot, int np) {
    if (BULK && tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&mbar[mslot])),
                   "r"(np * Jn * (Kn + 1) * 8)
                   : "memory");
  };
  auto stage_wait = [&](int mslot, int parity) {
    if (!BULK) return;
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar[mslot]);
    unsigned done = 0;
    for (int spin = 0; !done; spin++) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          "selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(mb), "r"(parity)
          : "memory");
      if (spin > (1 << 24)) __trap();
    }
  };
  if (BULK) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(&mbar[0])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(&mbar[1])));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }

  // the first layer's P+1 planes go out now, so that their latency overlaps
  // the table set-up below (ten-layer chunks: config 1)
  int rs0 = (P * i0) % NR;  // ring slot of the layer's first plane
  {
    int rs = rs0;
    stage_arm(i0 & 1, P + 1);
    for (int pa = 0; pa <= P; pa++) {
      const int I = P * i0 + pa;
      load_plane(I, rs, A.pbase ? A.pbase[I] : (int64_t)I * plane_stride, A.pkmin ? A.pkmin[I] : 0,
                 pa, i0 & 1);
      rs = rs + 1 >= NR ? 0 : rs + 1;
    }
  }
  if (i0 + 1 < i1) prefetch_layout(P * (i0 + 1) + 1, (i0 + 1) & 1);
  cp_commit();

#pragma unroll
  for (int q = 0; q < Q * Q; q++) Cx[q * NT + tid] = 0.0;
  // latent scratch of this CTA, addressed where the rare paths need it
  // (lcar: x-face carry [q * NT + tid]; ecg: increments [q * NT + cell])
  auto cta_id = [&]() {
    return ((int64_t)(blockIdx.z + A.zoff) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  };
#define lcar (A.lcarry + cta_id() * (Q * Q * NT) + tid)
#define ecg (A.ecg + cta_id() * (EW * NT))
  bool lat_had = false;
  unsigned ymask = 0u;
  if (F.source) {
    const int kl = tid / CY, jl = tid % CY;
    if (j0 + jl < A.ny && k0 + kl < A.nz) ymask = beam_column_mask<P>(A, j0 + jl, k0 + kl);
  }
  rec_ym[tid] = ymask;
  const int nbt = (F.source && __syncthreads_or(ymask != 0u)) ? min(A.nb, MB) : 0;
  for (int e = tid; e < nbt * CY; e += NT) {
    const int b = e / CY, r = e - (e / CY) * CY;
    src_factor_xy<P>(A, anchor<P>(A, 1, j0 + r), A.beams[b].y, Sy + (r * MB + b) * Q);
  }
  for (int e = tid; e < nbt * CZ; e += NT) {
    const int b = e / CZ, r = e - (e / CZ) * CZ;
    src_factor_z<P>(A, anchor<P>(A, 2, k0 + r), A.beams[b], Sz + (r * MB + b) * Q);
  }
  if (tid < nbt) beam_x[tid] = A.beams[tid].x;
  const int kl_top = A.nz - 1 - k0;
  const bool has_top = A.top_faces && kl_top < CZ;
  constexpr int CPW = (CY + NW - 1) / NW;
  auto side_work = [&](int il, int rs0) {
    if (has_top) {
      const int lane = tid & 31, warp = tid >> 5;
      face_phase<P>(A, lane, min(warp * CPW, CY), min(warp * CPW + CPW, CY), Fq, Fo,
                    [&](int r, int a, int b) {
                      int rs = rs0 + a;
                      rs = rs >= NR ? rs - NR : rs;
                      const int sh = BULK ? ((pinfo_sh[rs] >> (b & 1)) & 1) : 0;
                      return Tr[rs * PL + x2_rowoff(P * r + b) + P * kl_top + P + sh];
                    });
    }
    if (tid < nbt) src_factor_xy<P>(A, anchor<P>(A, 0, il), beam_x[tid], Sx + tid * Q);
  };

  // stability maxima (rec_amax: |T'| as its bit pattern, rec_smax: max T'):
  // thr = high word a node must reach to be able to raise either (smax <=
  // amax), so the exact update is a rare branch
  int thr = 0;
  auto track_exact = [&](double o) {
    const unsigned long long ab =
        (unsigned long long)__double_as_longlong(o) & 0x7fffffffffffffffull;
    const unsigned long long am = rec_amax[tid];
    const double sm_ = rec_smax[tid];
    rec_amax[tid] = ab > am ? ab : am;
    const double s2 = dmax(sm_, o);
    rec_smax[tid] = s2;
    thr = max(__double2hiint(s2), 0);
  };
  auto habs = [](double o) { return __double2hiint(o) & 0x7fffffff; };

  // latent increment of a node: the contributions of the (<= 4) cells around
  // it in the gather's order; cells without increments count as zero
  auto latent_sum = [&](int cpn, int tn, int a, int b, int c) {
    // tn: thread (cell) id of the own cell of the node (may be a ghost)
    double dc = 0.0;
    if (latf[cpn]) dc = __ldcg(ecg + (a * 9 + b * 3 + c) * NT + tn);
    if (b == 0 && latf[cpn - 1]) dc += __ldcg(ecg + (a * 9 + 6 + c) * NT + tn - 1);
    if (c == 0 && latf[cpn - ES]) dc += __ldcg(ecg + (a * 9 + b * 3 + 2) * NT + tn - CY);
    if (b == 0 && c == 0 && latf[cpn - ES - 1]) dc += __ldcg(ecg + (a * 9 + 8) * NT + tn - CY - 1);
    return dc;
  };

  // a seam partial (f, latent increment) to slot entry so: one 16-byte store
  // where the context keeps (f, dc) pairs (SArgs::seam_pair)
  auto seam_put = [&](int64_t so, double f, double dc) {
    if (LATENT && A.seam_pair) {
      reinterpret_cast<double2*>(A.fseam)[so] = make_double2(f, dc);
    } else {
      A.fseam[so] = f;
      if (LATENT) A.cseam[so] = dc;
    }
  };
  auto seam_get = [&](int64_t so, double& f, double& dc) {
    if (LATENT && A.seam_pair) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(A.fseam) + so);
      f = v.x;
      dc = v.y;
    } else {
      f = __ldcg(A.fseam + so);
      dc = LATENT ? __ldcg(A.cseam + so) : 0.0;
    }
  };

  // the four nodes (b, c < 2) of this thread's cell in plane I (element
  // plane a, ring slot rs); xc: 0 = ordinary plane, 1 / 2 = x seam with this
  // CTA on the low / high side (every node of the plane is a seam then)
  auto finalize_cell = [&](int a, int rs, int xc, bool latn) {
    const int4 r = rec4[tid];
    if (!(r.z & RF_LIVE)) return;
    const int cp = r.y;
    const int kmI = pinfo_k[rs];
    const int sI = A.NZ - kmI;
    const int j2 = r.w & 0xffff, k2 = r.w >> 16;
    const int64_t g0 = pinfo_b[rs] + (j2 * sI + k2);
    const bool s_y = (r.z & RF_SY) != 0;                          // b = 0 nodes on a y seam
    const bool s_z = (r.z & RF_SZ) != 0 && kmI < P * k0;          // c = 0 nodes on a z seam
    const double* e = E + a * 9 * EN + cp;
    double f00 = e[0 * EN];
    f00 += e[6 * EN - 1];
    f00 += e[2 * EN - ES];
    f00 += e[8 * EN - ES - 1];
    double f01 = e[1 * EN];
    f01 += e[7 * EN - 1];
    double f10 = e[3 * EN];
    f10 += e[5 * EN - ES];
    const double f11 = e[4 * EN];
    double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
    if (LATENT && ST_UNLIKELY(latn)) {
      d00 = latent_sum(cp, tid, a, 0, 0);
      d01 = latent_sum(cp, tid, a, 0, 1);
      d10 = latent_sum(cp, tid, a, 1, 0);
      d11 = latent_sum(cp, tid, a, 1, 1);
    }
    if (ST_UNLIKELY(xc != 0)) {
      // x seam plane: partials to this CTA's slots
      const int xb = xc == 2 ? 1 : 0;
      const int64_t s00 = (int64_t)(xb + (s_y ? 2 : 0) + (s_z ? 4 : 0)) * A.snv + g0;
      const int64_t s01 = (int64_t)(xb + (s_y ? 2 : 0)) * A.snv + g0 + 1;
      const int64_t s10 = (int64_t)(xb + (s_z ? 4 : 0)) * A.snv + g0 + sI;
      const int64_t s11 = (int64_t)xb * A.snv + g0 + sI + 1;
      seam_put(s00, f00, d00);
      seam_put(s01, f01, d01);
      seam_put(s10, f10, d10);
      seam_put(s11, f11, d11);
      return;
    }
    const double imIs = pinfo_im[rs];
    const int psh = BULK ? pinfo_sh[rs] : 0;
    const double* tp = Tr + rs * PL + r.x + (psh & 1);            // even row of the cell
    const double* tq = Tr + rs * PL + r.x + (psh >> 1) + R1;      // odd row
    const double mz0e = k2 == kmI ? A.imv_end : rec_mz[tid];
    const double yb0 = rec_my[tid] * imIs, yb1 = imr1 * imIs;
    double c00 = mz0e * yb0, c01 = imr1 * yb0, c10 = mz0e * yb1, c11 = imr1 * yb1;
    if (LATENT && ST_UNLIKELY(latn)) {
      if (d00 > 0.0) c00 = c00 / fma(c00, d00, 1.0);
      if (d01 > 0.0) c01 = c01 / fma(c01, d01, 1.0);
      if (d10 > 0.0) c10 = c10 / fma(c10, d10, 1.0);
      if (d11 > 0.0) c11 = c11 / fma(c11, d11, 1.0);
    }
    double o00 = tp[0] + A.dt * (c00 * f00);
    double o01 = tp[1] + A.dt * (c01 * f01);
    double o10 = tq[0] + A.dt * (c10 * f10);
    double o11 = tq[1] + A.dt * (c11 * f11);
    if (r.z & RF_DIR) {
      o00 = A.P.T_inf;
      o10 = A.P.T_inf;
    }
    // a seam node's partial goes out with the perimeter pass
    double* po = A.out + g0;
    if (!(s_y || s_z)) po[0] = o00;
    if (!s_y) po[1] = o01;
    if (!s_z) po[sI] = o10;
    po[sI + 1] = o11;
    const int h00 = (s_y || s_z) ? 0 : habs(o00), h01 = s_y ? 0 : habs(o01);
    const int h10 = s_z ? 0 : habs(o10), h11 = habs(o11);
    // a warp-uniform branch (the vote keeps it from being if-converted into
    // always-issued predicated code)
    if (__any_sync(__activemask(), max(max(h00, h01), max(h10, h11)) >= thr)) {
      if (!(s_y || s_z)) track_exact(o00);
      if (!s_y) track_exact(o01);
      if (!s_z) track_exact(o10);
      track_exact(o11);
    }
  };

  // the tile's perimeter nodes of plane I, one per lane: the high edges (J =
  // Jn-1 or K = Kn-1: a seam partial to the slot where the edge is shared
  // with the next tile, the finished node where it is the domain boundary)
  // and, in an ordinary plane, the low edges that are seams
  auto finalize_edges = [&](int a, int rs, int xc, bool latn) {
    const int kmI = pinfo_k[rs];
    const int sI = A.NZ - kmI;
    const bool z_lo = tz_lo && kmI < P * k0;
    const int n = (xc == 0 && (ty_lo || z_lo)) ? nper : nhi;
    if (tid >= n) return;
    const int64_t gb = pinfo_b[rs] + ((P * j0) * sI + P * k0);
    const double* ea = E + a * 9 * EN;
#pragma unroll 1
    for (int it = tid; it < n; it += NT) {
      const int4 pr = peri[it];
      const int J = pr.z & 255, K = (pr.z >> 8) & 255, fl = pr.z >> 16;
      const bool zs = (fl & PF_LOK) && z_lo;
      const bool seam = xc != 0 || (fl & PF_SEAM) || zs;
      if (!(fl & PF_HI) && !seam) continue;  // a low edge on the domain boundary: its cells' own
      double f = ea[pr.x & 0xffff];
      f += ea[(unsigned)pr.x >> 16];
      f += ea[pr.y & 0xffff];
      f += ea[(unsigned)pr.y >> 16];
      double dc = 0.0;
      if (LATENT && ST_UNLIKELY(latn)) {
        const int bj = J >> 1, bk = K >> 1;
        dc = latent_sum((bk + 1) * ES + bj + 1, bk * CY + bj, a, J & 1, K & 1);
      }
      const int64_t idx = gb + (J * sI + K);
      if (seam) {
        const int slot = (xc == 2 ? 1 : 0) + ((fl & PF_SLOT2) ? 2 : 0) + (zs ? 4 : 0);
        seam_put((int64_t)slot * A.snv + idx, f, dc);
      } else {
        const int Jg = P * j0 + J, Kg = P * k0 + K;
        const double my = (J & 1) ? imr1 : ((Jg == 0 || Jg == A.NY - 1) ? A.imv_end : A.imv_int);
        const double mz = (K & 1) ? imr1 : ((Kg == kmI || Kg == A.NZ - 1) ? A.imv_end : A.imv_int);
        double ci = mz * (my * pinfo_im[rs]);
        if (LATENT && dc > 0.0) ci = ci / fma(ci, dc, 1.0);
        const int sh = BULK ? ((pinfo_sh[rs] >> (J & 1)) & 1) : 0;
        double o = Tr[rs * PL + pr.w + sh] + A.dt * (ci * f);
        if (A.dir_bottom && Kg == 0) o = A.P.T_inf;
        A.out[idx] = o;
        if (__any_sync(__activemask(), habs(o) >= thr)) track_exact(o);
      }
    }
  };

  // prologue: the first layer's planes were issued above; wait, then its side work
  cp_wait<0>();
  stage_wait(i0 & 1, 0);
  __syncthreads();
  side_work(i0, rs0);

  // one loop body for the layers and the chunk's last plane (tail: i == i1,
  // the carried x face as element plane 0)
  // x-seam state of the chunk's first / last plane (recomputed where used:
  // two registers less across the cell evaluation)
#define xc1 ((i1 < ext || (A.iface_hi && ext == A.nx)) ? 1 : 0)
#define xc0 ((i0 > 0 || A.iface_lo) ? 2 : 0)
  __shared__ int nlat_s;  // layers that gathered latent increments
  if (tid == 0) nlat_s = 0;
#pragma unroll 1
  for (int i = i0; i <= i1; i++) {
    const bool tail = i == i1;
    cp_wait<0>();
    __syncthreads();
    if (i + 1 < i1) {
      const int buf = (i + 1) & 1;
      int rs = rs0 + P + 1;
      rs = rs >= NR ? rs - NR : rs;
      stage_arm(buf, P);
#pragma unroll
      for (int pa = 0; pa < P; pa++) {
        long long bI;
        int kmI;
        if (A.pbase) {
          bI = pf_b[buf][pa];
          kmI = pf_k[buf][pa];
        } else {
          bI = (int64_t)(P * (i + 1) + 1 + pa) * plane_stride;
          kmI = 0;
        }
        load_plane(P * (i + 1) + 1 + pa, rs, bI, kmI, pa, buf);
        rs = rs + 1 >= NR ? 0 : rs + 1;
      }
    }
    if (i + 2 < i1) prefetch_layout(P * (i + 2) + 1, i & 1);
    cp_commit();
    bool lf = false;
    const int4 r = rec4[tid];
    const bool live = (r.z & RF_LIVE) != 0;
    const int cp = r.y;
    if (live && !tail) {
      double t[Q3], G[Q3];
      // T at the Gauss points from the layer's three staged planes
      auto gauss_T = [&](double* tt) {
        int rs = rs0;
#pragma unroll
        for (int a = 0; a < Q; a++) {
          const int psh = BULK ? pinfo_sh[rs] : 0;
          const double* tpe = Tr + rs * PL + r.x + (psh & 1);   // rows b = 0, 2
          const double* tpo = Tr + rs * PL + r.x + (psh >> 1);  // row b = 1
#pragma unroll
          for (int b = 0; b < Q; b++)
#pragma unroll
            for (int c = 0; c < Q; c++)
              tt[(a * Q + b) * Q + c] = ((b & 1) ? tpo : tpe)[(b == 0 ? 0 : (b == 1 ? R1 : R2)) + c];
          rs = rs + 1 >= NR ? 0 : rs + 1;
        }
        interp3<P>(tt);
      };
      gauss_T(t);
      // latent test right away (candidates by the high words, a superset of
      // the open interval, then the exact test), so that t dies with the
      // gradients instead of staying live across the projection; the rare
      // latent cell recomputes it
#ifndef ST_X2_LAT_EARLY
#define ST_X2_LAT_EARLY 0  // A/B hook: 1 = test before the cell evaluation, the rare latent cell
                           // recomputes t (measured slower: 13.2 vs 12.5 ms on config 4)
#endif
      bool lat = false;
      if (LATENT && ST_X2_LAT_EARLY) {
        bool cand = false;
#pragma unroll
        for (int q = 0; q < Q3; q++)
          cand |= (unsigned)(__double2hiint(t[q]) - A.lat_hi0) <= (unsigned)A.lat_hiw;
        if (ST_UNLIKELY(cand)) lat = any_abs_lt<Q3>(t, A.lat_mid, A.lat_half);
      }
      {
        const int kl = tid / CY, jl = tid % CY;
        cell_element<P, false, true>(
            A, F, i, j0 + jl, k0 + kl, 0, t, G, rec_ym[tid], [&](int, int, int) { return 0.0; }, Sx,
            Sy + jl * MB * Q, Sz + kl * MB * Q, Fo + jl * Q * Q);
      }
#ifndef ST_X2_ESTORE_FIRST
#define ST_X2_ESTORE_FIRST 0  // A/B hook: plane-1 element stores before the x-carry exchange
#endif
      if (ST_X2_ESTORE_FIRST) {
#pragma unroll
        for (int q = Q * Q; q < EW; q++) E[q * EN + cp] = G[q];
      }
#pragma unroll
      for (int q = 0; q < Q * Q; q++) {
        G[q] += Cx[q * NT + tid];
        Cx[q * NT + tid] = G[P * Q * Q + q];
      }
#pragma unroll
      for (int q = 0; q < (ST_X2_ESTORE_FIRST ? Q * Q : EW); q++) E[q * EN + cp] = G[q];
      if (LATENT && !ST_X2_LAT_EARLY) {
        bool cand = false;
#pragma unroll
        for (int q = 0; q < Q3; q++)
          cand |= (unsigned)(__double2hiint(t[q]) - A.lat_hi0) <= (unsigned)A.lat_hiw;
        if (ST_UNLIKELY(cand)) lat = any_abs_lt<Q3>(t, A.lat_mid, A.lat_half);
      }
      if (LATENT) {
        lf = lat || lat_had;
        if (ST_UNLIKELY(lat)) {
          if (ST_X2_LAT_EARLY) gauss_T(t);
#pragma unroll
          for (int q = 0; q < Q3; q++) t[q] = fabs(t[q] - A.lat_mid) < A.lat_half ? A.lw3[q] : 0.0;
          project3<P>(t);
#pragma unroll
          for (int q = 0; q < Q * Q; q++) {
            if (lat_had) t[q] += lcar[q * NT];
            lcar[q * NT] = t[P * Q * Q + q];
          }
#pragma unroll
          for (int q = 0; q < EW; q++) ecg[q * NT + tid] = t[q];
        } else if (ST_UNLIKELY(lat_had)) {
#pragma unroll
          for (int q = 0; q < Q * Q; q++) ecg[q * NT + tid] = lcar[q * NT];
#pragma unroll
          for (int q = Q * Q; q < EW; q++) ecg[q * NT + tid] = 0.0;
        }
        latf[cp] = lf ? 1 : 0;
        lat_had = lat;
      }
    } else if (live) {
#pragma unroll
      for (int q = 0; q < Q * Q; q++) E[q * EN + cp] = Cx[q * NT + tid];
      if (LATENT) {
        lf = lat_had;
        if (lat_had)
#pragma unroll
          for (int q = 0; q < Q * Q; q++) ecg[q * NT + tid] = lcar[q * NT];
        latf[cp] = lat_had ? 1 : 0;
      }
    }
    cp_wait<0>();
    // the next layer's planes (its (i + 1 - i0) / 2-th use of the barrier)
    if (i + 1 < i1) stage_wait((i + 1) & 1, ((i + 1 - i0) >> 1) & 1);
    const bool latn = LATENT ? __syncthreads_or(lf) != 0 : (__syncthreads(), false);
    if (LATENT && latn && tid == 0) nlat_s++;
    int rs1 = rs0 + P;  // first plane of the next layer
    rs1 = rs1 >= NR ? rs1 - NR : rs1;
    if (i + 1 < i1) side_work(i + 1, rs1);
    const int na = tail ? 1 : P;
    int rs = rs0;
    ST_UNROLL_N(ST_X2_FIN_UNROLL)
    for (int a = 0; a < na; a++) {
      const int xc = tail ? xc1 : ((a == 0 && i == i0) ? xc0 : 0);
      finalize_cell(a, rs, xc, latn);
      finalize_edges(a, rs, xc, latn);
      rs = rs + 1 >= NR ? 0 : rs + 1;
    }
    rs0 = rs1;
  }
#ifndef ST_X2_INSEAM
#define ST_X2_INSEAM 1  // A/B hook: compile the opt-in in-kernel seam completion
#endif
  if (ST_X2_INSEAM && A.seamcnt != nullptr) {
    // ---- seam completion of the chunk's ordinary planes ----
    // x extents of the tile rows below / above
    const int ext_lo = (A.text && blockIdx.y > 0) ? A.text[blockIdx.y - 1] : A.nx;
    const int ext_hi = (A.text && blockIdx.y + 1 < gridDim.y) ? A.text[blockIdx.y + 1] : A.nx;
    // groups: faces y-low, y-high, z-low, z-high (0-3), corner lines (J, K) =
    // (0, 0), (0, hi), (hi, 0), (hi, hi) (4-7); a group's contributors are the
    // CTAs of this chunk that share the line / face
    __shared__ unsigned char glast[8];
    __syncthreads();  // the chunk's partial stores are issued
    if (tid < 8) {
      const int g = tid;
      const bool ylo = g == 0 || g == 4 || g == 5, yhi = g == 1 || g == 6 || g == 7;
      const bool zlo = g == 2 || g == 4 || g == 6, zhi = g == 3 || g == 5 || g == 7;
      const bool ys = (ylo && ty_lo) || (yhi && ty_hi);
      const bool zs = (zlo && tz_lo && ext_lo > i0) || (zhi && tz_hi);
      const int need = (ys ? 2 : 1) * (zs ? 2 : 1);
      bool last = false;
      if (need > 1) {
        const int gy = 2 * (int)blockIdx.x + (ylo ? 0 : (yhi ? 2 : 1));
        const int gz = 2 * (int)blockIdx.y + (zlo ? 0 : (zhi ? 2 : 1));
        __threadfence();
        last = atomicInc((unsigned*)A.seamcnt + ((chunk * A.GY + gy) * A.GZ + gz),
                         (unsigned)need - 1u) == (unsigned)need - 1u;
        if (last) __threadfence();
      }
      glast[g] = last ? 1 : 0;
    }
    __syncthreads();
    // plane range of the chunk without its x-seam planes
    const int Ia = P * i0 + (xc0 != 0 ? 1 : 0), Ib = P * i1 - (xc1 != 0 ? 1 : 0);
    auto xplane = [&](int I, int e) { return I > 0 && I % (P * A.Lx) == 0 && I < P * e; };
#pragma unroll 1
    for (int g = 0; g < 8; g++) {
      if (!glast[g]) continue;
      const bool ylo = g == 0 || g == 4 || g == 5, yhi = g == 1 || g == 6 || g == 7;
      const bool zlo = g == 2 || g == 4 || g == 6, zhi = g == 3 || g == 5 || g == 7;
      const bool yn = (ylo && ty_lo) || (yhi && ty_hi);
      // nodes of the group in a plane: a face's interior line or a corner
      const int nn = g < 2 ? Kn - 2 : (g < 4 ? Jn - 2 : 1);
      const int items = (Ib - Ia + 1) * nn;
      constexpr int U = 4;  // loads of U nodes in flight per thread
#pragma unroll 1
      for (int itb = tid; itb < items; itb += U * NT) {
        double s0[U], s2[U], s4[U], s6[U], c0[U], c2[U], c4[U], c6[U], Tn[U];
        int64_t idx[U];
        int Iu[U], JK[U], km[U];
        bool zn[U], on[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int it = itb + u * NT;
          on[u] = it < items;
          s0[u] = s2[u] = s4[u] = s6[u] = c0[u] = c2[u] = c4[u] = c6[u] = Tn[u] = 0.0;
          idx[u] = 0;
          Iu[u] = JK[u] = km[u] = 0;
          zn[u] = false;
          if (!on[u]) continue;
          const int pl = it / nn, e = it - pl * nn;
          const int I = Ia + pl;
          const int J = g < 2 ? (g == 0 ? 0 : Jn - 1) : (g < 4 ? e + 1 : (yhi ? Jn - 1 : 0));
          const int K = g < 2 ? e + 1 : (g < 4 ? (g == 2 ? 0 : Kn - 1) : (zhi ? Kn - 1 : 0));
          const int kmI = A.pkmin ? A.pkmin[I] : 0;
          const int sI = A.NZ - kmI;
          const bool z = (zlo && tz_lo && kmI < P * k0 && !xplane(I, ext_lo)) ||
                         (zhi && tz_hi && !xplane(I, ext_hi));
          // a z-low line above a row that has ended is no seam at this plane
          if (!(yn || z) || ((zlo || zhi) && !yn && !z)) {
            on[u] = false;
            continue;
          }
          // (a corner line whose z seam is with the seam pass at this plane
          // is with the seam pass as a whole)
          if ((zlo && tz_lo && kmI < P * k0 && xplane(I, ext_lo)) ||
              (zhi && tz_hi && xplane(I, ext_hi))) {
            on[u] = false;
            continue;
          }
          Iu[u] = I;
          JK[u] = J | (K << 8);
          km[u] = kmI;
          zn[u] = z;
          idx[u] = (A.pbase ? A.pbase[I] : (int64_t)I * plane_stride) +
                   ((P * j0 + J) * sI + P * k0 + K);
          seam_get(idx[u], s0[u], c0[u]);
          if (yn) seam_get(2 * A.snv + idx[u], s2[u], c2[u]);
          if (z) seam_get(4 * A.snv + idx[u], s4[u], c4[u]);
          if (yn && z) seam_get(6 * A.snv + idx[u], s6[u], c6[u]);
          Tn[u] = A.T[idx[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          if (!on[u]) continue;
          const int I = Iu[u], J = JK[u] & 255, K = JK[u] >> 8, kmI = km[u];
          // the seam pass's order: x side, then z side, then y side
          const double f = ((s0[u] + s2[u]) + s4[u]) + s6[u];
          const double dc = LATENT ? ((c0[u] + c2[u]) + c4[u]) + c6[u] : 0.0;
          const int Jg = P * j0 + J, Kg = P * k0 + K;
          const double my = (J & 1) ? imr1 : ((Jg == 0 || Jg == A.NY - 1) ? A.imv_end : A.imv_int);
          // z line of the node: extents of the tile rows below / above it
          const int e_low = zlo ? ext_lo : ext, e_up = zlo ? ext : ext_hi;
          double ci;
          if (zn[u] && e_low < e_up && I == P * e_low) {
            // re-entrant edge (the lower row ends here, the upper one goes
            // on): row sum over the three cells present (operators.py:325-339)
            const double mxz = ((A.m1_p * A.m1_p) + (A.m1_p * A.m1_0)) + (A.m1_0 * A.m1_0);
            ci = (1.0 / mxz) * (my * A.inv_rcdw);
          } else {
            const double mz =
                (K & 1) ? imr1 : ((Kg == kmI || Kg == A.NZ - 1) ? A.imv_end : A.imv_int);
            ci = mz * (my * plane_imx(I));
          }
          if (LATENT && dc > 0.0) ci = ci / fma(ci, dc, 1.0);
          double o = Tn[u] + A.dt * (ci * f);
          if (A.dir_bottom && Kg == 0) o = A.P.T_inf;
          A.out[idx[u]] = o;
          if (habs(o) >= thr) track_exact(o);
        }
      }
    }
  }
  if (LATENT && tid == 0 && nlat_s > 0 && A.latstat)
    atomicAdd(A.latstat, (unsigned long long)nlat_s);
  block_max2(__longlong_as_double((long long)rec_amax[tid]), rec_smax[tid], A.red);
#undef lcar
#undef ecg
#undef xc0
#undef xc1
#undef nhi
#undef nper
}
