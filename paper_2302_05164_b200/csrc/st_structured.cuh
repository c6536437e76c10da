// Structured backend: kernel argument block and the device helpers shared
// by the host-side backend (st_structured.cu) and the per-degree hot-kernel
// translation units (st_hot_p{1..4}.cu, compiled in parallel).
#pragma once
#include "st_common.cuh"
#include "st_basis_tables.h"

namespace st {

constexpr int kMQ = 5;

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
  // seam partial sums: 8 slot arrays of nv doubles (slot = x side + 2 y
  // side + 4 z side of the writing CTA), plain stores, no clearing
  // seam partials, slot-major: slot s of node idx at s * snv + idx (the
  // partials of consecutive seam nodes are stored coalesced); cseam holds
  // the latent capacity increments in the same layout
  double* fseam;
  double* cseam;
  // k_xslab contexts with latent heat: (f, dc) as one double2 per entry
  // in fseam instead (one 16-byte store per seam node, measured faster
  // there; k_xmarch is faster with the split arrays)
  int seam_pair;
  // k_xmarch latent x-face carry, per (CTA, thread) slot (Q^2 doubles
  // entry-major); only touched by cells with latent Gauss points
  double* lcarry;
  // k_xmarch2: latent increments of the cells that have any, per (CTA,
  // entry, thread) (global scratch, L2 resident), and the latent interval as
  // a window of high words (candidates for the exact test)
  double* ecg;
  int lat_hi0, lat_hiw;
  // k_xmarch2 launches (x2, set by the host per launch); with seamcnt != 0
  // the kernel completes the seams of ordinary planes itself: one arrival
  // counter per (plane, seam group), index (I GY + gy) GZ + gz with gy / gz
  // = 2 line for a tile seam line, 2 tile + 1 inside a tile; m1_0 / m1_p: 1D
  // lumped masses of a cell's end nodes (re-entrant edge of a fitted part)
  int x2;
  // CTA-layers that gathered latent increments, accumulated over launches
  // (the host picks the kernel for latent-dense fields from it)
  unsigned long long* latstat;
  int* seamcnt;
  int GY, GZ;
  double m1_0, m1_p;
  int64_t snv;
  // rank interfaces: own pre-summed plane (packed after the sweep) and the
  // neighbour's, per side (0: local plane 0, 1: local plane NX-1)
  double* ipf[2];
  double* ipc[2];
  const double* irf[2];
  const double* irc[2];
  int nb;
  const DevBeam* beams;
  double dt;
  DevParams P;
  unsigned long long* red;
  // uniform consolidated history (r_c = rc_value >= 1 >= g): the law
  // k = (r_p k_p + g k_m) + r_s k_s collapses to k = kA + g kB
  double kA, kB;
  // k_xmarch: -(h/2) kA, -(h/2) kB (a frozen conductivity: -(h/2) k, 0)
  // and -(h/2) for the stored-history law
  double kAh, kBh, mhh;
  double glo;     // -T_s / (T_l - T_s): g = clamp(T * inv_dT_l + glo)
  double lat_mid, lat_half;  // latent interval as |T - mid| < half
  double hw3[125];  // (h/2) W_qa W_qb W_qc      (diffusion weight)
  double lw3[125];  // rho L/dT (h/2)^3 W3        (latent capacity bump)
  // C^-1 of the constant lumped capacity as a tensor product of inverse
  // 1D lumped masses (row sums, operators.py:325-334):
  // C^-1(I,J,K) = inv_rcdw im(I) im(J) im(K)
  double inv_rcdw;
  double imr[5];          // interior node residue a = 1..P-1
  double imv_int, imv_end;  // cell vertex inside / at the end of the line
  // x-slab of a larger box: global plane offset / count, rank interfaces
  int gI0, gNX, iface_lo, iface_hi;
  // fitted part (cell row k holds cells i < xext[k], non-decreasing in k;
  // nullptrs for a full box): node (I, J, K) lives at pbase[I] + J (NZ -
  // pkmin[I]) + K; text[t] = x extent (cells) of tile row t; ioff_hi = id
  // of the first node of plane NX-1
  const int64_t* pbase;
  const int* pkmin;
  const int* text;
  int64_t ioff_hi;
  // first x chunk of this launch (a step may be launched as chunk ranges:
  // rank-interface chunks first, interior after, st_explicit_step_begin)
  int zoff;
};

// seam slot access (see SArgs::fseam)
__device__ __forceinline__ void seam_store(const SArgs& A, int64_t idx, int slot, double f,
                                           double dc, bool latent) {
  const int64_t so = (int64_t)slot * A.snv + idx;
  if (latent && A.seam_pair) {
    reinterpret_cast<double2*>(A.fseam)[so] = make_double2(f, dc);
  } else {
    A.fseam[so] = f;
    if (latent) A.cseam[so] = dc;
  }
}
__device__ __forceinline__ void seam_add(const SArgs& A, int64_t idx, int slot, double& f,
                                         double& dc, bool latent) {
  const int64_t so = (int64_t)slot * A.snv + idx;
  if (latent && A.seam_pair) {
    const double2 v = reinterpret_cast<const double2*>(A.fseam)[so];
    f += v.x;
    dc += v.y;
  } else {
    f += A.fseam[so];
    if (latent) dc += A.cseam[so];
  }
}


// inverse 1D lumped mass of node L on a line of N nodes
template <int P>
__device__ __forceinline__ double inv_mass1(const SArgs& A, int L, int N) {
  const int a = L % P;
  if (a != 0) return A.imr[a];
  return (L == 0 || L == N - 1) ? A.imv_end : A.imv_int;
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
        // compile-time coefficients (st_basis_tables.h): nvcc keeps IEEE
        // products by 0.0 (0 x inf = NaN), so the exact zeros of the
        // GLL/Gauss tables are skipped here explicitly (the tests resolve
        // after unrolling); a leading 1.0 is a copy.  Bitwise the same for
        // finite inputs.
        double acc = 0.0;
        bool init = false;
#pragma unroll
        for (int m = 0; m < Q; m++) {
          const double cf = TR ? Basis<P>::V(q, m) : Basis<P>::V(m, q);
          if (cf == 0.0) continue;
          acc = init ? fma(cf, in[m], acc) : (cf == 1.0 ? in[m] : cf * in[m]);
          init = true;
        }
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


// node update with its complete f (operators.py:359-368); with the latent
// extension the lumped capacity is C_const + dC(T)
__device__ __forceinline__ double finalize_node(const SArgs& A, double ci, bool bottom, double T,
                                                double f, double dc, bool latent) {
  // the latent increment of the lumped capacity only counts when positive:
  // Lagrange bases of degree >= 2 are negative at some Gauss points, so a
  // cell partly in the latent interval can lump a negative increment
  // 1 / (1/ci + dc) with one division
  if (latent && dc > 0.0) ci = ci / fma(ci, dc, 1.0);
  double o = T + A.dt * (ci * f);
  o = (A.dir_bottom && bottom) ? A.P.T_inf : o;
  // selects, not branches (measured faster in every hot kernel): rhs mode
  // (mode 1) returns f
  return A.mode == 1 ? f : o;
}

// A/B hook (compile time): k_xmarch2 stages its node planes with bulk
// asynchronous copies (cp.async.bulk + mbarrier, one copy per tile row,
// UBLKCP / SYNCS in SASS) instead of 8-byte cp.async per lane.  The reference
// numbering gives node rows an odd length (2 nz + 1 doubles), so a row starts
// on 8 bytes only: the copy takes the 16-byte aligned superset of the row and
// the consumers add a per-plane, per-row-parity shift of 0 or 1 doubles.
// Bitwise the same fields (profiles/scripts/r2_s4_bulk.sh runs the GPU tests
// on it), measured slower on config 4 (13.7 against 12.5 ms, equal on config
// 1), so the cp.async staging ships.
#ifndef ST_X2_BULK
#define ST_X2_BULK 0
#endif
// staged plane of k_xmarch2 (17 tile rows of 33 nodes): offset of tile row J
// and plane size in doubles.  Bulk rows start on 16 bytes (pitch 34) and every
// second row is skewed by 2 more, which keeps the threads' row stride an odd
// multiple of 4 banks as with the odd pitch 33 of the cp.async staging.
__host__ __device__ constexpr int x2_rowoff(int J) {
  return ST_X2_BULK ? 34 * J + 2 * (J >> 1) : 33 * J;
}
constexpr int kX2Plane = x2_rowoff(16) + (ST_X2_BULK ? 34 : 33);

// the lean Q2 explicit-step kernel (k_xmarch2) replaces k_xmarch<2> for
// explicit steps with a uniform history (ST_XMARCH2=0: the general kernel);
// read per launch, tests toggle it
static inline bool use_xmarch2() {
  const char* e = getenv("ST_XMARCH2");
  return !(e && e[0] == '0');
}

// tile of k_xmarch (CY x CZ cells, one thread per cell)
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

// tile of k_xslab (CY x CZ cells, p+1 threads per cell), min CTAs per SM,
// and the ring: SHORT keeps only the layer's P+1 planes (prefetch after
// step 1, finalisation reads T from global), otherwise 2P+1 planes
template <int P>
struct SlabTile;
template <>
struct SlabTile<1> {
  static constexpr int CY = 4, CZ = 32, MINB = 2;
  static constexpr bool SHORT = false;
};
template <>
struct SlabTile<2> {
  static constexpr int CY = 4, CZ = 8, MINB = 5;
  static constexpr bool SHORT = false;
};
template <>
struct SlabTile<3> {
  // full (2P+1)-plane ring (67 KB): 3 CTAs per SM still fit, 5 % faster than
  // the short ring at config-2 size
  static constexpr int CY = 4, CZ = 8, MINB = 3;
  static constexpr bool SHORT = false;
};
template <>
struct SlabTile<4> {
  // two CTAs per SM (168 registers, short ring: 112 KB of shared memory)
  static constexpr int CY = 4, CZ = 8, MINB = 2;
  static constexpr bool SHORT = true;
};

// beams the p >= 2 k_xmarch tables per step (separable source factors)
constexpr int kMaxTabBeams = 8;

// Hot kernels of degree P (defined in st_hot_p<P>.cu):
//   hot_resident: resident CTAs per SM of the kernel a context launches
//   hot_launch:   one launch of k_xmarch / k_xslab over `grid`
template <int P>
int hot_resident(bool slab, bool lat);
template <int P>
cudaError_t hot_launch(const SArgs& A, bool slab, bool lat, bool rcf, dim3 grid,
                       cudaStream_t stream);

}  // namespace st
