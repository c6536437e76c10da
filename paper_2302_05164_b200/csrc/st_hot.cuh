// Per-degree hot-kernel translation unit body: st_hot_p<P>.cu defines
// ST_HOT_P and includes this file, so the four degrees compile in parallel
// and only the changed degree's kernels are rebuilt.
#pragma once
#include "st_structured.cuh"

#ifndef ST_HOT_P
#error "define ST_HOT_P before including st_hot.cuh"
#endif

namespace st {

// 1D tables of this TU's degree for runtime-indexed lookups (k_xslab:
// the slab index s of a thread), initialised at compile time from the
// generated tables (st_basis_tables.h)
struct DevTab {
  double V[kMQ][kMQ], D[kMQ][kMQ], Dq[kMQ][kMQ], W[kMQ], U[kMQ];
};
template <int P>
constexpr DevTab make_devtab() {
  DevTab t{};
  for (int a = 0; a <= P; a++) {
    t.W[a] = Basis<P>::W(a);
    t.U[a] = Basis<P>::U(a);
    for (int q = 0; q <= P; q++) {
      t.V[a][q] = Basis<P>::V(a, q);
      t.D[a][q] = Basis<P>::D(a, q);
      t.Dq[a][q] = Basis<P>::Dq(a, q);
    }
  }
  return t;
}
static __constant__ DevTab kTab = make_devtab<ST_HOT_P>();

}  // namespace st

#include "st_xmarch.cuh"

namespace st {

template <int P, int CY, int CZ, bool LAT>
static constexpr size_t march_smem() {
  constexpr int PL = (P * CY + 1) * (P * CZ + 1);
  constexpr int EW = P * (P + 1) * (P + 1);
  constexpr int Q = P + 1;
  // COOP tables of k_xmarch (p >= 2): Sy, Sz, Sx, facet fluxes and terms
  constexpr int TAB = P >= 2 ? (CY + CZ + 1) * kMaxTabBeams * Q + 2 * CY * Q * Q : 0;
  return (size_t)((2 * P + 1) * PL + (LAT ? 2 : 1) * EW * CY * CZ + Q * Q * CY * CZ + TAB) *
         sizeof(double);
}

static constexpr size_t march2_smem() {
  constexpr int P = 2, CY = 8, CZ = 16, Q = 3;
  return (size_t)((2 * P + 1) * kX2Plane + P * Q * Q * (CY + 2) * (CZ + 2) +
                  Q * Q * CY * CZ + (CY + CZ + 1) * kMaxTabBeams * Q + 2 * CY * Q * Q) *
         sizeof(double);
}

template <int P, bool LAT>
static cudaError_t hot_kernel(bool slab, bool rcf, bool x2, const void** fn, size_t* smem,
                              int* threads) {
#if ST_HOT_P == 2
  {
    if (x2) {
      *fn = (const void*)k_xmarch2<LAT>;
      *smem = march2_smem();
      *threads = 128;
      static bool attr2 = false;
      if (attr2) return cudaSuccess;
      cudaError_t e =
          cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
      attr2 = e == cudaSuccess;
      return e;
    }
  }
#endif
  if (slab) {
    constexpr int CY = SlabTile<P>::CY, CZ = SlabTile<P>::CZ;
    *fn = rcf ? (const void*)k_xslab<P, CY, CZ, LAT, true> : (const void*)k_xslab<P, CY, CZ, LAT, false>;
    *smem = (size_t)slab_smem_doubles<P, CY, CZ, LAT>() * sizeof(double);
    *threads = (P + 1) * CY * CZ;
  } else {
    constexpr int CY = Tile<P>::CY, CZ = Tile<P>::CZ;
    *fn = rcf ? (const void*)k_xmarch<P, CY, CZ, LAT, true> : (const void*)k_xmarch<P, CY, CZ, LAT, false>;
    *smem = march_smem<P, CY, CZ, LAT>();
    *threads = CY * CZ;
  }
  // dynamic shared memory above 48 KB is opt-in per kernel (once)
  static bool attr[2][2] = {};
  if (attr[slab][rcf]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  attr[slab][rcf] = e == cudaSuccess;
  return e;
}

template <int P>
int hot_resident(bool slab, bool lat) {
  const void* fn;
  size_t smem;
  int threads, nb = 0;
  const bool x2 = P == 2 && !slab && use_xmarch2();
  cudaError_t e = lat ? hot_kernel<P, true>(slab, false, x2, &fn, &smem, &threads)
                      : hot_kernel<P, false>(slab, false, x2, &fn, &smem, &threads);
  if (e == cudaSuccess) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem);
  cudaGetLastError();
  return nb > 0 ? nb : 1;
}

template <int P>
cudaError_t hot_launch(const SArgs& A, bool slab, bool lat, bool rcf, dim3 grid,
                       cudaStream_t stream) {
  const void* fn;
  size_t smem;
  int threads;
  const bool x2 = P == 2 && A.x2 != 0;
  cudaError_t e = lat ? hot_kernel<P, true>(slab, rcf, x2, &fn, &smem, &threads)
                      : hot_kernel<P, false>(slab, rcf, x2, &fn, &smem, &threads);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<SArgs*>(&A)};
  return cudaLaunchKernel(fn, grid, dim3(threads), args, smem, stream);
}

template int hot_resident<ST_HOT_P>(bool, bool);
template cudaError_t hot_launch<ST_HOT_P>(const SArgs&, bool, bool, bool, dim3, cudaStream_t);

}  // namespace st
