// Pointwise physics on the device.  Each function restates one
// reference law with the same operation order (material.py, physics.py);
// fp64 throughout.
#pragma once

#include "st_internal.h"
#include <cstdlib>

namespace st {

// select-based max / clamp: two compares and selects instead of the
// NaN-propagating fmax/fmin sequences (a NaN state is caught separately by
// the divergence flag, so NaN semantics do not matter here)
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }
// the same clamp on the integer pipe: sign bit for x < 0, bit-pattern
// compare with 1.0 for x > 1 (non-negative doubles order like their bits);
// used where it measured faster (k_xmarch p >= 2)
__device__ __forceinline__ double clamp01_int(double x) {
  const long long b = __double_as_longlong(x);
  const long long one = 0x3FF0000000000000LL;
  return __longlong_as_double(b < 0 ? 0LL : (b > one ? one : b));
}
// the same result from the high word alone (4 SASS instructions instead of
// 8: ISETP, 2 VIMNMX, SEL): x < 0 (sign bit) -> +0, x >= 1 (high word >=
// 0x3FF00000; 1 + tiny has the same high word and clamps to 1) -> 1.0,
// else x unchanged; NaNs go to 0 / 1 by sign like clamp01_int
__device__ __forceinline__ double clamp01_hi(double x) {
  const int hi = __double2hiint(x);
  const unsigned lo = (unsigned)__double2loint(x);
  const int h = min(max(hi, 0), 0x3FF00000);
  const unsigned l = ((unsigned)hi < 0x3FF00000u) ? lo : 0u;
  return __hiloint2double(h, (int)l);
}


// any(|x_i - mid| < half) over N values as one chain of predicated
// compares (setp ... .or, DSETP.OR in SASS), 8 per inline-asm block: the
// predicate stays in a predicate register instead of the min-reduction
// nvcc forms from an |=-loop
__device__ __forceinline__ unsigned any_abs_lt8(unsigned p, const double* x, double mid,
                                                double half) {
  unsigned r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
      "setp.lt.or.f64 q, %2, %10, q;\n\tsetp.lt.or.f64 q, %3, %10, q;\n\t"
      "setp.lt.or.f64 q, %4, %10, q;\n\tsetp.lt.or.f64 q, %5, %10, q;\n\t"
      "setp.lt.or.f64 q, %6, %10, q;\n\tsetp.lt.or.f64 q, %7, %10, q;\n\t"
      "setp.lt.or.f64 q, %8, %10, q;\n\tsetp.lt.or.f64 q, %9, %10, q;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(p), "d"(fabs(x[0] - mid)), "d"(fabs(x[1] - mid)), "d"(fabs(x[2] - mid)),
        "d"(fabs(x[3] - mid)), "d"(fabs(x[4] - mid)), "d"(fabs(x[5] - mid)),
        "d"(fabs(x[6] - mid)), "d"(fabs(x[7] - mid)), "d"(half));
  return r;
}
template <int N>
__device__ __forceinline__ bool any_abs_lt(const double* x, double mid, double half) {
  unsigned p = 0;
#pragma unroll
  for (int i = 0; i + 8 <= N; i += 8) p = any_abs_lt8(p, x + i, mid, half);
#pragma unroll
  for (int i = N - N % 8; i < N; i++) p |= fabs(x[i] - mid) < half ? 1u : 0u;
  return p != 0;
}

// g(T) (material.py:46-57): 0 below T_s, 1 above T_l, ramp between.
__device__ __forceinline__ double liquid_fraction(const DevParams& P, double T) {
  double ramp = (T - P.T_s) / P.dT_l;
  return T < P.T_s ? 0.0 : (T > P.T_l ? 1.0 : ramp);
}

// Same law with the ramp as a multiply by 1/(T_l - T_s) (hot kernels).
__device__ __forceinline__ double liquid_fraction_fast(const DevParams& P, double T) {
  double ramp = (T - P.T_s) * P.inv_dT_l;
  return T < P.T_s ? 0.0 : (T > P.T_l ? 1.0 : ramp);
}

// k = (r_p k_p + r_m k_m) + r_s k_s, r_s clamped at 0 (material.py:68-85).
__device__ __forceinline__ double conductivity(const DevParams& P, double g, double rc) {
  double r_p = 1.0 - rc;
  double r_s = rc - g;
  r_s = r_s < 0.0 ? 0.0 : r_s;
  return (r_p * P.k_p + g * P.k_m) + r_s * P.k_s;
}

// dk/dT at frozen r_c (material.py:88-94).
__device__ __forceinline__ double conductivity_derivative(const DevParams& P, double T) {
  return (T > P.T_s && T < P.T_l) ? P.dk_slope : 0.0;
}

// rho * c_app(T): rho c (+ rho L/(T_lat_l-T_lat_s) strictly inside the
// latent interval when the extension is on).
__device__ __forceinline__ double heat_capacity(const DevParams& P, double T) {
  double v = P.rhoc;
  if (P.latent && T > P.T_lat_s && T < P.T_lat_l) v = P.rhoc + P.lat_bump;
  return v;
}

// Evaporation term (physics.py:186-202) at a clamped temperature above
// T_v.  Out of line: it only runs on vapourising facets, and inlining its
// exp / sqrt / divisions into every facet quadrature point of the hot
// kernels costs instruction cache on every step.
static __device__ __noinline__ double evaporation_term(double Tc, double cp082, double C_T, double inv_Tv,
                                                double C_M, double h_v, double c_mat,
                                                double T_h0) {
  double mdot = cp082 * exp(-C_T * (1.0 / Tc - inv_Tv)) * sqrt(C_M / Tc);
  return mdot * (h_v + c_mat * (Tc - T_h0));
}

// Outward surface flux: radiation (physics.py:174-183) + evaporation
// (physics.py:186-202) + convection (extension).
__device__ __forceinline__ double surface_flux(const DevParams& P, double T) {
  double T2 = T * T;
  double q = P.eps_sigma * (T2 * T2 - P.Ti4);
  if (P.evap_on) {
    double Tc = T < P.T_max ? T : P.T_max;
    Tc = Tc < 1.0 ? 1.0 : Tc;
    if (Tc > P.T_v)
      q = q + evaporation_term(Tc, P.cp082, P.C_T, P.inv_Tv, P.C_M, P.h_v, P.c_mat, P.T_h0);
  }
  if (P.h_conv != 0.0) q = q + P.h_conv * (T - P.T_inf);
  return q;
}

// Gaussian slab source at one point (physics.py:154-171).
__device__ __forceinline__ double beam_source(const DevParams& P, const DevBeam& b,
                                              double x, double y, double z) {
  double dx = x - b.x;
  double dy = y - b.y;
  double r2 = dx * dx + dy * dy;
  bool in_slab = (z >= b.z_top - P.h_powder) && (z <= b.z_top);
  double q = b.peak * exp((-2.0 * r2) / P.R2);
  return in_slab ? q : 0.0;
}

// Cell-level hit test of the reference (operators.py:295-307): xy box
// distance to the beam axis within cutoff, and overlap with the slab.
__device__ __forceinline__ bool beam_hits_cell(const DevParams& P, const DevBeam& b,
                                               double ax, double ay, double az,
                                               double h) {
  if (b.peak == 0.0) return false;
  double dx = fmax(fmax(ax - b.x, b.x - ax - h), 0.0);
  double dy = fmax(fmax(ay - b.y, b.y - ay - h), 0.0);
  double zlo = b.z_top - P.h_powder, zhi = b.z_top;
  return (dx * dx + dy * dy <= P.cut2) && (az <= zhi) && (az + h >= zlo);
}

// order-preserving bit key of a double (for atomicMax of signed values)
__device__ __forceinline__ unsigned long long order_key(double x) {
  unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__host__ __device__ inline double key_to_double(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ULL) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}

// block-wide max of (|x|, x) into two global order keys; every thread of
// the block must call it; one atomic pair per block
__device__ __forceinline__ void block_max2(double absval, double val,
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
    for (int i = 1; i < nw; i++) {
      ka = s_a[i] > ka ? s_a[i] : ka;
      ks = s_s[i] > ks ? s_s[i] : ks;
    }
    // same-address atomics serialise in L2: only blocks that raise the
    // running maximum issue one (the slot only ever grows)
    const volatile unsigned long long* vs = slot;
    if (ka > vs[0]) atomicMax(slot, ka);
    if (ks > vs[1]) atomicMax(slot + 1, ks);
  }
}

// programmatic dependent launch (PDL) of the unstructured scan loop's chain
// k_rhs_cells -> k_step_nodes (-> k_distribute) -> next step: a kernel
// launched with the attribute may start while its predecessor drains; each
// CTA waits for the predecessor's completion (and memory flush) before it
// reads or writes anything, then lets its own successor be staged.  With a
// plain launch both instructions are no-ops.  (Measured on the structured
// k_xmarch -> k_seam_list chain too: neutral per step, e2e 33.7 -> 30.3
// GDoF/s, so the structured path launches plainly.)
__device__ __forceinline__ void pdl_wait_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// The scan kernels split the two: pdl_release() first thing, so that the
// successor is staged (and runs its own table prefetch) while this kernel
// still waits -- it is only released once every CTA of this kernel is
// resident, and it touches nothing but static tables before its own
// pdl_wait(), which returns when this kernel (and with it every earlier one)
// has completed and flushed.
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

static inline bool use_pdl() {
  static const bool on = !(getenv("ST_NO_PDL") && getenv("ST_NO_PDL")[0] == '1');
  return on;
}

}  // namespace st
