// Shared device helpers for the LJ 12-6 force path (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "b200md.h"

#define LMD_CHECK_LAUNCH()                                   \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return lmd::set_cuda_error(e_);   \
  } while (0)

namespace lmd {

int set_cuda_error(cudaError_t e);

// Kernel constants derived from LJParams exactly as the reference does
// (executor.py:160-161): eps24 = 24*eps, sigma2 = sigma*sigma, rc2 = cutoff*cutoff.
struct LJK {
  double rc2, sigma2, eps24, eps48, eps4;
  // folded powers of sigma: f = u^4 (c12 u^3 - c6), e = u^3 (e12 u^3 - e6), u = 1/r2
  double c12, c6, e12, e6;
  long long rc2_bits;  // bit pattern of rc2 (positive doubles order like int64)
};

inline LJK make_ljk(const lmd_lj* p) {
  LJK k;
  k.rc2 = p->cutoff * p->cutoff;
  {
    union {
      double d;
      long long i;
    } u;
    u.d = k.rc2;
    k.rc2_bits = u.i;
  }
  k.sigma2 = p->sigma * p->sigma;
  k.eps24 = 24.0 * p->epsilon;
  k.eps48 = 48.0 * p->epsilon;
  k.eps4 = 4.0 * p->epsilon;
  const double s6 = k.sigma2 * k.sigma2 * k.sigma2;
  k.c12 = k.eps48 * s6 * s6;
  k.c6 = k.eps24 * s6;
  k.e12 = k.eps4 * s6 * s6;
  k.e6 = k.eps4 * s6;
  return k;
}

// r2 exactly as the reference computes it ((dx*dx + dy*dy) + dz*dz, no FMA;
// executor.py:93-94), so every cutoff decision is bit-identical.
__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Cutoff decision identical to the reference's `r2 >= rc2` test at two FP64
// slots less than r2_exact: r2 is formed with FMAs (|error| of a few ulp), the
// comparison happens on the bit patterns on the integer pipes, and only
// candidates within kR2Band ulps of rc2 are re-evaluated with the exact,
// unfused reference expression.  Returns the r2 used for the force.
constexpr long long kR2Band = 64;
__device__ __forceinline__ bool within_cutoff(double dx, double dy, double dz, const LJK& k,
                                              double& r2) {
  r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const long long b = __double_as_longlong(r2);
  if (b < k.rc2_bits - kR2Band) return true;
  if (b > k.rc2_bits + kR2Band) return false;
  r2 = r2_exact(dx, dy, dz);
  return r2 < k.rc2;
}

// 1/x for normal positive x: MUFU.RCP64H seed + one cubic Newton step
// (3 DFMA), ~1 ulp; the force tolerance is 1e-12 relative.
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  e = fma(e, e, e);
  return fma(y, e, y);
}

// Force scalar f with F_i += f * d (d = r_i - r_j), for r2 < rc2:
// f = 24 eps (2 s6^2 - s6) / r2, s6 = (sigma^2 / r2)^3 (kernels.py:112-126).
__device__ __forceinline__ double lj_scalar(double r2, const LJK& k, double& s6) {
  double inv = rcp_fast(r2);
  double s2 = k.sigma2 * inv;
  s6 = s2 * s2 * s2;
  return (s6 * inv) * fma(k.eps48, s6, -k.eps24);
}

// pattern (a, b) at warp width 32, lane -> (i_off, j_off) exactly as
// kernels.py:250-265 (_lane_templates).
template <int P>
struct Pattern;
template <>
struct Pattern<LMD_ONE_BY_V> {
  static constexpr int A = 1, B = 32;
  __device__ static int ioff(int l) { return 0; }
  __device__ static int joff(int l) { return l; }
};
template <>
struct Pattern<LMD_V_BY_ONE> {
  static constexpr int A = 32, B = 1;
  __device__ static int ioff(int l) { return l; }
  __device__ static int joff(int l) { return 0; }
};
template <>
struct Pattern<LMD_TWO_BY_HALF> {
  static constexpr int A = 2, B = 16;
  __device__ static int ioff(int l) { return l >> 4; }
  __device__ static int joff(int l) { return l & 15; }
};
template <>
struct Pattern<LMD_HALF_BY_TWO> {
  static constexpr int A = 16, B = 2;
  __device__ static int ioff(int l) { return l & 15; }
  __device__ static int joff(int l) { return l >> 4; }
};

// Sum over the lanes that share an i (i.e. over the j_off lanes).
template <int P>
__device__ __forceinline__ double reduce_j(double v) {
  if (P == LMD_ONE_BY_V) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  } else if (P == LMD_TWO_BY_HALF) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  } else if (P == LMD_HALF_BY_TWO) {
    v += __shfl_xor_sync(0xffffffffu, v, 16);
  }
  return v;
}

// Sum over the lanes that share a j (i.e. over the i_off lanes): the
// transposed store of the Newton3 j-side (kernels.py:9-16).
template <int P>
__device__ __forceinline__ double reduce_i(double v) {
  if (P == LMD_V_BY_ONE) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  } else if (P == LMD_TWO_BY_HALF) {
    v += __shfl_xor_sync(0xffffffffu, v, 16);
  } else if (P == LMD_HALF_BY_TWO) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One 256-bit read-only load per particle (LDG.E.ENL2.256 on sm_100a): a
// pos4 record is exactly one 32-byte sector.
__device__ __forceinline__ double4 ld_pos4(const double* pos4, long long k) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "l"(pos4 + 4 * k));
  return r;
}

// Deterministic fixed-order reduction of per-warp (epot, virial) partials.
int reduce_ev(const double* partials, int64_t nslots, lmd_stats* stats, cudaStream_t s);

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lmd
