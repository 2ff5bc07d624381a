// The LJ functor on two arbitrary buffers: compute_pair_vectorized
// (kernels.py:377-424) / _pair_sweep (kernels.py:197-239) on the device.
//
// i-side: one warp per chunk of A i-particles, j-fills of B lanes (the
// pattern's register fill, kernels.py:250-265), reduction over the j lanes.
// j-side (Newton3): the two-pass atomics-free scatter -- a second launch
// with one warp per chunk of j-particles re-evaluates the same pairs
// (identical operands and operations, so bitwise the same f*d) and
// subtracts them, reduced over the i lanes.  Deterministic, no FP atomics.
#include "common.cuh"

namespace lmd {

constexpr int kPairWarps = 4;

template <int P, bool EV>
__global__ void __launch_bounds__(32 * kPairWarps)
    pair_sweep_i_kernel(int ni, const double* __restrict__ pi4, int nj,
                        const double* __restrict__ pj4, int same, int newton3, LJK k,
                        double* __restrict__ fx, double* __restrict__ fy,
                        double* __restrict__ fz, double* __restrict__ ev,
                        lmd_stats* __restrict__ stats) {
  using Pat = Pattern<P>;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * kPairWarps + (threadIdx.x >> 5);
  const int io = Pat::ioff(lane), jo = Pat::joff(lane);
  const long long il = warp * Pat::A + io;
  const bool warp_live = warp * Pat::A < ni;
  long long pairs = 0;
  int overlap = 0;
  double e_acc = 0.0, v_acc = 0.0;
  const double w = newton3 ? 1.0 : 0.5;
  if (warp_live) {
    const bool iact = il < ni;
    const double4 pi = ld_pos4(pi4, iact ? il : 0);
    const bool iown = iact && pi.w == (double)LMD_OWNED;
    double ax = 0.0, ay = 0.0, az = 0.0;
    // uniform j start: same && newton3 walks the strict upper triangle
    for (int cj = 0; cj < nj; cj += Pat::B) {
      const int q = cj + jo;
      bool ok = iown && q < nj;
      if (same) ok = ok && (newton3 ? q > il : q != il);
      if (!ok) continue;
      const double4 pj = ld_pos4(pj4, q);
      if (pj.w == (double)LMD_DUMMY) continue;
      const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
      const double r2 = r2_exact(dx, dy, dz);
      if (r2 >= k.rc2) continue;
      if (r2 == 0.0) {
        overlap = 1;
        continue;
      }
      double s6;
      const double f = lj_scalar(r2, k, s6);
      ax = fma(f, dx, ax);
      ay = fma(f, dy, ay);
      az = fma(f, dz, az);
      ++pairs;
      if (EV) {
        e_acc = fma(w * s6, fma(k.eps4, s6, -k.eps4), e_acc);
        v_acc = fma(w * f, r2, v_acc);
      }
    }
    ax = reduce_j<P>(ax);
    ay = reduce_j<P>(ay);
    az = reduce_j<P>(az);
    if (iown && jo == 0) {
      fx[il] += ax;
      fy[il] += ay;
      fz[il] += az;
    }
  }
  pairs = warp_sum_ll(pairs);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && warp_live) {
    if (pairs) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pairs);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
  if (EV) {
    e_acc = warp_sum(e_acc);
    v_acc = warp_sum(v_acc);
    if (lane == 0) {
      ev[2 * warp] = warp_live ? e_acc : 0.0;
      ev[2 * warp + 1] = warp_live ? v_acc : 0.0;
    }
  }
}

// j-side of Newton3: warp per chunk of A' = B j-particles (transposed fill).
template <int P>
__global__ void __launch_bounds__(32 * kPairWarps)
    pair_sweep_j_kernel(int ni, const double* __restrict__ pi4, int nj,
                        const double* __restrict__ pj4, int same, LJK k,
                        double* __restrict__ fx, double* __restrict__ fy,
                        double* __restrict__ fz) {
  using Pat = Pattern<P>;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * kPairWarps + (threadIdx.x >> 5);
  // transposed roles: lanes sharing a j are the i_off lanes
  const int jo = Pat::joff(lane), io = Pat::ioff(lane);
  const long long q = warp * Pat::B + jo;
  if (warp * Pat::B >= nj) return;
  const bool jact = q < nj;
  const double4 pj = ld_pos4(pj4, jact ? q : 0);
  const bool jreal = jact && pj.w != (double)LMD_DUMMY;
  double bx = 0.0, by = 0.0, bz = 0.0;
  for (int ci = 0; ci < ni; ci += Pat::A) {
    const int p = ci + io;
    bool ok = jreal && p < ni;
    if (same) ok = ok && q > p;
    if (!ok) continue;
    const double4 pi = ld_pos4(pi4, p);
    if (pi.w != (double)LMD_OWNED) continue;
    const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
    const double r2 = r2_exact(dx, dy, dz);
    if (r2 >= k.rc2 || r2 == 0.0) continue;
    double s6;
    const double f = lj_scalar(r2, k, s6);
    bx = fma(f, dx, bx);
    by = fma(f, dy, by);
    bz = fma(f, dz, bz);
  }
  bx = reduce_i<P>(bx);
  by = reduce_i<P>(by);
  bz = reduce_i<P>(bz);
  if (jreal && io == 0) {
    fx[q] -= bx;
    fy[q] -= by;
    fz[q] -= bz;
  }
}

__global__ void buffer_counts_kernel(int n, const double* __restrict__ p4,
                                     long long* __restrict__ out) {
  // out = {owned, nondummy, self_pair_slots(newton3)}; one block, ordered scan
  __shared__ long long s_nd[1024];
  long long owned = 0, nd = 0;
  // pass 1: totals
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double w = p4[4 * (long long)k + 3];
    owned += w == (double)LMD_OWNED;
    nd += w != (double)LMD_DUMMY;
  }
  s_nd[threadIdx.x] = nd;
  __syncthreads();
  __shared__ long long tot_owned, tot_nd;
  if (threadIdx.x == 0) {
    long long a = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) a += s_nd[t];
    tot_nd = a;
  }
  __syncthreads();
  s_nd[threadIdx.x] = owned;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) a += s_nd[t];
    tot_owned = a;
  }
  __syncthreads();
  // self slots with newton3: sum over owned p of (#nondummy after p); a
  // single thread walks in order (functor buffers are small)
  if (threadIdx.x == 0) {
    long long seen = 0, acc = 0;
    for (int k = 0; k < n; ++k) {
      const double w = p4[4 * (long long)k + 3];
      seen += w != (double)LMD_DUMMY;
      if (w == (double)LMD_OWNED) acc += tot_nd - seen;
    }
    out[0] = tot_owned;
    out[1] = tot_nd;
    out[2] = acc;
  }
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int64_t lmd_pair_sweep_ev_slots(int64_t ni, int pattern) {
  const int A = pattern == LMD_ONE_BY_V ? 1 : pattern == LMD_V_BY_ONE ? 32
              : pattern == LMD_TWO_BY_HALF ? 2 : 16;
  return cdiv(cdiv(ni, A), kPairWarps) * kPairWarps;
}

int lmd_pair_sweep(int64_t ni, const double* pos4_i, int64_t nj, const double* pos4_j,
                   int same, int newton3, int pattern, int flags, const lmd_lj* lj,
                   double* fxi, double* fyi, double* fzi, double* fxj, double* fyj, double* fzj,
                   double* ev_scratch, lmd_stats* stats, void* stream) {
  if (ni < 0 || nj < 0 || ni > 0x7fffffffLL || nj > 0x7fffffffLL) return LMD_ERR_CONFIG;
  if (same && (ni != nj || pos4_i != pos4_j)) return LMD_ERR_CONFIG;
  if (ni == 0 || nj == 0) return LMD_OK;
  const LJK k = make_ljk(lj);
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  const int64_t slots = lmd_pair_sweep_ev_slots(ni, pattern);
  const unsigned bi = (unsigned)(slots / kPairWarps);
#define LMD_LAUNCH_PAIR(P)                                                                   \
  do {                                                                                       \
    using Pat = Pattern<P>;                                                                  \
    if (ev)                                                                                  \
      pair_sweep_i_kernel<P, true><<<bi, 32 * kPairWarps, 0, s>>>(                           \
          (int)ni, pos4_i, (int)nj, pos4_j, same, newton3, k, fxi, fyi, fzi, ev_scratch,     \
          stats);                                                                            \
    else                                                                                     \
      pair_sweep_i_kernel<P, false><<<bi, 32 * kPairWarps, 0, s>>>(                          \
          (int)ni, pos4_i, (int)nj, pos4_j, same, newton3, k, fxi, fyi, fzi, ev_scratch,     \
          stats);                                                                            \
    LMD_CHECK_LAUNCH();                                                                      \
    if (newton3) {                                                                           \
      const unsigned bj = (unsigned)cdiv(cdiv(nj, Pat::B), kPairWarps);                      \
      pair_sweep_j_kernel<P><<<bj, 32 * kPairWarps, 0, s>>>((int)ni, pos4_i, (int)nj, pos4_j, \
                                                             same, k, fxj, fyj, fzj);        \
      LMD_CHECK_LAUNCH();                                                                    \
    }                                                                                        \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_LAUNCH_PAIR(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_LAUNCH_PAIR(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_LAUNCH_PAIR(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_LAUNCH_PAIR(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_LAUNCH_PAIR
  if (ev) return reduce_ev(ev_scratch, slots, stats, s);
  return LMD_OK;
}

int lmd_buffer_counts(int64_t n, const double* pos4, int64_t* out3, void* stream) {
  if (n < 0 || n > 0x7fffffffLL) return LMD_ERR_CONFIG;
  buffer_counts_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>((int)n, pos4, (long long*)out3);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
