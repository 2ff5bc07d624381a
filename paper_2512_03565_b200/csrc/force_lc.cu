// K2 linked-cell LJ force (Newton3 off, full 27-cell shell) and the
// geometric KernelStats of the reference's cell schedules (sm_100a).
//
// Reference semantics: executor.py:72-115 (_sweep_span) over the units of
// traversals.py:173-241 (lc_c01 / lc_c18 / lc_c08).  With Newton3 off every
// owned particle i accumulates f(i, j) over all non-dummy j != i of its own
// and its 26 neighbour cells (owned view, else halo view -- containers.py:
// 178-184); halo particles receive nothing.  The three traversals differ
// only in unit order and in which side is i, which changes the summation
// order (within the 1e-12 force tolerance) and the lane statistics; the
// latter are computed exactly by lmd_lc_stats.
#include "common.cuh"

namespace lmd {

constexpr int kWarpsPerBlock = 4;

// One warp per owned cell.  The unit (cell C, neighbour D) is swept as the
// reference's chunked double loop: ceil(nC/A) i-chunks x ceil(nD/B) j-fills,
// lane l holding pair (i_off(l), j_off(l)).
template <int P, bool EV>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    lc_force_kernel(long long d0, long long d1, long long d2, long long t0, long long t1,
                    LJK k, const double* __restrict__ pos4, const int32_t* __restrict__ cstart,
                    const int32_t* __restrict__ ccount, const uint8_t* __restrict__ dup,
                    double* __restrict__ fx,
                    double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                    lmd_stats* __restrict__ stats) {
  using Pat = Pattern<P>;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const long long nowned = d0 * d1 * d2;
  double e_acc = 0.0, v_acc = 0.0;
  int pairs = 0, pairs_halo = 0, overlap = 0;   // per lane; widened in the warp sums
  if (warp < nowned) {
    const long long cx = warp % d0 + 1;
    const long long cy = (warp / d0) % d1 + 1;
    const long long cz = warp / (d0 * d1) + 1;
    const long long lin = cx + t0 * (cy + t1 * cz);
    const int ns = ccount[lin];
    const int ss = cstart[lin];
    // lane d < 27 holds neighbour cell d (itertools.product order, traversals.py:84)
    int nb_s = 0, nb_n = 0, nb_m = 1;
    if (lane < 27) {
      const int dx = lane / 9 - 1, dy = (lane / 3) % 3 - 1, dz = lane % 3 - 1;
      const long long nl = (cx + dx) + t0 * ((cy + dy) + t1 * (cz + dz));
      nb_s = cstart[nl];
      nb_n = ccount[nl];
      // reference unit multiplicity of the cell pair (lc_c08 / lc_c18 only)
      if (dup && nl != lin) nb_m = 1 + dup[nl < lin ? nl : lin];
    }
    const int io = Pat::ioff(lane), jo = Pat::joff(lane);
    for (int ci = 0; ci < ns; ci += Pat::A) {
      const int il = ci + io;
      const bool iact = il < ns;
      const int i = ss + (iact ? il : 0);
      const double4 pi = ld_pos4(pos4, i);
      double ax = 0.0, ay = 0.0, az = 0.0;
      for (int d = 0; d < 27; ++d) {
        const int js = __shfl_sync(0xffffffffu, nb_s, d);
        const int jn = __shfl_sync(0xffffffffu, nb_n, d);
        const int mult = __shfl_sync(0xffffffffu, nb_m, d);
        const double fm = (double)mult;
        for (int cj = 0; cj < jn; cj += Pat::B) {
          const int jl = cj + jo;
          const int j = js + jl;
          if (!iact || jl >= jn || j == i) continue;
          const double4 pj = ld_pos4(pos4, j);
          if (pj.w == (double)LMD_DUMMY) continue;
          const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
          const double r2 = r2_exact(dx, dy, dz);
          if (r2 >= k.rc2) continue;
          if (r2 == 0.0) {
            overlap = 1;
            continue;
          }
          double s6;
          const double f = lj_scalar(r2, k, s6) * fm;
          ax = fma(f, dx, ax);
          ay = fma(f, dy, ay);
          az = fma(f, dz, az);
          pairs += mult;
          if (pj.w != (double)LMD_OWNED) pairs_halo += mult;
          if (EV) {
            e_acc = fma((0.5 * fm) * s6, fma(k.eps4, s6, -k.eps4), e_acc);
            v_acc = fma(0.5 * f, r2, v_acc);
          }
        }
      }
      ax = reduce_j<P>(ax);
      ay = reduce_j<P>(ay);
      az = reduce_j<P>(az);
      if (iact && jo == 0) {
        fx[i] = ax;
        fy[i] = ay;
        fz[i] = az;
      }
    }
  }
  const long long pr = warp_sum_ll((long long)pairs);
  const long long ph = warp_sum_ll((long long)pairs_halo);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && warp < nowned) {
    if (pr) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pr);
    if (ph) atomicAdd((unsigned long long*)&stats->pairs_owned_halo, (unsigned long long)ph);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
  if (EV) {
    e_acc = warp_sum(e_acc);
    v_acc = warp_sum(v_acc);
    if (lane == 0) {
      ev[2 * warp] = e_acc;
      ev[2 * warp + 1] = v_acc;
    }
  }
}

// Thread per particle for every interaction order (a, b) = (A, B): a warp
// holds A consecutive particles of the cell-sorted backing (spanning cells,
// instead of one cell's ~12 particles in 32 i lanes) and B lanes per
// particle split its candidate stream -- lane (io, jo) takes, in each of the
// 27 neighbour cells, the candidates jo, jo + B, ... (N x 1 = one lane per
// particle, 1 x N = one warp per particle).  Each lane tests its candidates
// branch-free into a hit mask (the backing holds no DUMMY records: owned
// checked at rebuild, images tagged HALO) and evaluates LJ for the set bits
// only; the B partial forces are reduced with shuffles.  Same unit order,
// per-pair arithmetic and unit multiplicity as lc_force_kernel.
template <int P, bool EV>
__global__ void __launch_bounds__(128)
    lc_tpi_kernel(int n_owned, long long t0, long long t1, LJK k, const double* __restrict__ pos4,
                  const int32_t* __restrict__ cell_of, const int32_t* __restrict__ cstart,
                  const int32_t* __restrict__ ccount, const uint8_t* __restrict__ dup,
                  double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz,
                  double* __restrict__ ev, lmd_stats* __restrict__ stats) {
  using Pat = Pattern<P>;
  constexpr int A = Pat::A, B = Pat::B;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int io = Pat::ioff(lane), jo = Pat::joff(lane);
  const long long il = warp * A + io;
  const bool iact = il < n_owned;
  const int i = iact ? (int)il : 0;
  double e_acc = 0.0, v_acc = 0.0;
  int pairs = 0, pairs_halo = 0, overlap = 0;
  double ax = 0.0, ay = 0.0, az = 0.0;
  if (warp * A < n_owned) {
    const long long lin = cell_of[i];
    const double4 pi = ld_pos4(pos4, i);
    for (int d = 0; d < 27; ++d) {
      const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
      const long long nl = lin + dx + t0 * (dy + t1 * dz);
      const int js = cstart[nl], jn = ccount[nl];
      const double fm = (dup && nl != lin) ? 1.0 + (double)dup[nl < lin ? nl : lin] : 1.0;
      const int m = fm > 1.5 ? 2 : 1;
      const int nq = (iact && jn > jo) ? (jn - jo + B - 1) / B : 0;
      const int jb = js + jo;
      for (int q0 = 0; q0 < nq; q0 += 32) {
        const int cnt = min(nq - q0, 32);
        unsigned mask = 0u;
#pragma unroll 2
        for (int q = 0; q < cnt; ++q) {
          const double4 pj = ld_pos4(pos4, jb + B * (q0 + q));
          const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
          mask |= (r2 < k.rc2 ? 1u : 0u) << q;
        }
        const int rel = i - jb;                       // the self pair, if on this stream
        if (rel >= 0 && rel % B == 0) {
          const unsigned self = (unsigned)(rel / B - q0);
          if (self < 32u) mask &= ~(1u << self);
        }
        while (mask) {
          const int j = jb + B * (q0 + __ffs(mask) - 1);
          mask &= mask - 1u;
          const double4 pj = ld_pos4(pos4, j);
          const double ddx = pi.x - pj.x, ddy = pi.y - pj.y, ddz = pi.z - pj.z;
          const double r2 = r2_exact(ddx, ddy, ddz);
          if (r2 == 0.0) {
            overlap = 1;
            continue;
          }
          double s6;
          const double f = lj_scalar(r2, k, s6) * fm;
          ax = fma(f, ddx, ax);
          ay = fma(f, ddy, ay);
          az = fma(f, ddz, az);
          pairs += m;
          if (pj.w != (double)LMD_OWNED) pairs_halo += m;
          if (EV) {
            e_acc = fma((0.5 * fm) * s6, fma(k.eps4, s6, -k.eps4), e_acc);
            v_acc = fma(0.5 * f, r2, v_acc);
          }
        }
      }
    }
  }
  ax = reduce_j<P>(ax);
  ay = reduce_j<P>(ay);
  az = reduce_j<P>(az);
  if (iact && jo == 0) {
    fx[i] = ax;
    fy[i] = ay;
    fz[i] = az;
  }
  const long long pr = warp_sum_ll((long long)pairs);
  const long long ph = warp_sum_ll((long long)pairs_halo);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0) {
    if (pr) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pr);
    if (ph) atomicAdd((unsigned long long*)&stats->pairs_owned_halo, (unsigned long long)ph);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
  if (EV) {
    e_acc = warp_sum(e_acc);
    v_acc = warp_sum(v_acc);
    if (lane == 0) {
      ev[2 * warp] = e_acc;
      ev[2 * warp + 1] = v_acc;
    }
  }
}

// --------------------------------------------------------- geometric stats
struct CellView {
  int n;      // entries of buffer_at(lin)
  int owned;  // owned entries of that view
  int state;  // occupancy: 0 empty, 1 owned, 2 halo-only
};
__device__ __forceinline__ CellView view_of(const int32_t* oc, const int32_t* hc, long long l) {
  CellView v;
  int o = oc[l], h = hc[l];
  if (o > 0) {
    v.n = o;
    v.owned = o;
    v.state = 1;
  } else {
    v.n = h;
    v.owned = 0;
    v.state = h > 0 ? 2 : 0;
  }
  return v;
}
__device__ __forceinline__ long long cdivd(long long a, long long b) { return (a + b - 1) / b; }

// in-block ranks of _block_offset_rank (traversals.py:94-105)
__device__ __forceinline__ void c08_ranks(int dx, int dy, int dz, int& r1, int& r2) {
  r1 = 4 * (dx < 0 ? -dx : 0) + 2 * (dy < 0 ? -dy : 0) + (dz < 0 ? -dz : 0);
  r2 = 4 * (dx > 0 ? dx : 0) + 2 * (dy > 0 ? dy : 0) + (dz > 0 ? dz : 0);
}

__global__ void lc_stats_kernel(long long t0, long long t1, long long t2, int trav, int newton3,
                                int a, int b, const int32_t* __restrict__ oc,
                                const int32_t* __restrict__ hc, lmd_stats* __restrict__ stats) {
  // A cell holding owned particles and images appears twice in the
  // reference's anchor list (traversals.py:133), so its forward pairs are
  // emitted twice; pair_mult carries that multiplicity.
  const long long ncell = t0 * t1 * t2;
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long inv = 0, useful = 0;
  if (q < ncell) {
    const long long x = q % t0, y = (q / t0) % t1, z = q / (t0 * t1);
    const CellView A = view_of(oc, hc, q);
    if (trav == LMD_LC_C01) {
      // traversals.py:173-187: every owned cell x its 27 occupied neighbours
      if (A.state == 1) {
        for (int d = 0; d < 27; ++d) {
          const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
          const long long nl = (x + dx) + t0 * ((y + dy) + t1 * (z + dz));
          const CellView B = view_of(oc, hc, nl);
          if (B.state == 0) continue;
          inv += cdivd(A.n, a) * cdivd(B.n, b);
          if (nl == q) useful += (long long)A.owned * (A.n - 1 > 0 ? A.n - 1 : 0);
          else useful += (long long)A.owned * B.n;
        }
      }
    } else if (A.state != 0) {
      const long long pair_mult = (oc[q] > 0 && hc[q] > 0) ? 2 : 1;
      // traversals.py:190-241: self unit per owned cell, then each unordered
      // occupied adjacent pair once from its lower-linear-index anchor
      if (A.state == 1) {
        inv += cdivd(A.n, a) * cdivd(A.n, b);
        useful += newton3 ? (long long)A.n * (A.n - 1) / 2 : (long long)A.owned * (A.n - 1);
      }
      for (int dz = 0; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const bool fwd = dz > 0 || (dz == 0 && dy > 0) || (dz == 0 && dy == 0 && dx > 0);
            if (!fwd) continue;
            const long long nx = x + dx, ny = y + dy, nz = z + dz;
            if (nx < 0 || nx >= t0 || ny < 0 || ny >= t1 || nz < 0 || nz >= t2) continue;
            const long long nl = nx + t0 * (ny + t1 * nz);
            const CellView B = view_of(oc, hc, nl);
            if (B.state == 0 || (A.state == 2 && B.state == 2)) continue;
            if (A.state == 2 || B.state == 2) {
              // _emit_pair halo rule: the owned side is i, never N3
              const CellView& I = A.state == 2 ? B : A;
              const CellView& J = A.state == 2 ? A : B;
              inv += pair_mult * cdivd(I.n, a) * cdivd(J.n, b);
              useful += pair_mult * I.owned * J.n;
            } else if (newton3) {
              bool swap = false;
              if (trav == LMD_LC_C08) {
                int r1, r2;
                c08_ranks(dx, dy, dz, r1, r2);
                swap = r2 < r1;
              }
              const CellView& I = swap ? B : A;
              const CellView& J = swap ? A : B;
              inv += pair_mult * cdivd(I.n, a) * cdivd(J.n, b);
              useful += pair_mult * I.owned * J.n;
            } else {
              inv += pair_mult * (cdivd(A.n, a) * cdivd(B.n, b) + cdivd(B.n, a) * cdivd(A.n, b));
              useful += pair_mult * ((long long)A.owned * B.n + (long long)B.owned * A.n);
            }
          }
    }
  }
  inv = warp_sum_ll(inv);
  useful = warp_sum_ll(useful);
  if ((threadIdx.x & 31) == 0 && (inv || useful)) {
    atomicAdd((unsigned long long*)&stats->kernel_invocations, (unsigned long long)inv);
    atomicAdd((unsigned long long*)&stats->useful_interactions, (unsigned long long)useful);
  }
}

__global__ void lane_slots_kernel(lmd_stats* stats, int V) {
  stats->lane_slots = stats->kernel_invocations * (long long)V;
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int64_t lmd_lc_ev_slots(const lmd_grid* g) {
  int64_t nowned = g->dims[0] * g->dims[1] * g->dims[2];
  return cdiv(nowned, kWarpsPerBlock) * kWarpsPerBlock;
}

int lmd_force_lc(const lmd_grid* g, const lmd_lj* lj, int pattern, int flags,
                 const double* pos4, const int32_t* cell_start, const int32_t* cell_count,
                 const uint8_t* dup, double* fx, double* fy, double* fz, double* ev_scratch,
                 lmd_stats* stats, void* stream) {
  const LJK k = make_ljk(lj);
  const int64_t nowned = g->dims[0] * g->dims[1] * g->dims[2];
  const unsigned blocks = (unsigned)cdiv(nowned, kWarpsPerBlock);
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  cudaStream_t s = (cudaStream_t)stream;
#define LMD_LC_ARGS                                                                           \
  g->dims[0], g->dims[1], g->dims[2], g->tdims[0], g->tdims[1], k, pos4, cell_start,          \
      cell_count, dup, fx, fy, fz, ev_scratch, stats
#define LMD_LAUNCH_LC(P)                                                                      \
  do {                                                                                        \
    if (ev) lc_force_kernel<P, true><<<blocks, 32 * kWarpsPerBlock, 0, s>>>(LMD_LC_ARGS);        \
    else lc_force_kernel<P, false><<<blocks, 32 * kWarpsPerBlock, 0, s>>>(LMD_LC_ARGS);          \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_LAUNCH_LC(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_LAUNCH_LC(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_LAUNCH_LC(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_LAUNCH_LC(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_LAUNCH_LC
#undef LMD_LC_ARGS
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, lmd_lc_ev_slots(g), stats, s);
  return LMD_OK;
}

static inline int order_A(int p) {
  return p == LMD_ONE_BY_V ? 1 : p == LMD_V_BY_ONE ? 32 : p == LMD_TWO_BY_HALF ? 2 : 16;
}

int64_t lmd_lc_tpi_ev_slots(int64_t n_owned, int pattern) {
  return cdiv(cdiv(n_owned, order_A(pattern)), 4) * 4;
}

int lmd_force_lc_particles(const lmd_grid* g, const lmd_lj* lj, int pattern, int flags,
                           const double* pos4, int64_t n_owned, const int32_t* cell_of,
                           const int32_t* cell_start, const int32_t* cell_count,
                           const uint8_t* dup, double* fx, double* fy, double* fz,
                           double* ev_scratch, lmd_stats* stats, void* stream) {
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL) return LMD_ERR_CONFIG;
  const LJK k = make_ljk(lj);
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)cdiv(cdiv(n_owned, order_A(pattern)), 4);
#define LMD_TPI(P)                                                                          \
  do {                                                                                      \
    if (ev)                                                                                 \
      lc_tpi_kernel<P, true><<<blocks, 128, 0, s>>>((int)n_owned, g->tdims[0], g->tdims[1], \
                                                    k, pos4, cell_of, cell_start,           \
                                                    cell_count, dup, fx, fy, fz,            \
                                                    ev_scratch, stats);                     \
    else                                                                                    \
      lc_tpi_kernel<P, false><<<blocks, 128, 0, s>>>((int)n_owned, g->tdims[0],             \
                                                     g->tdims[1], k, pos4, cell_of,         \
                                                     cell_start, cell_count, dup, fx, fy,   \
                                                     fz, ev_scratch, stats);                \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_TPI(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_TPI(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_TPI(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_TPI(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_TPI
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, lmd_lc_tpi_ev_slots(n_owned, pattern), stats, s);
  return LMD_OK;
}

int lmd_lc_stats(const lmd_grid* g, int traversal, int newton3, int a, int b, int vector_width,
                 const int32_t* o_count, const int32_t* h_count, lmd_stats* stats,
                 void* stream) {
  if (vector_width < 4 || (vector_width & (vector_width - 1)) != 0) return LMD_ERR_CONFIG;
  if (a < 1 || b < 1 || a * b != vector_width) return LMD_ERR_CONFIG;
  if (traversal != LMD_LC_C01 && traversal != LMD_LC_C08 && traversal != LMD_LC_C18)
    return LMD_ERR_CONFIG;
  if (traversal == LMD_LC_C01 && newton3) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)cdiv(g->ncell, 256);
  lc_stats_kernel<<<blocks, 256, 0, s>>>(g->tdims[0], g->tdims[1], g->tdims[2], traversal,
                                         newton3, a, b, o_count, h_count, stats);
  LMD_CHECK_LAUNCH();
  lane_slots_kernel<<<1, 1, 0, s>>>(stats, vector_width);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
