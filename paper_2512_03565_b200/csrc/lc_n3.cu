// Colored Newton3 linked-cell traversals lc_c08 / lc_c18 (sm_100a).
//
// Reference: traversals.py:190-241 (_schedule_c18 / _schedule_c08) with the
// concurrency contract of traversals.py:1-6 -- units of one color but
// different bases may run concurrently, the units of one base run in order.
// Here: one kernel launch per color, one warp per base.  A base's write set
// (c08: its 2x2x2 block; c18: its cell and the 13 forward neighbours) is
// accumulated in the warp's shared memory -- i-side and j-side (dual write,
// kernels.py:9-16 transposed store) -- and added to the global forces once
// at the end.  Same-color write sets are disjoint, so no atomics and the
// summation order is fixed: deterministic forces.
#include "common.cuh"

namespace lmd {

constexpr int kN3Warps = 4;

struct CellTab {
  const int32_t* start;  // merged (buffer_at) view
  const int32_t* count;
  const int32_t* ocount;  // owned count (state 1 if > 0)
  const int32_t* hcount;
  const uint8_t* dup;
};

__device__ __forceinline__ int cell_state(const CellTab& t, long long l) {
  return t.ocount[l] > 0 ? 1 : (t.hcount[l] > 0 ? 2 : 0);
}

// One unit: i particles [is, is+ni) (owned cell), j particles [js, js+nj);
// `n3` dual-writes; `same` = self unit (strict upper triangle when n3).
// i slots / j slots index the warp's shared accumulators (-1: not written).
template <int P, bool EV>
__device__ __forceinline__ void n3_unit(int lane, const double* __restrict__ pos4, int is, int ni,
                                        int js, int nj, bool n3, bool same, int mult,
                                        int i_slot0, int j_slot0, double* __restrict__ acc,
                                        int acc_stride, const LJK& k, long long& pairs,
                                        long long& pairs_halo, int& overlap, double& e_acc,
                                        double& v_acc, int n_owned) {
  using Pat = Pattern<P>;
  const int io = Pat::ioff(lane), jo = Pat::joff(lane);
  for (int ci = 0; ci < ni; ci += Pat::A) {
    const int il = ci + io;
    const bool iact = il < ni;
    const double4 pi = ld_pos4(pos4, is + (iact ? il : 0));
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int cj = 0; cj < nj; cj += Pat::B) {
      const int jl = cj + jo;
      double bx = 0.0, by = 0.0, bz = 0.0;
      bool valid = iact && jl < nj;
      if (same) valid = valid && (n3 ? jl > il : jl != il);
      if (valid) {
        const double4 pj = ld_pos4(pos4, js + jl);
        if (pj.w != (double)LMD_DUMMY) {
          const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
          double r2;
          if (within_cutoff(dx, dy, dz, k, r2)) {
            if (r2 == 0.0) {
              overlap = 1;
            } else {
              double s6;
              const double f = lj_scalar(r2, k, s6) * (double)mult;
              ax = fma(f, dx, ax);
              ay = fma(f, dy, ay);
              az = fma(f, dz, az);
              if (n3) {
                bx = -f * dx;
                by = -f * dy;
                bz = -f * dz;
              }
              pairs += mult;
              const bool jhalo = js + jl >= n_owned;
              if (jhalo) pairs_halo += mult;
              if (EV) {
                const double w = (n3 ? 1.0 : 0.5) * mult;
                e_acc = fma(w * s6, fma(k.eps4, s6, -k.eps4), e_acc);
                v_acc = fma((n3 ? 1.0 : 0.5) * f, r2, v_acc);
              }
            }
          }
        }
      }
      if (n3) {
        // transposed store: reduce the j contributions over the i lanes
        bx = reduce_i<P>(bx);
        by = reduce_i<P>(by);
        bz = reduce_i<P>(bz);
        if (io == 0 && jl < nj) {
          double* a = acc + (j_slot0 + jl);
          a[0] += bx;
          a[acc_stride] += by;
          a[2 * acc_stride] += bz;
        }
        __syncwarp();
      }
    }
    ax = reduce_j<P>(ax);
    ay = reduce_j<P>(ay);
    az = reduce_j<P>(az);
    if (jo == 0 && iact) {
      double* a = acc + (i_slot0 + il);
      a[0] += ax;
      a[acc_stride] += ay;
      a[2 * acc_stride] += az;
    }
    __syncwarp();
  }
}

// c08 in-block ranks (traversals.py:94-105)
__device__ __forceinline__ void c08_rank(int dx, int dy, int dz, int& r1, int& r2) {
  r1 = 4 * (dx < 0 ? -dx : 0) + 2 * (dy < 0 ? -dy : 0) + (dz < 0 ? -dz : 0);
  r2 = 4 * (dx > 0 ? dx : 0) + 2 * (dy > 0 ? dy : 0) + (dz > 0 ? dz : 0);
}

// forward direction f (0..12) in itertools.product order (traversals.py:80-83)
__device__ __forceinline__ void fwd_dir(int f, int& dx, int& dy, int& dz) {
  int n = 0;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b)
      for (int c = -1; c <= 1; ++c) {
        const bool fwd = c > 0 || (c == 0 && b > 0) || (c == 0 && b == 0 && a > 0);
        if (!fwd) continue;
        if (n == f) {
          dx = a;
          dy = b;
          dz = c;
          return;
        }
        ++n;
      }
}

// Write-set cell w of a base: c08 -> block cell offsets (w in 0..7, bit 2 x,
// bit 1 y, bit 0 z); c18 -> 0 = the anchor, 1..13 = forward neighbours.
template <bool C08>
__device__ __forceinline__ void wset_offset(int w, int& ox, int& oy, int& oz) {
  if (C08) {
    ox = (w >> 2) & 1;
    oy = (w >> 1) & 1;
    oz = w & 1;
  } else if (w == 0) {
    ox = oy = oz = 0;
  } else {
    fwd_dir(w - 1, ox, oy, oz);
  }
}

template <int P, bool EV, bool C08>
__global__ void __launch_bounds__(32 * kN3Warps)
    lc_n3_kernel(long long t0, long long t1, long long t2, int color, long long nbx,
                 long long nby, long long nbz, LJK k, const double* __restrict__ pos4,
                 CellTab tab, int n_owned, int cap, double* __restrict__ fx,
                 double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                 lmd_stats* __restrict__ stats) {
  constexpr int W = C08 ? 8 : 14;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int stride = W * cap;
  double* acc = smem + (long long)wid * 3 * stride;
  const long long b = (long long)blockIdx.x * kN3Warps + wid;
  const long long nb = nbx * nby * nbz;
  long long pairs = 0, pairs_halo = 0;
  int overlap = 0;
  double e_acc = 0.0, v_acc = 0.0;
  if (b < nb) {
    // base coordinates of this color: c08 anchors step 2 (parity = color
    // bits), c18 anchors step 3/3/2 (color = x%3 + 3(y%3) + 9(z%2))
    long long ax, ay, az;
    if (C08) {
      ax = 2 * (b % nbx) + (color & 1);
      ay = 2 * ((b / nbx) % nby) + ((color >> 1) & 1);
      az = 2 * (b / (nbx * nby)) + ((color >> 2) & 1);
    } else {
      ax = 3 * (b % nbx) + color % 3;
      ay = 3 * ((b / nbx) % nby) + (color / 3) % 3;
      az = 2 * (b / (nbx * nby)) + color / 9;
    }
    if (ax < t0 && ay < t1 && az < t2) {
      // zero the write-set accumulators
      for (int s = lane; s < 3 * stride; s += 32) acc[s] = 0.0;
      __syncwarp();
      const long long alin = ax + t0 * (ay + t1 * az);
      // self unit of the anchor cell (only owned cells have one)
      if (cell_state(tab, alin) == 1) {
        const int s0 = tab.start[alin], n0 = tab.count[alin];
        n3_unit<P, EV>(lane, pos4, s0, n0, s0, n0, true, true, 1, 0, 0, acc, stride, k, pairs,
                       pairs_halo, overlap, e_acc, v_acc, n_owned);
      }
      for (int f = 0; f < 13; ++f) {
        int dx, dy, dz;
        fwd_dir(f, dx, dy, dz);
        // the pair (a, b = a + d) anchored at a (lower linear index)
        long long ax0, ay0, az0;
        if (C08) {
          ax0 = ax + (dx < 0 ? 1 : 0);
          ay0 = ay + (dy < 0 ? 1 : 0);
          az0 = az + (dz < 0 ? 1 : 0);
        } else {
          ax0 = ax;
          ay0 = ay;
          az0 = az;
        }
        const long long bx0 = ax0 + dx, by0 = ay0 + dy, bz0 = az0 + dz;
        if (ax0 >= t0 || ay0 >= t1 || az0 >= t2) continue;
        if (bx0 < 0 || bx0 >= t0 || by0 < 0 || by0 >= t1 || bz0 < 0 || bz0 >= t2) continue;
        const long long la = ax0 + t0 * (ay0 + t1 * az0), lb = bx0 + t0 * (by0 + t1 * bz0);
        const int sa = cell_state(tab, la), sb = cell_state(tab, lb);
        if (sa == 0 || sb == 0 || (sa == 2 && sb == 2)) continue;
        const int mult = 1 + (tab.dup ? tab.dup[la] : 0);
        // write-set slots of the two cells
        int wa, wb;
        if (C08) {
          wa = 4 * (int)(ax0 - ax) + 2 * (int)(ay0 - ay) + (int)(az0 - az);
          wb = 4 * (int)(bx0 - ax) + 2 * (int)(by0 - ay) + (int)(bz0 - az);
        } else {
          wa = 0;
          wb = 1 + f;
        }
        long long li = la, lj = lb;
        int wi = wa, wj = wb;
        bool n3 = true;
        if (sa == 2 || sb == 2) {
          // _emit_pair halo rule: the owned side is i, never Newton3
          if (sa == 2) {
            li = lb;
            lj = la;
            wi = wb;
            wj = wa;
          }
          n3 = false;
        } else if (C08) {
          int r1, r2;
          c08_rank(dx, dy, dz, r1, r2);
          if (r2 < r1) {
            li = lb;
            lj = la;
            wi = wb;
            wj = wa;
          }
        }
        n3_unit<P, EV>(lane, pos4, tab.start[li], tab.count[li], tab.start[lj], tab.count[lj],
                       n3, false, mult, wi * cap, wj * cap, acc, stride, k, pairs, pairs_halo,
                       overlap, e_acc, v_acc, n_owned);
      }
      // flush the write set (owned cells only; images are never written)
      for (int w = 0; w < W; ++w) {
        int ox, oy, oz;
        wset_offset<C08>(w, ox, oy, oz);
        const long long cx = ax + ox, cy = ay + oy, cz = az + oz;
        if (cx >= t0 || cy >= t1 || cz >= t2) continue;
        const long long l = cx + t0 * (cy + t1 * cz);
        if (cell_state(tab, l) != 1) continue;
        const int s0 = tab.start[l], n0 = tab.count[l];
        for (int q = lane; q < n0; q += 32) {
          fx[s0 + q] += acc[w * cap + q];
          fy[s0 + q] += acc[stride + w * cap + q];
          fz[s0 + q] += acc[2 * stride + w * cap + q];
        }
      }
    }
  }
  pairs = warp_sum_ll(pairs);
  pairs_halo = warp_sum_ll(pairs_halo);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && b < nb) {
    if (pairs) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pairs);
    if (pairs_halo)
      atomicAdd((unsigned long long*)&stats->pairs_owned_halo, (unsigned long long)pairs_halo);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
  if (EV) {
    e_acc = warp_sum(e_acc);
    v_acc = warp_sum(v_acc);
    if (lane == 0) {
      ev[2 * b] = e_acc;
      ev[2 * b + 1] = v_acc;
    }
  }
}

static inline long long cdivll(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace lmd

using namespace lmd;

extern "C" {

int64_t lmd_lc_n3_ev_slots(const lmd_grid* g) {
  // largest per-color base count over c08 and c18, rounded to the block
  const long long c08 = cdivll(g->tdims[0], 2) * cdivll(g->tdims[1], 2) * cdivll(g->tdims[2], 2);
  const long long c18 = cdivll(g->tdims[0], 3) * cdivll(g->tdims[1], 3) * cdivll(g->tdims[2], 2);
  const long long m = c08 > c18 ? c08 : c18;
  return cdivll(m, kN3Warps) * kN3Warps;
}

int lmd_force_lc_n3(const lmd_grid* g, const lmd_lj* lj, int traversal, int pattern, int flags,
                    const double* pos4, int64_t n_owned, const int32_t* cell_start,
                    const int32_t* cell_count, const int32_t* o_count, const int32_t* h_count,
                    const uint8_t* dup, int max_cell, double* fx, double* fy, double* fz,
                    double* ev_scratch, lmd_stats* stats, void* stream) {
  if (traversal != LMD_LC_C08 && traversal != LMD_LC_C18) return LMD_ERR_CONFIG;
  if (max_cell < 1) max_cell = 1;
  const bool c08 = traversal == LMD_LC_C08;
  const int W = c08 ? 8 : 14;
  const size_t smem = (size_t)kN3Warps * 3 * W * max_cell * sizeof(double);
  if (smem > 227 * 1024) return LMD_ERR_CONFIG;
  const LJK k = make_ljk(lj);
  const CellTab tab = {cell_start, cell_count, o_count, h_count, dup};
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  const long long t0 = g->tdims[0], t1 = g->tdims[1], t2 = g->tdims[2];
  const int ncolors = c08 ? 8 : 18;
  if (cudaMemsetAsync(fx, 0, n_owned * sizeof(double), s) != cudaSuccess ||
      cudaMemsetAsync(fy, 0, n_owned * sizeof(double), s) != cudaSuccess ||
      cudaMemsetAsync(fz, 0, n_owned * sizeof(double), s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  for (int color = 0; color < ncolors; ++color) {
    long long nbx, nby, nbz;
    if (c08) {
      nbx = cdivll(t0 - (color & 1), 2);
      nby = cdivll(t1 - ((color >> 1) & 1), 2);
      nbz = cdivll(t2 - ((color >> 2) & 1), 2);
    } else {
      nbx = cdivll(t0 - color % 3, 3);
      nby = cdivll(t1 - (color / 3) % 3, 3);
      nbz = cdivll(t2 - color / 9, 2);
    }
    const long long nb = nbx * nby * nbz;
    if (nb <= 0) continue;
    const unsigned blocks = (unsigned)cdivll(nb, kN3Warps);
    double* evc = ev_scratch;  // per-color partials reduced right away
#define LMD_N3(PP, EVB, C8)                                                                   \
  do {                                                                                        \
    auto kern = lc_n3_kernel<PP, EVB, C8>;                                                    \
    if (smem > 48 * 1024)                                                                     \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    kern<<<blocks, 32 * kN3Warps, smem, s>>>(t0, t1, t2, color, nbx, nby, nbz, k, pos4, tab,  \
                                             (int)n_owned, max_cell, fx, fy, fz, evc, stats); \
  } while (0)
#define LMD_N3_P(PP)                              \
  do {                                            \
    if (c08) {                                    \
      if (ev) LMD_N3(PP, true, true);             \
      else LMD_N3(PP, false, true);               \
    } else {                                      \
      if (ev) LMD_N3(PP, true, false);            \
      else LMD_N3(PP, false, false);              \
    }                                             \
  } while (0)
    switch (pattern) {
      case LMD_ONE_BY_V: LMD_N3_P(LMD_ONE_BY_V); break;
      case LMD_V_BY_ONE: LMD_N3_P(LMD_V_BY_ONE); break;
      case LMD_TWO_BY_HALF: LMD_N3_P(LMD_TWO_BY_HALF); break;
      case LMD_HALF_BY_TWO: LMD_N3_P(LMD_HALF_BY_TWO); break;
      default: return LMD_ERR_CONFIG;
    }
#undef LMD_N3_P
#undef LMD_N3
    LMD_CHECK_LAUNCH();
    if (ev) {
      const int rc = reduce_ev(evc, cdivll(nb, kN3Warps) * kN3Warps, stats, s);
      if (rc) return rc;
    }
  }
  return LMD_OK;
}

}  // extern "C"
