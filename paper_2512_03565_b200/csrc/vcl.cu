// K5-K7: Verlet cluster lists on the device (sm_100a).
//
// Reference: VerletClusterContainer (containers.py:302-479) and the vcl
// schedule (traversals.py:244-266).
//   K5 build: column key cx + width*cy with cx = floor((x-lo)/col)+1
//      (containers.py:335-341); lexsort((z, col)) as two stable radix sorts
//      (z as order-preserving bits, then col); each column chunked into
//      M-slot clusters, dummy-padded, dummies parked at the AABB minimum
//      (containers.py:343-406).
//   K6 cluster pairs: AABB gap^2 <= (rc+skin)^2 summed x, y, z exactly as
//      _box_distance_sq (containers.py:271-299) -- but binned by column and
//      z (clusters of a column are z-ordered) instead of the dense O(C^2)
//      matrix.  Lists come out in ascending cluster id, the reference order.
//   K7 force: one warp per owned cluster; its j-stream is itself, its full
//      neighbour list, then its halo links; lanes = (i slot) x (j slot).
#include <cub/cub.cuh>
#include <math.h>

#include "common.cuh"

namespace lmd {

__global__ void vcl_keys_kernel(int64_t n, const double* __restrict__ x,
                                const double* __restrict__ y, const double* __restrict__ z,
                                double lo0, double lo1, double col, long long width,
                                int32_t* __restrict__ colkey,
                                unsigned long long* __restrict__ zkey) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double fx = floor(__ddiv_rn(__dadd_rn(x[k], -lo0), col));
  const double fy = floor(__ddiv_rn(__dadd_rn(y[k], -lo1), col));
  const long long cx = (long long)fmax(fmin(fx, 1e9), -1e9) + 1;
  const long long cy = (long long)fmax(fmin(fy, 1e9), -1e9) + 1;
  colkey[k] = (int32_t)(cx + width * cy);
  // numpy orders -0.0 == +0.0 (ties by index): canonicalise, then map the
  // double onto an unsigned key with the same order
  double zz = z[k];
  if (zz == 0.0) zz = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(zz);
  b = (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
  zkey[k] = b;
}

__global__ void gather_i32_kernel(int64_t n, const int32_t* __restrict__ idx,
                                  const int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) dst[k] = src[idx[k]];
}

__global__ void iota32_kernel(int64_t n, int32_t* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) out[k] = (int32_t)k;
}

// run (column) starts over the sorted column keys
__global__ void run_flags_kernel(int64_t n, const int32_t* __restrict__ key,
                                 int32_t* __restrict__ flag) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) flag[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

// per run: start, count, clusters = ceil(count / M); run id from inclusive scan
__global__ void run_info_kernel(int64_t n, int M, const int32_t* __restrict__ key,
                                const int32_t* __restrict__ run_id,
                                int32_t* __restrict__ run_start, int32_t* __restrict__ run_nclu) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int r = run_id[k] - 1;
  if (k == 0 || key[k] != key[k - 1]) run_start[r] = (int32_t)k;
  if (k == n - 1 || key[k + 1] != key[k]) {
    // the run ends here; its start is written by the thread that owns it,
    // so store the end (exclusive) and convert after a second pass
    run_nclu[r] = (int32_t)(k + 1);
  }
}

__global__ void run_nclu_kernel(int nruns, int M, const int32_t* __restrict__ run_start,
                                int32_t* __restrict__ run_nclu) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  const int cnt = run_nclu[r] - run_start[r];
  run_nclu[r] = (cnt + M - 1) / M;
}

__global__ void slots_kernel(int64_t n, int M, const int32_t* __restrict__ run_id,
                             const int32_t* __restrict__ run_start,
                             const int32_t* __restrict__ run_coff,
                             const int32_t* __restrict__ sorted_key, int32_t* __restrict__ slot,
                             int32_t* __restrict__ cluster_key) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int r = run_id[k] - 1;
  const int rank = (int)k - run_start[r];
  const int c = run_coff[r] + rank / M;
  slot[k] = c * M + rank % M;
  if (rank % M == 0) cluster_key[c] = sorted_key[k];
}

__global__ void fill_dummy_kernel(int64_t m, double4* __restrict__ pos4) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) pos4[k] = make_double4(0.0, 0.0, 0.0, (double)LMD_DUMMY);
}

__global__ void scatter_slots_kernel(int64_t n, const int32_t* __restrict__ order,
                                     const int32_t* __restrict__ slot,
                                     const double* __restrict__ x, const double* __restrict__ y,
                                     const double* __restrict__ z, double own_value,
                                     double4* __restrict__ pos4) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int o = order[k];
  pos4[slot[k]] = make_double4(x[o], y[o], z[o], own_value);
}

// containers.py:393-406: min/max over real entries, dummies parked at the min
__global__ void aabb_kernel(int ncl, int M, double4* __restrict__ pos4, double* __restrict__ amin,
                            double* __restrict__ amax) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int t = 0; t < M; ++t) {
    const double4 p = pos4[(long long)c * M + t];
    if (p.w == (double)LMD_DUMMY) continue;
    const double v[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (v[ax] < lo[ax]) lo[ax] = v[ax];
      if (v[ax] > hi[ax]) hi[ax] = v[ax];
    }
  }
  for (int t = 0; t < M; ++t) {
    double4& p = pos4[(long long)c * M + t];
    if (p.w == (double)LMD_DUMMY) {
      p.x = lo[0];
      p.y = lo[1];
      p.z = lo[2];
    }
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    amin[3 * (long long)c + ax] = lo[ax];
    amax[3 * (long long)c + ax] = hi[ax];
  }
}

__global__ void column_table_kernel(int ncl, const int32_t* __restrict__ ckey,
                                    int32_t* __restrict__ tbeg, int32_t* __restrict__ tend,
                                    int tsize) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncl) return;
  const int k = ckey[c];
  if (k < 0 || k >= tsize) return;
  if (c == 0 || ckey[c - 1] != k) tbeg[k] = c;
  if (c == ncl - 1 || ckey[c + 1] != k) tend[k] = c + 1;
}

// _box_distance_sq (containers.py:271-273): per axis gap = max(0, max(a_min
// - b_max, b_min - a_max)); squares summed x, y, z in order
__device__ __forceinline__ double box_d2(const double* __restrict__ amin,
                                         const double* __restrict__ amax, long long a,
                                         const double* __restrict__ bmin,
                                         const double* __restrict__ bmax, long long b) {
  double s = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double u = __dadd_rn(amin[3 * a + ax], -bmax[3 * b + ax]);
    const double v = __dadd_rn(bmin[3 * b + ax], -amax[3 * a + ax]);
    const double m = u > v ? u : v;
    const double g = m > 0.0 ? m : 0.0;
    s = ax == 0 ? __dmul_rn(g, g) : __dadd_rn(s, __dmul_rn(g, g));
  }
  return s;
}

struct ColTab {
  const int32_t* beg;
  const int32_t* end;
  long long width, tsize;
};

// Visit candidate clusters (ascending id) of cluster a within the 5x5
// neighbouring columns whose AABB gap^2 <= limit.
template <typename F>
__device__ __forceinline__ void search(long long a, int32_t akey, const double* __restrict__ amin,
                                       const double* __restrict__ amax,
                                       const double* __restrict__ bmin,
                                       const double* __restrict__ bmax, const ColTab& tab,
                                       double rl, double limit, F&& visit) {
  const long long w = tab.width;
  const long long ax = akey % w, ay = akey / w;
  const double zlo = amin[3 * a + 2] - 2.0 * rl, zhi = amax[3 * a + 2] + 2.0 * rl;
  for (long long dy = -2; dy <= 2; ++dy) {
    for (long long dx = -2; dx <= 2; ++dx) {
      const long long cx = ax + dx, cy = ay + dy;
      if (cx < 0 || cx >= w || cy < 0) continue;
      const long long key = cx + w * cy;
      if (key >= tab.tsize) continue;
      int b0 = tab.beg[key], b1 = tab.end[key];
      if (b0 >= b1) continue;
      // clusters of a column are z-ordered: binary search the first whose
      // zmax >= zlo (a conservative window; the exact test follows)
      int lo = b0, hi = b1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (bmax[3 * (long long)mid + 2] < zlo) lo = mid + 1;
        else hi = mid;
      }
      for (int b = lo; b < b1; ++b) {
        if (bmin[3 * (long long)b + 2] > zhi) break;
        if (box_d2(amin, amax, a, bmin, bmax, b) <= limit) visit(b);
      }
    }
  }
}

// Count (list == nullptr) or fill the candidate clusters of every owned
// cluster a against one cluster set (owned: excluding a itself; or the halo
// clusters), in ascending id.  n3count (owned set only) = #{b > a}.
__global__ void vcl_pairs_kernel(int ncl, const int32_t* __restrict__ ckey,
                                 const double* __restrict__ amin, const double* __restrict__ amax,
                                 const double* __restrict__ bmin, const double* __restrict__ bmax,
                                 ColTab tab, int exclude_self, double rl, double limit,
                                 int32_t* __restrict__ count, int32_t* __restrict__ n3count,
                                 const long long* __restrict__ off, int32_t* __restrict__ list) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= ncl) return;
  int c = 0, c3 = 0;
  int32_t* out = list ? list + off[a] : nullptr;
  search(a, ckey[a], amin, amax, bmin, bmax, tab, rl, limit, [&](int b) {
    if (exclude_self && b == a) return;
    if (out) out[c] = b;
    ++c;
    c3 += b > a;
  });
  if (!list) {
    count[a] = c;
    if (n3count) n3count[a] = c3;
  }
}

// ------------------------------------------------------------------ force
// Warp per owned cluster, stream mapping: lane (il, g) = (lane % MP, lane / MP)
// (MP = M rounded up to a power of two <= 32) holds i slot il of the
// cluster; the G = 32 / MP lane groups take the cluster's units (self, list
// entries, halo links) round-robin, and each lane tests its i against all
// M slots of its unit branch-free into a hit mask, then evaluates LJ for the
// set bits only.  With ~10 % of cluster-pair tests inside rc, the LJ path runs
// a few times per unit instead of on nearly every fill.  Same pairs; each
// lane's summation order is fixed by the list, so results are deterministic.
// F32: the cutoff tests run in FP32 on a float4 copy of the records
// (pos4f) against rc^2 + the conversion / arithmetic error bound, so every
// pair inside the cutoff passes; the pairs that pass are then decided by the
// reference's exact FP64 r2 in the LJ loop -- same pairs, 7 FP32 instructions
// per test instead of 8 FP64 ones on the scarce FP64 pipe.
template <int MP, bool EV, bool F32>
__global__ void __launch_bounds__(128)
    vcl_stream_kernel(int ncl, int M, const double* __restrict__ pos4,
                      const float4* __restrict__ pos4f, float rc2_hi,
                      const long long* __restrict__ off, const int32_t* __restrict__ nlist,
                      const int32_t* __restrict__ list, const long long* __restrict__ hoff,
                      const int32_t* __restrict__ hnlist, const int32_t* __restrict__ hlist,
                      LJK k, double* __restrict__ fx, double* __restrict__ fy,
                      double* __restrict__ fz, double* __restrict__ ev,
                      lmd_stats* __restrict__ stats) {
  constexpr int G = 32 / MP;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  int pairs = 0, pairs_halo = 0, overlap = 0;
  double e_acc = 0.0, v_acc = 0.0;
  const int il = lane % MP, g = lane / MP;
  if (warp < ncl) {
    const int a = (int)warp;
    const long long n_owned_slots = (long long)ncl * M;
    const int nl = nlist[a];
    const int nhl = hnlist ? hnlist[a] : 0;
    const int32_t* lst = list + off[a];
    const int32_t* hlst = hlist ? hlist + hoff[a] : nullptr;
    const int units = 1 + nl + nhl;
    for (int ci = 0; ci < M; ci += MP) {
      const int islot = ci + il;
      const bool ilive = islot < M;
      const long long gi = (long long)a * M + (ilive ? islot : 0);
      const double4 pi = ld_pos4(pos4, gi);
      const bool iown = ilive && pi.w == (double)LMD_OWNED;
      const float pxf = (float)pi.x, pyf = (float)pi.y, pzf = (float)pi.z;
      double ax = 0.0, ay = 0.0, az = 0.0;
      // R = 32 / MP units per lane fill one 32-bit hit mask (unit r at bits
      // [r * MP, r * MP + M)), so the LJ loop runs once per set bit over R
      // units' worth of tests; M > 16 keeps one unit per mask, in 32-slot chunks
      constexpr int R = MP >= 32 ? 1 : 32 / MP;
      auto unit_cluster = [&](int u) {
        return u == 0 ? a : (u <= nl ? lst[u - 1] : ncl + hlst[u - 1 - nl]);
      };
      for (int u0 = 0; u0 < units; u0 += G * R) {
        const int bc0 = (u0 + g < units) ? unit_cluster(u0 + g) : a;   // unit r = 0
        for (int c0 = 0; c0 < M; c0 += 32) {
          const int cnt = min(M - c0, 32);
          unsigned mask = 0u;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int u = u0 + g + r * G;
            if (!iown || u >= units) continue;
            const int bc = r == 0 ? bc0 : unit_cluster(u);
            const long long base = (long long)bc * M + c0;
            unsigned m = 0u;
#pragma unroll 4
            for (int q = 0; q < cnt; ++q) {
              if (F32) {
                const float4 pj = __ldg(pos4f + base + q);
                const float dx = pxf - pj.x, dy = pyf - pj.y, dz = pzf - pj.z;
                const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                m |= (pj.w != (float)LMD_DUMMY && r2 < rc2_hi ? 1u : 0u) << q;
              } else {
                const double4 pj = ld_pos4(pos4, base + q);
                const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
                m |= (pj.w != (double)LMD_DUMMY && r2 < k.rc2 ? 1u : 0u) << q;
              }
            }
            if (bc == a) {   // self unit: not with itself
              const unsigned self = (unsigned)(gi - base);
              if (self < 32u) m &= ~(1u << self);
            }
            mask |= m << (r * MP);
          }
          while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1u;
            const int r = bit / MP, q = bit - r * MP;
            const long long gj =
                (long long)(r == 0 ? bc0 : unit_cluster(u0 + g + r * G)) * M + c0 + q;
            const double4 pj = ld_pos4(pos4, gj);
            const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
            const double r2 = r2_exact(dx, dy, dz);
            if (F32 && r2 >= k.rc2) continue;   // passed the FP32 band only
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
            pairs_halo += gj >= n_owned_slots;
            if (EV) {
              e_acc = fma(0.5 * s6, fma(k.eps4, s6, -k.eps4), e_acc);
              v_acc = fma(0.5 * f, r2, v_acc);
            }
          }
        }
      }
#pragma unroll
      for (int o = MP; o < 32; o <<= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, o);
        ay += __shfl_xor_sync(0xffffffffu, ay, o);
        az += __shfl_xor_sync(0xffffffffu, az, o);
      }
      if (g == 0 && ilive) {
        fx[gi] = ax;
        fy[gi] = ay;
        fz[gi] = az;
      }
    }
  }
  const long long pr = warp_sum_ll((long long)pairs);
  const long long ph = warp_sum_ll((long long)pairs_halo);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && warp < ncl) {
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

// float4 copies of the (x, y, z, ownership) records for the FP32 tests
// (packing two records per load for FADD2 / FFMA2 arithmetic was measured:
// no gain at M = 8 / 32, slower at M = 4 -- the LJ loop over the set bits,
// not the tests, bounds the kernel then)
__global__ void vcl_to_f32_kernel(long long n, const double4* __restrict__ pos4,
                                  float4* __restrict__ out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double4 p = pos4[k];
  out[k] = make_float4((float)p.x, (float)p.y, (float)p.z, (float)p.w);
}

// Interaction orders as warp mappings.  One warp per owned cluster a; the
// 32 lanes form the order's A x B template (Pattern<P>: lane -> (i_off,
// j_off), kernels.py:250-265): a fill evaluates A i-slots of the base
// cluster against B j-slots.  With B >= M the B j-lanes cover B / M whole
// units (neighbour clusters) per fill, else a unit takes ceil(M / B) fills;
// the base cluster takes ceil(M / A) i-blocks and lanes whose i-slot is >= M
// stay blank -- so, as in the paper, how well the
// order's A matches the cluster size M decides how many lanes do work.  Each
// lane first tests its pair of up to 32 fills into a hit mask (exact r2
// cutoff decision), then evaluates LJ for the set bits; the i force is
// reduced over the lanes sharing the i-slot (reduce_j<P>).
template <int P, bool EV>
__global__ void __launch_bounds__(128)
    vcl_order_kernel(int ncl, int M, int mshift, const double* __restrict__ pos4,
                     const long long* __restrict__ off, const int32_t* __restrict__ nlist,
                     const int32_t* __restrict__ list, const long long* __restrict__ hoff,
                     const int32_t* __restrict__ hnlist, const int32_t* __restrict__ hlist,
                     const double* __restrict__ amin, const double* __restrict__ amax,
                     const double* __restrict__ hmin, const double* __restrict__ hmax,
                     double skip2, LJK k, double* __restrict__ fx, double* __restrict__ fy,
                     double* __restrict__ fz, double* __restrict__ ev,
                     lmd_stats* __restrict__ stats) {
  constexpr int A = Pattern<P>::A, B = Pattern<P>::B;
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  int pairs = 0, pairs_halo = 0, overlap = 0;
  double e_acc = 0.0, v_acc = 0.0;
  const int io = Pattern<P>::ioff(lane), jo = Pattern<P>::joff(lane);
  // M a power of two (mshift >= 0): shifts; else divisions
  const bool pack = B >= M;
  const int upf = pack ? (mshift >= 0 ? B >> mshift : B / M) : 1;   // units per fill
  const int jf_n = pack ? 1 : (M + B - 1) / B;                       // fills per unit
  const int ju = pack ? (mshift >= 0 ? jo >> mshift : jo / M) : 0;
  const int js0 = pack ? (mshift >= 0 ? jo & (M - 1) : jo % M) : jo;
  if (warp < ncl) {
    const int a = (int)warp;
    const long long n_owned_slots = (long long)ncl * M;
    const int nl = nlist[a];
    const int nhl = hnlist ? hnlist[a] : 0;
    const int32_t* lst = list + off[a];
    const int32_t* hlst = hlist ? hlist + hoff[a] : nullptr;
    const int units = 1 + nl + nhl;
    const int groups = (units + upf - 1) / upf;  // unit groups (one fill row each)
    auto unit_cluster = [&](int u) {
      return u == 0 ? a : (u <= nl ? __ldg(lst + u - 1) : ncl + __ldg(hlst + u - 1 - nl));
    };
    for (int ib = 0; ib < M; ib += A) {
      const int islot = ib + io;
      const bool ilive = islot < M;
      const long long gi = (long long)a * M + (ilive ? islot : 0);
      const double4 pi = ld_pos4(pos4, gi);
      const bool iown = ilive && pi.w == (double)LMD_OWNED;
      double ax = 0.0, ay = 0.0, az = 0.0;
      // fills in (unit group, j-fill) order; 32 fills per hit mask
      for (int g0 = 0; g0 < groups; g0 += 32 / jf_n > 0 ? (32 / jf_n) : 1) {
        const int gstep = 32 / jf_n > 0 ? 32 / jf_n : 1;
        const int gn = min(gstep, groups - g0);
        unsigned mask = 0u;
        for (int gq = 0; gq < gn; ++gq) {
          const int u = (g0 + gq) * upf + ju;
          if (!iown || u >= units) continue;
          const int bc = unit_cluster(u);
          // with several fills per unit: skip the unit when this lane's i is
          // farther than rc + skin / 2 from the cluster's box (rebuild-time
          // AABB; members moved < skin / 2 since) -- no hit possible
          if (jf_n >= 4) {
            const double* lo = bc < ncl ? amin + 3LL * bc : hmin + 3LL * (bc - ncl);
            const double* hi = bc < ncl ? amax + 3LL * bc : hmax + 3LL * (bc - ncl);
            const double gx = fmax(0.0, fmax(__ldg(lo) - pi.x, pi.x - __ldg(hi)));
            const double gy = fmax(0.0, fmax(__ldg(lo + 1) - pi.y, pi.y - __ldg(hi + 1)));
            const double gz = fmax(0.0, fmax(__ldg(lo + 2) - pi.z, pi.z - __ldg(hi + 2)));
            if (gx * gx + gy * gy + gz * gz > skip2) continue;
          }
          for (int jf = 0; jf < jf_n; ++jf) {
            const int jslot = jf * B + js0;
            if (jslot >= M) break;
            const long long gj = (long long)bc * M + jslot;
            const double4 pj = ld_pos4(pos4, gj);
            const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
            const bool hit = pj.w != (double)LMD_DUMMY && r2 < k.rc2 && gj != gi;
            mask |= (hit ? 1u : 0u) << (gq * jf_n + jf);
          }
        }
        while (mask) {
          const int q = __ffs(mask) - 1;
          mask &= mask - 1u;
          const int gq = q / jf_n, jf = q - gq * jf_n;
          const int u = (g0 + gq) * upf + ju, jslot = jf * B + js0;
          const long long gj = (long long)unit_cluster(u) * M + jslot;
          const double4 pj = ld_pos4(pos4, gj);
          const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
          const double r2 = r2_exact(dx, dy, dz);
          if (r2 == 0.0) {
            overlap = 1;
            continue;
          }
          double s6;
          const double fs = lj_scalar(r2, k, s6);
          ax = fma(fs, dx, ax);
          ay = fma(fs, dy, ay);
          az = fma(fs, dz, az);
          ++pairs;
          pairs_halo += gj >= n_owned_slots;
          if (EV) {
            e_acc = fma(0.5 * s6, fma(k.eps4, s6, -k.eps4), e_acc);
            v_acc = fma(0.5 * fs, r2, v_acc);
          }
        }
      }
      ax = reduce_j<P>(ax);
      ay = reduce_j<P>(ay);
      az = reduce_j<P>(az);
      if (jo == 0 && ilive) {
        fx[gi] = ax;
        fy[gi] = ay;
        fz[gi] = az;
      }
    }
  }
  const long long pr = warp_sum_ll((long long)pairs);
  const long long ph = warp_sum_ll((long long)pairs_halo);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && warp < ncl) {
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

// KernelStats of the vcl schedule (traversals.py:244-266 + executor.py:38-69):
// per owned cluster a self unit, one unit per list entry (N3: z > k only)
// and one per halo link; invocations ceil(M/a)*ceil(M/b) each; useful from
// owned / non-dummy counts of the cluster views.
__global__ void vcl_stats_kernel(int ncl, int M, int newton3, int a, int b,
                                 const double* __restrict__ pos4, const long long* __restrict__ off,
                                 const int32_t* __restrict__ nlist,
                                 const int32_t* __restrict__ n3count,
                                 const int32_t* __restrict__ list,
                                 const long long* __restrict__ hoff,
                                 const int32_t* __restrict__ hcount,
                                 const int32_t* __restrict__ hlist,
                                 const int32_t* __restrict__ nd_of,
                                 lmd_stats* __restrict__ stats) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  long long inv = 0, useful = 0;
  if (c < ncl) {
    const long long per_unit = (long long)((M + a - 1) / a) * ((M + b - 1) / b);
    int owned = 0, nd = 0;
    long long self_n3 = 0;
    // owned / non-dummy counts; self slots (particles.py:125-143)
    for (int t = 0; t < M; ++t) {
      const double w = pos4[4 * ((long long)c * M + t) + 3];
      nd += w != (double)LMD_DUMMY;
      owned += w == (double)LMD_OWNED;
    }
    int seen = 0;
    for (int t = 0; t < M; ++t) {
      const double w = pos4[4 * ((long long)c * M + t) + 3];
      seen += w != (double)LMD_DUMMY;
      if (w == (double)LMD_OWNED) self_n3 += nd - seen;
    }
    const int nh = hcount ? hcount[c] : 0;
    const int units_owned = newton3 ? n3count[c] : nlist[c];
    inv = per_unit * (1 + units_owned + nh);
    useful = newton3 ? self_n3 : (long long)owned * (nd - 1 > 0 ? nd - 1 : 0);
    const int32_t* lst = list + off[c];
    for (int u = 0; u < nlist[c] + nh; ++u) {
      const bool halo = u >= nlist[c];
      const int z = halo ? ncl + hlist[hoff[c] + (u - nlist[c])] : lst[u];
      if (!halo && newton3 && z < c) continue;
      useful += (long long)owned * nd_of[z];
    }
  }
  inv = warp_sum_ll(inv);
  useful = warp_sum_ll(useful);
  if ((threadIdx.x & 31) == 0 && (inv || useful)) {
    atomicAdd((unsigned long long*)&stats->kernel_invocations, (unsigned long long)inv);
    atomicAdd((unsigned long long*)&stats->useful_interactions, (unsigned long long)useful);
  }
}

// non-dummy slots per cluster (owned and halo clusters), read once instead of
// once per list entry by vcl_stats_kernel
__global__ void cluster_nd_kernel(int64_t nclt, int M, const double* __restrict__ pos4,
                                  int32_t* __restrict__ nd) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nclt) return;
  int k = 0;
  for (int t = 0; t < M; ++t) k += pos4[4 * (c * M + t) + 3] != (double)LMD_DUMMY;
  nd[c] = k;
}

__global__ void vcl_lane_slots_kernel(lmd_stats* stats, int V) {
  stats->lane_slots = stats->kernel_invocations * (long long)V;
}

__global__ void vcl_collect_kernel(int64_t n, const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ slot, const double* __restrict__ fx,
                                   const double* __restrict__ fy, const double* __restrict__ fz,
                                   double* __restrict__ ox, double* __restrict__ oy,
                                   double* __restrict__ oz) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int o = order[k], s = slot[k];
  ox[o] = fx[s];
  oy[o] = fy[s];
  oz[o] = fz[s];
}

static inline unsigned g1(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace lmd

using namespace lmd;

extern "C" {

size_t lmd_vcl_temp_bytes(int64_t n) {
  size_t a = 0, b = 0, c = 0;
  const int m = (int)(n > 0 ? n : 1);
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, m);
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, m);
  cub::DeviceScan::InclusiveSum(nullptr, c, (const int32_t*)nullptr, (int32_t*)nullptr, m);
  size_t d = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, d, (const int32_t*)nullptr, (int32_t*)nullptr, m);
  size_t e = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, e, (const long long*)nullptr, (long long*)nullptr, m);
  size_t r = a > b ? a : b;
  r = r > c ? r : c;
  r = r > d ? r : d;
  return r > e ? r : e;
}

/* K5 step 1: lexsort((z, col)) order of n particles.  Scratch: colkey, ckey2,
 * tmp_idx, order (n int32 each), zkey, zkey2 (n uint64 each). */
int lmd_vcl_order(int64_t n, const double* x, const double* y, const double* z, double lo0,
                  double lo1, double col, int64_t width, int32_t* colkey, int32_t* ckey2,
                  uint64_t* zkey, uint64_t* zkey2, int32_t* tmp_idx, int32_t* order,
                  int32_t* sorted_colkey, void* temp, size_t temp_bytes, void* stream) {
  if (n <= 0) return LMD_OK;
  if (n > 0x7fffffffLL) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  vcl_keys_kernel<<<g1(n, 256), 256, 0, s>>>(n, x, y, z, lo0, lo1, col, width, colkey,
                                              (unsigned long long*)zkey);
  LMD_CHECK_LAUNCH();
  iota32_kernel<<<g1(n, 256), 256, 0, s>>>(n, tmp_idx);
  LMD_CHECK_LAUNCH();
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, bytes, (const unsigned long long*)zkey,
                                                  (unsigned long long*)zkey2, tmp_idx, order,
                                                  (int)n, 0, 64, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  // col keys in z order, then a stable sort by col (LSD: the z order survives ties)
  gather_i32_kernel<<<g1(n, 256), 256, 0, s>>>(n, order, colkey, ckey2);
  LMD_CHECK_LAUNCH();
  bytes = temp_bytes;
  e = cub::DeviceRadixSort::SortPairs(temp, bytes, ckey2, sorted_colkey, order, tmp_idx, (int)n, 0,
                                      32, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (cudaMemcpyAsync(order, tmp_idx, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  return LMD_OK;
}

/* K5 step 2: chunk the sorted columns into M-slot clusters
 * (containers.py:343-367).  run_id/run_start/run_nclu/run_coff: n int32
 * scratch.  Writes slot[k] (padded slot of the k-th sorted particle) and
 * cluster_key[c]; *ncl_out (host) = number of clusters (synchronises). */
int lmd_vcl_chunk(int64_t n, int M, const int32_t* sorted_colkey, int32_t* flag, int32_t* run_id,
                  int32_t* run_start, int32_t* run_nclu, int32_t* run_coff, int32_t* slot,
                  int32_t* cluster_key, int64_t* ncl_out, void* temp, size_t temp_bytes,
                  void* stream) {
  *ncl_out = 0;
  if (n <= 0) return LMD_OK;
  if (M < 2) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  run_flags_kernel<<<g1(n, 256), 256, 0, s>>>(n, sorted_colkey, flag);
  LMD_CHECK_LAUNCH();
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceScan::InclusiveSum(temp, bytes, flag, run_id, (int)n, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  int32_t nruns = 0;
  if (cudaMemcpyAsync(&nruns, run_id + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  run_info_kernel<<<g1(n, 256), 256, 0, s>>>(n, M, sorted_colkey, run_id, run_start, run_nclu);
  LMD_CHECK_LAUNCH();
  run_nclu_kernel<<<g1(nruns, 256), 256, 0, s>>>(nruns, M, run_start, run_nclu);
  LMD_CHECK_LAUNCH();
  bytes = temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(temp, bytes, run_nclu, run_coff, nruns, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  int32_t last[2] = {0, 0};
  if (cudaMemcpyAsync(&last[0], run_coff + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(&last[1], run_nclu + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  *ncl_out = (int64_t)last[0] + last[1];
  slots_kernel<<<g1(n, 256), 256, 0, s>>>(n, M, run_id, run_start, run_coff, sorted_colkey, slot,
                                           cluster_key);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

/* K5 step 3: padded backing (containers.py:369-376) -- all slots dummy, then
 * pos4[slot[k]] = particle order[k] -- and the AABBs with dummies parked at
 * the minimum (containers.py:393-406). */
int lmd_vcl_backing(int64_t n, int64_t ncl, int M, const int32_t* order, const int32_t* slot,
                    const double* x, const double* y, const double* z, double own_value,
                    double* pos4, double* amin, double* amax, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = ncl * M;
  if (m > 0) {
    fill_dummy_kernel<<<g1(m, 256), 256, 0, s>>>(m, reinterpret_cast<double4*>(pos4));
    LMD_CHECK_LAUNCH();
  }
  if (n > 0) {
    scatter_slots_kernel<<<g1(n, 256), 256, 0, s>>>(n, order, slot, x, y, z, own_value,
                                                     reinterpret_cast<double4*>(pos4));
    LMD_CHECK_LAUNCH();
  }
  if (ncl > 0) {
    aabb_kernel<<<g1(ncl, 128), 128, 0, s>>>((int)ncl, M, reinterpret_cast<double4*>(pos4), amin,
                                             amax);
    LMD_CHECK_LAUNCH();
  }
  return LMD_OK;
}

/* Column table: tbeg/tend[key] = cluster range of a column (tsize entries,
 * caller-zeroed). */
int lmd_vcl_column_table(int64_t ncl, const int32_t* cluster_key, int32_t* tbeg, int32_t* tend,
                         int64_t tsize, void* stream) {
  if (ncl <= 0) return LMD_OK;
  column_table_kernel<<<g1(ncl, 256), 256, 0, (cudaStream_t)stream>>>(
      (int)ncl, cluster_key, tbeg, tend, (int)tsize);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

/* K6: candidate clusters of every owned cluster against one cluster set
 * (amin/amax: owned AABBs; bmin/bmax + tbeg/tend: the target set and its
 * column table; exclude_self for the owned set).  Pass list == NULL to count
 * (count, and n3count = #{b > a} if non-NULL), then the exclusive-scan
 * offsets of count and the list buffer to fill (ascending id). */
int lmd_vcl_pairs(int64_t ncl, const int32_t* cluster_key, const double* amin, const double* amax,
                  const double* bmin, const double* bmax, const int32_t* tbeg,
                  const int32_t* tend, int64_t width, int64_t tsize, int exclude_self, double rl,
                  double limit, int32_t* count, int32_t* n3count, const int64_t* off,
                  int32_t* list, void* stream) {
  if (ncl <= 0) return LMD_OK;
  ColTab t = {tbeg, tend, width, tsize};
  vcl_pairs_kernel<<<g1(ncl, 128), 128, 0, (cudaStream_t)stream>>>(
      (int)ncl, cluster_key, amin, amax, bmin, bmax, t, exclude_self, rl, limit, count, n3count,
      (const long long*)off, list);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int64_t lmd_vcl_ev_slots(int64_t ncl) { return cdiv(ncl, 4) * 4; }

/* K7: force over the cluster lists (Newton3 off: every owned cluster against
 * itself, its full list and its halo links).  pos4 = [owned padded | halo
 * padded]; forces written per owned slot. */
int lmd_force_vcl_order(int64_t ncl, int M, int pattern, int flags, const lmd_lj* lj,
                        const double* pos4, const int64_t* off, const int32_t* nlist,
                        const int32_t* list, const int64_t* hoff, const int32_t* hnlist,
                        const int32_t* hlist, const double* amin, const double* amax,
                        const double* hmin, const double* hmax, double* fx, double* fy,
                        double* fz, double* ev_scratch, lmd_stats* stats, void* stream) {
  if (ncl <= 0) return LMD_OK;
  if (M < 2 || M > 32 || pattern < 0 || pattern > 3 || !amin || !amax) return LMD_ERR_CONFIG;
  const LJK k = make_ljk(lj);
  int mshift = -1;
  for (int b = 0; b < 6; ++b)
    if ((1 << b) == M) mshift = b;
  // skip a unit when the i particle is farther than rc + skin/2 from its box
  const double skip_r = lj->cutoff + 0.5 * lj->skin;
  const double skip2 = skip_r * skip_r * (1.0 + 1e-12);
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  const unsigned blocks = (unsigned)cdiv(ncl, 4);
#define LMD_VCLO(PV)                                                                          \
  do {                                                                                        \
    if (ev)                                                                                   \
      vcl_order_kernel<PV, true><<<blocks, 128, 0, s>>>(                                      \
          (int)ncl, M, mshift, pos4, (const long long*)off, nlist, list,                      \
          (const long long*)hoff, hnlist, hlist, amin, amax, hmin, hmax, skip2, k, fx, fy, fz, \
          ev_scratch, stats);                                                                 \
    else                                                                                      \
      vcl_order_kernel<PV, false><<<blocks, 128, 0, s>>>(                                     \
          (int)ncl, M, mshift, pos4, (const long long*)off, nlist, list,                      \
          (const long long*)hoff, hnlist, hlist, amin, amax, hmin, hmax, skip2, k, fx, fy, fz, \
          ev_scratch, stats);                                                                 \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_VCLO(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_VCLO(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_VCLO(LMD_TWO_BY_HALF); break;
    default: LMD_VCLO(LMD_HALF_BY_TWO); break;
  }
#undef LMD_VCLO
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, lmd_vcl_ev_slots(ncl), stats, s);
  return LMD_OK;
}

int lmd_force_vcl(int64_t ncl, int M, int flags, const lmd_lj* lj, const double* pos4,
                  const int64_t* off, const int32_t* nlist, const int32_t* list,
                  const int64_t* hoff, const int32_t* hnlist, const int32_t* hlist, double* fx,
                  double* fy, double* fz, double* ev_scratch, lmd_stats* stats,
                  int64_t n_records, float* pos4f, double max_abs, void* stream) {
  if (ncl <= 0) return LMD_OK;
  if (M < 2) return LMD_ERR_CONFIG;
  const LJK k = make_ljk(lj);
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  const unsigned blocks = (unsigned)cdiv(ncl, 4);
  const int mp = M >= 32 ? 32 : M > 8 ? 16 : M > 4 ? 8 : M > 2 ? 4 : 2;
  // FP32 tests (pos4f != NULL): |FP32 r2 - exact r2| <= err for coordinates
  // up to max_abs (conversion 2^-24 |x| per coordinate, twice per difference,
  // times 2 |d| summed over the axes; a few ulp of r2 for the arithmetic),
  // doubled for safety
  float rc2_hi = 0.f;
  const bool f32 = pos4f != nullptr && n_records > 0 && max_abs > 0.0 && isfinite(max_abs);
  if (f32) {
    const double eps = 5.9604644775390625e-8, rc = lj->cutoff;
    const double err = 2.0 * (4.0 * 1.7320508075688772 * (rc + 1.0) * eps * max_abs +
                              8.0 * eps * (k.rc2 + 1.0));
    rc2_hi = (float)(k.rc2 + err);
    rc2_hi = nextafterf(rc2_hi, INFINITY);
    vcl_to_f32_kernel<<<(unsigned)cdiv(n_records, 256), 256, 0, s>>>(
        n_records, (const double4*)pos4, (float4*)pos4f);
    LMD_CHECK_LAUNCH();
  }
#define LMD_VCLK2(MPV, EVB, FB)                                                             \
  vcl_stream_kernel<MPV, EVB, FB><<<blocks, 128, 0, s>>>(                                   \
      (int)ncl, M, pos4, (const float4*)pos4f, rc2_hi, (const long long*)off, nlist, list,  \
      (const long long*)hoff, hnlist, hlist, k, fx, fy, fz, ev_scratch, stats)
#define LMD_VCLK(MPV)                  \
  do {                                 \
    if (ev) {                          \
      if (f32) LMD_VCLK2(MPV, true, true);   \
      else LMD_VCLK2(MPV, true, false);      \
    } else {                           \
      if (f32) LMD_VCLK2(MPV, false, true);  \
      else LMD_VCLK2(MPV, false, false);     \
    }                                  \
  } while (0)
  switch (mp) {
    case 2: LMD_VCLK(2); break;
    case 4: LMD_VCLK(4); break;
    case 8: LMD_VCLK(8); break;
    case 16: LMD_VCLK(16); break;
    default: LMD_VCLK(32); break;
  }
#undef LMD_VCLK
#undef LMD_VCLK2
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, lmd_vcl_ev_slots(ncl), stats, s);
  return LMD_OK;
}

int lmd_vcl_stats(int64_t ncl, int M, int newton3, int a, int b, int vector_width,
                  const double* pos4, const int64_t* off, const int32_t* nlist,
                  const int32_t* n3count, const int32_t* list, const int64_t* hoff,
                  const int32_t* hcount, const int32_t* hlist, int64_t ncl_total,
                  int32_t* nd_scratch, lmd_stats* stats, void* stream) {
  if (vector_width < 4 || (vector_width & (vector_width - 1)) != 0) return LMD_ERR_CONFIG;
  if (a < 1 || b < 1 || a * b != vector_width) return LMD_ERR_CONFIG;
  if (ncl_total < ncl) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  if (ncl > 0) {
    cluster_nd_kernel<<<g1(ncl_total, 256), 256, 0, s>>>(ncl_total, M, pos4, nd_scratch);
    LMD_CHECK_LAUNCH();
    vcl_stats_kernel<<<g1(ncl, 128), 128, 0, s>>>(
        (int)ncl, M, newton3, a, b, pos4, (const long long*)off, nlist, n3count, list,
        (const long long*)hoff, hcount, hlist, nd_scratch, stats);
    LMD_CHECK_LAUNCH();
  }
  vcl_lane_slots_kernel<<<1, 1, 0, s>>>(stats, vector_width);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

/* collect_forces (containers.py:475-479): out[order[k]] = f[slot[k]]. */
int lmd_vcl_collect(int64_t n, const int32_t* order, const int32_t* slot, const double* fx,
                    const double* fy, const double* fz, double* ox, double* oy, double* oz,
                    void* stream) {
  if (n <= 0) return LMD_OK;
  vcl_collect_kernel<<<g1(n, 256), 256, 0, (cudaStream_t)stream>>>(n, order, slot, fx, fy, fz, ox,
                                                                    oy, oz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
