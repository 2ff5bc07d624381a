// K3c/K4c: Verlet lists over i-clusters -- CI particles per lane share one list.
//
// The per-particle VL kernel (vl.cu) is bound by the L1 data path: every
// list entry is a 32-byte gather that serves exactly one pair test.  Here
// the owned particles of each cell (cell-sorted backing, so consecutive) are
// cut into clusters of up to CI consecutive particles; a cluster's list is
// the UNION of its members' lists (candidate j listed iff some member has
// r2 < (rc+skin)^2, exact r2), and the lane that owns the cluster tests
// every gathered j against all CI members.  Per-particle list lengths
// (count[i], the member's own hits) are written too, so the lane statistics
// are the same closed forms as for plain lists.  Full lists only (Newton3
// off): the pair set, forces and pair counts are those of vl.cu.
//
// Layout: clusters play the role of i in vl.cu -- tiles of A clusters,
// entry k of tile cluster il at fill step k / B on lane lane_of(il, k % B),
// lane-chunked by kChunk steps, fixed per-tile capacity cap_steps.
#include "vl_common.cuh"

namespace lmd {

template <int CI>
__global__ void vl_ci_build_kernel(GridK g, int ncl, int ntiles, int A, int B, int pattern,
                                   double rl2, int32_t sentinel, const double* __restrict__ pos4,
                                   const int32_t* __restrict__ cl_first,
                                   const int32_t* __restrict__ cl_len,
                                   const int32_t* __restrict__ os, const int32_t* __restrict__ oc,
                                   const int32_t* __restrict__ hs, const int32_t* __restrict__ hc,
                                   int cap_steps, int32_t* __restrict__ count,
                                   long long* __restrict__ toff, int32_t* __restrict__ kmax,
                                   int32_t* __restrict__ max_count, int32_t* __restrict__ nbr) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = c / A, il = c - t * A;
  const long long stride = (long long)cap_steps * 32;
  int32_t* out = nbr + (long long)t * stride;
  const int cap = cap_steps * B;
  int k = 0;
  if (c < ncl) {
    const int f = cl_first[c], len = cl_len[c];
    double4 pm[CI];
    int cnt[CI];
#pragma unroll
    for (int m = 0; m < CI; ++m) {
      pm[m] = ld_pos4(pos4, f + (m < len ? m : 0));
      cnt[m] = 0;
    }
    const long long lin = cell_of_owned(pm[0], g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2, g.d0,
                                        g.d1, g.d2, g.t0, g.t1);
    for (int view = 0; view < 2; ++view) {
      const int32_t* vs = view ? hs : os;
      const int32_t* vc = view ? hc : oc;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const long long nl = lin + dx + g.t0 * (dy + g.t1 * dz);
            const int cc = vc[nl];
            if (cc == 0) continue;
            const int s0 = vs[nl];
            for (int j = s0; j < s0 + cc; ++j) {
              const double4 pj = ld_pos4(pos4, j);
              if (pj.w == (double)LMD_DUMMY) continue;
              bool any = false;
#pragma unroll
              for (int m = 0; m < CI; ++m) {
                const bool hit = m < len && j != f + m &&
                                 r2_exact(pm[m].x - pj.x, pm[m].y - pj.y, pm[m].z - pj.z) < rl2;
                cnt[m] += hit;
                any |= hit;
              }
              if (any) {
                if (k < cap) {
                  const int st = k / B, l = lane_of(pattern, il, k % B);
                  out[(long long)(st / kChunk) * (32 * kChunk) + l * kChunk + st % kChunk] = j;
                }
                ++k;
              }
            }
          }
    }
#pragma unroll
    for (int m = 0; m < CI; ++m)
      if (m < len) count[f + m] = cnt[m];
  }
  int m = k;
  for (int off = 1; off < A; off <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  int steps = (m + B - 1) / B;
  steps = (steps + kChunk - 1) / kChunk * kChunk;
  if (steps > cap_steps) steps = cap_steps;
  if (t < ntiles) {
    for (int q = min(k, cap); q < steps * B; ++q) {
      const int st = q / B, l = lane_of(pattern, il, q % B);
      out[(long long)(st / kChunk) * (32 * kChunk) + l * kChunk + st % kChunk] = sentinel;
    }
    if (il == 0) {
      kmax[t] = steps * B;
      toff[t] = (long long)t * stride;
    }
  }
  int w = m;
  for (int off = 16; off > 0; off >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, off));
  if ((threadIdx.x & 31) == 0 && w > 0) atomicMax(max_count, w);
}

// One pair (member i at pi, candidate j at pj), Newton3 off.
template <bool EV>
__device__ __forceinline__ void ci_pair(const double3& pi, const double4& pj, bool live,
                                        const LJK& k, double& ax, double& ay,
                                        double& az, Acc& a) {
  const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
  double r2;
  if (!live || !within_cutoff(dx, dy, dz, k, r2)) return;
  if (r2 == 0.0) {
    a.overlap = 1;
    return;
  }
  double s6;
  const double f = lj_scalar(r2, k, s6);
  ax = fma(f, dx, ax);
  ay = fma(f, dy, ay);
  az = fma(f, dz, az);
  ++a.pairs;
  if (EV) {
    a.e = fma(0.5 * s6, fma(k.eps4, s6, -k.eps4), a.e);
    a.v = fma(0.5 * f, r2, a.v);
  }
}

template <int CI>
struct CiBounds {
  static constexpr int kMinBlocks = CI == 2 ? 5 : 4;
};

template <int P, bool EV, int CI>
__global__ void __launch_bounds__(32 * kVLWarps, CiBounds<CI>::kMinBlocks)
    vl_ci_force_kernel(int n_owned, int ncl, int ntiles, const double* __restrict__ pos4,
                       const int32_t* __restrict__ cl_first, const int32_t* __restrict__ cl_len,
                       const long long* __restrict__ toff, const int32_t* __restrict__ kmax,
                       const int32_t* __restrict__ nbr, LJK k, double* __restrict__ fx,
                       double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                       lmd_stats* __restrict__ stats) {
  using Pat = Pattern<P>;
  constexpr int U = 2;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * kVLWarps + (threadIdx.x >> 5);
  Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0};
  if (t < ntiles) {
    const int io = Pat::ioff(lane), jo = Pat::joff(lane);
    const int c = t * Pat::A + io;
    const bool cact = c < ncl;
    const int f = cact ? cl_first[c] : 0;
    const int len = cact ? cl_len[c] : 0;
    double3 pi[CI];
    double ax[CI], ay[CI], az[CI];
#pragma unroll
    for (int m = 0; m < CI; ++m) {
      const double4 p = ld_pos4(pos4, f + (m < len ? m : 0));
      pi[m] = make_double3(p.x, p.y, p.z);
      ax[m] = ay[m] = az[m] = 0.0;
    }
    const int4* chunks = reinterpret_cast<const int4*>(nbr + toff[t]) + lane;
    const int nchunks = kmax[t] / Pat::B / kChunk;
    int4 nxt = nchunks > 0 ? __ldg(chunks) : make_int4(0, 0, 0, 0);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int4 cur = nxt;
      if (ch + 1 < nchunks) nxt = __ldg(chunks + (long long)(ch + 1) * 32);
      const int j[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
      for (int g0 = 0; g0 < 4; g0 += U) {
        double4 pj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pj[u] = ld_pos4(pos4, j[g0 + u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int jj = j[g0 + u];
#pragma unroll
          for (int m = 0; m < CI; ++m)
            ci_pair<EV>(pi[m], pj[u], m < len && jj != f + m, k, ax[m], ay[m], az[m], a);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < CI; ++m) {
      const double rx = reduce_j<P>(ax[m]), ry = reduce_j<P>(ay[m]), rz = reduce_j<P>(az[m]);
      if (m < len && jo == 0) {
        fx[f + m] = rx;
        fy[f + m] = ry;
        fz[f + m] = rz;
      }
    }
  }
  flush_acc(a, lane, t < ntiles, EV, (long long)blockIdx.x * kVLWarps + (threadIdx.x >> 5), ev,
            stats);
}

template <int P, bool EV>
static void launch_ci(int ci, int64_t n_owned, int64_t ncl, int64_t ntiles, const double* pos4,
                      const int32_t* cl_first, const int32_t* cl_len, const int64_t* tile_off,
                      const int32_t* kmax, const int32_t* nbr, const LJK& k, double* fx,
                      double* fy, double* fz, double* ev, lmd_stats* stats, cudaStream_t s) {
  const unsigned blocks = (unsigned)cdiv(ntiles, kVLWarps);
#define LMD_CI(C)                                                                                \
  vl_ci_force_kernel<P, EV, C><<<blocks, 32 * kVLWarps, 0, s>>>(                                 \
      (int)n_owned, (int)ncl, (int)ntiles, pos4, cl_first, cl_len, (const long long*)tile_off, \
      kmax, nbr, k, fx, fy, fz, ev, stats)
  if (ci == 2) LMD_CI(2);
  else LMD_CI(4);
#undef LMD_CI
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int lmd_vl_ci_build(const lmd_grid* g, double rl2, int pattern, int ci, int64_t n_clusters,
                    const int32_t* cl_first, const int32_t* cl_len, int32_t sentinel,
                    const double* pos4, const int32_t* o_start, const int32_t* o_count,
                    const int32_t* h_start, const int32_t* h_count, int32_t cap_steps,
                    int32_t* count, int64_t* tile_off, int32_t* kmax, int32_t* max_count,
                    int32_t* nbr, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(max_count, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (ci != 2 && ci != 4) return LMD_ERR_CONFIG;
  if (n_clusters <= 0) return LMD_OK;
  if (n_clusters > 0x7fffffffLL || cap_steps <= 0 || cap_steps % kChunk) return LMD_ERR_CONFIG;
  const int A = pattern_A(pattern), B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_clusters, A);
  const unsigned blocks = (unsigned)cdiv(ntiles * A, 128);
#define LMD_CIB(C)                                                                              \
  vl_ci_build_kernel<C><<<blocks, 128, 0, s>>>(                                                 \
      make_gridk(g), (int)n_clusters, (int)ntiles, A, B, pattern, rl2, sentinel, pos4, cl_first, \
      cl_len, o_start, o_count, h_start, h_count, cap_steps, count, (long long*)tile_off, kmax,  \
      max_count, nbr)
  if (ci == 2) LMD_CIB(2);
  else LMD_CIB(4);
#undef LMD_CIB
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int64_t lmd_vl_ci_ev_slots(int64_t n_clusters, int pattern) {
  return cdiv(cdiv(n_clusters, pattern_A(pattern)), kVLWarps) * kVLWarps;
}

int lmd_force_vl_ci(int pattern, int ci, int flags, const lmd_lj* lj, int64_t n_owned,
                    int64_t n_clusters, const int32_t* cl_first, const int32_t* cl_len,
                    const double* pos4, const int64_t* tile_off, const int32_t* kmax,
                    const int32_t* nbr, double* fx, double* fy, double* fz, double* ev_scratch,
                    lmd_stats* stats, void* stream) {
  if (ci != 2 && ci != 4) return LMD_ERR_CONFIG;
  if (n_clusters <= 0) return LMD_OK;
  const LJK k = make_ljk(lj);
  const int64_t ntiles = cdiv(n_clusters, pattern_A(pattern));
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
#define LMD_CIP(P)                                                                            \
  do {                                                                                        \
    if (ev)                                                                                   \
      launch_ci<P, true>(ci, n_owned, n_clusters, ntiles, pos4, cl_first, cl_len, tile_off,   \
                         kmax, nbr, k, fx, fy, fz, ev_scratch, stats, s);                     \
    else                                                                                      \
      launch_ci<P, false>(ci, n_owned, n_clusters, ntiles, pos4, cl_first, cl_len, tile_off,  \
                          kmax, nbr, k, fx, fy, fz, ev_scratch, stats, s);                    \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_CIP(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_CIP(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_CIP(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_CIP(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_CIP
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, cdiv(ntiles, kVLWarps) * kVLWarps, stats, s);
  return LMD_OK;
}

}  // extern "C"
