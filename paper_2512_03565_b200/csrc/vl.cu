// K3/K4: Verlet lists with a skin -- build and force (sm_100a).
//
// Extension: the reference excludes plain Verlet lists; the
// north star adds them.  Semantics (mirrored by oracle/lj_oracle.c:vl_build):
// candidates are the owned particles and the images of the 27 cells of the
// rc+skin grid (no buffer_at shadowing), listed iff r2 < (rc+skin)^2 with the
// reference's exact r2.  Half lists (Newton3): owned j > i only, images always.
//
// List layout = the interaction order: owned particles (cell-sorted) form
// i-tiles of A consecutive particles (A = distinct i per warp fill).  Entry k
// of tile particle il is consumed at fill step s = k / B by the lane l with
// (i_off(l), j_off(l)) = (il, k % B).  Each lane's entries are stored in
// chunks of kChunk consecutive steps -- entry (s, l) at
// tile_off[t] + (s / kChunk) * 32 * kChunk + l * kChunk + s % kChunk -- so a
// lane fetches kChunk indices with one 128-bit load and a warp reads 512
// contiguous bytes per chunk.  Tiles are padded to a whole number of chunks
// with a sentinel particle far away.  Lists are ascending in j.
#include <cub/cub.cuh>

#include "vl_common.cuh"

namespace lmd {

template <int P>
struct Tile {
  static constexpr int A = Pattern<P>::A, B = Pattern<P>::B;
};

// visits every candidate j (index into the combined backing) of owned i
template <typename F>
__device__ __forceinline__ void for_candidates(int i, const double4& pi, int newton3, long long t0,
                                               long long t1, long long lin,
                                               const int32_t* __restrict__ os,
                                               const int32_t* __restrict__ oc,
                                               const int32_t* __restrict__ hs,
                                               const int32_t* __restrict__ hc,
                                               const double* __restrict__ pos4, double rl2,
                                               F&& visit) {
  for (int view = 0; view < 2; ++view) {
    const int32_t* vs = view ? hs : os;
    const int32_t* vc = view ? hc : oc;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const long long nl = lin + dx + t0 * (dy + t1 * dz);
          const int s = vs[nl], c = vc[nl];
          for (int j = s; j < s + c; ++j) {
            if (!view && (j == i || (newton3 && j < i))) continue;
            const double4 pj = ld_pos4(pos4, j);
            if (pj.w == (double)LMD_DUMMY) continue;
            const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
            if (r2 < rl2) visit(j);
          }
        }
  }
}

__global__ void vl_count_kernel(GridK g, int n, int newton3, double rl2,
                                const double* __restrict__ pos4, const int32_t* __restrict__ os,
                                const int32_t* __restrict__ oc, const int32_t* __restrict__ hs,
                                const int32_t* __restrict__ hc, int32_t* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = ld_pos4(pos4, i);
  int c = 0;
  if (pi.w == (double)LMD_OWNED) {
    const long long lin = cell_of_owned(pi, g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2, g.d0, g.d1,
                                        g.d2, g.t0, g.t1);
    for_candidates(i, pi, newton3, g.t0, g.t1, lin, os, oc, hs, hc, pos4, rl2,
                   [&](int) { ++c; });
  }
  count[i] = c;
}

__global__ void vl_tile_kernel(int n, int A, int B, const int32_t* __restrict__ count,
                               long long* __restrict__ tile_len, int32_t* __restrict__ kmax) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int ntiles = (n + A - 1) / A;
  if (t >= ntiles) return;
  int m = 0;
  for (int k = t * A; k < t * A + A && k < n; ++k) m = max(m, count[k]);
  int steps = (m + B - 1) / B;
  steps = (steps + kChunk - 1) / kChunk * kChunk;
  kmax[t] = steps * B;
  tile_len[t] = (long long)steps * 32;
}

__global__ void vl_fill_kernel(GridK g, int n, int A, int B, int pattern, int newton3, double rl2,
                               const double* __restrict__ pos4, const int32_t* __restrict__ os,
                               const int32_t* __restrict__ oc, const int32_t* __restrict__ hs,
                               const int32_t* __restrict__ hc, const long long* __restrict__ toff,
                               int32_t* __restrict__ nbr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = i / A, il = i - t * A;
  int32_t* out = nbr + toff[t];
  int k = 0;
  const double4 pi = ld_pos4(pos4, i);
  if (pi.w == (double)LMD_OWNED) {
    const long long lin = cell_of_owned(pi, g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2, g.d0, g.d1,
                                        g.d2, g.t0, g.t1);
    for_candidates(i, pi, newton3, g.t0, g.t1, lin, os, oc, hs, hc, pos4, rl2, [&](int j) {
      const int st = k / B, l = lane_of(pattern, il, k % B);
      out[(long long)(st / kChunk) * (32 * kChunk) + l * kChunk + st % kChunk] = j;
      ++k;
    });
  }
}

// Single-pass build into a fixed per-tile capacity: tile t owns the slots
// [t * cap_steps * 32, (t + 1) * cap_steps * 32), so no count pass and no
// prefix scan are needed.  Thread per owned particle; a tile's A particles
// are A aligned lanes of one warp, which agree on the tile's step count with
// a shuffle reduction, and each thread pads its own slots with the sentinel
// up to that count.  Entries past the capacity are dropped and reported
// through *max_count (the caller rebuilds with a larger capacity).
template <int P>
__global__ void vl_build_kernel(GridK g, int n, int ntiles, int newton3,
                                double rl2, int32_t sentinel, const double* __restrict__ pos4,
                                const int32_t* __restrict__ os, const int32_t* __restrict__ oc,
                                const int32_t* __restrict__ hs, const int32_t* __restrict__ hc,
                                int cap_steps, int32_t* __restrict__ count,
                                int32_t* __restrict__ count_half,
                                long long* __restrict__ toff, int32_t* __restrict__ kmax,
                                int32_t* __restrict__ max_count, int32_t* __restrict__ nbr) {
  constexpr int A = Pattern<P>::A, B = Pattern<P>::B, pattern = P;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = i / A, il = i - t * A;
  const long long stride = (long long)cap_steps * 32;
  int32_t* out = nbr + (long long)t * stride;
  const int cap = cap_steps * B;
  int k = 0, kh = 0;
  if (i < n) {
    const double4 pi = ld_pos4(pos4, i);
    if (pi.w == (double)LMD_OWNED) {
      const long long lin = cell_of_owned(pi, g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2, g.d0,
                                          g.d1, g.d2, g.t0, g.t1);
      for (int view = 0; view < 2; ++view) {
        const int32_t* vs = view ? hs : os;
        const int32_t* vc = view ? hc : oc;
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              const long long nl = lin + dx + g.t0 * (dy + g.t1 * dz);
              const int c = vc[nl];
              if (c == 0) continue;
              int j = vs[nl];
              const int e = j + c;
              if (!view && newton3) j = max(j, i + 1);
              // hits of up to 32 consecutive candidates are collected as a
              // bit mask and emitted afterwards in ascending order, so the
              // (warp-divergent) emit path runs once per hit, not once per
              // candidate that some lane of the warp accepted
              // branch-free candidate loop: the backing holds no DUMMY
              // records (owned checked at rebuild, images / ghosts tagged
              // HALO, the sentinel is in no cell) and the self pair is
              // cleared from the mask afterwards
              for (int j0 = j; j0 < e; j0 += 32) {
                const int cnt = min(e - j0, 32);
                unsigned mask = 0u;
#pragma unroll 2
                for (int q = 0; q < cnt; ++q) {
                  const double4 pj = ld_pos4(pos4, j0 + q);
                  const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
                  mask |= (r2 < rl2 ? 1u : 0u) << q;
                }
                if (!view) {
                  const unsigned self = (unsigned)(i - j0);
                  if (self < 32u) mask &= ~(1u << self);
                }
                while (mask) {
                  const int jj = j0 + __ffs(mask) - 1;
                  mask &= mask - 1u;
                  kh += view || jj > i;
                  if (k < cap) {
                    const int st = k / B, l = lane_of(pattern, il, k % B);
                    out[(long long)(st / kChunk) * (32 * kChunk) + l * kChunk + st % kChunk] = jj;
                  }
                  ++k;
                }
              }
            }
      }
    }
    count[i] = k;
    if (count_half) count_half[i] = kh;
  }
  // the tile's longest list (aligned groups of A lanes)
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

// Line-aligned entry order (optional pass after the build).  The force
// kernel is bound by the L1 data pipe, which retires about one distinct
// 128-B line per cycle per warp gather; with each lane's list in ascending
// order the 32 lanes of a fill touch ~21 distinct lines.  This pass permutes
// every lane's own slot sequence (so every entry stays with its particle;
// valid for every interaction order): each lane keeps a window of its next W
// entries in shared memory and, at each step, takes the entry whose line
// occurs most often across the warp's windows (ties: smaller index), which
// makes lanes gather from shared lines in the same fill (~14.6 lines at
// W = 16 in a host simulation).  Counts live in a 1024-entry table indexed
// by line mod 1024 (collisions only blur the heuristic).  Deterministic:
// choices are made from counts frozen by __syncwarp, and the slot written
// at step s was read into the window before (in place).
template <int W>
__global__ void __launch_bounds__(32 * kVLWarps)
    vl_align_kernel(int ntiles, int B, const long long* __restrict__ toff,
                    const int32_t* __restrict__ kmax, int32_t* __restrict__ nbr) {
  __shared__ int cnt_s[kVLWarps][1024];
  __shared__ int win_s[kVLWarps][W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * kVLWarps + w;
  if (t >= ntiles) return;
  int* cnt = cnt_s[w];
  for (int q = lane; q < 1024; q += 32) cnt[q] = 0;
  __syncwarp();
  const int steps = kmax[t] / B;
  int32_t* base = nbr + toff[t];
  auto slot = [&](int st) -> long long {
    return (long long)(st / kChunk) * (32 * kChunk) + lane * kChunk + st % kChunk;
  };
  int nxt = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    int v = -1;
    if (nxt < steps) v = base[slot(nxt++)];
    win_s[w][q][lane] = v;
    if (v >= 0) atomicAdd(&cnt[(v >> 2) & 1023], 1);
  }
  __syncwarp();
  for (int st = 0; st < steps; ++st) {
    int best = 0, bc = -1, bv = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = win_s[w][q][lane];
      if (v >= 0) {
        const int c = cnt[(v >> 2) & 1023];
        if (c > bc || (c == bc && v < bv)) {
          bc = c;
          bv = v;
          best = q;
        }
      }
    }
    __syncwarp();
    base[slot(st)] = bv;
    atomicSub(&cnt[(bv >> 2) & 1023], 1);
    int v = -1;
    if (nxt < steps) v = base[slot(nxt++)];
    win_s[w][best][lane] = v;
    if (v >= 0) atomicAdd(&cnt[(v >> 2) & 1023], 1);
    __syncwarp();
  }
}

__global__ void fill_i32_kernel(int64_t n, int32_t v, int32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = v;
}

// ------------------------------------------------------------------ force
// N3: 0 = full lists; 1 = half lists, the j side by FP64 atomics; 2 = full
// lists with the reference's Newton3 pair bookkeeping (pairs with an image j
// counted apart, the host halves the owned-owned ones): no atomics,
// deterministic.
template <bool EV, int N3>
__device__ __forceinline__ void vl_pair(const double4& pi, const double4& pj, int j, int n_owned,
                                        const LJK& k, Acc& a, double* __restrict__ fx,
                                        double* __restrict__ fy, double* __restrict__ fz) {
  const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
  double r2;
  if (!within_cutoff(dx, dy, dz, k, r2)) return;
  if (r2 == 0.0) {
    a.overlap = 1;
    return;
  }
  double s6;
  const double f = lj_scalar(r2, k, s6);
  a.ax = fma(f, dx, a.ax);
  a.ay = fma(f, dy, a.ay);
  a.az = fma(f, dz, a.az);
  ++a.pairs;
  const bool jhalo = j >= n_owned;
  if (N3 == 2) a.halo += jhalo;
  if (N3 == 1 && !jhalo) {
    atomicAdd(fx + j, -f * dx);
    atomicAdd(fy + j, -f * dy);
    atomicAdd(fz + j, -f * dz);
  }
  if (EV) {
    const double w = (N3 == 1 && !jhalo) ? 1.0 : 0.5;
    a.e = fma(w * s6, fma(k.eps4, s6, -k.eps4), a.e);
    a.v = fma(w * f, r2, a.v);
  }
}

// One i-tile: lane (io, jo) walks entries k = jo, jo + B, ... of particle
// t*A + io.  Indices for U fills are loaded first, then the U positions
// (256-bit gathers), then the U interactions, so each lane keeps 2U loads in
// flight.  Writes the tile's i forces; pair counts etc. accumulate in `a`.
struct SoA {
  const double* __restrict__ x;
  const double* __restrict__ y;
  const double* __restrict__ z;
};

// gather modes: 0 = 256-bit pos4 record, 1 = SoA x, y, z (64-bit each)
template <int GM>
__device__ __forceinline__ double4 ld_j(const double* __restrict__ pos4, const SoA& q, int j) {
  if (GM == 1) return make_double4(__ldg(q.x + j), __ldg(q.y + j), __ldg(q.z + j), 0.0);
  return ld_pos4(pos4, j);
}

template <int P, bool EV, int N3, int U, int SOA>
__device__ __forceinline__ void vl_tile(int t, int lane, int n_owned,
                                        const int32_t* __restrict__ out_perm,
                                        const double* __restrict__ pos4, const SoA& q,
                                        const long long* __restrict__ toff,
                                        const int32_t* __restrict__ kmax,
                                        const int32_t* __restrict__ nbr, const LJK& k, Acc& a,
                                        double* __restrict__ fx, double* __restrict__ fy,
                                        double* __restrict__ fz) {
  using Pat = Pattern<P>;
  // U = positions gathered per group (2 or 4) within a 4-step index chunk
  static_assert(U == 2 || U == 4, "gather group must divide the index chunk");
  const int io = Pat::ioff(lane), jo = Pat::joff(lane);
  const int i = t * Pat::A + io;
  const bool iact = i < n_owned;
  const double4 pi = ld_pos4(pos4, iact ? i : 0);
  const int4* chunks = reinterpret_cast<const int4*>(nbr + toff[t]) + lane;
  const int nchunks = kmax[t] / Pat::B / kChunk;
  const double ax0 = a.ax, ay0 = a.ay, az0 = a.az;
  a.ax = a.ay = a.az = 0.0;
  // software pipeline: the next chunk's indices are in flight while the
  // current chunk's positions are gathered and evaluated
  int4 nxt = nchunks > 0 ? __ldg(chunks) : make_int4(0, 0, 0, 0);
  for (int c = 0; c < nchunks; ++c) {
    const int4 cur = nxt;
    if (c + 1 < nchunks) nxt = __ldg(chunks + (long long)(c + 1) * 32);
    const int j[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
    for (int g = 0; g < 4; g += U) {
      double4 pj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pj[u] = ld_j<SOA>(pos4, q, j[g + u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        vl_pair<EV, N3>(pi, pj[u], j[g + u], n_owned, k, a, fx, fy, fz);
    }
  }
  if (!iact) a.ax = a.ay = a.az = 0.0;
  const double rx = reduce_j<P>(a.ax), ry = reduce_j<P>(a.ay), rz = reduce_j<P>(a.az);
  if (iact && jo == 0) {
    if (N3 == 1) {
      atomicAdd(fx + i, rx);
      atomicAdd(fy + i, ry);
      atomicAdd(fz + i, rz);
    } else {
      // out_perm: write straight into the caller's order (collect_forces fused)
      const int o = out_perm ? out_perm[i] : i;
      fx[o] = rx;
      fy[o] = ry;
      fz[o] = rz;
    }
  }
  a.ax = ax0;
  a.ay = ay0;
  a.az = az0;
}

// One warp per i-tile.  The 2-wide gather variant trades memory-level
// parallelism per warp for occupancy (64 registers, 8 blocks per SM).
template <int P, bool EV, int N3, int U, int SOA>
__global__ void __launch_bounds__(32 * kVLWarps, 8)
    vl_force_kernel(int n_owned, int ntiles, const int32_t* __restrict__ out_perm,
                    const double* __restrict__ pos4, SoA q,
                    const long long* __restrict__ toff, const int32_t* __restrict__ kmax,
                    const int32_t* __restrict__ nbr, LJK k, double* __restrict__ fx,
                    double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                    lmd_stats* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * kVLWarps + (threadIdx.x >> 5);
  Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0};
  if (t < ntiles)
    vl_tile<P, EV, N3, U, SOA>(t, lane, n_owned, out_perm, pos4, q, toff, kmax, nbr, k, a, fx, fy,
                               fz);
  flush_acc(a, lane, t < ntiles, EV, (long long)blockIdx.x * kVLWarps + (threadIdx.x >> 5), ev,
            stats);
}

__global__ void vl_stats_kernel(int n, int a, int b, const int32_t* __restrict__ count,
                                lmd_stats* __restrict__ stats) {
  // i-tiles of `a` consecutive backing slots; each tile's j-stream is its
  // longest list, chunked by b (oracle/lj_oracle.c: orc_force_phase_vl)
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int ntiles = (n + a - 1) / a;
  long long inv = 0, useful = 0;
  if (t < ntiles) {
    int m = 0;
    for (int q = t * a; q < t * a + a && q < n; ++q) {
      m = max(m, count[q]);
      useful += count[q];
    }
    inv = (m + b - 1) / b;
  }
  inv = warp_sum_ll(inv);
  useful = warp_sum_ll(useful);
  if ((threadIdx.x & 31) == 0 && (inv || useful)) {
    atomicAdd((unsigned long long*)&stats->kernel_invocations, (unsigned long long)inv);
    atomicAdd((unsigned long long*)&stats->useful_interactions, (unsigned long long)useful);
  }
}

__global__ void lane_slots_kernel_vl(lmd_stats* stats, int V) {
  stats->lane_slots = stats->kernel_invocations * (long long)V;
}

__global__ void gather_soa_kernel(int64_t n, const int32_t* __restrict__ perm,
                                  const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, double* __restrict__ ox,
                                  double* __restrict__ oy, double* __restrict__ oz) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t s = perm ? perm[k] : (int32_t)k;
  ox[k] = x[s];
  oy[k] = y[s];
  oz[k] = z[s];
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int lmd_vl_count(const lmd_grid* g, double rl2, int newton3, int64_t n_owned, const double* pos4,
                 const int32_t* o_start, const int32_t* o_count, const int32_t* h_start,
                 const int32_t* h_count, int32_t* count, void* stream) {
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL) return LMD_ERR_CONFIG;
  vl_count_kernel<<<(unsigned)cdiv(n_owned, 128), 128, 0, (cudaStream_t)stream>>>(
      make_gridk(g), (int)n_owned, newton3, rl2, pos4, o_start, o_count, h_start, h_count, count);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int64_t lmd_vl_num_tiles(int64_t n_owned, int pattern) {
  return cdiv(n_owned, pattern_A(pattern));
}

size_t lmd_vl_scan_temp_bytes(int64_t ntiles) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const long long*)nullptr, (long long*)nullptr,
                                (int)(ntiles > 0 ? ntiles : 1));
  return bytes;
}

int lmd_vl_layout(int64_t n_owned, int pattern, const int32_t* count, int64_t* tile_len,
                  int64_t* tile_off, int32_t* kmax, void* temp, size_t temp_bytes,
                  void* stream) {
  if (n_owned <= 0) return LMD_OK;
  const int A = pattern_A(pattern), B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_owned, A);
  cudaStream_t s = (cudaStream_t)stream;
  vl_tile_kernel<<<(unsigned)cdiv(ntiles, 256), 256, 0, s>>>((int)n_owned, A, B, count,
                                                             (long long*)tile_len, kmax);
  LMD_CHECK_LAUNCH();
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, bytes, (const long long*)tile_len,
                                                (long long*)tile_off, (int)ntiles, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  return LMD_OK;
}

int lmd_vl_fill(const lmd_grid* g, double rl2, int newton3, int pattern, int64_t n_owned,
                int32_t sentinel, const double* pos4, const int32_t* o_start,
                const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                const int64_t* tile_off, int64_t total, int32_t* nbr, void* stream) {
  if (n_owned <= 0) return LMD_OK;
  const int A = pattern_A(pattern), B = pattern_B(pattern);
  cudaStream_t s = (cudaStream_t)stream;
  fill_i32_kernel<<<1184, 256, 0, s>>>(total, sentinel, nbr);
  LMD_CHECK_LAUNCH();
  vl_fill_kernel<<<(unsigned)cdiv(n_owned, 128), 128, 0, s>>>(
      make_gridk(g), (int)n_owned, A, B, pattern, newton3, rl2, pos4, o_start, o_count, h_start,
      h_count, (const long long*)tile_off, nbr);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_vl_build(const lmd_grid* g, double rl2, int newton3, int pattern, int64_t n_owned,
                 int32_t sentinel, const double* pos4, const int32_t* o_start,
                 const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                 int32_t cap_steps, int32_t* count, int32_t* count_half, int64_t* tile_off,
                 int32_t* kmax, int32_t* max_count, int32_t* nbr, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(max_count, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL || cap_steps <= 0 || cap_steps % kChunk) return LMD_ERR_CONFIG;
  const int A = pattern_A(pattern), B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_owned, A);
  const unsigned blocks = (unsigned)cdiv(ntiles * A, 128);
#define LMD_VLB(P)                                                                             \
  vl_build_kernel<P><<<blocks, 128, 0, s>>>(make_gridk(g), (int)n_owned, (int)ntiles, newton3, \
                                            rl2, sentinel, pos4, o_start, o_count, h_start,    \
                                            h_count, cap_steps, count, count_half,             \
                                            (long long*)tile_off, kmax, max_count, nbr)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_VLB(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_VLB(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_VLB(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_VLB(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_VLB
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_vl_align(int pattern, int64_t n_units, int window, const int64_t* tile_off,
                 const int32_t* kmax, int32_t* nbr, void* stream) {
  if (n_units <= 0) return LMD_OK;
  const int B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_units, pattern_A(pattern));
  const unsigned blocks = (unsigned)cdiv(ntiles, kVLWarps);
  cudaStream_t s = (cudaStream_t)stream;
  switch (window) {
    case 8: vl_align_kernel<8><<<blocks, 32 * kVLWarps, 0, s>>>((int)ntiles, B, (const long long*)tile_off, kmax, nbr); break;
    case 16: vl_align_kernel<16><<<blocks, 32 * kVLWarps, 0, s>>>((int)ntiles, B, (const long long*)tile_off, kmax, nbr); break;
    case 32: vl_align_kernel<32><<<blocks, 32 * kVLWarps, 0, s>>>((int)ntiles, B, (const long long*)tile_off, kmax, nbr); break;
    default: return LMD_ERR_CONFIG;
  }
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int64_t lmd_vl_ev_slots(int64_t n_owned, int pattern) {
  return cdiv(lmd_vl_num_tiles(n_owned, pattern), kVLWarps) * kVLWarps;
}

}  // extern "C"

template <int P, bool EV, int N3, int GM>
static void launch_vl(int64_t n_owned, int64_t ntiles, const int32_t* out_perm,
                      const double* pos4, const SoA& q,
                      const int64_t* tile_off, const int32_t* kmax, const int32_t* nbr,
                      const LJK& k, double* fx, double* fy, double* fz, double* ev,
                      lmd_stats* stats, cudaStream_t s) {
  const unsigned blocks = (unsigned)cdiv(ntiles, kVLWarps);
  vl_force_kernel<P, EV, N3, 2, GM><<<blocks, 32 * kVLWarps, 0, s>>>(
      (int)n_owned, (int)ntiles, out_perm, pos4, q, (const long long*)tile_off, kmax, nbr, k, fx, fy, fz, ev,
      stats);
}

template <int P, bool EV, int N3>
static void launch_vl_g(int gm, int64_t n_owned, int64_t ntiles, const int32_t* out_perm,
                        const double* pos4,
                        const SoA& q, const int64_t* tile_off, const int32_t* kmax,
                        const int32_t* nbr, const LJK& k, double* fx, double* fy, double* fz,
                        double* ev, lmd_stats* stats, cudaStream_t s) {
  if (gm == 1)
    launch_vl<P, EV, N3, 1>(n_owned, ntiles, out_perm, pos4, q, tile_off, kmax, nbr, k, fx, fy, fz, ev,
                            stats, s);
  else
    launch_vl<P, EV, N3, 0>(n_owned, ntiles, out_perm, pos4, q, tile_off, kmax, nbr, k, fx, fy, fz, ev,
                            stats, s);
}

extern "C" {

int lmd_force_vl(int pattern, int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                 const double* pos4, const double* soa, int64_t ntot, const int64_t* tile_off,
                 const int32_t* kmax, const int32_t* nbr, const int32_t* out_perm, double* fx,
                 double* fy, double* fz, double* ev_scratch, lmd_stats* stats, void* stream) {
  if (n_owned <= 0) return LMD_OK;
  if (newton3 < 0 || newton3 > 2) return LMD_ERR_CONFIG;
  if (out_perm && newton3 == 1) return LMD_ERR_CONFIG;
  const LJK k = make_ljk(lj);
  const int64_t ntiles = lmd_vl_num_tiles(n_owned, pattern);
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  // gathers: soa != NULL -> x, y, z from SoA arrays soa[0..ntot), soa[ntot..), ...;
  // else the 256-bit pos4 record (a 128 + 64-bit x, y, z variant measured 20 %
  // slower)
  const int gm = soa ? 1 : 0;
  const SoA q = {soa, soa ? soa + ntot : nullptr, soa ? soa + 2 * ntot : nullptr};
#define LMD_VLK(P, EVB, N3B)                                                                  \
  launch_vl_g<P, EVB, N3B>(gm, n_owned, ntiles, out_perm, pos4, q, tile_off, kmax, nbr, k, fx, \
                           fy, fz,                                                            \
                           ev_scratch, stats, s)
#define LMD_VL_P(P)                                   \
  do {                                                \
    if (ev) {                                         \
      if (newton3 == 1) LMD_VLK(P, true, 1);          \
      else if (newton3 == 2) LMD_VLK(P, true, 2);     \
      else LMD_VLK(P, true, 0);                       \
    } else {                                          \
      if (newton3 == 1) LMD_VLK(P, false, 1);         \
      else if (newton3 == 2) LMD_VLK(P, false, 2);    \
      else LMD_VLK(P, false, 0);                      \
    }                                                 \
  } while (0)
  switch (pattern) {
    case LMD_ONE_BY_V: LMD_VL_P(LMD_ONE_BY_V); break;
    case LMD_V_BY_ONE: LMD_VL_P(LMD_V_BY_ONE); break;
    case LMD_TWO_BY_HALF: LMD_VL_P(LMD_TWO_BY_HALF); break;
    case LMD_HALF_BY_TWO: LMD_VL_P(LMD_HALF_BY_TWO); break;
    default: return LMD_ERR_CONFIG;
  }
#undef LMD_VL_P
#undef LMD_VLK
  LMD_CHECK_LAUNCH();
  if (ev) {
    const int64_t slots = cdiv(ntiles, kVLWarps) * kVLWarps;
    return reduce_ev(ev_scratch, slots, stats, s);
  }
  return LMD_OK;
}

int lmd_vl_stats(int64_t n_owned, int a, int b, int vector_width, const int32_t* count,
                 lmd_stats* stats, void* stream) {
  if (vector_width < 4 || (vector_width & (vector_width - 1)) != 0) return LMD_ERR_CONFIG;
  if (a < 1 || b < 1 || a * b != vector_width) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_owned > 0) {
    const int64_t ntiles = cdiv(n_owned, a);
    vl_stats_kernel<<<(unsigned)cdiv(ntiles, 256), 256, 0, s>>>((int)n_owned, a, b, count, stats);
    LMD_CHECK_LAUNCH();
  }
  lane_slots_kernel_vl<<<1, 1, 0, s>>>(stats, vector_width);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_gather_soa(int64_t n, const int32_t* perm, const double* x, const double* y,
                   const double* z, double* ox, double* oy, double* oz, void* stream) {
  if (n <= 0) return LMD_OK;
  gather_soa_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(n, perm, x, y, z,
                                                                             ox, oy, oz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
