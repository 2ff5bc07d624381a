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
#include <type_traits>

#include "vl_common.cuh"

namespace lmd {

template <int P>
struct Tile {
  static constexpr int A = Pattern<P>::A, B = Pattern<P>::B;
};

// Single-pass build into a fixed per-tile capacity: tile t owns the slots
// [t * cap_steps * 32, (t + 1) * cap_steps * 32), so no count pass and no
// prefix scan are needed.  Thread per owned particle; a tile's A particles
// are A aligned lanes of one warp, which agree on the tile's step count with
// a shuffle reduction, and each thread pads its own slots with the sentinel
// up to that count.  Entries past the capacity are dropped and reported
// through *max_count (the caller rebuilds with a larger capacity).
// IDX = uint16_t: staged lists with every group staged (local rows < 2^16),
// 8 steps per 128-bit chunk; idle slots 0xffff.
#ifndef LMD_BUILD_MIN_BLOCKS
#define LMD_BUILD_MIN_BLOCKS 12
#endif
template <int P, typename IDX = int32_t>
__global__ void __launch_bounds__(128, LMD_BUILD_MIN_BLOCKS) vl_build_kernel(GridK g, int n, int ntiles, int newton3,
                                double rl2, int32_t sentinel, const double* __restrict__ pos4,
                                const int32_t* __restrict__ os, const int32_t* __restrict__ oc,
                                const int32_t* __restrict__ hs, const int32_t* __restrict__ hc,
                                int cap_steps, int32_t* __restrict__ count,
                                int32_t* __restrict__ count_half,
                                long long* __restrict__ toff, int32_t* __restrict__ kmax,
                                int32_t* __restrict__ max_count, int32_t* __restrict__ nbr,
                                const int32_t* __restrict__ groups, int G) {
  constexpr int A = Pattern<P>::A, B = Pattern<P>::B, pattern = P;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = i / A, il = i - t * A;
  constexpr int CH = 16 / sizeof(IDX);  // steps per 128-bit chunk
  const long long stride = (long long)cap_steps * 32;
  IDX* out = reinterpret_cast<IDX*>(nbr) + (long long)t * stride;
  const int cap = cap_steps * B;
  int k = 0, kh = 0;
  if (i < n) {
    const double4 pi = ld_pos4(pos4, i);
    if (pi.w == (double)LMD_OWNED) {
      const long long lin = cell_of_owned(pi, g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2, g.d0,
                                          g.d1, g.d2, g.t0, g.t1);
      // staged: the group's record and this particle's row within the group
      // (groups gathering global indices have all offsets 0)
      const int32_t* grec = groups ? groups + (long long)(i / G) * kGroupRec : nullptr;
      const int grow = grec ? (lin / g.t0 == __ldg(grec + kGrpRow) ? 0 : 1) : 0;
      for (int view = 0; view < 2; ++view) {
        const int32_t* vs = view ? hs : os;
        const int32_t* vc = view ? hc : oc;
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy) {
            // the 3 cells dx = -1..1 of this row are consecutive linear
            // cells: their particles form one contiguous index range
            const long long nl0 = lin - 1 + g.t0 * (dy + g.t1 * dz);
            int j = 0x7fffffff, e = -1;
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
              const int c = vc[nl0 + dx];
              if (c) {
                const int s0 = vs[nl0 + dx];
                j = min(j, s0);
                e = max(e, s0 + c);
              }
            }
            if (e < 0) continue;
            // staged lists: index into the group's shared-memory copy of
            // this (view, dy, dz) run (vl_group_kernel); 0 for global
            const int roff =
                grec ? __ldg(grec + kGrpOff + view * 18 + grow * 9 + (dz + 1) * 3 + (dy + 1))
                     : 0;
            if (!view && newton3) j = max(j, i + 1);
            // hits of up to 64 consecutive candidates are collected as a
            // bit mask and emitted afterwards in ascending order, so the
            // (warp-divergent) emit path runs once per hit, not once per
            // candidate that some lane of the warp accepted; one range per
            // row (not per cell) keeps the lanes' emission loops balanced.
            // Branch-free candidate loop: the backing holds no DUMMY records
            // (owned checked at rebuild, images / ghosts tagged HALO, the
            // sentinel is in no cell) and the self pair is cleared afterwards
            for (int j0 = j; j0 < e; j0 += 64) {
              const int cnt = min(e - j0, 64);
              unsigned long long mask = 0ull;
              // shift-and-add accumulation (2 integer instructions per
              // candidate); bit-reversed below to candidate order
              unsigned long long racc = 0ull;
#pragma unroll 2
              for (int q = 0; q < cnt; ++q) {
                const double4 pj = ld_pos4(pos4, j0 + q);
                const double r2 = r2_exact(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z);
                racc = racc + racc + (r2 < rl2 ? 1ull : 0ull);
              }
              mask = __brevll(racc << (64 - cnt));
              if (!view) {
                const unsigned self = (unsigned)(i - j0);
                if (self < 64u) mask &= ~(1ull << self);
              }
              // half-list length: every image hit, owned hits with j > i
              {
                const int d = i + 1 - j0;
                kh += __popcll(view || d <= 0 ? mask : (d >= 64 ? 0ull : mask & (~0ull << d)));
              }
              while (mask) {
                const int jj = j0 + __ffsll((long long)mask) - 1;
                mask &= mask - 1ull;
                if (k < cap) {
                  const int st = k / B, l = lane_of(pattern, il, k % B);
                  out[(long long)(st / CH) * (32 * CH) + l * CH + st % CH] = (IDX)(jj + roff);
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
  steps = (steps + CH - 1) / CH * CH;
  if (steps > cap_steps) steps = cap_steps;
  if (t < ntiles) {
    for (int q = min(k, cap); q < steps * B; ++q) {
      const int st = q / B, l = lane_of(pattern, il, q % B);
      out[(long long)(st / CH) * (32 * CH) + l * CH + st % CH] = (IDX)sentinel;
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

// Group run table for the staged lists (one warp per group; lane l scans
// runs l and l + 32 for their first and last particle).
__global__ void vl_group_kernel(GridK g, int n, int G, int scap, const double* __restrict__ pos4,
                                const int32_t* __restrict__ os, const int32_t* __restrict__ oc,
                                const int32_t* __restrict__ hs, const int32_t* __restrict__ hc,
                                int32_t* __restrict__ groups, int32_t* __restrict__ smax) {
  const int lane = threadIdx.x & 31;
  const long long grp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long ngroups = ((long long)n + G - 1) / G;
  if (grp >= ngroups) return;
  const long long i0 = grp * G, i1 = min((long long)n, i0 + G) - 1;
  const long long lo = cell_of_owned(ld_pos4(pos4, i0), g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2,
                                     g.d0, g.d1, g.d2, g.t0, g.t1);
  const long long hi = cell_of_owned(ld_pos4(pos4, i1), g.lo0, g.lo1, g.lo2, g.cl0, g.cl1, g.cl2,
                                     g.d0, g.d1, g.d2, g.t0, g.t1);
  const long long row_lo = lo / g.t0, row_hi = hi / g.t0;
  // the group's particles must lie in row_lo or row_hi (rows in between are
  // ring rows when the group crosses a z-plane); otherwise it gathers globally
  bool two = true;
  if (row_hi - row_lo > 1)
    for (long long i = i0 + lane; i <= i1; i += 32) {
      const long long r = cell_of_owned(ld_pos4(pos4, i), g.lo0, g.lo1, g.lo2, g.cl0, g.cl1,
                                        g.cl2, g.d0, g.d1, g.d2, g.t0, g.t1) / g.t0;
      two &= r == row_lo || r == row_hi;
    }
  const int R = row_hi == row_lo ? 1 : (__all_sync(0xffffffffu, two) ? 2 : 3);
  int start[2] = {0, 0}, len[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
    if (r >= kGroupRuns || R > 2) continue;
    const int view = r / 18, rr = (r % 18) / 9, q = r % 9, dz = q / 3 - 1, dy = q % 3 - 1;
    if (rr >= R) continue;
    const int32_t* vs = view ? hs : os;
    const int32_t* vc = view ? hc : oc;
    const long long xa = rr == 0 ? lo % g.t0 : 1;
    const long long xb = rr == R - 1 ? hi % g.t0 : g.d0;
    const long long nrow = (rr == 0 ? row_lo : row_hi) + dy + g.t1 * dz;
    int first = -1, last = -1;
    for (long long c = nrow * g.t0 + xa - 1; c <= nrow * g.t0 + xb + 1; ++c) {
      const int k = vc[c];
      if (k) {
        if (first < 0) first = vs[c];
        last = vs[c] + k;
      }
    }
    if (first >= 0) {
      start[h] = first & ~1;                 // 16-B aligned bulk copies
      len[h] = (last - start[h] + 1) & ~1;
    }
  }
  // exclusive scan of the run lengths (runs 0..31, then 32..35) -> bases
  int incl = len[0];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int totA = __shfl_sync(0xffffffffu, incl, 31);
  int incl2 = len[1];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl2, d);
    if (lane >= d) incl2 += v;
  }
  const int base[2] = {incl - len[0], totA + incl2 - len[1]};
  const int S = totA + __shfl_sync(0xffffffffu, incl2, 31);
  const int halo_base = __shfl_sync(0xffffffffu, base[0], 18);  // run 18 = first image run
  const bool glob = R > 2 || S > scap;
  int32_t* rec = groups + grp * kGroupRec;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
    if (r < kGroupRuns) {
      rec[kGrpStart + r] = glob ? 0 : start[h];
      rec[kGrpLen + r] = glob ? 0 : len[h];
      rec[kGrpOff + r] = glob ? 0 : base[h] - start[h];
    }
  }
  if (lane == 0) {
    rec[kGrpS] = glob ? 0 : S;
    rec[kGrpHalo] = glob ? n : halo_base;
    rec[kGrpGlobal] = glob ? 1 : 0;
    rec[kGrpRow] = (int)row_lo;
    rec[kGrpRow + 1] = (int)row_hi;
    atomicMax(smax, glob ? 0 : S);
    if (glob) atomicAdd(smax + 1, 1);
  }
}

// Bank-conflict-aware entry order (optional pass after the build, for the
// SoA gathers).  Measured (tools/bank_probe.cu, profiles/r01_bank_probe.jsonl):
// a warp's 64-bit gather -- shared memory or L1-resident global alike -- is
// served per half-warp, costing the largest number of lanes of that half
// that hit one 8-byte bank pair (16 pairs per 128 B), i.e. 2 cycles when
// conflict-free and ~6-8.5 for random indices.  With SoA arrays whose rows
// start on 128 B, x[j], y[j], z[j] sit in bank pair j & 15.  This pass
// permutes every lane's own slot sequence so that, step by step, the lanes
// of each half-warp gather from distinct bank pairs:
//   * each lane buckets its entries by bank pair (shared memory);
//   * at step s, lane l of a half first takes its Latin-square pair
//     (l + s) & 15 if it still holds one (conflict-free by construction);
//     then `rounds` proposal rounds: a lane proposes the first pair, rotated
//     to start at (l + s) & 15, that it holds and no winner of its half has
//     taken; the lowest proposing lane wins (prefix OR over the half);
//   * a lane that lost every round idles (slot -1) if it can still finish
//     within the tile's T steps, otherwise it takes a conflicting entry.
// Entries never leave their lane, the step count T is unchanged, every
// choice is a function of warp-uniform state: the list is a deterministic
// permutation of the build's.  Idle slots are -1 (ld_j<1> skips the load).
__device__ __forceinline__ int first_rot16(unsigned m, int k) {
  const unsigned r = ((m >> k) | (m << (16 - k))) & 0xffffu;
  return r ? ((__ffs(r) - 1 + k) & 15) : -1;
}

__global__ void vl_bank_kernel(int ntiles, int B, int32_t sentinel, int rounds, int tcap,
                               const long long* __restrict__ toff,
                               const int32_t* __restrict__ kmax, int32_t* __restrict__ nbr) {
  extern __shared__ int32_t bank_sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int t = blockIdx.x * nw + w;
  if (t >= ntiles) return;  // warp-uniform
  const int T = kmax[t] / B;
  int32_t* cur = bank_sm + (size_t)w * (64 * 16 + (size_t)tcap * 32);
  int32_t* cnt = cur + 16 * 32;
  int32_t* ent = cnt + 16 * 32;
  int4* base4 = reinterpret_cast<int4*>(nbr + toff[t]);
#pragma unroll
  for (int b = 0; b < 16; ++b) cnt[b * 32 + lane] = 0;
  int n = 0;
  for (int c = 0; c < T / kChunk; ++c) {
    const int4 v = base4[c * 32 + lane];
    const int j[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j[u] != sentinel && j[u] >= 0) {
        ++cnt[(j[u] & 15) * 32 + lane];
        ++n;
      }
  }
  unsigned avail = 0u;
  int acc = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const int c = cnt[b * 32 + lane];
    cur[b * 32 + lane] = acc;
    acc += c;
    avail |= (c ? 1u : 0u) << b;
  }
  for (int c = 0; c < T / kChunk; ++c) {
    const int4 v = base4[c * 32 + lane];
    const int j[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j[u] != sentinel && j[u] >= 0) {
        const int p = cur[(j[u] & 15) * 32 + lane]++;
        ent[p * 32 + lane] = j[u];
      }
  }
  // cursors back to the bucket starts
#pragma unroll
  for (int b = 0; b < 16; ++b) cur[b * 32 + lane] -= cnt[b * 32 + lane];
  const int half = lane >> 4, hl = lane & 15;
  int lrem = n;
  for (int s0 = 0; s0 < T; s0 += kChunk) {
  int out[kChunk];
#pragma unroll
  for (int u = 0; u < kChunk; ++u) {
    const int s = s0 + u;
    const int rot = (hl + s) & 15;
    int pick = -1;
    bool pending = lrem > 0;
    // the lane's own bank pair of this step (a Latin square: conflict-free)
    if (pending && ((avail >> rot) & 1u)) {
      pick = rot;
      pending = false;
    }
    unsigned usedw = __reduce_or_sync(0xffffffffu, pick >= 0 ? 1u << (pick + 16 * half) : 0u);
    for (int r = 0; r < rounds; ++r) {
      const unsigned used = (usedw >> (16 * half)) & 0xffffu;
      const int b = pending ? first_rot16(avail & ~used, rot) : -1;
      if (!__any_sync(0xffffffffu, b >= 0)) break;
      // lowest lane of the half proposing a pair wins it: prefix OR
      const unsigned p = b >= 0 ? 1u << (b + 16 * half) : 0u;
      unsigned incl = p;
#pragma unroll
      for (int d = 1; d < 16; d <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
        if (hl >= d) incl |= v;
      }
      unsigned lower = __shfl_up_sync(0xffffffffu, incl, 1);
      if (hl == 0) lower = 0u;
      const bool win = p != 0u && !(lower & p);
      usedw |= __reduce_or_sync(0xffffffffu, win ? p : 0u);
      if (win) {
        pick = b;
        pending = false;
      }
    }
    if (pending && T - s <= lrem) pick = first_rot16(avail, rot);  // no slack left
    int j = -1;
    if (pick >= 0) {
      const int p = cur[pick * 32 + lane]++;
      j = ent[p * 32 + lane];
      if (--cnt[pick * 32 + lane] == 0) avail &= ~(1u << pick);
      --lrem;
    }
    out[u] = j;
  }
  base4[(s0 / kChunk) * 32 + lane] = make_int4(out[0], out[1], out[2], out[3]);
  }
}

// Lane-local variant (rounds == 0): lane l of a half takes its Latin-square
// pair (l + s) & 15 at step s when it still holds one, idles while it has
// slack, and otherwise takes the first pair it holds in rotated order.  No
// cross-lane communication, so every lane schedules independently; per-lane
// bank counts and bucket cursors live in registers as packed bytes (tiles of
// more than 255 steps are left in build order), only the bucketed entries
// are in shared memory.
__device__ __forceinline__ unsigned get_byte4(const unsigned (&v)[4], int b) {
  const unsigned w = (b & 8) ? ((b & 4) ? v[3] : v[2]) : ((b & 4) ? v[1] : v[0]);
  return (w >> ((b & 3) * 8)) & 0xffu;
}
__device__ __forceinline__ void add_byte4(unsigned (&v)[4], int b, unsigned x) {
  const unsigned inc = x << ((b & 3) * 8);
  if (b < 4) v[0] += inc;
  else if (b < 8) v[1] += inc;
  else if (b < 12) v[2] += inc;
  else v[3] += inc;
}

// entries of one 128-bit list chunk: 4 int32 or 8 uint16 (0xffff / -1 /
// sentinel = no entry -> -1)
template <bool I16>
__device__ __forceinline__ void unpack_chunk(const int4& v, int32_t sentinel, int* j) {
  if (I16) {
    const unsigned w4[4] = {(unsigned)v.x, (unsigned)v.y, (unsigned)v.z, (unsigned)v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned lo = w4[e] & 0xffffu, hi = w4[e] >> 16;
      j[2 * e] = lo == 0xffffu ? -1 : (int)lo;
      j[2 * e + 1] = hi == 0xffffu ? -1 : (int)hi;
    }
  } else {
    const int w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) j[e] = (w4[e] == sentinel || w4[e] < 0) ? -1 : w4[e];
  }
}

template <bool I16>
__global__ void __launch_bounds__(256)
    vl_bank_local_kernel(int ntiles, int B, int32_t sentinel, int tcap,
                         const long long* __restrict__ toff, const int32_t* __restrict__ kmax,
                         int32_t* __restrict__ nbr) {
  constexpr int CH = I16 ? 8 : 4;  // entries per 128-bit chunk
  extern __shared__ __align__(128) uint16_t bank_ent[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int t = blockIdx.x * nw + w;
  if (t >= ntiles) return;  // warp-uniform
  const int T = kmax[t] / B;
  if (T > tcap || T == 0) return;  // workspace bound; keep the build order
  // per warp: counts and cursors per (bank pair, lane) as 16-bit words,
  // then the entries bucketed by bank pair (16-bit local rows)
  uint16_t* cnt = bank_ent + (size_t)w * (48 * 32 + (size_t)tcap * 32);
  uint16_t* cur = cnt + 16 * 32;
  uint16_t* end = cur + 16 * 32;
  uint16_t* ent = end + 16 * 32;
  int4* base4 = I16 ? reinterpret_cast<int4*>(reinterpret_cast<uint16_t*>(nbr) + toff[t])
                    : reinterpret_cast<int4*>(nbr + toff[t]);
  const int nch = T / CH;
#pragma unroll
  for (int b = 0; b < 16; ++b) cnt[b * 32 + lane] = 0;
  int n = 0;
  bool wide = false;
  // pass 1: bank counts (4 chunk loads in flight)
  for (int c0 = 0; c0 < nch; c0 += 4) {
    int4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      v[q] = c0 + q < nch ? base4[(c0 + q) * 32 + lane] : make_int4(-1, -1, -1, -1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int j[CH];
      unpack_chunk<I16>(v[q], sentinel, j);
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (j[u] >= 0) {
          ++cnt[(j[u] & 15) * 32 + lane];
          wide |= j[u] > 0xfffe;
          ++n;
        }
    }
  }
  // tiles of groups that gather global indices keep the build order
  if (__any_sync(0xffffffffu, wide)) return;
  // bucket starts / ends and the avail mask
  unsigned avail = 0u;
  int acc = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const int c = cnt[b * 32 + lane];
    cur[b * 32 + lane] = (uint16_t)acc;
    acc += c;
    end[b * 32 + lane] = (uint16_t)acc;
    avail |= (c ? 1u : 0u) << b;
  }
  // pass 2: scatter into the buckets
  for (int c0 = 0; c0 < nch; c0 += 4) {
    int4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      v[q] = c0 + q < nch ? base4[(c0 + q) * 32 + lane] : make_int4(-1, -1, -1, -1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int j[CH];
      unpack_chunk<I16>(v[q], sentinel, j);
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (j[u] >= 0) {
          const int b = j[u] & 15;
          const int p = cur[b * 32 + lane];
          cur[b * 32 + lane] = (uint16_t)(p + 1);
          ent[p * 32 + lane] = (uint16_t)j[u];
        }
    }
  }
  // cursors back to the bucket starts
#pragma unroll
  for (int b = 0; b < 16; ++b) cur[b * 32 + lane] = (uint16_t)(end[b * 32 + lane] - cnt[b * 32 + lane]);
  const int hl = lane & 15;
  int lrem = n;
  for (int s0 = 0; s0 < T; s0 += CH) {
    int out[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int s = s0 + u;
      const int rot = (hl + s) & 15;
      int pick = -1;
      if (lrem > 0) {
        if ((avail >> rot) & 1u) pick = rot;
        else if (T - s <= lrem) pick = first_rot16(avail, rot);  // no slack left
      }
      int j = -1;
      if (pick >= 0) {
        const int p = cur[pick * 32 + lane];
        j = ent[p * 32 + lane];
        cur[pick * 32 + lane] = (uint16_t)(p + 1);
        if (p + 1 == end[pick * 32 + lane]) avail &= ~(1u << pick);
        --lrem;
      }
      out[u] = j;
    }
    int4 o;
    if (I16) {
      unsigned w4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w4[e] = ((unsigned)out[2 * e] & 0xffffu) | (((unsigned)out[2 * e + 1] & 0xffffu) << 16);
      o = make_int4((int)w4[0], (int)w4[1], (int)w4[2], (int)w4[3]);
    } else {
      o = make_int4(out[0], out[1], out[2], out[3]);
    }
    base4[(s0 / CH) * 32 + lane] = o;
  }
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
// GM = 1: j < 0 is an idle slot of a bank-scheduled list (vl_bank_kernel):
// no load (the lane drops out of the gather, so it adds no bank conflict),
// a position far outside every cutoff.
template <int GM>
__device__ __forceinline__ double4 ld_j(const double* __restrict__ pos4, const SoA& q, int j) {
  if (GM == 1) {
    if (j < 0) return make_double4(1.0e300, 1.0e300, 1.0e300, 0.0);
    return make_double4(__ldg(q.x + j), __ldg(q.y + j), __ldg(q.z + j), 0.0);
  }
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

// ------------------------------------------------------------ staged force
// One block per group of G = 32 * W owned particles (W tiles, thread per i):
// thread 0 arms an mbarrier and issues one TMA bulk copy per (run, axis) of
// the SoA positions into shared memory (no register staging, no LSU
// writeback), every warp then walks its tile's bank-scheduled local
// indices with conflict-free 64-bit shared-memory loads.  Groups whose runs
// exceed the capacity gather their global indices from the SoA arrays.
// rows per axis of the shared-memory copy, by group size; the last row is a
// dummy far away (idle slots), so a group stages at most rows - 16 rows
template <int W>
struct StageRows {
  static constexpr int value = W == 4 ? 2304 : (W == 8 ? 4096 : 7168);
};
static inline int stage_rows(int group_size) {
  return group_size == 128 ? StageRows<4>::value
                           : (group_size == 256 ? StageRows<8>::value : StageRows<16>::value);
}

// One list slot of the staged kernel, branch-free apart from the rare exact
// re-evaluation near the cutoff: the LJ expression runs for every lane (the
// warp would run it anyway whenever one lane hits) and is masked.
// Four list slots of the staged kernel, branch-free: r2 is always the
// reference's unfused expression (two FP64 instructions more than the FMA
// form, but no near-cutoff re-evaluation branch), the cutoff test compares
// bit patterns on the integer pipe, the LJ expression runs for every lane
// (the warp would run it anyway whenever one lane hits) and the
// accumulation is predicated.
template <bool EV, int N3>
__device__ __forceinline__ void staged_pairs4(const double4& pi, const double* xj,
                                              const double* yj, const double* zj,
                                              const unsigned* j, int hb, const LJK& k, Acc& a) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double dx = pi.x - xj[u], dy = pi.y - yj[u], dz = pi.z - zj[u];
    const double r2 = r2_exact(dx, dy, dz);
    const unsigned long long b = (unsigned long long)__double_as_longlong(r2);
    // 0 < r2 < rc2 in one unsigned compare of the bit patterns (r2 >= +0)
    const bool hit = b - 1ull < (unsigned long long)k.rc2_bits - 1ull;
    // overlap: r2 == 0 (the numba -1 sentinel); the high word is 0 only for
    // r2 < 2^-1022, i.e. coincident particles -- tracked as a running min
    a.hi_min = min(a.hi_min, (unsigned)(b >> 32));
    const bool in = hit;
    // u = 1/r2; f = 24 eps (2 s6^2 - s6) / r2 = u^4 (c12 u^3 - c6) with the
    // powers of sigma folded into c12, c6: 5 FP64 instructions after the
    // reciprocal (kernels.py:112-126 evaluates the same expression)
    const double ur = rcp_fast(r2);
    const double u2 = ur * ur;
    const double u3 = u2 * ur;
    double f = (u2 * u2) * fma(k.c12, u3, -k.c6);
    f = hit ? f : 0.0;  // one select; the accumulation then runs unpredicated
    a.ax = fma(f, dx, a.ax);
    a.ay = fma(f, dy, a.ay);
    a.az = fma(f, dz, a.az);
    if (EV) {
      const double hu = hit ? 0.5 * u3 : 0.0;
      a.e = fma(hu, fma(k.e12, u3, -k.e6), a.e);
      a.v = fma(0.5 * f, r2, a.v);
    }
    a.pairs += in;
    if (N3 == 2) a.halo += (in && (int)j[u] >= hb);
  }
}

#ifndef LMD_STAGED_PREFETCH
#define LMD_STAGED_PREFETCH 4
#endif
#ifndef LMD_STAGED_BATCH
#define LMD_STAGED_BATCH 2
#endif
constexpr int kStagedPrefetch = LMD_STAGED_PREFETCH;  // index chunks in flight
constexpr int kStagedBatch = LMD_STAGED_BATCH;        // chunks evaluated together

template <bool EV, int N3, int ROWS, bool STAGED, bool I16>
__device__ __forceinline__ void vl_staged_tile(int t, int lane, int n_owned, int hb,
                                               unsigned dummy, unsigned long long* bar,
                                               const int32_t* __restrict__ out_perm,
                                               const double* __restrict__ pos4,
                                               const double* __restrict__ xs,
                                               const double* __restrict__ ys,
                                               const double* __restrict__ zs,
                                               const long long* __restrict__ toff,
                                               const int32_t* __restrict__ kmax,
                                               const int32_t* __restrict__ nbr, const LJK& k,
                                               Acc& a, double* __restrict__ fx,
                                               double* __restrict__ fy, double* __restrict__ fz) {
  const int i = t * 32 + lane;
  const bool iact = i >= 0 && i < n_owned;
  // I16: 16-bit local rows, 8 steps per 128-bit chunk (else 32-bit, 4 steps)
  constexpr int CH = I16 ? 8 : 4;
  const int4* chunks =
      (I16 ? reinterpret_cast<const int4*>(reinterpret_cast<const uint16_t*>(nbr) + toff[t])
           : reinterpret_cast<const int4*>(nbr + toff[t])) +
      lane;
  const int nchunks = kmax[t] / CH;
  // the tile's whole index list towards L2 first (one bulk prefetch), so the
  // streamed chunk loads below see L2, not HBM, latency
  if (lane == 0 && nchunks > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(chunks),
                 "r"((unsigned)nchunks * 512u)
                 : "memory");
  const double4 pi = ld_pos4(pos4, iact ? i : 0);
  // Index chunks stream kStagedPrefetch chunks ahead in a register ring
  // addressed statically (the loop is unrolled by the ring size, so no
  // register move waits on an outstanding load).  Slots are evaluated in
  // batches of kStagedBatch chunks; the positions of batch b + 1 are loaded
  // while batch b is evaluated.
  constexpr int NB = I16 ? 1 : kStagedBatch, R = 2 * NB, NS = CH * NB;
  int4 ring[R];
#pragma unroll
  for (int d = 0; d < R; ++d)
    ring[d] = d < nchunks ? __ldg(chunks + (long long)d * 32) : make_int4(-1, -1, -1, -1);
  if (bar) mbar_wait(bar, 0);  // the staged rows have landed
  auto load_batch = [&](int d0, unsigned* j, double* x, double* y, double* z) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int4 v = ring[(d0 + q) % R];
      // idle slots (-1 / 0xffff) read the dummy row
      if (I16) {
        const unsigned w4[4] = {(unsigned)v.x, (unsigned)v.y, (unsigned)v.z, (unsigned)v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          j[8 * q + 2 * e] = min(w4[e] & 0xffffu, dummy);
          j[8 * q + 2 * e + 1] = min(w4[e] >> 16, dummy);
        }
      } else {
        j[4 * q + 0] = min((unsigned)v.x, dummy);
        j[4 * q + 1] = min((unsigned)v.y, dummy);
        j[4 * q + 2] = min((unsigned)v.z, dummy);
        j[4 * q + 3] = min((unsigned)v.w, dummy);
      }
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      if (STAGED) {
        x[u] = xs[j[u]];
        y[u] = xs[j[u] + ROWS];
        z[u] = xs[j[u] + 2 * ROWS];
      } else {
        x[u] = __ldg(xs + j[u]);
        y[u] = __ldg(ys + j[u]);
        z[u] = __ldg(zs + j[u]);
      }
    }
  };
  // two batch buffers used in turn (ping-pong: no register moves)
  unsigned jA[NS], jB[NS];
  double xA[NS], yA[NS], zA[NS], xB[NS], yB[NS], zB[NS];
  auto refill = [&](int d, int c) {
#pragma unroll
    for (int q = 0; q < NB; ++q)
      ring[d + q] = c + q + R < nchunks ? __ldg(chunks + (long long)(c + q + R) * 32)
                                        : make_int4(-1, -1, -1, -1);
  };
  load_batch(0, jA, xA, yA, zA);
  for (int c0 = 0; c0 < nchunks; c0 += R) {
    // batch A = chunks c0 .. c0 + NB - 1 (ring slots 0 .. NB - 1)
    refill(0, c0);
    load_batch(NB, jB, xB, yB, zB);
#pragma unroll
    for (int q = 0; q < NS / 4; ++q)
      staged_pairs4<EV, N3>(pi, xA + 4 * q, yA + 4 * q, zA + 4 * q, jA + 4 * q, hb, k, a);
    if (c0 + NB >= nchunks) break;
    // batch B = chunks c0 + NB .. c0 + R - 1 (ring slots NB .. R - 1)
    refill(NB, c0 + NB);
    load_batch(0, jA, xA, yA, zA);
#pragma unroll
    for (int q = 0; q < NS / 4; ++q)
      staged_pairs4<EV, N3>(pi, xB + 4 * q, yB + 4 * q, zB + 4 * q, jB + 4 * q, hb, k, a);
  }
  if (iact) {
    const int o = out_perm ? out_perm[i] : i;
    fx[o] = a.ax;
    fy[o] = a.ay;
    fz[o] = a.az;
  }
}

// 16 warps per SM (shared memory bounds it): up to 128 registers per thread
template <bool EV, int N3, int W, bool I16>
__global__ void __launch_bounds__(32 * W, 16 / W)
    vl_staged_kernel(int n_owned, int ntiles, int sentinel, const int32_t* __restrict__ out_perm,
                     const double* __restrict__ pos4, SoA q, const int32_t* __restrict__ groups,
                     const long long* __restrict__ toff, const int32_t* __restrict__ kmax,
                     const int32_t* __restrict__ nbr,
                     LJK k, double* __restrict__ fx,
                     double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                     lmd_stats* __restrict__ stats, int dbg) {
  constexpr int ROWS = StageRows<W>::value;
  extern __shared__ __align__(128) double st_sm[];
  double* xs = st_sm;  // y at + ROWS, z at + 2 ROWS
  __shared__ unsigned long long bar;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t* rec = groups + (long long)blockIdx.x * kGroupRec;
  const bool glob = rec[kGrpGlobal] != 0;
  const int hb = rec[kGrpHalo];
  if (!glob && !(dbg & 2)) {
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    if (threadIdx.x == 32 % (32 * W)) {
      xs[ROWS - 1] = 1.0e30;
      xs[2 * ROWS - 1] = 1.0e30;
      xs[3 * ROWS - 1] = 1.0e30;
    }
    __syncthreads();
    // warp 0: lane 0 arms the barrier, then lane l issues the three bulk
    // copies of runs l and l + 32 (one thread issuing them all serialises)
    if (threadIdx.x < 32) {
      if (lane == 0) mbar_expect_tx(&bar, (unsigned)rec[kGrpS] * 3u * 8u);
      __syncwarp();
      for (int r = lane; r < kGroupRuns; r += 32) {
        const int len = rec[kGrpLen + r];
        if (len) {
          const int st = rec[kGrpStart + r];
          const int base = st + rec[kGrpOff + r];
          bulk_g2s(xs + base, q.x + st, (unsigned)len * 8u, &bar);
          bulk_g2s(xs + ROWS + base, q.y + st, (unsigned)len * 8u, &bar);
          bulk_g2s(xs + 2 * ROWS + base, q.z + st, (unsigned)len * 8u, &bar);
        }
      }
    }
  }
  const int t = blockIdx.x * W + w;
  if (t >= ntiles) return;  // warp-uniform; no block barrier follows
  if (dbg & 1) {            // timing probe: staging only
    if (!glob && !(dbg & 2)) mbar_wait(&bar, 0);
    return;
  }
  Acc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0};
  if (glob)
    vl_staged_tile<EV, N3, ROWS, false, I16>(t, lane, n_owned, hb, (unsigned)sentinel, nullptr,
                                             out_perm, pos4,
                                        q.x, q.y, q.z, toff, kmax, nbr, k, a, fx, fy, fz);
  else
    vl_staged_tile<EV, N3, ROWS, true, I16>(t, lane, n_owned, hb, (unsigned)(ROWS - 1),
                                       (dbg & 2) ? nullptr : &bar, out_perm,
                                       pos4, xs, xs, xs, toff, kmax, nbr, k, a, fx, fy, fz);
  a.overlap |= a.hi_min == 0u;
  flush_acc(a, lane, true, EV, t, ev, stats);
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

int64_t lmd_vl_num_tiles(int64_t n_owned, int pattern) {
  return cdiv(n_owned, pattern_A(pattern));
}

static int vl_build_impl(const lmd_grid* g, double rl2, int newton3, int pattern, int64_t n_owned,
                         int32_t sentinel, const double* pos4, const int32_t* o_start,
                         const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                         int32_t cap_steps, int32_t* count, int32_t* count_half,
                         int64_t* tile_off, int32_t* kmax, int32_t* max_count, int32_t* nbr,
                         const int32_t* staged_groups, int staged_G, void* stream,
                         bool idx16 = false) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(max_count, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL || cap_steps <= 0 || cap_steps % (idx16 ? 8 : kChunk))
    return LMD_ERR_CONFIG;
  const int A = pattern_A(pattern), B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_owned, A);
  const unsigned blocks = (unsigned)cdiv(ntiles * A, 128);
  const int32_t* groups = staged_groups;
  if (idx16) {
    if (pattern != LMD_V_BY_ONE || !groups) return LMD_ERR_CONFIG;
    vl_build_kernel<LMD_V_BY_ONE, uint16_t><<<blocks, 128, 0, s>>>(
        make_gridk(g), (int)n_owned, (int)ntiles, newton3, rl2, 0xffff, pos4, o_start, o_count,
        h_start, h_count, cap_steps, count, count_half, (long long*)tile_off, kmax, max_count,
        nbr, groups, staged_G);
    LMD_CHECK_LAUNCH();
    return LMD_OK;
  }
  const int G = staged_G;
#define LMD_VLB(P)                                                                          \
  vl_build_kernel<P><<<blocks, 128, 0, s>>>(make_gridk(g), (int)n_owned, (int)ntiles, newton3, \
                                            rl2, sentinel, pos4, o_start, o_count, h_start,    \
                                            h_count, cap_steps, count, count_half,             \
                                            (long long*)tile_off, kmax, max_count, nbr,        \
                                            groups, G)
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

int lmd_vl_build(const lmd_grid* g, double rl2, int newton3, int pattern, int64_t n_owned,
                 int32_t sentinel, const double* pos4, const int32_t* o_start,
                 const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                 int32_t cap_steps, int32_t* count, int32_t* count_half, int64_t* tile_off,
                 int32_t* kmax, int32_t* max_count, int32_t* nbr, void* stream) {
  return vl_build_impl(g, rl2, newton3, pattern, n_owned, sentinel, pos4, o_start, o_count,
                       h_start, h_count, cap_steps, count, count_half, tile_off, kmax, max_count,
                       nbr, nullptr, 0, stream);
}

int lmd_vl_build_staged(const lmd_grid* g, double rl2, int newton3, int64_t n_owned,
                        const double* pos4, const int32_t* o_start, const int32_t* o_count,
                        const int32_t* h_start, const int32_t* h_count, int32_t group_size,
                        const int32_t* groups, int32_t index_bits, int32_t cap_steps,
                        int32_t* count, int32_t* count_half, int64_t* tile_off, int32_t* kmax,
                        int32_t* max_count, int32_t* nbr, void* stream) {
  if (group_size <= 0 || group_size % 32) return LMD_ERR_CONFIG;
  if (index_bits != 16 && index_bits != 32) return LMD_ERR_CONFIG;
  return vl_build_impl(g, rl2, newton3, LMD_V_BY_ONE, n_owned, -1, pos4, o_start, o_count,
                       h_start, h_count, cap_steps, count, count_half, tile_off, kmax, max_count,
                       nbr, groups, group_size, stream, index_bits == 16);
}

size_t lmd_vl_bank_smem_per_warp(int32_t cap_steps) {
  return (size_t)(64 * 16 + (size_t)cap_steps * 32) * sizeof(int32_t);
}

int lmd_vl_bank_schedule(int pattern, int64_t n_units, int32_t sentinel, int rounds,
                         int32_t cap_steps, int32_t max_steps, int32_t index_bits,
                         const int64_t* tile_off, const int32_t* kmax, int32_t* nbr,
                         void* stream) {
  if (n_units <= 0) return LMD_OK;
  if (rounds < 0 || rounds > 16 || cap_steps <= 0 || cap_steps % kChunk) return LMD_ERR_CONFIG;
  if (index_bits != 16 && index_bits != 32) return LMD_ERR_CONFIG;
  if (index_bits == 16 && (rounds != 0 || cap_steps % 8)) return LMD_ERR_CONFIG;
  const int B = pattern_B(pattern);
  const int64_t ntiles = cdiv(n_units, pattern_A(pattern));
  cudaStream_t st = (cudaStream_t)stream;
  if (rounds == 0) {
    // workspace sized by the longest tile of this list (tcap steps, <= 255)
    const int tcap = max_steps;
    if (tcap <= 0 || tcap > 255) return LMD_ERR_CONFIG;
    const size_t per = (48 * 32 + (size_t)tcap * 32) * sizeof(uint16_t);
    int nwl = (int)(72 * 1024 / per);
    nwl = nwl < 1 ? 1 : (nwl > 8 ? 8 : nwl);
    auto kern = index_bits == 16 ? vl_bank_local_kernel<true> : vl_bank_local_kernel<false>;
    cudaError_t e0 =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per * nwl));
    if (e0 != cudaSuccess) return set_cuda_error(e0);
    kern<<<(unsigned)cdiv(ntiles, nwl), 32 * nwl, per * nwl, st>>>(
        (int)ntiles, B, sentinel, tcap, (const long long*)tile_off, kmax, nbr);
    LMD_CHECK_LAUNCH();
    return LMD_OK;
  }
  const size_t per_warp = lmd_vl_bank_smem_per_warp(cap_steps);
  const size_t budget = 200 * 1024;
  if (per_warp > budget) return LMD_ERR_CONFIG;
  int nw = (int)(96 * 1024 / per_warp);
  nw = nw < 1 ? 1 : (nw > 8 ? 8 : nw);
  const size_t smem = per_warp * nw;
  cudaError_t e = cudaFuncSetAttribute(vl_bank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return set_cuda_error(e);
  vl_bank_kernel<<<(unsigned)cdiv(ntiles, nw), 32 * nw, smem, (cudaStream_t)stream>>>(
      (int)ntiles, B, sentinel, rounds, cap_steps, (const long long*)tile_off, kmax, nbr);
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

int lmd_vl_groups(const lmd_grid* g, int64_t n_owned, int32_t group_size, int32_t capacity,
                  const double* pos4, const int32_t* o_start, const int32_t* o_count,
                  const int32_t* h_start, const int32_t* h_count, int32_t* groups,
                  int32_t* smax, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(smax, 0, 2 * sizeof(int32_t), s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL || group_size <= 0 || group_size % 32 || capacity <= 0)
    return LMD_ERR_CONFIG;
  const int64_t ngroups = cdiv(n_owned, group_size);
  vl_group_kernel<<<(unsigned)cdiv(ngroups * 32, 256), 256, 0, s>>>(
      make_gridk(g), (int)n_owned, group_size, capacity, pos4, o_start, o_count, h_start, h_count,
      groups, smax);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int32_t lmd_vl_staged_capacity(int32_t group_size) {
  if (group_size != 128 && group_size != 256 && group_size != 512) return 0;
  return stage_rows(group_size) - 16;
}

int lmd_force_vl_staged(int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                        const double* pos4, const double* soa, int64_t stride, int32_t sentinel,
                        int32_t group_size, const int32_t* groups, int32_t index_bits,
                        const int64_t* tile_off, const int32_t* kmax, const int32_t* nbr,
                        const int32_t* out_perm, double* fx, double* fy, double* fz,
                        double* ev_scratch, lmd_stats* stats, void* stream) {
  if (n_owned <= 0) return LMD_OK;
  if (newton3 != 0 && newton3 != 2) return LMD_ERR_CONFIG;
  if (!soa || stride % 16 || sentinel < 0 || sentinel >= stride) return LMD_ERR_CONFIG;
  if (group_size != 128 && group_size != 256 && group_size != 512) return LMD_ERR_CONFIG;
  if (index_bits != 16 && index_bits != 32) return LMD_ERR_CONFIG;
  const bool idx16 = index_bits == 16;
  const LJK k = make_ljk(lj);
  const int64_t ntiles = cdiv(n_owned, 32);
  const int64_t ngroups = cdiv(n_owned, group_size);
  cudaStream_t s = (cudaStream_t)stream;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  const SoA q = {soa, soa + stride, soa + 2 * stride};
  const size_t smem = (size_t)stage_rows(group_size) * 3 * sizeof(double);
#define LMD_VLS(EVB, N3B, W)                                                                   \
  do {                                                                                         \
    auto kern = idx16 ? vl_staged_kernel<EVB, N3B, W, true> : vl_staged_kernel<EVB, N3B, W, false>; \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                         (int)smem);                                          \
    if (e != cudaSuccess) return set_cuda_error(e);                                            \
    kern<<<(unsigned)ngroups, 32 * W, smem, s>>>((int)n_owned, (int)ntiles, (int)sentinel,     \
                                                 out_perm, pos4, q, groups,                    \
                                                 (const long long*)tile_off, kmax, nbr, k, fx, \
                                                 fy, fz, ev_scratch, stats, (flags >> 8) & 3); \
  } while (0)
#define LMD_VLS_W(EVB, N3B)                                 \
  do {                                                      \
    switch (group_size) {                                   \
      case 128: LMD_VLS(EVB, N3B, 4); break;                \
      case 256: LMD_VLS(EVB, N3B, 8); break;                \
      case 512: LMD_VLS(EVB, N3B, 16); break;               \
      default: return LMD_ERR_CONFIG;                       \
    }                                                       \
  } while (0)
  if (ev) {
    if (newton3) LMD_VLS_W(true, 2);
    else LMD_VLS_W(true, 0);
  } else {
    if (newton3) LMD_VLS_W(false, 2);
    else LMD_VLS_W(false, 0);
  }
#undef LMD_VLS_W
#undef LMD_VLS
  LMD_CHECK_LAUNCH();
  if (ev) return reduce_ev(ev_scratch, ntiles, stats, s);
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
