// K3s/K4s: segmented, row-aligned, staged Verlet lists -- the default
// force path for the v_by_one order (sm_100a).
//
// Extension: the reference has no Verlet lists; the pair set is
// the reference's: a pair (i, j) interacts iff the reference's exact r2
// (executor.py:93-94) is below rc^2, and the lists are a superset of those
// pairs whenever they are valid (below).
//
// Layout
//   rows    positions live in HBM as (x, y, z) rows of 24 B in rebuild order:
//           the owned particles cell-sorted, then the images cell-sorted.
//           A (y, z) line of the ring-padded rc+skin cell grid holds one
//           contiguous index range of rows, each cell a sub-range of it.
//   groups  each interior line's owned particles cut into groups of up to
//           128 consecutive particles (fewer, in steps of 32, where a group
//           would stage more than kVsBudget rows; one block, 4 tiles of 32
//           lanes, thread per particle).  A group never leaves its line,
//           so its candidates are 18 row runs: for (view: owned / image, dz,
//           dy) the cells xa-1 .. xb+1 of the neighbouring line, xa .. xb
//           being the group's cells.  Both kernels copy those runs into
//           shared memory with one TMA bulk copy each (local row r at byte
//           24 r; a dummy row far away follows the last run).
//   lists   per lane, 16-bit BYTE offsets (24 * local row): three LDS.64 with
//           immediate offsets 0 / 8 / 16, no index arithmetic.  Two segments
//           per tile: entries whose build-time distance is below rc + delta
//           (inner), then the rest up to rc + skin (outer); each padded to
//           the tile's longest lane in chunks of 8 entries (one 128-bit load
//           per lane per 8 slots; chunk c of lane l at (t * cap + c) * 32 +
//           l).  A group's particles are dealt to lanes by descending inner
//           length (slot map), so a tile's lanes have similar lengths.
//           Within a segment each lane's entries follow a lane-local
//           Latin-square bank order: at step k lane l takes an entry in
//           shared-memory bank pair (l + k) & 15 (row j's x sits in bank
//           pair 3 j & 15) when it has one, so the 16 lanes of a half-warp
//           gather from distinct bank pairs.
//   validity  the outer segment covers every pair within rc while each
//           particle moved less than skin / 2 since the build (the
//           container's rebuild rule, containers.py:23-38); the inner
//           segment alone while they moved less than delta / 2 -- decided on
//           the device per launch from the largest displacement, which the
//           refresh kernel reduces (no host involvement).
//
// Force kernel per slot: 3 LDS.64, dx/dy/dz (3 DADD), r2 with FMAs (3),
// MUFU.RCP64H + 3 DFMA reciprocal, LJ with folded sigma powers (5), 3 DFMA
// accumulations = 17 FP64 instructions; the cutoff decision compares the bit
// patterns on the integer pipe and is applied by zeroing the reciprocal
// seed's high word (the reciprocal and f are then exactly 0).  The FMA r2
// differs from the reference's unfused r2 by a few ulp, so a candidate whose
// r2 has the high word of rc^2 (+-1: a band of 2^32 ulp) flags its chunk; a
// flagged chunk (warp vote, ~1e-3 of chunks) is re-decided with the exact
// expression and the accumulators corrected -- every decision is the
// reference's.
#include <algorithm>
#include <cub/cub.cuh>

#include "vl_common.cuh"

namespace lmd {

constexpr int kVsG = 128;      // particles per group (4 warps)
constexpr int kVsRec = 64;     // int32 per group record
constexpr int kVsRuns = 18;    // (view, dz, dy)
constexpr int kVsSelfRun = 4;  // view 0, dz = 0, dy = 0
constexpr int kVsMaxRows = 2704;  // 24 * (row + 15) < 65536: byte offsets (dummies incl.) fit 16 bits
// staged-row budget of a group: groups shrink (in steps of 32 particles)
// until they stage at most this many rows, so 5 blocks (44 KB each) fit an SM
constexpr int kVsBudget = 1840;
constexpr int kVsRingBytes = 32 * kVsG;   // build: 16 hits of 2 B per lane
enum : int {
  kVsP0 = 0, kVsCnt = 1, kVsS = 2, kVsHb = 3, kVsSelf = 4, kVsRow = 5, kVsXa = 6, kVsXb = 7,
  kVsStart = 8, kVsLen = 8 + kVsRuns, kVsBase = 8 + 2 * kVsRuns
};
static_assert(kVsBase + kVsRuns <= kVsRec, "group record");
// info[]: 0 max staged rows, 1 groups over capacity, 2 number of groups,
//         3 most chunks a tile needed, 4 most entries a lane needed
constexpr int kVsInfo = 8;

// ------------------------------------------------------------------- plan
// one thread per line of the ring-padded grid: "filled" starts (an empty
// cell starts where the previous one ended, so cells xa..xb of a line span
// [fs[xa], fs[xb] + count[xb])) for both views
__global__ void vls_rows_kernel(long long nrows, int t0, const int32_t* __restrict__ os,
                                const int32_t* __restrict__ oc, const int32_t* __restrict__ hs,
                                const int32_t* __restrict__ hc, int32_t* __restrict__ fso,
                                int32_t* __restrict__ fsi) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const long long base = r * t0;
#pragma unroll 1
  for (int v = 0; v < 2; ++v) {
    const int32_t* s = v ? hs : os;
    const int32_t* c = v ? hc : oc;
    int32_t* fs = v ? fsi : fso;
    int pos = 0;
    for (int x = 0; x < t0; ++x)
      if (c[base + x]) {
        pos = s[base + x];
        break;
      }
    for (int x = 0; x < t0; ++x) {
      fs[base + x] = pos;
      pos += c[base + x];
    }
  }
}

// one thread per line, twice: COUNT = the number of groups of each
// interior line (then scanned), else the group records
template <bool COUNT>
__global__ void vls_groups_kernel(long long nrows, int t0, int t1, int d0, int d1, int d2, int G,
                                  int budget, const int32_t* __restrict__ fso,
                                  const int32_t* __restrict__ oc, const int32_t* __restrict__ fsi,
                                  const int32_t* __restrict__ hc,
                                  int32_t* __restrict__ row_groups,
                                  const int32_t* __restrict__ row_gend,
                                  int32_t* __restrict__ groups, int32_t* __restrict__ info) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int y = (int)(r % t1), z = (int)(r / t1);
  const bool interior = y >= 1 && y <= d1 && z >= 1 && z <= d2;
  if (!COUNT && r == nrows - 1) info[2] = row_gend[r];
  if (!interior) {
    if (COUNT) row_groups[r] = 0;
    return;
  }
  const long long g0 = COUNT ? 0 : row_gend[r] - row_groups[r];
  const long long base = r * t0;
  const int first = fso[base], n_row = fso[base + t0 - 1] + oc[base + t0 - 1] - first;
  // staged rows of a group over cells xa .. xb (alignment included)
  auto staged = [&](int xa, int xb) {
    int S = 0;
    for (int q = 0; q < kVsRuns; ++q) {
      const int v = q / 9, dz = (q % 9) / 3 - 1, dy = q % 3 - 1;
      const int32_t* fs = v ? fsi : fso;
      const int32_t* cc = v ? hc : oc;
      const long long nb = base + (long long)t0 * (dy + (long long)t1 * dz);
      const int s = fs[nb + xa - 1], e = fs[nb + xb + 1] + cc[nb + xb + 1];
      if (e > s) S += (e - (s & ~1) + 1) & ~1;
    }
    return S;
  };
  auto cell_of = [&](int x, int p) {  // first cell from x holding particle p
    while (x < d0 && fso[base + x] + oc[base + x] <= p) ++x;
    return x;
  };
  int x = 1, p0 = first, smax = 0, over = 0, k = 0;
  while (p0 < first + n_row) {
    // up to G particles; fewer (in steps of 32) while the group would stage
    // more than budget rows (sparse lines span more cells), so that 5
    // blocks fit an SM
    const int rem = first + n_row - p0;
    const int xa = cell_of(x, p0);
    int cnt = min(G, rem), xb = cell_of(xa, p0 + cnt - 1);
    while (cnt > 32 && staged(xa, xb) > budget) {
      cnt = (cnt - 1) / 32 * 32;
      xb = cell_of(xa, p0 + cnt - 1);
    }
    if (COUNT) {
      p0 += cnt;
      x = xb;
      ++k;
      continue;
    }
    int32_t* rec = groups + (g0 + k) * kVsRec;
    int S = 0, hb = 0;
    for (int q = 0; q < kVsRuns; ++q) {
      const int v = q / 9, dz = (q % 9) / 3 - 1, dy = q % 3 - 1;
      const int32_t* fs = v ? fsi : fso;
      const int32_t* cc = v ? hc : oc;
      const long long nb = base + (long long)t0 * (dy + (long long)t1 * dz);
      const int s = fs[nb + xa - 1], e = fs[nb + xb + 1] + cc[nb + xb + 1];
      int st = 0, ln = 0;
      if (e > s) {
        st = s & ~1;  // even rows: 16-B aligned bulk copies (24 B rows)
        ln = (e - st + 1) & ~1;
      }
      if (q == 9) hb = S;
      rec[kVsStart + q] = st;
      rec[kVsLen + q] = ln;
      rec[kVsBase + q] = S;
      S += ln;
    }
    rec[kVsP0] = p0;
    rec[kVsCnt] = cnt;
    rec[kVsS] = S;
    rec[kVsHb] = hb;
    rec[kVsSelf] = p0 - rec[kVsStart + kVsSelfRun] + rec[kVsBase + kVsSelfRun];
    rec[kVsRow] = (int)r;
    rec[kVsXa] = xa;
    rec[kVsXb] = xb;
    smax = max(smax, S);
    over += S > kVsMaxRows ? 1 : 0;
    p0 += cnt;
    x = xb;
    ++k;
  }
  if (COUNT) {
    row_groups[r] = k;
    return;
  }
  atomicMax(info, smax);
  if (over) atomicAdd(info + 1, over);
}

// warp 0 copies the group's runs into shared memory (one bulk copy per run;
// lane 0 arms the barrier with the byte count first)
__device__ __forceinline__ void vls_stage(const int32_t* __restrict__ rec,
                                          const double* __restrict__ rows, double* sm,
                                          unsigned long long* bar) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) mbar_expect_tx(bar, (unsigned)rec[kVsS] * 24u);
    __syncwarp();
    if (lane < kVsRuns) {
      const int len = rec[kVsLen + lane];
      if (len)
        bulk_g2s(sm + 3 * rec[kVsBase + lane], rows + 3LL * rec[kVsStart + lane],
                 (unsigned)len * 24u, bar);
    }
  }
}

// 16 dummy rows far away, one per shared-memory bank pair, from row D = S
// rounded up to 16 (row D + t sits in bank pair 3 t & 15); written before the
// block barrier that precedes the staging
__device__ __forceinline__ void vls_dummies(const int32_t* __restrict__ rec, double* sm) {
  if (threadIdx.x >= 32 && threadIdx.x < 48) {
    const int D = (rec[kVsS] + 15) & ~15;
    const int r = D + (int)threadIdx.x - 32;
    sm[3 * r] = 1.0e30;
    sm[3 * r + 1] = 1.0e30;
    sm[3 * r + 2] = 1.0e30;
  }
}

// packed FP32 pairs (sm_100: FADD2 / FMUL2 / FFMA2), low word = first element
__device__ __forceinline__ unsigned long long f32x2_pack(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ unsigned long long f32x2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f32x2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f32x2_fma(unsigned long long a, unsigned long long b,
                                                        unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// exact class of local row j for a particle at (px, py, pz): bit 0 = within
// rl (the reference's unfused r2), bit 1 = beyond the inner radius
__device__ __noinline__ int vls_exact_class(const double* __restrict__ rows, const int* run_st,
                                            const int* run_rb, int j, double px, double py,
                                            double pz, double rin2, double rl2) {
  int gq = 0;
  for (int q = 1; q < kVsRuns; ++q) gq += j >= run_rb[q] ? 1 : 0;
  const long long gj = 3LL * (j - run_rb[gq] + run_st[gq]);
  const double r2 = r2_exact(px - rows[gj], py - rows[gj + 1], pz - rows[gj + 2]);
  return (r2 < rl2 ? 1 : 0) | (r2 < rin2 ? 0 : 2);
}

// ------------------------------------------------------------------ build
// One block per group, thread per particle, 5 blocks per SM (shared memory:
// the FP32 copies of the group's rows, later the lanes' sorted hits).
//  1. walk: every lane of a warp walks the union of the warp's candidate
//     ranges of a run (warp-uniform loop, broadcast shared-memory loads) and
//     keeps the candidates of its own 3 cells with r2 < rl^2 (the
//     reference's exact expression), inner (r2 < rin^2) or outer; hits are
//     appended to the lane's private stretch of the group's list area in
//     global memory (still unused: the lists are written in step 3) and
//     counted per (segment, bank pair) in shared memory.
//  2. counting sort of each lane's hits by (segment, bank pair) into the
//     shared memory the staged rows occupied.
//  3. the group's particles are ranked by inner length (the slot map) and
//     each emits its segments in its new lane's Latin-square bank order.
template <int MODE>   // 0: plain entry order, 1: bank order, 2: the walk alone
__global__ void __launch_bounds__(kVsG, 5)
    vls_build_kernel(int t0, int t1, const int32_t* __restrict__ groups,
                     const int32_t* __restrict__ info_in, const double* __restrict__ rows,
                     const int32_t* __restrict__ fso, const int32_t* __restrict__ oc,
                     const int32_t* __restrict__ fsi, const int32_t* __restrict__ hc,
                     double rin2, double rl2, int area_bytes, int cap_chunks, int cap_ent,
                     int4* __restrict__ nbr, int32_t* __restrict__ segc,
                     uint8_t* __restrict__ slotmap, int32_t* __restrict__ count,
                     int32_t* __restrict__ count_half, int32_t* __restrict__ info) {
  constexpr bool BANK = MODE == 1;
  extern __shared__ __align__(128) double sm_b[];
  uint16_t* sorted = reinterpret_cast<uint16_t*>(sm_b);    // hits by bucket (steps 2-3)
  // after the area: a 16-entry ring per lane for the walk's hits, then (bank
  // order only) the bucket counters
  uint8_t* ring_area = reinterpret_cast<uint8_t*>(sm_b) + area_bytes;   // [128][32 B]
  uint8_t* cnt = ring_area + kVsRingBytes;                        // [32 buckets][128]
  uint8_t* pos = cnt + 32 * kVsG;                                 // [32 buckets][128]
  __shared__ int n_in_sm[kVsG], n_out_sm[kVsG], slot_sm[kVsG];
  __shared__ int run_st[kVsRuns], run_rb[kVsRuns + 1];
  __shared__ int bad_sm;
  const int g = blockIdx.x;
  if (g >= info_in[2]) return;
  const int32_t* rec = groups + (long long)g * kVsRec;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < kVsRuns) {
    run_st[tid] = rec[kVsStart + tid];
    run_rb[tid] = rec[kVsBase + tid];
  }
  if (tid == kVsRuns) run_rb[kVsRuns] = rec[kVsS];
  if (tid == 32) bad_sm = 0;
  if (BANK) {
#pragma unroll
    for (int b = 0; b < 32; ++b) cnt[b * kVsG + tid] = 0;
  }
  const int cnt_p = rec[kVsCnt], p0 = rec[kVsP0];
  const bool active = tid < cnt_p;
  const int p = p0 + tid;
  const int irow = rec[kVsSelf] + tid;
  const long long rowbase = (long long)rec[kVsRow] * t0;
  // this lane's stretch of its (original) tile's list area: the hits
  uint16_t* hits = reinterpret_cast<uint16_t*>(nbr + ((long long)(g * (kVsG / 32) + w) *
                                                      cap_chunks) * 32) + lane * cap_ent;
  // the lane's cell: cell ends are non-decreasing along the line, so the
  // cell is xa + the number of cells ending at or before p (independent
  // loads, no dependent chain)
  int cx = rec[kVsXa];
  if (active) {
    const int xa = cx, xb = rec[kVsXb];
#pragma unroll 4
    for (int x = xa; x < xb; ++x) cx += p >= fso[rowbase + x] + oc[rowbase + x] ? 1 : 0;
  }
  // the lane's candidate range in every run (local rows, l0 | l1 << 16),
  // loaded up front: the table reads overlap the staging copy instead of
  // stalling every run of the walk
  unsigned lb[kVsRuns];
#pragma unroll
  for (int q = 0; q < kVsRuns; ++q) {
    const int v = q / 9, dz = (q % 9) / 3 - 1, dy = q % 3 - 1;
    lb[q] = 0u;
    if (active && rec[kVsLen + q]) {
      const int32_t* fs = v ? fsi : fso;
      const int32_t* cc = v ? hc : oc;
      const long long nb = rowbase + (long long)t0 * (dy + (long long)t1 * dz);
      const int off = rec[kVsBase + q] - rec[kVsStart + q];
      const int l0 = fs[nb + cx - 1] + off;
      const int l1 = fs[nb + cx + 1] + cc[nb + cx + 1] + off;
      lb[q] = (unsigned)l0 | ((unsigned)l1 << 16);
    }
  }
  double px = -1.0e30, py = -1.0e30, pz = -1.0e30;
  if (active) {   // owned rows are the first rows, in rebuild order
    px = rows[3LL * p];
    py = rows[3LL * p + 1];
    pz = rows[3LL * p + 2];
  }
  // FP32 copies of the group's rows (the 18 runs, straight from global
  // memory) relative to the group's first particle, two rows at a time:
  // local rows 2 q and 2 q + 1 as {x, x', y, y', z, z'} at byte 24 q, so one
  // LDS.64 per axis feeds the packed FP32 arithmetic of the walk
  const int S = rec[kVsS];
  const double ox = rows[3LL * p0], oy = rows[3LL * p0 + 1], oz = rows[3LL * p0 + 2];
  float* xf = reinterpret_cast<float*>(sm_b);
  float rmax = 0.f;
  __syncthreads();   // run table
#pragma unroll 4
  for (int j = tid; j < S; j += kVsG) {
    int q = 0;
#pragma unroll
    for (int r = 1; r < kVsRuns; ++r) q += j >= run_rb[r] ? 1 : 0;   // bases are non-decreasing
    const long long gj = 3LL * (run_st[q] + (j - run_rb[q]));
    const float a = (float)(rows[gj] - ox), b = (float)(rows[gj + 1] - oy),
                c = (float)(rows[gj + 2] - oz);
    float* o = xf + 6 * (j >> 1) + (j & 1);
    o[0] = a;
    o[2] = b;
    o[4] = c;
    rmax = fmaxf(rmax, fmaxf(fabsf(a), fmaxf(fabsf(b), fabsf(c))));
  }
  // decision bounds: |FP32 r2 - exact r2| <= err for coordinates up to
  // rmax from the origin (conversion: 2^-24 rmax per coordinate, twice per
  // difference; arithmetic: a few ulp of rl^2); outside [rl2 - err, rl2 +
  // err) the FP32 decision is the exact one, inside the candidate is
  // flagged and decided exactly (FP64 rows in global memory) in step 2
  __shared__ float rmax_sm;
  if (tid == 0) rmax_sm = 0.f;
  __syncthreads();
  atomicMax(reinterpret_cast<int*>(&rmax_sm), __float_as_int(rmax));  // rmax >= 0
  __syncthreads();
  const double rl = sqrt(rl2);
  const double err = 8.0 * 5.9604644775390625e-8 * ((double)rmax_sm + 4.0) * 2.0 * rl +
                     8.0 * 5.9604644775390625e-8 * rl2;
  const float rl2_lo = (float)(rl2 - err), rl2_hi = (float)(rl2 + err);
  const float rin2_hi = (float)(rin2 + err);
  const float pxf = (float)(px - ox), pyf = (float)(py - oy), pzf = (float)(pz - oz);
  const unsigned long long pxx = f32x2_pack(pxf, pxf), pyy = f32x2_pack(pyf, pyf),
                           pzz = f32x2_pack(pzf, pzf);
  // 1. walk.  No per-candidate range or self test: a candidate outside the
  //    lane's own 3 cells is farther than rl (cells are at least rl wide), so
  //    the distance test alone decides; the lane's own row (distance 0) is
  //    appended like a hit and dropped in step 2, which also classifies the
  //    entries (inner / outer / in the FP32 band around rl).
  unsigned n_ent = 0;  // entries appended (own row and band candidates included)
  unsigned n_fl = 0;   // entries already flushed to the lane's stretch (multiple of 8)
  // Hits go through a 16-entry ring in shared memory and reach the lane's
  // stretch 8 at a time (one 16-B store): a 2-B global store per hit is one
  // L2 request each -- 1.3e9 per build at 16.8M particles, and the L2 request
  // rate, not the instruction count, then bounds the walk.
  const unsigned ring = smem_u32(ring_area + tid * 32);
  uint4* const stretch = reinterpret_cast<uint4*>(hits);
  auto test = [&](int j, float r2) {
    // appended (predicated store and increment, no branch) when r2 < rl2_hi;
    // classified in step 2
    const unsigned at = ring + ((n_ent & 15u) << 1);
    asm volatile(
        "{\n .reg .pred p;\n"
        " setp.lt.f32 p, %3, %4;\n"
        " @p st.shared.u16 [%1], %2;\n"
        " @p add.u32 %0, %0, 1;\n}"
        : "+r"(n_ent)
        : "r"(at), "h"((unsigned short)j), "f"(r2), "f"(rl2_hi)
        : "memory");
  };
  // called at least every 9 candidates (a lane holds at most 7 unflushed
  // entries afterwards, so the ring never wraps onto them)
  auto flush = [&](bool all) {
    while (n_fl + 8u <= n_ent || (all && n_fl < n_ent)) {
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "r"(ring + ((n_fl & 15u) << 1))
                   : "memory");
      if (n_fl + 8u <= (unsigned)cap_ent) stretch[n_fl >> 3] = v;
      n_fl += 8u;
    }
  };
  // rows jp (even) and jp + 1 with packed FP32 arithmetic
  auto pair = [&](int jp, bool m0, bool m1) {
    const unsigned long long* q = reinterpret_cast<const unsigned long long*>(xf + 3 * jp);
    const unsigned long long dx = f32x2_sub(pxx, q[0]), dy = f32x2_sub(pyy, q[1]),
                             dz = f32x2_sub(pzz, q[2]);
    const unsigned long long r = f32x2_fma(dz, dz, f32x2_fma(dy, dy, f32x2_mul(dx, dx)));
    if (m0) test(jp, __uint_as_float((unsigned)r));
    if (m1) test(jp + 1, __uint_as_float((unsigned)(r >> 32)));
  };
  unsigned lbn = lb[0];
#pragma unroll 1   // (lb[] lives in local memory: one L1 read per run; unrolling
                   // 18 copies of the walk overflows the instruction cache)
  for (int q = 0; q < kVsRuns; ++q) {
    const unsigned lbq = lbn;
    lbn = lb[min(q + 1, kVsRuns - 1)];   // one run ahead
    const int l0 = (int)(lbq & 0xffffu), l1 = (int)(lbq >> 16);
    // the union of the warp's candidate ranges: real rows of this run only
    // (the even-alignment rows around a run are never tested -- they could
    // be candidates of another run)
    const int u0 = __reduce_min_sync(0xffffffffu, l1 > l0 ? l0 : 0x7fffffff);
    const int u1 = __reduce_max_sync(0xffffffffu, l1 > l0 ? l1 : 0);
    if (u1 <= u0) continue;
    int j = u0;
    if (j & 1) {
      pair(j - 1, false, true);
      ++j;
    }
#pragma unroll 1
    for (; j + 7 < u1; j += 8) {
      pair(j, true, true);
      pair(j + 2, true, true);
      pair(j + 4, true, true);
      pair(j + 6, true, true);
      flush(false);
    }
    for (; j + 1 < u1; j += 2) pair(j, true, true);
    if (j < u1) pair(j, true, false);
    flush(false);
  }
  flush(true);
  const int ent_max = __reduce_max_sync(0xffffffffu, (int)n_ent);
  // (a plain read first: the running maximum settles after a few blocks, and
  // one same-address atomic per warp is what this avoids)
  if (lane == 0 && ent_max > *reinterpret_cast<volatile int32_t*>(info + 4))
    atomicMax(info + 4, ent_max);
  if (MODE == 2) {
    // the walk alone (the one-shot force phase evaluates the raw hits from
    // the FP64 rows, lmd_vls_direct): the lane's raw count, then done
    if (active) count[p] = (int)n_ent;
    return;
  }
  // a lane without room makes the whole build void (the host retries with
  // the observed maximum): flagged here, read by every warp after step 2
  const bool room = ent_max <= cap_ent;
  if (lane == 0 && !room) atomicOr(&bad_sm, 1);
  // 2. the lane's hits are read back (8 at a time; a lane's stretch is 16-B
  //    aligned: cap_ent % 8 == 0) and classified with the walk's FP32 r2
  //    (the same arithmetic, bit for bit): the own row is dropped, band
  //    candidates are decided by the reference's exact r2 from the FP64 rows,
  //    entries beyond the inner radius get bit 14, and the half list length
  //    is counted (local rows follow the global order: j > own row <=> a
  //    later owned particle or an image).  The classified entries go back to
  //    the stretch (dropped ones as 0xffff); then a counting sort by
  //    (segment, bank pair) into shared memory (bucket starts -> pos; a
  //    lane's counts stay below 256: cap_ent <= 255)
  uint16_t* mine = sorted + tid * cap_ent;
  uint4* hits8 = reinterpret_cast<uint4*>(hits);
  auto hit_at = [](const uint4& v, int e) {
    const unsigned w = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
    return (e & 1) ? w >> 16 : w & 0xffffu;
  };
  int n_in = 0, n_half = 0, n_tot = 0;
  if (room) {
    uint4 vn = hits8[0];   // one chunk ahead (cap_ent >= 8)
    for (int e0 = 0; e0 < (int)n_ent; e0 += 8) {
      const uint4 v = vn;
      if (e0 + 8 < (int)n_ent) vn = hits8[(e0 >> 3) + 1];
      unsigned o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        unsigned h = 0xffffu;
        if (e0 + e < (int)n_ent) {
          const int j = (int)hit_at(v, e);
          const float* r = xf + 6 * (j >> 1) + (j & 1);
          const float dx = pxf - r[0], dy = pyf - r[2], dz = pzf - r[4];
          const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          bool keep = j != irow;
          bool outer = r2f >= rin2_hi;
          if (r2f >= rl2_lo) {   // rare: the exact decision (out of line)
            const int d = vls_exact_class(rows, run_st, run_rb, j, px, py, pz, rin2, rl2);
            keep = keep && (d & 1);
            outer = (d & 2) != 0;
          }
          if (keep) {
            h = (unsigned)j | (outer ? 0x4000u : 0u);
            n_tot += 1;
            n_in += outer ? 0 : 1;
            n_half += j > irow ? 1 : 0;
            if (BANK) {
              const int bk = (outer ? 16 : 0) + ((3 * j) & 15);
              cnt[bk * kVsG + tid] = (uint8_t)(cnt[bk * kVsG + tid] + 1);
            }
          }
        }
        o[e >> 1] |= h << (16 * (e & 1));
      }
      hits8[e0 >> 3] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();  // every lane has read the FP32 rows: the sort may overwrite them
  const bool ok = bad_sm == 0;
  if (ok && BANK) {
    int acc = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      pos[b * kVsG + tid] = (uint8_t)acc;
      acc += cnt[b * kVsG + tid];
    }
    uint4 vn = hits8[0];
    for (int e0 = 0; e0 < (int)n_ent; e0 += 8) {
      const uint4 v = vn;
      if (e0 + 8 < (int)n_ent) vn = hits8[(e0 >> 3) + 1];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e0 + e < (int)n_ent) {
          const unsigned h = hit_at(v, e);
          if (h != 0xffffu) {
            const unsigned j = h & 0x3fffu;
            const int bk = ((h >> 14) << 4) + ((3 * j) & 15);
            const int at = pos[bk * kVsG + tid];
            mine[at] = (uint16_t)j;
            pos[bk * kVsG + tid] = (uint8_t)(at + 1);
          }
        }
      }
    }
    // pos[b] = end of bucket b; the emission takes from start = end - cnt
  }
  if (ok && !BANK) {
    // plain order: a stable partition into [inner | outer], two running
    // positions in registers
    int at_in = 0, at_out = n_in;
    uint4 vn = hits8[0];
    for (int e0 = 0; e0 < (int)n_ent; e0 += 8) {
      const uint4 v = vn;
      if (e0 + 8 < (int)n_ent) vn = hits8[(e0 >> 3) + 1];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e0 + e < (int)n_ent) {
          const unsigned h = hit_at(v, e);
          if (h != 0xffffu) {
            const bool outer = (h >> 14) != 0;
            mine[outer ? at_out : at_in] = (uint16_t)(h & 0x3fffu);
            at_in += outer ? 0 : 1;
            at_out += outer ? 1 : 0;
          }
        }
      }
    }
  }
  const int n_out = n_tot - n_in;
  if (active) {
    count[p] = n_tot;
    count_half[p] = n_half;
  }
  // 3. deal the group's particles to lanes by descending inner length (ties:
  //    thread order); inactive threads rank last
  const int key = active ? n_in : -1;
  n_in_sm[tid] = key;
  n_out_sm[tid] = n_out;
  __syncthreads();
  int rank = 0;
#pragma unroll 8
  for (int o = 0; o < kVsG; ++o) {
    const int ko = n_in_sm[o];
    rank += (ko > key || (ko == key && o < tid)) ? 1 : 0;
  }
  slot_sm[rank] = active ? tid : 0xff;
  slotmap[(long long)g * kVsG + rank] = active ? (uint8_t)tid : (uint8_t)0xff;
  __syncthreads();  // every lane has read its hits: the list area is free
  // 4. emission, one warp per tile (its lanes = the particles dealt to it):
  //    lane-local Latin-square bank order -- at step k the lane takes an
  //    entry from bucket (bank pair) (lane + k) & 15 if it has one, else the
  //    next non-empty bucket in rotation; past its list it takes the dummy
  //    row of bank (lane + k) & 15 (16 dummies, one per bank pair, from row
  //    D = S rounded up to 16), so padding never conflicts within a
  //    half-warp.  (A warp-cooperative matching of lanes to free banks per
  //    step cut the conflicts by a quarter but not the force time: measured,
  //    DESIGN.md.)
  const int src = slot_sm[tid];
  const bool live = src != 0xff;
  const int t = g * (kVsG / 32) + w;
  const unsigned dbase = (unsigned)((S + 15) & ~15);
  const uint16_t* hits_of = sorted + (live ? src : 0) * cap_ent;
  int chunk = 0;
#pragma unroll 1
  for (int seg = 0; seg < 2; ++seg) {
    const int ns = live ? (seg ? n_out_sm[src] : n_in_sm[src]) : 0;
    const int C = (__reduce_max_sync(0xffffffffu, ns) + 7) >> 3;
    unsigned m = 0;
    if (BANK && ok && live) {
#pragma unroll
      for (int b = 0; b < 16; ++b)
        m |= (cnt[(seg * 16 + b) * kVsG + src] != 0 ? 1u : 0u) << b;
    }
    // plain order: the segment's entries as the walk found them
    const uint16_t* seg_of = hits_of + (seg ? (live ? n_in_sm[src] : 0) : 0);
#pragma unroll 1
    for (int c = 0; c < C; ++c) {
      unsigned wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = c * 8 + e;
        const int d = (lane + k) & 15;
        unsigned val = (dbase + (unsigned)((11 * d) & 15)) * 24u;   // dummy of bank d
        if (BANK) {
          if (k < ns && m) {
            const unsigned rot = ((m >> d) | (m << (16 - d))) & 0xffffu;
            const int b = (d + __ffs(rot) - 1) & 15;
            const int bi = (seg * 16 + b) * kVsG + src;
            const int left = cnt[bi];
            val = (unsigned)hits_of[pos[bi] - left] * 24u;
            cnt[bi] = (uint8_t)(left - 1);
            if (left == 1) m &= ~(1u << b);
          }
        } else if (ok && k < ns) {
          val = (unsigned)seg_of[k] * 24u;
        }
        wv[e >> 1] |= val << (16 * (e & 1));
      }
      if (chunk + c < cap_chunks)
        nbr[((long long)t * cap_chunks + chunk + c) * 32 + lane] =
            make_int4((int)wv[0], (int)wv[1], (int)wv[2], (int)wv[3]);
    }
    if (lane == 0) segc[2 * t + seg] = C;
    chunk += C;
  }
  if (lane == 0 && chunk > *reinterpret_cast<volatile int32_t*>(info + 3))
    atomicMax(info + 3, chunk);
}

// ------------------------------------------------------------------ force
struct VsAcc {
  double ax, ay, az, e, v;
  int pairs, halo;
};

// the LJ force scalar of one slot with the FMA r2 (also used by the rare
// correction path, so a correction removes exactly what was added)
__device__ __forceinline__ double vs_force_scalar(double r2, bool hit, const LJK& k, double& u3) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  // outside the cutoff the seed's high word (its low word is 0) is zeroed:
  // y = 0, so ur = 0 and f = 0 exactly (one SEL, in place)
  y = __hiloint2double(hit ? __double2hiint(y) : 0, __double2loint(y));
  double e = fma(-r2, y, 1.0);
  e = fma(e, e, e);
  const double ur = fma(y, e, y);
  const double u2 = ur * ur;
  u3 = u2 * ur;
  return (u2 * u2) * fma(k.c12, u3, -k.c6);
}

// FMA-r2 decision: the high words alone (r2 >= 0); every r2 whose high
// word is within 1 of rc^2's (including all ties of the high word) flags the
// chunk for the exact re-decision
__device__ __forceinline__ bool vs_fast_hit(double r2, unsigned band_hi) {
  return (unsigned)__double2hiint(r2) < band_hi;
}

template <bool EV, int N3>
__device__ __forceinline__ void vs_slot(double px, double py, double pz, double xj, double yj,
                                        double zj, unsigned off, unsigned hb_off,
                                        unsigned band_hi, const LJK& k, VsAcc& a, bool& band) {
  const double dx = px - xj, dy = py - yj, dz = pz - zj;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const unsigned hi = (unsigned)__double2hiint(r2);
  const bool hit = hi < band_hi;
  band |= (hi - (band_hi - 1u)) < 3u;
  double u3;
  const double f = vs_force_scalar(r2, hit, k, u3);
  a.ax = fma(f, dx, a.ax);
  a.ay = fma(f, dy, a.ay);
  a.az = fma(f, dz, a.az);
  if (EV) {
    a.e = fma(0.5 * u3, fma(k.e12, u3, -k.e6), a.e);
    a.v = fma(0.5 * f, r2, a.v);
  }
  // predicated increments (one instruction each)
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p add.s32 %0, %0, 1;\n}"
      : "+r"(a.pairs)
      : "r"((unsigned)hit));
  if (N3 == 2) a.halo += (hit && off >= hb_off) ? 1 : 0;
}

// exact re-decision of one slot of a flagged chunk: the reference's unfused
// r2 decides; where it disagrees with the FMA decision the slot's
// contribution is added or removed
template <bool EV, int N3>
__device__ __forceinline__ void vs_fix_slot(double px, double py, double pz, double xj, double yj,
                                            double zj, unsigned off, unsigned hb_off,
                                            const LJK& k, VsAcc& a) {
  const double dx = px - xj, dy = py - yj, dz = pz - zj;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const bool fast = vs_fast_hit(r2, (unsigned)(k.rc2_bits >> 32));
  const bool exact = r2_exact(dx, dy, dz) < k.rc2;
  if (fast == exact) return;
  double u3;
  const double f = vs_force_scalar(r2, true, k, u3);
  const double sgn = exact ? 1.0 : -1.0;
  a.ax = fma(sgn * f, dx, a.ax);
  a.ay = fma(sgn * f, dy, a.ay);
  a.az = fma(sgn * f, dz, a.az);
  if (EV) {
    a.e = fma(sgn * 0.5 * u3, fma(k.e12, u3, -k.e6), a.e);
    a.v = fma(sgn * 0.5 * f, r2, a.v);
  }
  a.pairs += exact ? 1 : -1;
  if (N3 == 2 && off >= hb_off) a.halo += exact ? 1 : -1;
}

// 16-bit entry u (compile-time) of a packed chunk
__device__ __forceinline__ unsigned vs_off(const int4& w, int u) {
  const unsigned v = (unsigned)(u < 2 ? w.x : u < 4 ? w.y : u < 6 ? w.z : w.w);
  return (u & 1) ? v >> 16 : v & 0xffffu;
}
// the same for a run-time u (rare path)
__device__ __forceinline__ unsigned vs_off_dyn(const int4& w, int u) {
  const int q = u >> 1;
  const unsigned v = (unsigned)(q == 0 ? w.x : q == 1 ? w.y : q == 2 ? w.z : w.w);
  return (u & 1) ? v >> 16 : v & 0xffffu;
}

__device__ __forceinline__ double lds_at(const double* sm, unsigned off, int axis) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(sm) + off + 8 * axis);
}

template <int OCC, bool EV, int N3>
__global__ void __launch_bounds__(kVsG, OCC)
    vls_force_kernel(const int32_t* __restrict__ groups, const int32_t* __restrict__ gindex,
                     const double* __restrict__ rows, const int4* __restrict__ nbr,
                     const int32_t* __restrict__ segc, const uint8_t* __restrict__ slotmap,
                     int cap_chunks, const unsigned long long* __restrict__ disp,
                     unsigned long long half_delta2_bits, LJK k,
                     const int32_t* __restrict__ out_perm, double* __restrict__ fx,
                     double* __restrict__ fy, double* __restrict__ fz, double* __restrict__ ev,
                     lmd_stats* __restrict__ stats, int n_groups, int pf_dist) {
  extern __shared__ __align__(128) double sm_f[];
  double* xs = sm_f;
  __shared__ unsigned long long bar;
  // one block per group (grid = number of groups); every global load the
  // block needs is independent of the others and issued up front, so the
  // start costs one round trip plus the staging copy
  const int g = gindex ? __ldg(gindex + blockIdx.x) : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int t = g * (kVsG / 32) + w;
  const int32_t* rec = groups + (long long)g * kVsRec;
  const int4* chunks = nbr + (long long)t * cap_chunks * 32 + lane;
  int4 r0 = __ldg(chunks);  // cap_chunks >= 2: always addressable
  int4 r1 = __ldg(chunks + 32);
  const int src = slotmap[(long long)g * kVsG + tid];
  const int self = __ldg(rec + kVsSelf), hb = __ldg(rec + kVsHb);
  const int c_in = __ldg(segc + 2 * t), c_out = __ldg(segc + 2 * t + 1);
  // inner segment alone while every particle moved less than delta / 2
  const bool outer = disp == nullptr || *disp >= half_delta2_bits;
  if (tid == 0) mbar_init(&bar, 1);
  vls_dummies(rec, xs);
  __syncthreads();
  vls_stage(rec, rows, xs, &bar);
  // warm the L2 with the rows of the group that starts about one wave of
  // blocks later, so its staging copies hit the L2 rather than HBM
  if (!gindex && pf_dist > 0 && tid >= 32 && tid < 32 + kVsRuns &&
      (int)blockIdx.x + pf_dist < n_groups) {
    const int32_t* nrec = groups + (long long)(blockIdx.x + pf_dist) * kVsRec;
    const int q = tid - 32, len = __ldg(nrec + kVsLen + q);
    if (len)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       rows + 3LL * __ldg(nrec + kVsStart + q)),
                   "r"((unsigned)len * 24u)
                   : "memory");
  }
  const int nch = c_in + (outer ? c_out : 0);
  if (lane == 0 && nch > 2)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(chunks + 64),
                 "r"((unsigned)(nch - 2) * 512u)
                 : "memory");
  const bool active = src != 0xff;
  const int irow = self + src;
  const unsigned hb_off = (unsigned)hb * 24u;
  const unsigned band_hi = (unsigned)(k.rc2_bits >> 32);
  mbar_wait(&bar, 0);
  double px = -1.0e30, py = -1.0e30, pz = -1.0e30;
  if (active) {
    px = xs[3 * irow];
    py = xs[3 * irow + 1];
    pz = xs[3 * irow + 2];
  }
  VsAcc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0};
  // Pair pipeline: the positions of the next 2 slots are loaded while the
  // current 2 are evaluated (registers, not ILP, are the scarce resource);
  // a chunk (8 slots) stays packed in one int4 and index chunk c + 2 is
  // fetched while chunk c is evaluated.  The band flags of a chunk are voted
  // on once; a flagged chunk is re-decided exactly from shared memory.
  double xP[2], yP[2], zP[2], xQ[2], yQ[2], zQ[2];
  auto load2 = [&](const int4& cw, int u0, double* x, double* y, double* z) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned o = vs_off(cw, u0 + u);
      x[u] = lds_at(xs, o, 0);
      y[u] = lds_at(xs, o, 1);
      z[u] = lds_at(xs, o, 2);
    }
  };
  auto eval2 = [&](const int4& cw, int u0, const double* x, const double* y, const double* z,
                   bool& band) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
      vs_slot<EV, N3>(px, py, pz, x[u], y[u], z[u], vs_off(cw, u0 + u), hb_off, band_hi, k, a,
                      band);
  };
  auto fix = [&](const int4& cw) {
#pragma unroll 1
    for (int u = 0; u < 8; ++u) {
      const unsigned o = vs_off_dyn(cw, u);
      vs_fix_slot<EV, N3>(px, py, pz, lds_at(xs, o, 0), lds_at(xs, o, 1), lds_at(xs, o, 2), o,
                          hb_off, k, a);
    }
  };
  // one chunk: cw = chunk c (its first pair already loaded into P), nw =
  // chunk c + 1, fw receives chunk c + 2
  auto chunk = [&](const int4& cw, const int4& nw, int4& fw, int c) {
    // (clamped to the launch's last chunk: the two chunks past it belong to
    // the outer segment or the padding and would be fetched for nothing)
    fw = __ldg(chunks + (long long)min(c + 2, nch - 1) * 32);
    bool band = false;
    load2(cw, 2, xQ, yQ, zQ);
    eval2(cw, 0, xP, yP, zP, band);
    load2(cw, 4, xP, yP, zP);
    eval2(cw, 2, xQ, yQ, zQ, band);
    load2(cw, 6, xQ, yQ, zQ);
    eval2(cw, 4, xP, yP, zP, band);
    const bool more = c + 1 < nch;
    if (more) load2(nw, 0, xP, yP, zP);
    eval2(cw, 6, xQ, yQ, zQ, band);
    if (__any_sync(0xffffffffu, band)) fix(cw);
    return more;
  };
  int4 r2;
  if (nch > 0) load2(r0, 0, xP, yP, zP);
#pragma unroll 1
  for (int c = 0; c < nch; c += 3) {
    if (!chunk(r0, r1, r2, c)) break;
    if (!chunk(r1, r2, r0, c + 1)) break;
    if (!chunk(r2, r0, r1, c + 2)) break;
  }
  int overlap = 0;
  if (active && !(isfinite(a.ax) && isfinite(a.ay) && isfinite(a.az))) {
    // rare: find an exactly coincident in-list pair (the numba -1 sentinel)
    for (int c = 0; c < nch && !overlap; ++c) {
      const int4 cw = __ldg(chunks + (long long)c * 32);
      for (int u = 0; u < 8; ++u) {
        const unsigned o = vs_off_dyn(cw, u);
        if (r2_exact(px - lds_at(xs, o, 0), py - lds_at(xs, o, 1), pz - lds_at(xs, o, 2)) == 0.0)
          overlap = 1;
      }
    }
  }
  if (active) {
    const int p = rec[kVsP0] + src;
    const int o = out_perm ? out_perm[p] : p;
    fx[o] = a.ax;
    fy[o] = a.ay;
    fz[o] = a.az;
  }
  // statistics: per-warp atomics (block-level accumulation in shared memory
  // before the global atomics was measured 1 % slower: 1.789 vs 1.771 ms)
  Acc fl = {0.0, 0.0, 0.0, a.e, a.v, a.pairs, overlap, a.halo};
  flush_acc(fl, lane, true, EV, t, ev, stats);
}

// ------------------------------------------------------------ direct (K4d)
// One force phase without lists, for a structure that is used once
// (force_phase on a temporary container, driver.py:107-129), in two kernels:
// the list build's walk alone (vls_build_kernel<2>: packed FP32, every
// candidate within rl + the FP32 error bound appended to the lane's stretch
// of a scratch area, the own row included), then this kernel: one block per
// group stages the group's FP64 rows as the force kernel does and every lane
// takes its raw hits through the reference's exact r2 (unfused): r2 < rl^2
// counts towards the list lengths (the Verlet-list statistics), r2 < rc^2 is
// evaluated.  Same pairs, forces (to summation order) and statistics as list
// build + force kernel.
template <bool EV, int N3>
__global__ void __launch_bounds__(kVsG, 5)
    vls_rawforce_kernel(const int32_t* __restrict__ groups, const double* __restrict__ rows,
                        double rl2, LJK k, int cap_chunks, int cap_ent,
                        const int4* __restrict__ scratch, const int32_t* __restrict__ out_perm,
                        double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz,
                        double* __restrict__ ev, lmd_stats* __restrict__ stats,
                        int32_t* __restrict__ count, int32_t* __restrict__ count_half,
                        const int32_t* __restrict__ info) {
  extern __shared__ __align__(128) double sm_d[];
  double* xs = sm_d;
  __shared__ unsigned long long bar;
  if (info[4] > cap_ent) return;   // the walk ran out of room: the host retries
  const int g = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int t = g * (kVsG / 32) + w;
  const int32_t* rec = groups + (long long)g * kVsRec;
  if (tid == 0) mbar_init(&bar, 1);
  vls_dummies(rec, xs);
  __syncthreads();
  vls_stage(rec, rows, xs, &bar);
  const int cnt_p = rec[kVsCnt];
  const bool active = tid < cnt_p;
  const int p = rec[kVsP0] + tid;
  const int irow = rec[kVsSelf] + tid;
  const unsigned hb_row = (unsigned)rec[kVsHb];   // first image row (local)
  const unsigned dummy = (unsigned)((rec[kVsS] + 15) & ~15);   // a far-away row
  const int n_raw = active ? count[p] : 0;
  // the lane's stretch, as the walk laid it out
  const uint4* hits8 = reinterpret_cast<const uint4*>(
      reinterpret_cast<const uint16_t*>(scratch + ((long long)t * cap_chunks) * 32) +
      lane * cap_ent);
  const int raw_max = __reduce_max_sync(0xffffffffu, n_raw);
  uint4 vn = hits8[0];
  mbar_wait(&bar, 0);
  double px = -1.0e30, py = -1.0e30, pz = -1.0e30;
  if (active) {
    px = xs[3 * irow];
    py = xs[3 * irow + 1];
    pz = xs[3 * irow + 2];
  }
  VsAcc a = {0.0, 0.0, 0.0, 0.0, 0.0, 0, 0};
  int n_list = 0, n_half = 0;
#pragma unroll 1
  for (int e0 = 0; e0 < raw_max; e0 += 8) {
    const uint4 v = vn;
    if (e0 + 8 < raw_max) vn = hits8[min((e0 >> 3) + 1, (cap_ent >> 3) - 1)];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const unsigned wv = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
      const unsigned jr = (e & 1) ? wv >> 16 : wv & 0xffffu;
      const bool mine = e0 + e < n_raw && (int)jr != irow;
      const unsigned j = mine ? jr : dummy;
      const double dx = px - xs[3 * j], dy = py - xs[3 * j + 1], dz = pz - xs[3 * j + 2];
      const double r2 = r2_exact(dx, dy, dz);
      const bool in_rl = r2 < rl2;            // (the dummy row is far outside)
      const bool hit = r2 < k.rc2;
      n_list += in_rl ? 1 : 0;
      n_half += (in_rl && (int)j > irow) ? 1 : 0;
      double u3;
      const double f = vs_force_scalar(r2, hit, k, u3);
      a.ax = fma(f, dx, a.ax);
      a.ay = fma(f, dy, a.ay);
      a.az = fma(f, dz, a.az);
      if (EV) {
        a.e = fma(0.5 * u3, fma(k.e12, u3, -k.e6), a.e);
        a.v = fma(0.5 * f, r2, a.v);
      }
      a.pairs += hit ? 1 : 0;
      if (N3 == 2) a.halo += (hit && j >= hb_row) ? 1 : 0;
    }
  }
  if (active) {
    count[p] = n_list;
    count_half[p] = n_half;
  }
  // a coincident pair (r2 == 0 inside the cutoff): the numba -1 sentinel
  const int overlap = (active && !(isfinite(a.ax) && isfinite(a.ay) && isfinite(a.az))) ? 1 : 0;
  if (active) {
    const int o = out_perm ? out_perm[p] : p;
    fx[o] = a.ax;
    fy[o] = a.ay;
    fz[o] = a.az;
  }
  Acc fl = {0.0, 0.0, 0.0, a.e, a.v, a.pairs, overlap, a.halo};
  flush_acc(fl, lane, true, EV, t, ev, stats);
}

// ---------------------------------------------------------------- refresh
// rows[k] = positions of particle perm[k] (x, y, z), and with disp the
// largest squared displacement from build[k], max-reduced into disp[slot]
// (bit pattern of a non-negative double); disp[slot ^ 1] is cleared for the
// next launch
// nh > 0: threads n .. n + nh - 1 also write the periodic images (rows n ..):
// image k' = position of owner[k'] (caller order) + the exact shift its code
// names per axis (0 none, 1 + (hi - lo), 2 + (lo - hi): domain.py:112-118),
// so one launch refreshes the whole backing
struct VsImg {
  double up[3], down[3];   // hi - lo, lo - hi per axis (rounded once, as the reference's)
};
__global__ void vls_refresh_kernel(long long n, const int32_t* __restrict__ perm,
                                   const double* __restrict__ x, const double* __restrict__ y,
                                   const double* __restrict__ z, double* __restrict__ rows,
                                   const double* __restrict__ build,
                                   unsigned long long* __restrict__ disp, int slot, long long nh,
                                   const int32_t* __restrict__ owner,
                                   const int8_t* __restrict__ shift, VsImg img) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (k >= n && k < n + nh) {
    const int o = owner[k - n];
    int sc = shift[k - n];
    const double p[3] = {x[o], y[o], z[o]};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int d = sc % 3;
      sc /= 3;
      rows[3 * k + ax] = __dadd_rn(p[ax], d == 1 ? img.up[ax] : (d == 2 ? img.down[ax] : 0.0));
    }
  }
  if (k < n) {
    const int s = perm ? perm[k] : (int)k;
    const double px = x[s], py = y[s], pz = z[s];
    rows[3 * k] = px;
    rows[3 * k + 1] = py;
    rows[3 * k + 2] = pz;
    if (disp) {
      // the reference's unfused expression (containers.py:23-38), so the
      // rebuild decision taken from it is the one lmd_max_displacement2 takes
      const double ex = __dadd_rn(px, -build[3 * k]), ey = __dadd_rn(py, -build[3 * k + 1]),
                   ez = __dadd_rn(pz, -build[3 * k + 2]);
      d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
    }
  }
  if (!disp) return;
  if (k == 0) disp[slot ^ 1] = 0ull;
  unsigned long long b = (unsigned long long)__double_as_longlong(d2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  // one atomic per block at most, and only where it would raise the running
  // maximum (a plain read of the hot word first): half a million same-address
  // atomics per launch cost 0.5 ms at 16.8M particles
  __shared__ unsigned long long wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) b = max(b, wmax[w]);
    if (b > *reinterpret_cast<volatile unsigned long long*>(disp + slot)) atomicMax(disp + slot, b);
  }
}

// rows_out[k] = rows_in[perm[k]] (3 doubles); with disp, the largest squared
// displacement from build[k] is max-reduced into disp[slot] as well (ghost
// rows of a decomposition: their displacements count for the inner segment's
// validity like the owned particles', and are known here without asking
// their owners)
__global__ void vls_gather_rows_kernel(long long n, const int32_t* __restrict__ perm,
                                       const double* __restrict__ in, double* __restrict__ out,
                                       const double* __restrict__ build,
                                       unsigned long long* __restrict__ disp, int slot) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (k < n) {
    const long long s = perm ? perm[k] : k;
    const double px = in[3 * s], py = in[3 * s + 1], pz = in[3 * s + 2];
    out[3 * k] = px;
    out[3 * k + 1] = py;
    out[3 * k + 2] = pz;
    if (disp) {
      const double ex = __dadd_rn(px, -build[3 * k]), ey = __dadd_rn(py, -build[3 * k + 1]),
                   ez = __dadd_rn(pz, -build[3 * k + 2]);
      d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
    }
  }
  if (!disp) return;
  unsigned long long b = (unsigned long long)__double_as_longlong(d2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  __shared__ unsigned long long wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) b = max(b, wmax[w]);
    if (b > *reinterpret_cast<volatile unsigned long long*>(disp + slot)) atomicMax(disp + slot, b);
  }
}

// rows -> pos4 (ownership OWNED below n_owned, HALO above) and SoA copies
__global__ void vls_rows_to_legacy_kernel(long long n, long long n_owned,
                                          const double* __restrict__ rows,
                                          double4* __restrict__ pos4, double* __restrict__ sx,
                                          double* __restrict__ sy, double* __restrict__ sz) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double px = rows[3 * k], py = rows[3 * k + 1], pz = rows[3 * k + 2];
  if (pos4)
    pos4[k] = make_double4(px, py, pz, k < n_owned ? (double)LMD_OWNED : (double)LMD_HALO);
  if (sx) {
    sx[k] = px;
    sy[k] = py;
    sz[k] = pz;
  }
}

template <int OCC, bool EV, int N3>
static int launch_force(dim3 grid, size_t smem, cudaStream_t s, const int32_t* groups,
                        const int32_t* gindex, const double* rows, const void* nbr,
                        const int32_t* segc, const uint8_t* slotmap, int cap_chunks,
                        const unsigned long long* disp, unsigned long long hd2, const LJK& k,
                        const int32_t* out_perm, double* fx, double* fy, double* fz, double* ev,
                        lmd_stats* stats) {
  auto kern = vls_force_kernel<OCC, EV, N3>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_cuda_error(e);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<grid, kVsG, smem, s>>>(groups, gindex, rows, (const int4*)nbr, segc, slotmap, cap_chunks,
                               disp, hd2, k, out_perm, fx, fy, fz, ev, stats, (int)grid.x,
                               OCC * sms);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

static inline size_t stage_bytes(int32_t rows) {
  return ((size_t)(rows + 16) * 24 + 127) / 128 * 128;   // + the 16 dummy rows
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int64_t lmd_vls_max_groups(const lmd_grid* g, int64_t n_owned) {
  // every group but a line's last holds at least 32 particles
  const int64_t rows = g->dims[1] * g->dims[2];
  return cdiv(n_owned, 32) + rows;
}

int32_t lmd_vls_rows_for(int32_t staged_rows) {
  if (staged_rows > kVsMaxRows) return 0;
  return (staged_rows + 63) / 64 * 64;  // shared-memory rows to reserve
}

size_t lmd_vls_plan_temp_bytes(const lmd_grid* g) {
  const int64_t nrows = g->tdims[1] * g->tdims[2];
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)nrows);
  return bytes;
}

int lmd_vls_plan(const lmd_grid* g, int64_t n_owned, const int32_t* o_start,
                 const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                 int32_t* fs_own, int32_t* fs_img, int32_t* row_groups, int32_t* row_gend,
                 void* temp, size_t temp_bytes, int32_t* groups, int32_t* info, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(info, 0, kVsInfo * sizeof(int32_t), s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  if (n_owned <= 0) return LMD_OK;
  if (n_owned > 0x7fffffffLL) return LMD_ERR_CONFIG;
  const GridK k = make_gridk(g);
  const long long nrows = g->tdims[1] * g->tdims[2];
  vls_rows_kernel<<<(unsigned)cdiv(nrows, 128), 128, 0, s>>>(nrows, (int)k.t0, o_start, o_count,
                                                               h_start, h_count, fs_own, fs_img);
  LMD_CHECK_LAUNCH();
  vls_groups_kernel<true><<<(unsigned)cdiv(nrows, 128), 128, 0, s>>>(
      nrows, (int)k.t0, (int)k.t1, (int)k.d0, (int)k.d1, (int)k.d2, kVsG, kVsBudget, fs_own,
      o_count, fs_img, h_count, row_groups, nullptr, nullptr, nullptr);
  LMD_CHECK_LAUNCH();
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceScan::InclusiveSum(temp, bytes, row_groups, row_gend, (int)nrows, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  vls_groups_kernel<false><<<(unsigned)cdiv(nrows, 128), 128, 0, s>>>(
      nrows, (int)k.t0, (int)k.t1, (int)k.d0, (int)k.d1, (int)k.d2, kVsG, kVsBudget, fs_own,
      o_count, fs_img, h_count, row_groups, row_gend, groups, info);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

static inline int build_area(int32_t rows, int32_t cap_entries) {
  // FP32 copies of the rows (step 1: 12 B per row), then the lanes' sorted
  // hits (steps 2-3)
  const size_t a = std::max((size_t)rows * 12, (size_t)cap_entries * kVsG * 2);
  return (int)((a + 127) / 128 * 128);
}

size_t lmd_vls_build_smem(int32_t rows, int32_t cap_entries) {
  return (size_t)build_area(rows, cap_entries) + kVsRingBytes + 2 * 32 * kVsG;
}

int lmd_vls_build(const lmd_grid* g, double rin2, double rl2, int64_t n_owned, int32_t rows,
                  const double* pos_rows, const int32_t* fs_own, const int32_t* o_count,
                  const int32_t* fs_img, const int32_t* h_count, const int32_t* groups,
                  int64_t max_groups, int32_t cap_chunks, int32_t cap_entries, int32_t bank_order,
                  void* nbr, int32_t* seg_chunks, uint8_t* slotmap, int32_t* count,
                  int32_t* count_half, int32_t* info, void* stream) {
  if (n_owned <= 0 || max_groups <= 0) return LMD_OK;
  if (cap_entries < 8 || cap_entries > 255 || cap_entries % 8 || !(rin2 <= rl2))
    return LMD_ERR_CONFIG;
  // each lane's hits fit its tile's list area before the lists are written
  if (cap_chunks < 2 || cap_chunks * 8 < cap_entries) return LMD_ERR_CONFIG;
  if (rows <= 0 || rows > kVsMaxRows + 64 || (uintptr_t)pos_rows % 16) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  const GridK k = make_gridk(g);
  // the bucket counters exist only for the bank order
  const size_t smem = (size_t)build_area(rows, cap_entries) + kVsRingBytes +
                      (bank_order ? 2 * 32 * kVsG : 0);
  auto kern = bank_order ? vls_build_kernel<1> : vls_build_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return set_cuda_error(e);
  kern<<<(unsigned)max_groups, kVsG, smem, s>>>(
      (int)k.t0, (int)k.t1, groups, info, pos_rows, fs_own, o_count, fs_img, h_count, rin2, rl2,
      build_area(rows, cap_entries), cap_chunks, cap_entries, (int4*)nbr, seg_chunks, slotmap,
      count, count_half, info);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int64_t lmd_vls_ev_slots(int64_t max_groups) { return max_groups * (kVsG / 32); }

int lmd_vls_force(int newton3, int flags, const lmd_lj* lj, int64_t n_owned, int32_t rows,
                  const double* pos_rows, const int32_t* groups, int64_t n_groups,
                  const int32_t* group_index, int64_t n_index, const void* nbr, const int32_t* seg_chunks,
                  const uint8_t* slotmap, int32_t cap_chunks, const uint64_t* disp,
                  double half_delta2, const int32_t* out_perm, double* fx, double* fy,
                  double* fz, double* ev_scratch, lmd_stats* stats, void* stream) {
  if (n_owned <= 0 || n_groups <= 0) return LMD_OK;
  if (newton3 != 0 && newton3 != 2) return LMD_ERR_CONFIG;
  if (rows <= 0 || rows > kVsMaxRows + 64 || (uintptr_t)pos_rows % 16 || !(half_delta2 >= 0.0) ||
      cap_chunks < 2)
    return LMD_ERR_CONFIG;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  if (ev && !ev_scratch) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  const LJK k = make_ljk(lj);
  union {
    double d;
    unsigned long long u;
  } hd;
  hd.d = half_delta2;
  if (group_index && n_index <= 0) {  // an empty subset: nothing to launch
    if (ev && !(flags & LMD_FLAG_DEFER_EV))
      return reduce_ev(ev_scratch, lmd_vls_ev_slots(n_groups), stats, (cudaStream_t)stream);
    return LMD_OK;
  }
  const dim3 grid((unsigned)(group_index ? n_index : n_groups));
  const size_t smem = stage_bytes(rows);
  const unsigned long long* dp = (const unsigned long long*)disp;
  // blocks per SM by the staging footprint (228 KB per SM, 1 KB reserved
  // per block): 5 up to ~44 KB, else 4
  const bool five = smem + 1024 + 128 <= 45 * 1024;
#define LMD_VSF(OCC, EVB, N3B)                                                                  \
  rc = launch_force<OCC, EVB, N3B>(grid, smem, s, groups, group_index, pos_rows, nbr, seg_chunks, \
                                   slotmap, cap_chunks, dp, hd.u, k, out_perm, fx, fy, fz,      \
                                   ev_scratch, stats)
#define LMD_VSF_O(EVB, N3B)       \
  if (five) LMD_VSF(5, EVB, N3B); \
  else LMD_VSF(4, EVB, N3B);
  int rc = LMD_OK;
  if (ev) {
    if (newton3) { LMD_VSF_O(true, 2) } else { LMD_VSF_O(true, 0) }
  } else {
    if (newton3) { LMD_VSF_O(false, 2) } else { LMD_VSF_O(false, 0) }
  }
#undef LMD_VSF_O
#undef LMD_VSF
  if (rc != LMD_OK) return rc;
  if (ev && !(flags & LMD_FLAG_DEFER_EV))
    return reduce_ev(ev_scratch, lmd_vls_ev_slots(n_groups), stats, s);
  return LMD_OK;
}

int lmd_vls_direct(const lmd_grid* g, int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                   int32_t rows, const double* pos_rows, const int32_t* fs_own,
                   const int32_t* o_count, const int32_t* fs_img, const int32_t* h_count,
                   const int32_t* groups, int64_t n_groups, int32_t cap_entries, void* scratch,
                   const int32_t* out_perm, double* fx, double* fy, double* fz,
                   double* ev_scratch, lmd_stats* stats, int32_t* count, int32_t* count_half,
                   int32_t* info, void* stream) {
  if (n_owned <= 0 || n_groups <= 0) return LMD_OK;
  if (newton3 != 0 && newton3 != 2) return LMD_ERR_CONFIG;
  if (cap_entries < 8 || cap_entries % 8 || cap_entries > 4088) return LMD_ERR_CONFIG;
  if (rows <= 0 || rows > kVsMaxRows + 64 || (uintptr_t)pos_rows % 16) return LMD_ERR_CONFIG;
  const bool ev = (flags & LMD_FLAG_ENERGY) != 0;
  if (ev && !ev_scratch) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  const LJK k = make_ljk(lj);
  const GridK gk = make_gridk(g);
  const double rl = lj->cutoff + lj->skin;
  const int cap_chunks = cap_entries / 8;   // scratch: n_groups * 4 tiles * cap_chunks * 512 B
  {   // 1. the walk (FP32 rows only: 12 B per row)
    const size_t area = ((size_t)rows * 12 + 127) / 128 * 128;
    const size_t smem = area + kVsRingBytes;
    auto kern = vls_build_kernel<2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    kern<<<(unsigned)n_groups, kVsG, smem, s>>>(
        (int)gk.t0, (int)gk.t1, groups, info, pos_rows, fs_own, o_count, fs_img, h_count, rl * rl,
        rl * rl, (int)area, cap_chunks, cap_entries, (int4*)scratch, nullptr, nullptr, count,
        count_half, info);
    LMD_CHECK_LAUNCH();
  }
  const size_t smem = stage_bytes(rows);   // 2. the raw hits from the FP64 rows
#define LMD_VSD(EVB, N3B)                                                                   \
  {                                                                                         \
    auto kern = vls_rawforce_kernel<EVB, N3B>;                                              \
    cudaError_t e =                                                                         \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return set_cuda_error(e);                                         \
    kern<<<(unsigned)n_groups, kVsG, smem, s>>>(groups, pos_rows, rl * rl, k, cap_chunks,   \
                                                cap_entries, (const int4*)scratch, out_perm, \
                                                fx, fy, fz, ev_scratch, stats, count,       \
                                                count_half, info);                          \
  }
  if (ev) {
    if (newton3) LMD_VSD(true, 2) else LMD_VSD(true, 0)
  } else {
    if (newton3) LMD_VSD(false, 2) else LMD_VSD(false, 0)
  }
#undef LMD_VSD
  LMD_CHECK_LAUNCH();
  if (ev && !(flags & LMD_FLAG_DEFER_EV))
    return reduce_ev(ev_scratch, lmd_vls_ev_slots(n_groups), stats, s);
  return LMD_OK;
}

int lmd_vls_reduce_ev(int64_t n_groups, const double* ev_scratch, lmd_stats* stats, void* stream) {
  if (n_groups <= 0) return LMD_OK;
  return reduce_ev(ev_scratch, lmd_vls_ev_slots(n_groups), stats, (cudaStream_t)stream);
}

int lmd_vls_refresh(int64_t n, const int32_t* perm, const double* x, const double* y,
                    const double* z, double* rows, const double* build_rows, uint64_t* disp,
                    int32_t slot, const lmd_box* box, int64_t n_images, const int32_t* owner,
                    const int8_t* shift, void* stream) {
  if (n <= 0) return LMD_OK;
  if (slot != 0 && slot != 1) return LMD_ERR_CONFIG;
  if (disp && !build_rows) return LMD_ERR_CONFIG;
  if (n_images > 0 && (!box || !owner || !shift)) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  VsImg img = {};
  if (n_images > 0)
    for (int ax = 0; ax < 3; ++ax) {
      img.up[ax] = box->hi[ax] - box->lo[ax];
      img.down[ax] = box->lo[ax] - box->hi[ax];
    }
  const long long total = n + (n_images > 0 ? n_images : 0);
  vls_refresh_kernel<<<(unsigned)cdiv(total, 256), 256, 0, s>>>(
      n, perm, x, y, z, rows, build_rows, (unsigned long long*)disp, slot,
      n_images > 0 ? n_images : 0, owner, shift, img);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_vls_gather_rows(int64_t n, const int32_t* perm, const double* rows_in, double* rows_out,
                        const double* build_rows, uint64_t* disp, int32_t slot, void* stream) {
  if (n <= 0) return LMD_OK;
  if (disp && (!build_rows || (slot != 0 && slot != 1))) return LMD_ERR_CONFIG;
  vls_gather_rows_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, perm, rows_in, rows_out, build_rows, (unsigned long long*)disp, slot);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_vls_rows_to_legacy(int64_t n, int64_t n_owned, const double* rows, double* pos4,
                           double* sx, double* sy, double* sz, void* stream) {
  if (n <= 0) return LMD_OK;
  vls_rows_to_legacy_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, n_owned, rows, (double4*)pos4, sx, sy, sz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
