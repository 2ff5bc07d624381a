// Shared pieces of the Verlet-list build and force kernels (vl.cu, vl_ci.cu).
#pragma once

#include "common.cuh"

namespace lmd {

constexpr int kVLWarps = 4;
constexpr int kChunk = 4;  // fill steps per lane per 128-bit index load

// Staged Verlet lists (v_by_one): a group of G consecutive owned particles
// (G/32 tiles, one block) copies the SoA positions of its candidate runs
// into shared memory.  The group's particles lie in one or two cell rows
// (rows are (y, z) lines of the ring-padded grid, row = lin / t0); for row
// rr of the group and each (dy, dz), run r = view * 18 + rr * 9 +
// (dz + 1) * 3 + (dy + 1) covers the cells xa - 1 .. xb + 1 of the
// neighbouring row (xa .. xb = the group's cells in its row) of the owned
// (view 0) or image (view 1) backing: one contiguous index range.
// Per-group record of kGroupRec int32: run starts (even), lengths (even),
// local-index offsets (base - start), then S, the first image-run local
// index, a flag (1: more than two rows or S > capacity -- the group gathers
// from global memory with global indices) and the group's first row.
constexpr int kGroupRuns = 36;
constexpr int kGroupRec = 128;
constexpr int kGrpStart = 0, kGrpLen = 36, kGrpOff = 72, kGrpS = 108, kGrpHalo = 109,
              kGrpGlobal = 110, kGrpRow = 111;

// lane holding (i_off = il, j_off = jo) of a pattern (inverse of Pattern<P>)
__device__ __forceinline__ int lane_of(int pattern, int il, int jo) {
  switch (pattern) {
    case LMD_ONE_BY_V: return jo;
    case LMD_V_BY_ONE: return il;
    case LMD_TWO_BY_HALF: return il * 16 + jo;
    default: return il + 16 * jo;  // LMD_HALF_BY_TWO
  }
}

__device__ __forceinline__ long long cell_of_owned(const double4& p, double lo0, double lo1,
                                                   double lo2, double cl0, double cl1, double cl2,
                                                   long long d0, long long d1, long long d2,
                                                   long long t0, long long t1) {
  const double pp[3] = {p.x, p.y, p.z};
  const double lo[3] = {lo0, lo1, lo2}, cl[3] = {cl0, cl1, cl2};
  const long long d[3] = {d0, d1, d2};
  long long q[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double s = floor(__ddiv_rn(__dadd_rn(pp[ax], -lo[ax]), cl[ax]));
    long long v = !(s >= -4.0) ? -3 : (s > 1.0e15 ? 1000000000000000LL : (long long)s + 1);
    q[ax] = v < 1 ? 1 : (v > d[ax] ? d[ax] : v);
  }
  return q[0] + t0 * (q[1] + t1 * q[2]);
}

struct GridK {
  double lo0, lo1, lo2, cl0, cl1, cl2;
  long long d0, d1, d2, t0, t1;
};

// ------------------------------------------------------------------ force
// per-lane accumulators; counts are 32-bit (a lane sees at most a few
// thousand pairs per launch) and widened once in flush_acc.  `halo` (pairs
// with an image j) is counted only where Newton3 bookkeeping needs it.
struct Acc {
  double ax, ay, az, e, v;
  int pairs, overlap, halo;
  unsigned hi_min = 0xffffffffu;  // staged kernel: smallest r2 high word seen
};

__device__ __forceinline__ void flush_acc(const Acc& a, int lane, bool live, bool ev_on,
                                          long long warp_slot, double* __restrict__ ev,
                                          lmd_stats* __restrict__ stats) {
  const long long pairs = warp_sum_ll((long long)a.pairs);
  const long long halo = warp_sum_ll((long long)a.halo);
  const int overlap = __any_sync(0xffffffffu, a.overlap);
  if (lane == 0 && live) {
    if (pairs) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pairs);
    if (halo) atomicAdd((unsigned long long*)&stats->pairs_owned_halo, (unsigned long long)halo);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
  if (ev_on) {
    const double e = warp_sum(a.e), v = warp_sum(a.v);
    if (lane == 0) {
      ev[2 * warp_slot] = e;
      ev[2 * warp_slot + 1] = v;
    }
  }
}

// mbarrier + TMA bulk-copy helpers (PTX): one elected thread arms the
// barrier with the byte count, issues cp.async.bulk copies that complete
// their bytes on it, and consumers wait on phase 0.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

static inline GridK make_gridk(const lmd_grid* g) {
  GridK k;
  k.lo0 = g->lo[0];
  k.lo1 = g->lo[1];
  k.lo2 = g->lo[2];
  k.cl0 = g->cell_len[0];
  k.cl1 = g->cell_len[1];
  k.cl2 = g->cell_len[2];
  k.d0 = g->dims[0];
  k.d1 = g->dims[1];
  k.d2 = g->dims[2];
  k.t0 = g->tdims[0];
  k.t1 = g->tdims[1];
  return k;
}

static inline int pattern_A(int p) {
  return p == LMD_ONE_BY_V ? 1 : p == LMD_V_BY_ONE ? 32 : p == LMD_TWO_BY_HALF ? 2 : 16;
}
static inline int pattern_B(int p) { return 32 / pattern_A(p); }


}  // namespace lmd
