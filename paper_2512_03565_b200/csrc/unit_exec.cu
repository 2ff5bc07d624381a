// execute_packed on the device: the reference's batched operator
// (executor.py:118-171) over an explicit, colored unit list.
//
// Units are grouped by (color, base); one launch per color, one warp per
// base, the base's units in order (traversals.py:1-6: same-color units of
// different bases write disjoint buffers -- verify_coloring).  A unit sweeps
// i-span x j-span exactly like _sweep_span (executor.py:72-115): owned i
// only, non-dummy j, self exclusion / strict upper triangle, Newton3 dual
// write.  Forces accumulate (+=) in place; every write of a warp is ordered
// by __syncwarp, so the result is deterministic.
#include "common.cuh"

namespace lmd {

struct UnitArrays {
  const int64_t* i_off;
  const int64_t* i_len;
  const int64_t* j_off;
  const int64_t* j_len;
  const uint8_t* j_halo;
  const uint8_t* n3;
  const uint8_t* same;
};

template <int P>
__global__ void __launch_bounds__(128)
    packed_color_kernel(UnitArrays u, const int64_t* __restrict__ base_units,
                        const int64_t* __restrict__ base_start, long long nbases,
                        const double* __restrict__ own4, const double* __restrict__ halo4,
                        double* __restrict__ ofx, double* __restrict__ ofy,
                        double* __restrict__ ofz, double* __restrict__ hfx,
                        double* __restrict__ hfy, double* __restrict__ hfz, LJK k,
                        lmd_stats* __restrict__ stats) {
  using Pat = Pattern<P>;
  const int lane = threadIdx.x & 31;
  const long long b = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  long long pairs = 0;
  int overlap = 0;
  if (b < nbases) {
    const int io = Pat::ioff(lane), jo = Pat::joff(lane);
    for (long long q = base_start[b]; q < base_start[b + 1]; ++q) {
      const long long w = base_units[q];
      const long long i0 = u.i_off[w], ni = u.i_len[w], j0 = u.j_off[w], nj = u.j_len[w];
      const bool jh = u.j_halo[w] != 0, n3 = u.n3[w] != 0, same = u.same[w] != 0;
      const double* jpos = jh ? halo4 : own4;
      double* jfx = jh ? hfx : ofx;
      double* jfy = jh ? hfy : ofy;
      double* jfz = jh ? hfz : ofz;
      for (long long ci = 0; ci < ni; ci += Pat::A) {
        const long long il = ci + io;
        const bool ilive = il < ni;
        const double4 pi = ld_pos4(own4, i0 + (ilive ? il : 0));
        const bool iown = ilive && pi.w == (double)LMD_OWNED;
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (long long cj = 0; cj < nj; cj += Pat::B) {
          const long long jl = cj + jo;
          double bx = 0.0, by = 0.0, bz = 0.0;
          bool ok = iown && jl < nj;
          if (same) ok = ok && (n3 ? jl > il : jl != il);
          if (ok) {
            const double4 pj = ld_pos4(jpos, j0 + jl);
            if (pj.w != (double)LMD_DUMMY) {
              const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
              double r2;
              if (within_cutoff(dx, dy, dz, k, r2)) {
                if (r2 == 0.0) {
                  overlap = 1;
                } else {
                  double s6;
                  const double f = lj_scalar(r2, k, s6);
                  ax = fma(f, dx, ax);
                  ay = fma(f, dy, ay);
                  az = fma(f, dz, az);
                  if (n3) {
                    bx = -f * dx;
                    by = -f * dy;
                    bz = -f * dz;
                  }
                  ++pairs;
                }
              }
            }
          }
          if (n3) {
            bx = reduce_i<P>(bx);
            by = reduce_i<P>(by);
            bz = reduce_i<P>(bz);
            if (io == 0 && jl < nj) {
              jfx[j0 + jl] += bx;
              jfy[j0 + jl] += by;
              jfz[j0 + jl] += bz;
            }
            __syncwarp();
          }
        }
        ax = reduce_j<P>(ax);
        ay = reduce_j<P>(ay);
        az = reduce_j<P>(az);
        if (jo == 0 && iown) {
          ofx[i0 + il] += ax;
          ofy[i0 + il] += ay;
          ofz[i0 + il] += az;
        }
        __syncwarp();
      }
    }
  }
  pairs = warp_sum_ll(pairs);
  overlap = __any_sync(0xffffffffu, overlap);
  if (lane == 0 && b < nbases) {
    if (pairs) atomicAdd((unsigned long long*)&stats->pair_interactions, (unsigned long long)pairs);
    if (overlap) atomicOr(&stats->overlap, 1);
  }
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int lmd_execute_packed(int64_t n_units, const int64_t* i_off, const int64_t* i_len,
                       const int64_t* j_off, const int64_t* j_len, const uint8_t* j_halo,
                       const uint8_t* newton3, const uint8_t* same, int n_colors,
                       const int64_t* color_base_start, const int64_t* base_units,
                       const int64_t* base_start, int pattern, const lmd_lj* lj,
                       const double* own4, const double* halo4, double* ofx, double* ofy,
                       double* ofz, double* hfx, double* hfy, double* hfz, lmd_stats* stats,
                       void* stream) {
  if (n_units <= 0) return LMD_OK;
  const LJK k = make_ljk(lj);
  const UnitArrays u = {i_off, i_len, j_off, j_len, j_halo, newton3, same};
  cudaStream_t s = (cudaStream_t)stream;
  for (int c = 0; c < n_colors; ++c) {
    // color c owns bases [color_base_start[c], color_base_start[c+1]) (host array)
    const long long b0 = color_base_start[c], b1 = color_base_start[c + 1];
    const long long nb = b1 - b0;
    if (nb <= 0) continue;
    const unsigned blocks = (unsigned)cdiv(nb, 4);
#define LMD_PK(PP)                                                                           \
  packed_color_kernel<PP><<<blocks, 128, 0, s>>>(u, base_units, base_start + b0, nb, own4,   \
                                                 halo4, ofx, ofy, ofz, hfx, hfy, hfz, k, stats)
    switch (pattern) {
      case LMD_ONE_BY_V: LMD_PK(LMD_ONE_BY_V); break;
      case LMD_V_BY_ONE: LMD_PK(LMD_V_BY_ONE); break;
      case LMD_TWO_BY_HALF: LMD_PK(LMD_TWO_BY_HALF); break;
      case LMD_HALF_BY_TWO: LMD_PK(LMD_HALF_BY_TWO); break;
      default: return LMD_ERR_CONFIG;
    }
#undef LMD_PK
    LMD_CHECK_LAUNCH();
  }
  return LMD_OK;
}

}  // extern "C"
