// K1 cell binning / stable sort and K9 periodic images (sm_100a).
//
// Replaces containers.py:100-189 (LinkedCellsContainer.cell_coords,
// linear_index, rebuild, refresh, collect_forces) and domain.py:97-144
// (build_halo).  Sorting is CUB's LSD radix sort, which is stable, so the
// permutation equals np.argsort(kind="stable") bit for bit.
#include <cub/cub.cuh>
#include <math.h>
#include <stdio.h>

#include "common.cuh"

namespace lmd {

static thread_local cudaError_t g_last_cuda = cudaSuccess;
int set_cuda_error(cudaError_t e) {
  g_last_cuda = e;
  fprintf(stderr, "[b200md] CUDA error: %s\n", cudaGetErrorString(e));
  return LMD_ERR_CUDA;
}

// ---------------------------------------------------------------- K1 cells
__global__ void cell_index_kernel(int64_t n, const double* __restrict__ x,
                                  const double* __restrict__ y, const double* __restrict__ z,
                                  double lo0, double lo1, double lo2, double cl0, double cl1,
                                  double cl2, long long d0, long long d1, long long d2,
                                  long long t0, long long t1, int ring,
                                  int32_t* __restrict__ cell) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double p[3] = {x[k], y[k], z[k]};
  const double lo[3] = {lo0, lo1, lo2};
  const double cl[3] = {cl0, cl1, cl2};
  const long long d[3] = {d0, d1, d2};
  long long q[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    // np.floor((pos - min) / cell_length): IEEE sub and div (no reciprocal)
    double s = floor(__ddiv_rn(__dadd_rn(p[ax], -lo[ax]), cl[ax]));
    // .astype(np.int64) then +1 and np.clip; clamp before the cast so huge
    // or non-finite values cannot overflow the conversion
    long long v;
    if (!(s >= -4.0)) v = -3;
    else if (s > 1.0e15) v = 1000000000000000LL;
    else v = (long long)s + 1;
    long long lo_c = ring ? 0 : 1, hi_c = ring ? d[ax] + 1 : d[ax];
    v = v < lo_c ? lo_c : (v > hi_c ? hi_c : v);
    q[ax] = v;
  }
  cell[k] = (int32_t)(q[0] + t0 * (q[1] + t1 * q[2]));
}

__global__ void iota_kernel(int64_t n, int32_t* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) out[k] = (int32_t)k;
}

__global__ void cell_ranges_kernel(int64_t n, int32_t base, const int32_t* __restrict__ key,
                                   int32_t* __restrict__ start, int32_t* __restrict__ count) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t c = key[k];
  if (k == 0 || key[k - 1] != c) start[c] = base + (int32_t)k;
  if (k == n - 1 || key[k + 1] != c) {
    // count = end - start; the start of this run is found by the thread that
    // owns its first element, so record the end and subtract afterwards
    count[c] = base + (int32_t)k + 1;
  }
}

__global__ void cell_count_fix_kernel(int64_t ncell, const int32_t* __restrict__ start,
                                      int32_t* __restrict__ count) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  int32_t e = count[c];
  count[c] = e > 0 ? e - start[c] : 0;
}

__global__ void merge_tables_kernel(int64_t ncell, const int32_t* __restrict__ os,
                                    const int32_t* __restrict__ oc,
                                    const int32_t* __restrict__ hs,
                                    const int32_t* __restrict__ hc, int32_t* __restrict__ s,
                                    int32_t* __restrict__ c, uint8_t* __restrict__ dup) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= ncell) return;
  // a cell holding owned particles AND images (images of particles that sit
  // outside [lo, hi) mid-step): the reference lists it twice as an anchor
  if (dup) dup[q] = (oc[q] > 0 && hc[q] > 0) ? 1 : 0;
  if (oc[q] > 0) {
    s[q] = os[q];
    c[q] = oc[q];
  } else {
    s[q] = hs[q];
    c[q] = hc[q];
  }
}

// sx != nullptr: also the SoA copies (one read, both layouts)
__global__ void gather_pos4_kernel(int64_t n, const int32_t* __restrict__ perm,
                                   const double* __restrict__ x, const double* __restrict__ y,
                                   const double* __restrict__ z, const int8_t* __restrict__ own,
                                   double own_value, double4* __restrict__ pos4,
                                   double* __restrict__ sx = nullptr,
                                   double* __restrict__ sy = nullptr,
                                   double* __restrict__ sz = nullptr) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t s = perm ? perm[k] : (int32_t)k;
  double w = own ? (double)own[s] : own_value;
  const double px = x[s], py = y[s], pz = z[s];
  pos4[k] = make_double4(px, py, pz, w);
  if (sx) {
    sx[k] = px;
    sy[k] = py;
    sz[k] = pz;
  }
}

__global__ void scatter_forces_kernel(int64_t n, const int32_t* __restrict__ perm,
                                      const double* __restrict__ fx, const double* __restrict__ fy,
                                      const double* __restrict__ fz, double* __restrict__ ox,
                                      double* __restrict__ oy, double* __restrict__ oz) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t d = perm[k];
  ox[d] = fx[k];
  oy[d] = fy[k];
  oz[d] = fz[k];
}

// ------------------------------------------------------------- K9 images
struct BoxK {
  double lo[3], hi[3];
  int per[3];
};

__device__ __forceinline__ void near_flags(const BoxK& b, double margin, const double p[3],
                                           int nlo[3], int nhi[3]) {
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    // domain.py:102-103: (pos - lo < margin), (hi - pos < margin)
    nlo[ax] = b.per[ax] && (__dadd_rn(p[ax], -b.lo[ax]) < margin);
    nhi[ax] = b.per[ax] && (__dadd_rn(b.hi[ax], -p[ax]) < margin);
  }
}

__global__ void halo_count_kernel(BoxK b, double margin, int64_t n, const double* __restrict__ x,
                                  const double* __restrict__ y, const double* __restrict__ z,
                                  const int8_t* __restrict__ own, int32_t* __restrict__ count) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (own && own[k] != LMD_OWNED) {
    count[k] = 0;
    return;
  }
  const double p[3] = {x[k], y[k], z[k]};
  int nlo[3], nhi[3];
  near_flags(b, margin, p, nlo, nhi);
  int c = (1 + nlo[0] + nhi[0]) * (1 + nlo[1] + nhi[1]) * (1 + nlo[2] + nhi[2]) - 1;
  count[k] = c;
}

__global__ void halo_emit_kernel(BoxK b, double margin, int64_t n, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 const int8_t* __restrict__ own, const int32_t* __restrict__ off,
                                 double* __restrict__ hx, double* __restrict__ hy,
                                 double* __restrict__ hz, int32_t* __restrict__ owner,
                                 int8_t* __restrict__ shift) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (own && own[k] != LMD_OWNED) return;
  const double p[3] = {x[k], y[k], z[k]};
  int nlo[3], nhi[3];
  near_flags(b, margin, p, nlo, nhi);
  // shift options per axis in itertools.product order: 0, +L (near lo), -L (near hi)
  double opt[3][3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    opt[ax][0] = 0.0;
    opt[ax][1] = __dadd_rn(b.hi[ax], -b.lo[ax]);
    opt[ax][2] = __dadd_rn(b.lo[ax], -b.hi[ax]);
  }
  int w = off[k];
  for (int s0 = 0; s0 < 3; ++s0) {
    if ((s0 == 1 && !nlo[0]) || (s0 == 2 && !nhi[0])) continue;
    for (int s1 = 0; s1 < 3; ++s1) {
      if ((s1 == 1 && !nlo[1]) || (s1 == 2 && !nhi[1])) continue;
      for (int s2 = 0; s2 < 3; ++s2) {
        if ((s2 == 1 && !nlo[2]) || (s2 == 2 && !nhi[2])) continue;
        if (s0 == 0 && s1 == 0 && s2 == 0) continue;
        hx[w] = __dadd_rn(p[0], opt[0][s0]);
        hy[w] = __dadd_rn(p[1], opt[1][s1]);
        hz[w] = __dadd_rn(p[2], opt[2][s2]);
        owner[w] = (int32_t)k;
        shift[w] = (int8_t)(s0 + 3 * s1 + 9 * s2);
        ++w;
      }
    }
  }
}

__global__ void halo_refresh_kernel(BoxK b, int64_t nh, const int32_t* __restrict__ owner,
                                    const int8_t* __restrict__ shift, const double* __restrict__ x,
                                    const double* __restrict__ y, const double* __restrict__ z,
                                    double4* __restrict__ pos4, double* __restrict__ sx = nullptr,
                                    double* __restrict__ sy = nullptr,
                                    double* __restrict__ sz = nullptr) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nh) return;
  int32_t o = owner[k];
  int s = shift[k];
  const double p[3] = {x[o], y[o], z[o]};
  double q[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    int d = s % 3;
    s /= 3;
    double sh = d == 1 ? __dadd_rn(b.hi[ax], -b.lo[ax])
                       : (d == 2 ? __dadd_rn(b.lo[ax], -b.hi[ax]) : 0.0);
    q[ax] = __dadd_rn(p[ax], sh);
  }
  pos4[k] = make_double4(q[0], q[1], q[2], (double)LMD_HALO);
  if (sx) {
    sx[k] = q[0];
    sy[k] = q[1];
    sz[k] = q[2];
  }
}

__global__ void halo_refresh_soa_kernel(BoxK b, int64_t nh, const int32_t* __restrict__ owner,
                                        const int8_t* __restrict__ shift,
                                        const double* __restrict__ x, const double* __restrict__ y,
                                        const double* __restrict__ z, double* __restrict__ ox,
                                        double* __restrict__ oy, double* __restrict__ oz,
                                        int stride) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nh) return;
  int32_t o = owner[k];
  int s = shift[k];
  const double p[3] = {x[o], y[o], z[o]};
  double q[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    int d = s % 3;
    s /= 3;
    double sh = d == 1 ? __dadd_rn(b.hi[ax], -b.lo[ax])
                       : (d == 2 ? __dadd_rn(b.lo[ax], -b.hi[ax]) : 0.0);
    q[ax] = __dadd_rn(p[ax], sh);
  }
  ox[k * stride] = q[0];
  oy[k * stride] = q[1];
  oz[k * stride] = q[2];
}

// ------------------------------------------------ deterministic reductions
__global__ void reduce_ev_kernel(const double* __restrict__ part, int64_t nslots,
                                 lmd_stats* stats) {
  // one block of 1024 threads, fixed assignment and tree order
  __shared__ double se[32], sv[32];
  double e = 0.0, v = 0.0;
  for (int64_t k = threadIdx.x; k < nslots; k += blockDim.x) {
    e += part[2 * k];
    v += part[2 * k + 1];
  }
  e = warp_sum(e);
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    se[w] = e;
    sv[w] = v;
  }
  __syncthreads();
  if (w == 0) {
    e = l < (int)(blockDim.x >> 5) ? se[l] : 0.0;
    v = l < (int)(blockDim.x >> 5) ? sv[l] : 0.0;
    e = warp_sum(e);
    v = warp_sum(v);
    if (l == 0) {
      stats->epot += e;
      stats->virial += v;
    }
  }
}

int reduce_ev(const double* partials, int64_t nslots, lmd_stats* stats, cudaStream_t s) {
  reduce_ev_kernel<<<1, 1024, 0, s>>>(partials, nslots, stats);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

static inline BoxK make_boxk(const lmd_box* b) {
  BoxK k;
  for (int ax = 0; ax < 3; ++ax) {
    k.lo[ax] = b->lo[ax];
    k.hi[ax] = b->hi[ax];
    k.per[ax] = b->periodic[ax] != 0;
  }
  return k;
}

static inline unsigned grid1d(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace lmd

using namespace lmd;

extern "C" {

int lmd_version(void) { return 1; }

const char* lmd_status_string(int status) {
  switch (status) {
    case LMD_OK: return "ok";
    case LMD_ERR_CONFIG: return "configuration error";
    case LMD_ERR_DEGENERATE: return "degenerate domain";
    case LMD_ERR_CUDA: return cudaGetErrorString(g_last_cuda);
    case LMD_ERR_OVERLAP: return "zero distance between interacting particles";
    default: return "unknown status";
  }
}

int lmd_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

int lmd_grid_init(const lmd_box* box, double length, lmd_grid* g) {
  int64_t total = 1;
  for (int ax = 0; ax < 3; ++ax) {
    double L = box->hi[ax] - box->lo[ax];
    double d = floor(L / length);  // containers.py:77
    if (!(d >= 1.0)) return LMD_ERR_DEGENERATE;
    if (d > 2.0e9) return LMD_ERR_CONFIG;
    g->dims[ax] = (int64_t)d;
    g->cell_len[ax] = L / (double)g->dims[ax];  // containers.py:82
    g->tdims[ax] = g->dims[ax] + 2;
    g->lo[ax] = box->lo[ax];
    total *= g->tdims[ax];
  }
  if (total > 0x7fffffffLL) return LMD_ERR_CONFIG;
  g->ncell = total;
  return LMD_OK;
}

int lmd_cell_index(const lmd_grid* g, int ring, int64_t n, const double* x, const double* y,
                   const double* z, int32_t* cell, void* stream) {
  if (n <= 0) return LMD_OK;
  cell_index_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, x, y, z, g->lo[0], g->lo[1], g->lo[2], g->cell_len[0], g->cell_len[1], g->cell_len[2],
      g->dims[0], g->dims[1], g->dims[2], g->tdims[0], g->tdims[1], ring, cell);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

size_t lmd_sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n > 0 ? n : 1),
                                  0, 32);
  return bytes;
}

int lmd_sort_by_cell(int64_t n, int64_t ncell, const int32_t* cell, int32_t* cell_sorted,
                     int32_t* perm, int32_t* scratch_iota, void* temp, size_t temp_bytes,
                     void* stream) {
  if (n <= 0) return LMD_OK;
  if (n > 0x7fffffffLL) return LMD_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  iota_kernel<<<grid1d(n, 256), 256, 0, s>>>(n, scratch_iota);
  LMD_CHECK_LAUNCH();
  int end_bit = 1;
  while (end_bit < 31 && (1LL << end_bit) < ncell) ++end_bit;
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, bytes, cell, cell_sorted, scratch_iota,
                                                  perm, (int)n, 0, end_bit, s);
  if (e != cudaSuccess) return set_cuda_error(e);
  return LMD_OK;
}

int lmd_cell_ranges(int64_t n, int64_t ncell, int32_t base, const int32_t* cell_sorted,
                    int32_t* cell_start, int32_t* cell_count, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(cell_start, 0, ncell * sizeof(int32_t), s) != cudaSuccess ||
      cudaMemsetAsync(cell_count, 0, ncell * sizeof(int32_t), s) != cudaSuccess)
    return set_cuda_error(cudaGetLastError());
  if (n > 0) {
    cell_ranges_kernel<<<grid1d(n, 256), 256, 0, s>>>(n, base, cell_sorted, cell_start,
                                                      cell_count);
    LMD_CHECK_LAUNCH();
  }
  cell_count_fix_kernel<<<grid1d(ncell, 256), 256, 0, s>>>(ncell, cell_start, cell_count);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_merge_cell_tables(int64_t ncell, const int32_t* o_start, const int32_t* o_count,
                          const int32_t* h_start, const int32_t* h_count, int32_t* start,
                          int32_t* count, uint8_t* dup, void* stream) {
  merge_tables_kernel<<<grid1d(ncell, 256), 256, 0, (cudaStream_t)stream>>>(
      ncell, o_start, o_count, h_start, h_count, start, count, dup);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_gather_pos4(int64_t n, const int32_t* perm, const double* x, const double* y,
                    const double* z, const int8_t* own, double own_value, double* pos4,
                    void* stream) {
  if (n <= 0) return LMD_OK;
  gather_pos4_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, perm, x, y, z, own, own_value, reinterpret_cast<double4*>(pos4));
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_halo_count(const lmd_box* box, double margin, int64_t n, const double* x,
                   const double* y, const double* z, const int8_t* own, int32_t* count,
                   void* stream) {
  if (n <= 0) return LMD_OK;
  halo_count_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(make_boxk(box), margin, n,
                                                                      x, y, z, own, count);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

size_t lmd_scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(n > 0 ? n : 1));
  return bytes;
}

int lmd_exclusive_scan_i32(int64_t n, const int32_t* in, int32_t* out, void* temp,
                           size_t temp_bytes, void* stream) {
  if (n <= 0) return LMD_OK;
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, bytes, in, out, (int)n,
                                                (cudaStream_t)stream);
  if (e != cudaSuccess) return set_cuda_error(e);
  return LMD_OK;
}

int lmd_halo_emit(const lmd_box* box, double margin, int64_t n, const double* x,
                  const double* y, const double* z, const int8_t* own, const int32_t* offset,
                  double* hx, double* hy, double* hz, int32_t* owner, int8_t* shift,
                  void* stream) {
  if (n <= 0) return LMD_OK;
  halo_emit_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(
      make_boxk(box), margin, n, x, y, z, own, offset, hx, hy, hz, owner, shift);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_halo_refresh_pos4(const lmd_box* box, int64_t nh, const int32_t* owner,
                          const int8_t* shift, const double* x, const double* y,
                          const double* z, double* pos4_halo, void* stream) {
  if (nh <= 0) return LMD_OK;
  halo_refresh_kernel<<<grid1d(nh, 256), 256, 0, (cudaStream_t)stream>>>(
      make_boxk(box), nh, owner, shift, x, y, z, reinterpret_cast<double4*>(pos4_halo));
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_gather_pos4_soa(int64_t n, const int32_t* perm, const double* x, const double* y,
                        const double* z, double own_value, double* pos4, double* sx, double* sy,
                        double* sz, void* stream) {
  if (n <= 0) return LMD_OK;
  gather_pos4_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, perm, x, y, z, nullptr, own_value, reinterpret_cast<double4*>(pos4), sx, sy, sz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_halo_refresh_pos4_soa(const lmd_box* box, int64_t nh, const int32_t* owner,
                              const int8_t* shift, const double* x, const double* y,
                              const double* z, double* pos4_halo, double* sx, double* sy,
                              double* sz, void* stream) {
  if (nh <= 0) return LMD_OK;
  halo_refresh_kernel<<<grid1d(nh, 256), 256, 0, (cudaStream_t)stream>>>(
      make_boxk(box), nh, owner, shift, x, y, z, reinterpret_cast<double4*>(pos4_halo), sx, sy,
      sz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_halo_refresh_soa(const lmd_box* box, int64_t nh, const int32_t* owner,
                         const int8_t* shift, const double* x, const double* y, const double* z,
                         double* ox, double* oy, double* oz, void* stream) {
  if (nh <= 0) return LMD_OK;
  halo_refresh_soa_kernel<<<grid1d(nh, 256), 256, 0, (cudaStream_t)stream>>>(
      make_boxk(box), nh, owner, shift, x, y, z, ox, oy, oz, 1);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_halo_refresh_rows(const lmd_box* box, int64_t nh, const int32_t* owner,
                          const int8_t* shift, const double* x, const double* y, const double* z,
                          double* rows, void* stream) {
  if (nh <= 0) return LMD_OK;
  halo_refresh_soa_kernel<<<grid1d(nh, 256), 256, 0, (cudaStream_t)stream>>>(
      make_boxk(box), nh, owner, shift, x, y, z, rows, rows + 1, rows + 2, 3);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_scatter_forces(int64_t n, const int32_t* perm, const double* fx, const double* fy,
                       const double* fz, double* ox, double* oy, double* oz, void* stream) {
  if (n <= 0) return LMD_OK;
  scatter_forces_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(n, perm, fx, fy, fz,
                                                                          ox, oy, oz);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
