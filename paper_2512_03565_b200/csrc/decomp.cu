// Ghost-layer exchange helpers for the brick decomposition (SURVEY §8e,
// decomposition.py): the per-stage pack (gather + image shift) as one
// kernel, and the gather of row-major ghost positions into the pos4 backing.
#include "common.cuh"

namespace lmd {

// out[k] = source(idx[k]) with out[k][axis] += shift, where source indexes
// [owned (SoA ox, oy, oz) | ghosts received so far (row-major g)].
__global__ void ghost_pack_kernel(int64_t count, const int32_t* __restrict__ idx, int64_t n_owned,
                                  const double* __restrict__ ox, const double* __restrict__ oy,
                                  const double* __restrict__ oz, const double* __restrict__ g,
                                  int axis, double shift, double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const int64_t s = idx[k];
  double p[3];
  if (s < n_owned) {
    p[0] = ox[s];
    p[1] = oy[s];
    p[2] = oz[s];
  } else {
    const double* r = g + 3 * (s - n_owned);
    p[0] = r[0];
    p[1] = r[1];
    p[2] = r[2];
  }
  p[axis] = __dadd_rn(p[axis], shift);   // the image position pos + (hi - lo) / (lo - hi)
  out[3 * k] = p[0];
  out[3 * k + 1] = p[1];
  out[3 * k + 2] = p[2];
}

__global__ void gather_pos4_rows_kernel(int64_t n, const int32_t* __restrict__ perm,
                                        const double* __restrict__ rows, double own_value,
                                        double4* __restrict__ pos4) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t s = perm ? perm[k] : k;
  pos4[k] = make_double4(rows[3 * s], rows[3 * s + 1], rows[3 * s + 2], own_value);
}

__global__ void gather_rows_soa_kernel(int64_t n, const int32_t* __restrict__ perm,
                                       const double* __restrict__ rows, double* __restrict__ x,
                                       double* __restrict__ y, double* __restrict__ z) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t s = perm ? perm[k] : k;
  x[k] = rows[3 * s];
  y[k] = rows[3 * s + 1];
  z[k] = rows[3 * s + 2];
}

}  // namespace lmd

using namespace lmd;

extern "C" {

int lmd_ghost_pack(int64_t count, const int32_t* idx, int64_t n_owned, const double* ox,
                   const double* oy, const double* oz, const double* ghost_rows, int axis,
                   double shift, double* out_rows, void* stream) {
  if (count <= 0) return LMD_OK;
  if (axis < 0 || axis > 2) return LMD_ERR_CONFIG;
  ghost_pack_kernel<<<(unsigned)cdiv(count, 256), 256, 0, (cudaStream_t)stream>>>(
      count, idx, n_owned, ox, oy, oz, ghost_rows, axis, shift, out_rows);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_gather_pos4_rows(int64_t n, const int32_t* perm, const double* rows, double own_value,
                         double* pos4, void* stream) {
  if (n <= 0) return LMD_OK;
  gather_pos4_rows_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, perm, rows, own_value, reinterpret_cast<double4*>(pos4));
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_gather_rows_soa(int64_t n, const int32_t* perm, const double* rows, double* x, double* y,
                        double* z, void* stream) {
  if (n <= 0) return LMD_OK;
  gather_rows_soa_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(n, perm, rows,
                                                                                  x, y, z);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
