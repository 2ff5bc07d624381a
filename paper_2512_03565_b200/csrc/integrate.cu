// K11: velocity-Verlet halves and boundary handling, elementwise on the device.
//
// integrator.py:21-48 and domain.py:69-94, reproducing numpy's expression
// order (x += v*dt + f*(h*dt*dt); v += (f + fo)*(h*dt)) and np.mod's
// fmod-plus-sign-fix remainder so trajectories match the reference bit for bit.
#include <math.h>

#include "common.cuh"

namespace lmd {

__device__ __forceinline__ double np_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if ((b < 0.0) != (m < 0.0)) m += b;
  } else {
    m = copysign(0.0, b);
  }
  return m;
}

__global__ void boundaries_kernel(int64_t n, double lo0, double lo1, double lo2, double hi0,
                                  double hi1, double hi2, int p0, int p1, int p2,
                                  double* __restrict__ x, double* __restrict__ y,
                                  double* __restrict__ z, double* __restrict__ vx,
                                  double* __restrict__ vy, double* __restrict__ vz,
                                  int32_t* __restrict__ diverged) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double* X[3] = {x, y, z};
  double* V[3] = {vx, vy, vz};
  const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  const int per[3] = {p0, p1, p2};
  for (int ax = 0; ax < 3; ++ax) {
    const double L = hi[ax] - lo[ax];
    double p = X[ax][k];
    if (p > hi[ax] + L || p < lo[ax] - L) {
      atomicOr(diverged, 1);
      return;
    }
    if (per[ax]) {
      X[ax][k] = np_mod(p - lo[ax], L) + lo[ax];
    } else {
      if (p > hi[ax]) {
        p = 2.0 * hi[ax] - p;
        V[ax][k] = -V[ax][k];
      }
      if (p < lo[ax]) {
        p = 2.0 * lo[ax] - p;
        V[ax][k] = -V[ax][k];
      }
      X[ax][k] = p;
    }
  }
}

__global__ void verlet_kernel(int64_t n, int phase, double dt, double half_over_m,
                              double* __restrict__ x, double* __restrict__ y,
                              double* __restrict__ z, double* __restrict__ vx,
                              double* __restrict__ vy, double* __restrict__ vz,
                              double* __restrict__ fx, double* __restrict__ fy,
                              double* __restrict__ fz, double* __restrict__ ox,
                              double* __restrict__ oy, double* __restrict__ oz,
                              int32_t* __restrict__ nonfinite) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double* X[3] = {x, y, z};
  double* V[3] = {vx, vy, vz};
  double* F[3] = {fx, fy, fz};
  double* O[3] = {ox, oy, oz};
  bool bad = false;
  for (int ax = 0; ax < 3; ++ax) {
    if (phase == 0) {
      const double c = __dmul_rn(__dmul_rn(half_over_m, dt), dt);
      const double f = F[ax][k];
      const double xn = __dadd_rn(X[ax][k], __dadd_rn(__dmul_rn(V[ax][k], dt), __dmul_rn(f, c)));
      X[ax][k] = xn;
      O[ax][k] = f;
      F[ax][k] = 0.0;
      bad |= !isfinite(xn) || !isfinite(V[ax][k]);
    } else if (phase == 1) {
      const double c = __dmul_rn(half_over_m, dt);
      const double vn = __dadd_rn(V[ax][k], __dmul_rn(__dadd_rn(F[ax][k], O[ax][k]), c));
      V[ax][k] = vn;
      bad |= !isfinite(vn) || !isfinite(X[ax][k]);
    } else {
      // phase 2: this step's post-force half followed by the next step's
      // pre-force half in one pass (the same expressions in the same order,
      // so the trajectory is bit for bit that of the two launches)
      const double c1 = __dmul_rn(half_over_m, dt);
      const double c2 = __dmul_rn(__dmul_rn(half_over_m, dt), dt);
      const double f = F[ax][k];
      const double vn = __dadd_rn(V[ax][k], __dmul_rn(__dadd_rn(f, O[ax][k]), c1));
      const double x0 = X[ax][k];
      const double xn = __dadd_rn(x0, __dadd_rn(__dmul_rn(vn, dt), __dmul_rn(f, c2)));
      V[ax][k] = vn;
      X[ax][k] = xn;
      O[ax][k] = f;
      F[ax][k] = 0.0;
      bad |= !isfinite(vn) || !isfinite(x0) || !isfinite(xn);
    }
  }
  if (bad) atomicOr(nonfinite, 1);
}

}  // namespace lmd

using namespace lmd;

// max over particles of |r - r_ref|^2 with the reference's unfused
// (dx^2 + dy^2) + dz^2 (containers.py:23-38); r_ref rows are (x, y, z).
// Non-negative doubles order like their bit patterns: one 64-bit atomicMax
// per warp on the bits.
__global__ void max_disp2_kernel(int64_t n, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 const double* __restrict__ ref,
                                 unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double dx = __dadd_rn(x[k], -ref[3 * k]);
    const double dy = __dadd_rn(y[k], -ref[3 * k + 1]);
    const double dz = __dadd_rn(z[k], -ref[3 * k + 2]);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    m = fmax(m, d2);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

extern "C" {

int lmd_max_displacement2(int64_t n, const double* x, const double* y, const double* z,
                          const double* ref_xyz, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (n <= 0) return LMD_OK;
  const int64_t blocks = cdiv(n, 256) < 148 * 8 ? cdiv(n, 256) : 148 * 8;
  max_disp2_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, x, y, z, ref_xyz,
                                                    (unsigned long long*)out);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_apply_boundaries(const lmd_box* box, int64_t n, double* x, double* y, double* z,
                         double* vx, double* vy, double* vz, int32_t* diverged, void* stream) {
  if (n <= 0) return LMD_OK;
  boundaries_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, box->lo[0], box->lo[1], box->lo[2], box->hi[0], box->hi[1], box->hi[2],
      box->periodic[0], box->periodic[1], box->periodic[2], x, y, z, vx, vy, vz, diverged);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

int lmd_verlet_step(int64_t n, int phase, double dt, double mass, double* x, double* y,
                    double* z, double* vx, double* vy, double* vz, double* fx, double* fy,
                    double* fz, double* ox, double* oy, double* oz, int32_t* nonfinite,
                    void* stream) {
  if (phase < 0 || phase > 2) return LMD_ERR_CONFIG;
  if (n <= 0) return LMD_OK;
  verlet_kernel<<<(unsigned)cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(
      n, phase, dt, 0.5 / mass, x, y, z, vx, vy, vz, fx, fy, fz, ox, oy, oz, nonfinite);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
