// FP64 pipe peak microbenchmark (the roofline denominator; MEASURED_PEAKS.json
// has no FP64 entry).  Independent DFMA chains, 16 per thread, so the pipe and
// not the DFMA latency bounds the rate.
#include "common.cuh"

namespace lmd {

__global__ void dfma_burn_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = fma(r[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += r[k];
  if (s == 1234.5) out[threadIdx.x] = s;
}

}  // namespace lmd

extern "C" {

/* Launch blocks x threads threads running `iters` x 128 DFMA each (2 flops per DFMA);
 * the caller times the launch with events on `stream`. */
int lmd_dfma_burn(int blocks, int threads, int iters, double* scratch, void* stream) {
  lmd::dfma_burn_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(scratch, iters, 0.999999,
                                                                      1e-7);
  LMD_CHECK_LAUNCH();
  return LMD_OK;
}

}  // extern "C"
