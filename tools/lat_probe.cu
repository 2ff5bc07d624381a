// Dependent-chain latencies (one warp): DFMA, DMUL, MUFU.RCP64H + Newton,
// LDS.64 pointer chase.  Cycles per dependent step; JSON lines.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kN = 4096;
__global__ void dfma_chain(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rcp_chain(double* out, long long* cyc, double a) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) {
    double y;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void lds_chain(double* out, long long* cyc) {
  __shared__ int s[1024];
  for (int k = threadIdx.x; k < 1024; k += 32) s[k] = (k * 37 + 11) & 1023;
  __syncwarp();
  int p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 64);
  for (int r = 0; r < 2; ++r) {
    dfma_chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
    rcp_chain<<<1, 32>>>(out, cyc, 0.5);
    lds_chain<<<1, 32>>>(out, cyc);
    cudaDeviceSynchronize();
  }
  printf("{\"dfma_dep_cycles\": %.2f, \"rcp64h_plus_dadd_dep_cycles\": %.2f, \"lds32_dep_cycles\": %.2f}\n",
         (double)cyc[0] / kN, (double)cyc[1] / kN, (double)cyc[2] / kN);
  return 0;
}
