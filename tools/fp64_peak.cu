// FP64 pipe microbenchmark: measured peak for the roofline denominator.
// Independent DFMA chains (8 per thread) so the pipe, not latency, bounds it.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (OP == 0) r[k] = fma(r[k], a, b);
        else if (OP == 1) r[k] = __dadd_rn(r[k], b);
        else r[k] = __dmul_rn(r[k], a);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, p.multiProcessorCount, clk);
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"dfma", "dadd", "dmul"};
  for (int op = 0; op < 3; ++op) {
    int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2000;
    double best = 1e30;
    for (int rep = 0; rep < 12; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) dfma_kernel<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      else if (op == 1) dfma_kernel<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      else dfma_kernel<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2 && ms < best) best = ms;
    }
    double ops = (double)blocks * threads * iters * 16 * 8;
    double flops = ops * (op == 0 ? 2.0 : 1.0);
    printf(", \"%s_ops_per_s\": %.4e, \"%s_tflops\": %.3f", names[op], ops / (best * 1e-3), names[op], flops / (best * 1e-3) / 1e12);
  }
  printf("}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
