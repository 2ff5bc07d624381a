// Microbenchmark: data-pipe cost of 64-bit shared-memory and L1-resident
// global gathers under controlled lane -> bank-pair patterns.  Decides the
// conflict model the staged Verlet-list schedule is built for.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bank_probe tools/bank_probe.cu
//   tools/bank_probe   -> one JSON line per pattern: cycles per warp-load per SM
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kSlots = 2048;      // 16 KB of doubles
constexpr int kIters = 4096;
constexpr int kThreads = 256;

// slot of lane l at iteration it for pattern p (row offset varies per
// iteration so consecutive loads are different words)
__device__ __forceinline__ int slot_of(int p, int l, int it) {
  const int row = (it * 7) & 63;  // 64 rows of 16 bank-pairs -> 1024 slots
  int bp, r;
  switch (p) {
    case 0: bp = l & 15; r = row + (l >> 4); break;            // halves distinct, halves share banks
    case 1: bp = l & 15; r = row + 32 * (l >> 4); break;       // halves distinct, other half 32 rows away
    case 2: bp = l >> 1; r = row + (l & 1); break;              // 2-way within a half (16 bp over warp)
    case 3: bp = 0; r = row + l; break;                          // 32-way
    case 4: bp = (l & 7); r = row + (l >> 3); break;             // 4 lanes per bp (2 per half)
    case 5: bp = l & 15; r = row; break;                         // l and l+16 same word (broadcast)
    case 6: bp = (l * 5 + it) & 15; r = row + (l >> 4) * 3; break;  // distinct per half, rotated
    case 7: {  // pseudo-random
      unsigned h = (unsigned)(l * 2654435761u) ^ (unsigned)(it * 40503u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      return (int)(h % 1024u);
    }
    default: bp = l & 15; r = row; break;
  }
  return ((r & 63) * 16 + bp) % 1024;
}

template <int P>
__global__ void smem_kernel(double* out, long long* cyc) {
  __shared__ double s[kSlots];
  for (int k = threadIdx.x; k < kSlots; k += blockDim.x) s[k] = k * 0.5;
  __syncthreads();
  const int l = threadIdx.x & 31;
  int sl[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) sl[u] = slot_of(P, l, u);
  double acc = 0.0;
  int off = 0;
  long long t0 = clock64();
  for (int it = 0; it < kIters; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += s[(sl[u] + off) & 1023];
    off += 16 * 8;
  }
  long long t1 = clock64();
  if (acc == -1.0) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int P>
__global__ void gmem_kernel(const double* __restrict__ g, double* out, long long* cyc) {
  const int l = threadIdx.x & 31;
  const double* base = g + (blockIdx.x & 7) * kSlots;
  int sl[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) sl[u] = slot_of(P, l, u);
  double acc = 0.0;
  int off = 0;
  long long t0 = clock64();
  for (int it = 0; it < kIters; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += __ldg(base + ((sl[u] + off) & 1023));
    off += 16 * 8;
  }
  long long t1 = clock64();
  if (acc == -1.0) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <int P>
void run(const char* name, bool shared, double* g, double* out, long long* cyc, int sms) {
  const int blocks = sms * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    cudaEventRecord(a);
    if (shared) smem_kernel<P><<<blocks, kThreads>>>(out, cyc);
    else gmem_kernel<P><<<blocks, kThreads>>>(g, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double loads_per_sm = (double)blocks / sms * (kThreads / 32) * kIters;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("{\"mem\": \"%s\", \"pattern\": \"%s\", \"ms\": %.4f, \"sm_cycles_per_warp_load\": %.3f}\n",
         shared ? "shared" : "global", name, ms, cycles / loads_per_sm);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *g, *out;
  long long* cyc;
  cudaMalloc(&g, 8 * kSlots * sizeof(double));
  cudaMemset(g, 0, 8 * kSlots * sizeof(double));
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, 8);
  for (int sh = 1; sh >= 0; --sh) {
    run<0>("halves_distinct_bp_shared_between_halves", sh, g, out, cyc, sms);
    run<1>("halves_distinct_bp_far_rows", sh, g, out, cyc, sms);
    run<2>("2way_within_half", sh, g, out, cyc, sms);
    run<3>("32way", sh, g, out, cyc, sms);
    run<4>("4_lanes_per_bp", sh, g, out, cyc, sms);
    run<5>("broadcast_pairs", sh, g, out, cyc, sms);
    run<6>("rotated_distinct_per_half", sh, g, out, cyc, sms);
    run<7>("random", sh, g, out, cyc, sms);
  }
  return 0;
}
