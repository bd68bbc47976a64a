// Does DMMA (mma.sync m8n8k4 f64) share issue/throughput with DFMA/DMUL on B200?  Each thread runs
// TILES independent DMMA accumulations interleaved with NF independent DFMA chains per iteration;
// reports the time per iteration against the DMMA-only and DFMA-only costs (DESIGN.md §5 K4).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int TILES, int NF>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  double c[TILES > 0 ? TILES : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = 0; }
#pragma unroll
  for (int k = 0; k < NF; ++k) f[k] = threadIdx.x * 1e-3 + k;
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(av), "d"(bv));
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k] = fma(f[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int k = 0; k < NF; ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <int TILES, int NF>
int run(double* d, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  const int iters = 4000, threads = 256, grid = sms * 4;
  mix_kernel<TILES, NF><<<grid, threads>>>(d, 10, 1.0000001, 1e-7);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  mix_kernel<TILES, NF><<<grid, threads>>>(d, iters, 1.0000001, 1e-7);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)grid * threads / 32 * iters;
  const double mma_tf = 256.0 * 2 * TILES * warps / ms / 1e9;
  const double fma_tf = 2.0 * 32 * NF * warps / ms / 1e9;
  printf("DMMA x%-2d + DFMA x%-3d per iter: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", TILES, NF, ms,
         mma_tf, fma_tf, mma_tf + fma_tf);
  return 0;
}

int main() {
  double* d;
  CK(cudaMalloc(&d, 8));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s sms %d\n", prop.name, prop.multiProcessorCount);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;
  run<8, 0>(d, sms, e0, e1);
  run<0, 64>(d, sms, e0, e1);
  run<8, 16>(d, sms, e0, e1);
  run<8, 32>(d, sms, e0, e1);
  run<8, 64>(d, sms, e0, e1);
  run<16, 16>(d, sms, e0, e1);
  run<16, 32>(d, sms, e0, e1);
  return 0;
}
