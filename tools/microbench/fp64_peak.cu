// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA (vector) and DMMA (mma.sync m8n8k4 f64).
// Used to state the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int TILES>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(av), "d"(bv));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 8));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d\n", prop.name, sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocksPerSm : {1, 2, 4, 8}) {
    for (int threads : {256, 512}) {
      int grid = sms * blocksPerSm;
      dfma_kernel<8><<<grid, threads>>>(d, 100, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, threads>>>(d, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * grid * threads;
      printf("DFMA blocks/SM %d threads %d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSm, threads, flops / ms / 1e9, ms);
    }
  }
  for (int blocksPerSm : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      int grid = sms * blocksPerSm;
      dmma_kernel<4><<<grid, threads>>>(d, 100, 1.0, 1.0);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<4><<<grid, threads>>>(d, iters / 4, 1.0, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 4 * (double)(iters / 4) * grid * (threads / 32);
      printf("DMMA blocks/SM %d threads %d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSm, threads, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
