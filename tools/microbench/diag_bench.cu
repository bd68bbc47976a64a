// Micro-benchmark of the K5 diagonal-block factorisation (one warp, lane = row, row in registers):
// cycles per 32-column block for variants of the pivot computation.  nvcc -O3 -arch=sm_100a diag_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int KB = 32;
template <int V>
__global__ void k(const double* __restrict__ A, double* __restrict__ out, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  __shared__ double Pn[KB * KB];
  __shared__ double sc[KB];
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    for (int e = lane; e < KB * KB; e += 32) Pn[e] = A[e];
    __syncwarp();
    double row[KB];
#pragma unroll
    for (int c = 0; c < KB; ++c) row[c] = (c <= lane) ? Pn[c * KB + lane] : 0.0;
#pragma unroll
    for (int c = 0; c < KB; ++c) {
      const double sjj = __shfl_sync(0xffffffffu, row[c], c);
      double inv, p;
      if (V == 0) { p = sjj > 1e-12 ? sqrt(sjj) : 0.0; inv = p > 0.0 ? 1.0 / p : 0.0; }
      else if (V == 1) { inv = sjj > 1e-12 ? rsqrt(sjj) : 0.0; p = sjj * inv; }
      else if (V == 3) { inv = sjj > 1e-12 ? rsqrt(sjj) : 0.0; p = sjj * inv; }
      else if (V == 5) { inv = (double)rsqrtf((float)sjj); p = sjj * inv; }  // floor (inexact)
      else {  // fp32 rsqrt seed + two Newton steps in fp64
        const double y0 = (double)rsqrtf((float)sjj);
        double y = y0 * (1.5 - 0.5 * sjj * y0 * y0);
        y = y * (1.5 - 0.5 * sjj * y * y);
        inv = sjj > 1e-12 ? y : 0.0; p = sjj * inv;
      }
      row[c] = lane == c ? p : row[c] * inv;
      if (V <= 2 || V == 5) {
        if (p > 0.0) {
#pragma unroll
          for (int c2 = c + 1; c2 < KB; ++c2) {
            const double l2 = __shfl_sync(0xffffffffu, row[c], c2);
            if (lane >= c2) row[c2] -= row[c] * l2;
          }
        }
      } else {  // column broadcast through shared memory: one store per lane, broadcast loads
        sc[lane] = row[c];
        __syncwarp();
        if (p > 0.0) {
#pragma unroll
          for (int c2 = c + 1; c2 < KB; ++c2)
            if (lane >= c2) row[c2] -= row[c] * sc[c2];
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int c = 0; c < KB; ++c) acc += row[c];
  }
  long long t1 = clock64();
  out[lane] = acc;
  if (lane == 0) *cyc = (t1 - t0) / reps;
}
int main() {
  double h[KB * KB];
  for (int i = 0; i < KB; ++i)
    for (int j = 0; j < KB; ++j) h[j * KB + i] = (i == j ? KB + 1.0 : 1.0 / (1 + i + j));  // column-major SPD
  double *dA, *dout; long long* dc; cudaMalloc(&dA, sizeof h); cudaMalloc(&dout, 32 * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  long long c;
  k<0><<<1, 32>>>(dA, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("sqrt+div   : %lld cycles/block\n", c);
  k<1><<<1, 32>>>(dA, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("rsqrt      : %lld cycles/block\n", c);
  k<2><<<1, 32>>>(dA, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("f32 seed+NR: %lld cycles/block\n", c);
  k<3><<<1, 32>>>(dA, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("rsqrt+smem : %lld cycles/block\n", c);
  k<5><<<1, 32>>>(dA, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("f32 rsqrt  : %lld cycles/block\n", c);
  return 0;
}
