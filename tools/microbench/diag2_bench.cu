// Micro-benchmark of the K5 diagonal-block factorisation (one warp, lane = row, row in registers):
// the kept software-pipelined chol_block (csrc/solve.cu) vs a 16 + 16 split (columns 0..15, the rank-16
// update of rows/columns 16..31 from shared memory, columns 16..31) with the same arithmetic in the same
// order (results must be bit-identical).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a diag2_bench.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
constexpr int KB = 32;
__device__ __forceinline__ double rsqrt_pivot(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r * r, 1.0);
  return fma(fma(e, 0.375, 0.5), r * e, r);
}
// columns [C0, C1) of the right-looking factorisation, updates restricted to columns < C1
template <int KR, int C0, int C1>
__device__ __forceinline__ void chol_cols(double (&row)[KR], int bwd, const double* dv, double delta2, int lane,
                                          double& myinv, double& mys) {
  auto pivot = [&](int c, double sjj, double& inv, double& p) {
    const bool keep = c < bwd && dv[c] > 0.0 && sjj > delta2;
    const double r = rsqrt_pivot(keep ? sjj : 1.0);
    inv = keep ? r : 0.0;
    p = keep ? sjj * r : 0.0;
  };
  double sjj = __shfl_sync(0xffffffffu, row[C0], C0), inv, p;
  pivot(C0, sjj, inv, p);
#pragma unroll
  for (int c = C0; c < C1; ++c) {
    if (lane == c) { myinv = inv; mys = sjj; }
    row[c] = lane == c ? p : row[c] * inv;
    double sjj_n = 0.0, inv_n = 0.0, p_n = 0.0;
    if (c + 1 < C1) {
      const double l = __shfl_sync(0xffffffffu, row[c], c + 1);
      row[c + 1] = fma(lane >= c + 1 ? -row[c] : 0.0, l, row[c + 1]);
      sjj_n = __shfl_sync(0xffffffffu, row[c + 1], c + 1);
      pivot(c + 1, sjj_n, inv_n, p_n);
    }
#pragma unroll
    for (int b0 = c + 2; b0 < C1; b0 += 8) {
      double l2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (b0 + k < C1) l2[k] = __shfl_sync(0xffffffffu, row[c], b0 + k);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (b0 + k < C1) row[b0 + k] = fma(lane >= b0 + k ? -row[c] : 0.0, l2[k], row[b0 + k]);
    }
    sjj = sjj_n; inv = inv_n; p = p_n;
  }
}
template <int KR>
__device__ __forceinline__ void chol_block(double (&row)[KR], int bwd, const double* dv, double delta2, int lane,
                                           double& myinv, double& mys) {
  myinv = 0.0; mys = INFINITY;
  chol_cols<KR, 0, KR>(row, bwd, dv, delta2, lane, myinv, mys);
}
// 16 + 16: columns 0..15 (their updates only within 0..15), then every row's columns 16..31 take the 16
// updates of columns 0..15 in column order from the shared copy of rows 16..31, then columns 16..31
template <int KR>
__device__ __forceinline__ void chol_split(double (&row)[KR], int bwd, const double* dv, double delta2, int lane,
                                           double& myinv, double& mys, double* sm /* [16][16] */) {
  constexpr int H = KR / 2;
  myinv = 0.0; mys = INFINITY;
  chol_cols<KR, 0, H>(row, bwd, dv, delta2, lane, myinv, mys);
  if (lane >= H) {
#pragma unroll
    for (int c = 0; c < H; ++c) sm[(lane - H) * H + c] = row[c];
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < H; ++c) {
    const double rc = -row[c];
#pragma unroll
    for (int c2 = H; c2 < KR; c2 += 2) {  // L[c2][c], L[c2+1][c] (broadcast reads)
      const double a = sm[(c2 - H) * H + c], b = sm[(c2 + 1 - H) * H + c];
      row[c2] = fma(lane >= c2 ? rc : 0.0, a, row[c2]);
      row[c2 + 1] = fma(lane >= c2 + 1 ? rc : 0.0, b, row[c2 + 1]);
    }
  }
  __syncwarp();
  chol_cols<KR, H, KR>(row, bwd, dv, delta2, lane, myinv, mys);
}
// W-column blocks: columns [b, b+W) by chol_cols, then the rank-W update of columns >= b+W from the
// shared copy of rows >= b+W (same updates, same order as the right-looking loop)
template <int KR, int W, int B>
__device__ __forceinline__ void chol_splitw_step(double (&row)[KR], int bwd, const double* dv, double delta2, int lane,
                                                 double& myinv, double& mys, double* sm) {
  if constexpr (B < KR) {
    chol_cols<KR, B, B + W>(row, bwd, dv, delta2, lane, myinv, mys);
    if constexpr (B + W < KR) {
      if (lane >= B + W) {
#pragma unroll
        for (int c = 0; c < W; ++c) sm[(lane - B - W) * W + c] = row[B + c];
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const double rc = -row[B + c];
#pragma unroll
        for (int c2 = B + W; c2 < KR; ++c2)
          row[c2] = fma(lane >= c2 ? rc : 0.0, sm[(c2 - B - W) * W + c], row[c2]);
      }
      __syncwarp();
    }
    chol_splitw_step<KR, W, B + W>(row, bwd, dv, delta2, lane, myinv, mys, sm);
  }
}
template <int KR, int W>
__device__ __forceinline__ void chol_splitw(double (&row)[KR], int bwd, const double* dv, double delta2, int lane,
                                            double& myinv, double& mys, double* sm) {
  myinv = 0.0; mys = INFINITY;
  chol_splitw_step<KR, W, 0>(row, bwd, dv, delta2, lane, myinv, mys, sm);
}
template <int V>
__global__ void k(const double* __restrict__ A, const double* __restrict__ dv, double* __restrict__ out,
                  long long* cyc, int reps) {
  const int lane = threadIdx.x & 31;
  __shared__ double sm_all[8][16 * 24];
  double* sm = sm_all[threadIdx.x >> 5];
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    double row[KB];
#pragma unroll
    for (int c = 0; c < KB; ++c) row[c] = (c <= lane) ? A[c * KB + lane] + 1e-300 * it : 0.0;
    double myinv, mys;
    if (V == 0) chol_block<KB>(row, KB, dv, 1e-12, lane, myinv, mys);
    else if (V == 1) chol_split<KB>(row, KB, dv, 1e-12, lane, myinv, mys, sm);
    else if (V == 2) chol_splitw<KB, 8>(row, KB, dv, 1e-12, lane, myinv, mys, sm);
    else chol_splitw<KB, 16>(row, KB, dv, 1e-12, lane, myinv, mys, sm);
    if (it == reps - 1) {
#pragma unroll
      for (int c = 0; c < KB; ++c) out[lane * KB + c] = row[c];
    }
    acc += row[lane] + myinv;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
  out[KB * KB + lane] += acc;
}
int main() {
  double h[KB * KB], d[KB];
  for (int i = 0; i < KB; ++i) {
    d[i] = 1.0;
    for (int j = 0; j < KB; ++j) h[j * KB + i] = (i == j ? 1.0 : 0.9 / (1 + (i > j ? i - j : j - i)));
  }
  double *dA, *dd, *o0, *o1; long long* dc;
  cudaMalloc(&dA, sizeof h); cudaMalloc(&dd, sizeof d); cudaMalloc(&o0, 8 * (KB * KB + KB));
  cudaMalloc(&o1, 8 * (KB * KB + KB)); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice); cudaMemcpy(dd, d, sizeof d, cudaMemcpyHostToDevice);
  const char* names[4] = {"chol_block (kept, pipelined)", "chol_split (16+16)", "splitw W=8", "splitw W=16"};
  double ref[KB * KB];
  for (int warps = 1; warps <= 8; warps *= 8) {
    for (int v = 0; v < 4; ++v) {
      long long c = 0;
      double* o = v == 0 ? o0 : o1;
      for (int warm = 0; warm < 2; ++warm) {
        if (v == 0) k<0><<<1, 32 * warps>>>(dA, dd, o, dc, 200);
        if (v == 1) k<1><<<1, 32 * warps>>>(dA, dd, o, dc, 200);
        if (v == 2) k<2><<<1, 32 * warps>>>(dA, dd, o, dc, 200);
        if (v == 3) k<3><<<1, 32 * warps>>>(dA, dd, o, dc, 200);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      }
      double r[KB * KB];
      cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
      if (v == 0) memcpy(ref, r, sizeof r);
      printf("%d warp(s)  %-30s %6lld cycles/block  bit-identical %s\n", warps, names[v], c,
             memcmp(ref, r, sizeof r) == 0 ? "yes" : "NO");
    }
  }
  return 0;
}
