// unscoped.cu — SURVEY §8(f) row f2: the unscoped high-order fit (one node, max_depth = 0) up to
// degree 14 (𝓛 = 680), §3 / Fig. 1 (L_max = 6, 10, 14 on N_p = 8^6).
//
// The level path solves the normal equations from raw moments (K5), which squares the condition
// number of the monomial Vandermonde Λ; at p >= 12 that is beyond fp64.  The paper's own solve is a QR
// of Λ.  This path computes exactly that R without forming the monomial Gram:
//   1. V = the Vandermonde of the tensor Legendre basis s_a s_b s_c P_a(x) P_b(y) P_c(z) (s_k = √(2k+1)),
//      same polynomial space, well conditioned on space-filling point sets; the RHS f is its last column;
//   2. G = [V f]ᵀ[V f] by a split-K SYRK on the FP64 tensor cores (DMMA m8n8k4; fixed-order split
//      reduction);
//   3. bordered Cholesky G = R_Vᵀ R_V in one CTA: the last row gives y = Qᵀf and ρ = ‖f − V V⁺f‖;
//   4. the monomial basis is Λ = V C with C upper triangular in the Algorithm-2 order (x^a = Σ_k e_ak
//      s_k P_k(x) per axis; β ≤ α componentwise ⇒ index(β) ≤ index(α)), so Λ = Q (R_V C): the R of the
//      paper's QR is R = R_V C — a product of triangles, its diagonal a plain product (no cancellation);
//   5. the column-rejection walk of reading G9 on R D⁻¹ (D = column norms of R = those of Λ), the same
//      Householder re-triangularisation as K5q, restricted to the rows a reflector can touch, and the
//      back substitution R_S c̃ = (Qᵀf)_S;  a_α = c̃_α / D_α (monomial form, used by Horner);
//   6. r = f − Λ(u)·a over the points (Horner) with the octant energies Σr² for the node statistics.
// Evaluation uses the ordinary K7 path (one node).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "fmi.h"
#include "horner.cuh"

namespace fmi {

namespace {

constexpr int UMAXP = 14;
constexpr int UT = 64;    // SYRK tile
constexpr int UTHREADS = 256;

// x^a = Σ_k c_ue[a][k] · s_k P_k(x)
__constant__ double c_ue[(UMAXP + 1) * (UMAXP + 1)];

// ---- 1. Legendre rows: V[i][col], row-major with ld LDV (multiple of UT) --------------------------
template <int P>
__global__ void __launch_bounds__(UTHREADS)
    k_leg_rows(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
               const double* __restrict__ f, int64_t r0, int64_t nr, const uint8_t* __restrict__ el,
               const uint8_t* __restrict__ em, const uint8_t* __restrict__ en, int L, int LDV,
               double* __restrict__ V, double cx, double cy, double cz, double sc) {
  __shared__ double tp[3][32][P + 1];  // s_k P_k of the 32 rows' local coordinates, per axis
  const int64_t base = (int64_t)blockIdx.x * 32;
  if (threadIdx.x < 96) {
    const int row = threadIdx.x & 31, ax = threadIdx.x >> 5;
    const int64_t i = r0 + base + row;
    double u = 0.0;
    if (base + row < nr) {
      const double* src = ax == 0 ? ux : (ax == 1 ? uy : uz);
      u = to_local(src[i], ax == 0 ? cx : (ax == 1 ? cy : cz), sc);  // the node frame
    }
    double pm = 1.0, pk = u;  // Bonnet: (k+1) P_{k+1} = (2k+1) u P_k - k P_{k-1}
    tp[ax][row][0] = 1.0;
    if (P >= 1) tp[ax][row][1] = u * sqrt(3.0);
    for (int k = 1; k < P; ++k) {
      const double pn = ((2.0 * k + 1.0) * u * pk - k * pm) / (k + 1.0);
      pm = pk;
      pk = pn;
      tp[ax][row][k + 1] = pn * sqrt(2.0 * (k + 1) + 1.0);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * LDV; e += UTHREADS) {
    const int row = e / LDV, col = e - row * LDV;
    if (base + row >= nr) continue;
    double v = 0.0;
    if (col < L) v = tp[0][row][el[col]] * tp[1][row][em[col]] * tp[2][row][en[col]];
    else if (col == L) v = f[r0 + base + row];
    V[(base + row) * (int64_t)LDV + col] = v;
  }
}

// ---- 2. split-K SYRK: part[split] (+)= V[rows of split]ᵀ V[rows of split], lower tiles only ------------
// Tensor-core variant (FP64 DMMA, mma.sync m8n8k4): the Gram is a dense contraction, so each warp
// issues 8x8x4 double MMAs — 256 FMAs per instruction instead of 32.  CTA = 4 warps on a 64x64 tile
// (2x2 warps of 32x32 = 4x4 MMA sub-tiles), k-slices of 16 rows staged in shared memory (rows padded to
// 72 doubles: the four rows a fragment load touches fall in two bank phases).
constexpr int SYD_THREADS = 128, SYD_K = 16, SYD_LD = 72;
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(SYD_THREADS)
    k_syrk_dmma(const double* __restrict__ V, int64_t nr, int LDV, int nsplit, bool accumulate,
                double* __restrict__ part) {
  const int t = blockIdx.x;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  const int split = blockIdx.y;
  const int64_t k0 = nr * split / nsplit, k1 = nr * (split + 1) / nsplit;
  __shared__ __align__(16) double As[SYD_K][SYD_LD], Bs[SYD_K][SYD_LD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // the warp's 32x32 quadrant
  const int fr = lane & 3, fc = lane >> 2;  // fragment row (k) and column (m or n) of this lane
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int NQ = (SYD_K * UT) / SYD_THREADS;  // 8 loads per operand per thread
  double pa[NQ], pb[NQ];
  auto fetch = [&](int64_t kb) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = threadIdx.x + q * SYD_THREADS;
      const int kk = e / UT, c = e % UT;
      const int64_t row = kb + kk;
      pa[q] = row < k1 ? V[row * LDV + ti * UT + c] : 0.0;
      pb[q] = row < k1 ? V[row * LDV + tj * UT + c] : 0.0;
    }
  };
  if (k0 < k1) fetch(k0);
  for (int64_t kb = k0; kb < k1; kb += SYD_K) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = threadIdx.x + q * SYD_THREADS;
      As[e / UT][e % UT] = pa[q];
      Bs[e / UT][e % UT] = pb[q];
    }
    __syncthreads();
    if (kb + SYD_K < k1) fetch(kb + SYD_K);
#pragma unroll
    for (int ks = 0; ks < SYD_K; ks += 4) {
      double af[4], bf[4];  // A[m][k] = V[k][m], B[k][n] = V[k][n]
#pragma unroll
      for (int ms = 0; ms < 4; ++ms) af[ms] = As[ks + fr][wm * 32 + ms * 8 + fc];
#pragma unroll
      for (int ns = 0; ns < 4; ++ns) bf[ns] = Bs[ks + fr][wn * 32 + ns * 8 + fc];
#pragma unroll
      for (int ms = 0; ms < 4; ++ms)
#pragma unroll
        for (int ns = 0; ns < 4; ++ns) dmma884(acc[ms][ns][0], acc[ms][ns][1], af[ms], bf[ns]);
    }
    __syncthreads();
  }
  double* out = part + (int64_t)split * LDV * LDV;
#pragma unroll
  for (int ms = 0; ms < 4; ++ms)
#pragma unroll
    for (int ns = 0; ns < 4; ++ns)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t o = (int64_t)(ti * UT + wm * 32 + ms * 8 + fc) * LDV + tj * UT + wn * 32 + ns * 8 + 2 * fr + h;
        out[o] = accumulate ? out[o] + acc[ms][ns][h] : acc[ms][ns][h];
      }
}

// G[i][j] = Σ_split part[split][i][j] (fixed order), lower triangle of the leading n×n block
__global__ void k_sum_splits(const double* __restrict__ part, int nsplit, int LDV, int n, double* __restrict__ G,
                             double* __restrict__ diag0) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e / n), j = (int)(e % n);
  if (j > i) return;
  double s = 0.0;
  for (int p = 0; p < nsplit; ++p) s += part[(int64_t)p * LDV * LDV + (int64_t)i * LDV + j];
  G[(int64_t)i * LDV + j] = s;
  if (i == j) diag0[i] = s;
}

// ---- 3. bordered Cholesky (one CTA): lower factor in place; row n-1 = [yᵀ, ρ] -------------------------
// Right-looking, 32-column panels (the K5 scheme with runtime n): the panel (rows j0..n-1) is staged
// column-major in shared memory; warp 0 factors the diagonal block with each lane's row in registers
// (shuffles, no CTA barrier per column); the rows below are solved thread-per-row in registers; the
// trailing lower triangle (in global memory, L2-resident) is updated with 4x4 register tiles.
constexpr int CKB = 32;
constexpr int CTHREADS = 512;
__host__ __device__ inline int chol_ldp(int n) {
  const int r4 = (n + 3) & ~3;
  return r4 % 16 == 0 ? r4 + 2 : r4;
}

// A Schur pivot below kZeroPivot of the column's own squared norm (diag0) is a column in the span of the
// previous ones up to rounding (degenerate point sets, e.g. coplanar): it is set to 0 and its monomial
// counterparts are then rejected by the G9 walk.
constexpr double kZeroPivot = 1e-13;
// CholeskyQR2 trigger: nodes with fewer than kCholQR2Fill·𝓛 points (near-interpolation leaves: κ(V) of
// 1e5 at n ≈ 𝓛, p = 12) or a relative Schur pivot below kCholQR2Ratio get the second pass.  The smallest
// relative pivot underestimates κ² by orders of magnitude (2e-4 at κ = 1.7e5), so it alone cannot decide.
constexpr double kCholQR2Ratio = 1e-2;
constexpr double kCholQR2Fill = 16.0;
__global__ void __launch_bounds__(CTHREADS) k_chol_bordered(double* __restrict__ G, int n, int LDV,
                                                            const double* __restrict__ diag0,
                                                            int* __restrict__ nonpd, double* __restrict__ minrat) {
  extern __shared__ __align__(16) double Pn[];  // [CKB][LDP]
  __shared__ double sinv[CKB];
  const int LDP = chol_ldp(n);
  G += (int64_t)blockIdx.x * LDV * LDV;  // batched: node blockIdx.x of the batch
  diag0 += (int64_t)blockIdx.x * LDV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double rmin = INFINITY;  // warp 0: smallest Schur pivot / column norm² (1/κ² estimate), ρ excluded
  for (int j0 = 0; j0 < n; j0 += CKB) {
    const int bw = min(CKB, n - j0), R = n - j0;
    for (int e = tid; e < R * bw; e += CTHREADS) {
      const int r = e / bw, c = e - r * bw;
      Pn[c * LDP + r] = (r >= bw || c <= r) ? G[(int64_t)(j0 + r) * LDV + j0 + c] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      double row[CKB];
#pragma unroll
      for (int c = 0; c < CKB; ++c) row[c] = (c <= lane && lane < bw) ? Pn[c * LDP + lane] : 0.0;
#pragma unroll
      for (int c = 0; c < CKB; ++c) {
        if (c < bw) {
          const int j = j0 + c;
          const double d = __shfl_sync(0xffffffffu, row[c], c);
          double p;
          if (j == n - 1) {
            p = sqrt(fmax(d, 0.0));  // ρ: residual norm of the least-squares fit
          } else {
            const bool ok = d > kZeroPivot * diag0[j];
            p = ok ? sqrt(d) : 0.0;
            if (ok) rmin = fmin(rmin, d / diag0[j]);
            if (lane == 0 && !ok) atomicAdd(nonpd, 1);
          }
          const double inv = p > 0.0 ? 1.0 / p : 0.0;
          if (lane == 0) sinv[c] = inv;
          row[c] = lane == c ? p : row[c] * inv;
          if (p > 0.0) {
#pragma unroll
            for (int c2 = c + 1; c2 < CKB; ++c2) {
              const double l2 = __shfl_sync(0xffffffffu, row[c], c2);
              if (lane >= c2) row[c2] -= row[c] * l2;
            }
          }
        }
      }
      if (lane < bw) {
#pragma unroll
        for (int c = 0; c < CKB; ++c)
          if (c <= lane) Pn[c * LDP + lane] = row[c];
      }
    }
    __syncthreads();
    for (int r = bw + tid; r < R; r += CTHREADS) {
      double x[CKB];
#pragma unroll
      for (int c = 0; c < CKB; ++c) x[c] = c < bw ? Pn[c * LDP + r] : 0.0;
#pragma unroll
      for (int c = 0; c < CKB; ++c) {
        if (c < bw) {
          const double inv = sinv[c];
          const double lc = x[c] * inv;
          x[c] = lc;
          if (inv > 0.0) {
#pragma unroll
            for (int c2 = c + 1; c2 < CKB; ++c2)
              if (c2 < bw) x[c2] -= lc * Pn[c * LDP + c2];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CKB; ++c)
        if (c < bw) Pn[c * LDP + r] = x[c];
    }
    __syncthreads();
    for (int e = tid; e < R * bw; e += CTHREADS) {
      const int r = e / bw, c = e - r * bw;
      if (r >= bw || c <= r) G[(int64_t)(j0 + r) * LDV + j0 + c] = Pn[c * LDP + r];
    }
    // trailing update G[i][k] -= Σ_c P[i][c] P[k][c], j1 <= k <= i < n, 4x4 tiles
    const int j1 = j0 + bw, R2 = n - j1;
    if (R2 > 0) {
      const int nt4 = (R2 + 3) / 4;
      const int ntile = nt4 * (nt4 + 1) / 2;
      for (int t = tid; t < ntile; t += CTHREADS) {
        int ti = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        while (ti * (ti + 1) / 2 > t) --ti;
        const int tk = t - ti * (ti + 1) / 2;
        const int i0 = j1 + 4 * ti, k0 = j1 + 4 * tk;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        const double* pi = Pn + (i0 - j0);
        const double* pk = Pn + (k0 - j0);
        for (int c = 0; c < bw; ++c) {
          const double2 a01 = *reinterpret_cast<const double2*>(pi + c * LDP);
          const double2 a23 = *reinterpret_cast<const double2*>(pi + c * LDP + 2);
          const double2 b01 = *reinterpret_cast<const double2*>(pk + c * LDP);
          const double2 b23 = *reinterpret_cast<const double2*>(pk + c * LDP + 2);
          const double av[4] = {a01.x, a01.y, a23.x, a23.y};
          const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int i = i0 + a, k = k0 + b;
            if (i < n && k <= i) G[(int64_t)i * LDV + k] -= acc[a][b];
          }
      }
    }
    __syncthreads();
  }
  if (tid == 0 && minrat) minrat[blockIdx.x] = rmin;
}

// ---- 3b. CholeskyQR2 second pass for ill-conditioned nodes ------------------------------------------
// One Cholesky of the Gram carries an error ~κ(V)²·eps into R_V; nodes with few points per unknown
// (n ≈ 𝓛 at leaves) reach κ(V)² ~ 1e8.  The second pass makes R_V as accurate as the Householder R of
// the paper's QR whenever κ(V)² eps < 1: Q1 = V L1⁻ᵀ (row-wise forward substitution),
// L2 = chol(Q1ᵀQ1) (≈ I), R_V = (L1 L2)ᵀ.  Zero pivots of L1 give zero Q1 columns and zero L2
// columns, so a column in the span of its predecessors keeps its representation (row of L1).
//
// Q1 rows in place: x L1ᵀ = v, i.e. x_j = (v_j − Σ_{k<j} L1[j][k] x_k) / L1[j][j] (0 for a zero pivot);
// warp = QRB rows sharing every L1 row load, x kept in shared memory.
constexpr int QRB = 4, QWARPS = 4;
__global__ void __launch_bounds__(QWARPS * 32)
    k_rows_trsm(double* __restrict__ V, int64_t nr, int LDV, int n, const double* __restrict__ G) {
  extern __shared__ __align__(16) double xs[];  // [QWARPS][QRB][n]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * QWARPS + warp) * QRB;
  if (r0 >= nr) return;
  double* x = xs + (int64_t)warp * QRB * n;
  for (int e = lane; e < QRB * n; e += 32) {
    const int q = e / n, c = e - q * n;
    x[e] = r0 + q < nr ? V[(r0 + q) * LDV + c] : 0.0;
  }
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    const double* Lj = G + (int64_t)j * LDV;
    double acc[QRB];
#pragma unroll
    for (int q = 0; q < QRB; ++q) acc[q] = 0.0;
    for (int k = lane; k < j; k += 32) {
      const double l = Lj[k];
#pragma unroll
      for (int q = 0; q < QRB; ++q) acc[q] = fma(l, x[q * n + k], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < QRB; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    const double d = Lj[j];
    if (lane < QRB) {
      double a = acc[0];
#pragma unroll
      for (int q = 1; q < QRB; ++q) if (lane == q) a = acc[q];
      x[lane * n + j] = d > 0.0 ? (x[lane * n + j] - a) / d : 0.0;
    }
    __syncwarp();
  }
  for (int e = lane; e < QRB * n; e += 32) {
    const int q = e / n, c = e - q * n;
    if (r0 + q < nr) V[(r0 + q) * LDV + c] = x[e];
  }
}

// Lc[i][k] = Σ_{m=k..i} L1[i][m] L2[m][k] (lower, row-major, ld LDV)
__global__ void k_tri_product(const double* __restrict__ L1, const double* __restrict__ L2, int n, int LDV,
                              double* __restrict__ Lc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e / n), k = (int)(e % n);
  if (k > i) return;
  double v = 0.0;
  for (int m = k; m <= i; ++m) v = fma(L1[(int64_t)i * LDV + m], L2[(int64_t)m * LDV + k], v);
  Lc[(int64_t)i * LDV + k] = v;
}

// ---- 4. R = R_V C, augmented with [y; ρ] as column L; column-major A[col * LA + row] -----------------
__global__ void k_r_mono(const double* __restrict__ G, int L, int LDV, const uint8_t* __restrict__ el,
                         const uint8_t* __restrict__ em, const uint8_t* __restrict__ en, int P,
                         double* __restrict__ A) {
  const int LA = L + 1;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)LA * LA) return;
  G += (int64_t)blockIdx.y * LDV * LDV;  // batched: node blockIdx.y of the batch
  A += (int64_t)blockIdx.y * LA * LA;
  const int j = (int)(e / LA), i = (int)(e % LA);  // column j, row i
  double v = 0.0;
  if (j == L) {
    v = G[(int64_t)L * LDV + i];  // y_i (i < L) and ρ (i = L): the factor's last row
  } else if (i <= j) {
    const int aj = el[j], bj = em[j], cj = en[j];
    for (int k = i; k <= j; ++k) {
      const int ak = el[k], bk = em[k], ck = en[k];
      if (ak > aj || bk > bj || ck > cj) continue;
      const double c = c_ue[aj * (UMAXP + 1) + ak] * c_ue[bj * (UMAXP + 1) + bk] * c_ue[cj * (UMAXP + 1) + ck];
      if (c == 0.0) continue;
      v = fma(G[(int64_t)k * LDV + i], c, v);  // R_V[i][k] = L_factor[k][i]
    }
  }
  (void)P;
  A[(int64_t)j * LA + i] = v;
}

__device__ __forceinline__ double ublock_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// ---- 5. equilibration, column-rejection walk (G9) and back substitution (one CTA) ---------------------
__global__ void __launch_bounds__(UTHREADS)
    k_unscoped_solve(double* __restrict__ A, int L, double delta, double* __restrict__ work, int* __restrict__ kept,
                     NodeTable nt, int64_t node0) {
  const int LA = L + 1;
  // batched: node node0 + blockIdx.x, its R in A[blockIdx.x], 3L doubles and L ints of scratch
  A += (int64_t)blockIdx.x * LA * LA;
  double* dinv = work + (int64_t)blockIdx.x * 3 * L;
  double* piv = dinv + L;
  double* sol = dinv + 2 * L;
  kept += (int64_t)blockIdx.x * L;
  const int64_t node = node0 + blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarp = UTHREADS / 32;
  __shared__ double red[UTHREADS / 32];
  // D_j = ‖column j of R‖ = ‖column j of Λ‖ (Q orthonormal)
  for (int j = warp; j < L; j += nwarp) {
    double s = 0.0;
    for (int i = lane; i <= j; i += 32) { const double t = A[(int64_t)j * LA + i]; s = fma(t, t, s); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dinv[j] = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < L * LA; e += UTHREADS) A[e] *= dinv[e / LA];
  __syncthreads();
  // walk: k = rows consumed by the kept columns; column j's non-zeros are rows k..j
  int k = 0;
  for (int j = 0; j < L; ++j) {
    double* Aj = A + (int64_t)j * LA;
    double part = 0.0;
    for (int i = k + tid; i <= j; i += UTHREADS) { const double t = Aj[i]; part = fma(t, t, part); }
    const double nrm2 = ublock_sum(part, red);
    const double nrm = sqrt(nrm2);
    const bool keep = dinv[j] > 0.0 && nrm > delta;
    if (tid == 0) { kept[j] = keep ? k : -1; piv[j] = keep ? nrm : 0.0; }
    if (!keep) { __syncthreads(); continue; }
    if (j > k) {  // a reflector over rows k..j zeroes rows k+1..j of column j
      const double d = Aj[k];
      const double alpha = d >= 0.0 ? -nrm : nrm;
      const double v0 = d - alpha;
      const double vtv = nrm2 - d * d + v0 * v0;
      const double beta = vtv > 0.0 ? 2.0 / vtv : 0.0;
      for (int c = j + 1 + warp; c < LA; c += nwarp) {
        double* Ac = A + (int64_t)c * LA;
        double w = 0.0;
        for (int i = k + 1 + lane; i <= j; i += 32) w = fma(Aj[i], Ac[i], w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w = fma(v0, Ac[k], w);
        const double bw = beta * w;
        for (int i = k + 1 + lane; i <= j; i += 32) Ac[i] -= bw * Aj[i];
        if (lane == 0) Ac[k] -= bw * v0;
      }
      __syncthreads();
      if (tid == 0) Aj[k] = alpha;
    }
    __syncthreads();
    ++k;
  }
  // back substitution over the kept columns (row kept[j] holds column j's pivot), rhs = column L
  const double* Ar = A + (int64_t)L * LA;
  for (int i = tid; i < L; i += UTHREADS) sol[i] = kept[i] >= 0 ? Ar[kept[i]] : 0.0;
  __syncthreads();
  for (int j = L - 1; j >= 0; --j) {
    const int row = kept[j];
    if (row < 0) continue;  // uniform across the block
    const double* Aj = A + (int64_t)j * LA;
    const double cj = sol[j] / Aj[row];
    __syncthreads();
    for (int i = tid; i < j; i += UTHREADS)
      if (kept[i] >= 0) sol[i] -= Aj[kept[i]] * cj;
    if (tid == 0) sol[j] = cj;
    __syncthreads();
  }
  for (int i = tid; i < L; i += UTHREADS) {
    const double a = sol[i] * dinv[i];
    nt.coef[node * L + i] = a;
    nt.pcoef[node * L + i] = a;
  }
  if (tid == 0) {
    int rk = 0;
    double mn = INFINITY;
    for (int i = 0; i < L; ++i)
      if (kept[i] >= 0) { ++rk; mn = fmin(mn, piv[i]); }
    nt.rank[node] = rk;
    nt.minpiv[node] = rk ? mn : 0.0;
    nt.flag[node] = 1;  // fitted by the Householder-QR path
  }
}

// ---- 6. residual r -= Λ(u)·a over the root's points, Σr² per chunk (chunks lie in one octant) ----------
template <int P>
__global__ void __launch_bounds__(UTHREADS)
    k_unscoped_resid(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
                     double* __restrict__ r, NodeTable nt, int64_t first, const Chunk* __restrict__ chunks,
                     const int64_t* __restrict__ nchunks, double* __restrict__ partial) {
  constexpr int L = rank3(P);
  __shared__ __align__(16) double sa[(L + 1) & ~1];
  __shared__ double red[UTHREADS / 32];
  const int64_t cidx = blockIdx.x;
  if (cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  const int64_t node = first + (ck.owner >> 3);  // chunks of octant segments node*8 + o
  const Frame fr = node_frame(nt.cell[node]);
  for (int i = threadIdx.x; i < L; i += UTHREADS) sa[i] = nt.coef[node * L + i];
  __syncthreads();
  const SmemCoefVolatile cf(sa);
  double ss = 0.0;
  for (int64_t i = ck.start + threadIdx.x; i < ck.end; i += UTHREADS) {
    const double x = to_local(ux[i], fr.cx, fr.scale);
    const double y = to_local(uy[i], fr.cy, fr.scale);
    const double z = to_local(uz[i], fr.cz, fr.scale);
    const double v = r[i] - horner3<P>(cf, x, y, z);
    r[i] = v;
    ss = fma(v, v, ss);
  }
  const double t = ublock_sum(ss, red);
  if (threadIdx.x == 0) partial[cidx] = t;
}

// octant energies of the level's nodes in chunk order -> child_ss[(first + node)*8 + o]
__global__ void k_octant_ss(const double* __restrict__ partial, const int64_t* __restrict__ chunk_begin,
                            const int64_t* __restrict__ nchunks, NodeTable nt, int64_t first, int64_t nseg) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nseg) return;
  const int64_t c0 = chunk_begin[g], c1 = g + 1 < nseg ? chunk_begin[g + 1] : *nchunks;
  double s = 0.0;
  for (int64_t c = c0; c < c1; ++c) s += partial[c];
  nt.child_ss[first * 8 + g] = s;
}

// host: x^a = Σ_k e[a][k] · s_k P_k(x) from the monomial coefficients of the Legendre polynomials
std::vector<double> legendre_to_monomial_table() {
  constexpr int n = UMAXP + 1;
  std::vector<double> pc(n * n, 0.0);  // P_k(x) = Σ_j pc[k][j] x^j
  pc[0] = 1.0;
  pc[1 * n + 1] = 1.0;
  for (int k = 1; k + 1 < n; ++k)
    for (int j = 0; j < n; ++j) {
      double v = -k * pc[(k - 1) * n + j];
      if (j > 0) v += (2.0 * k + 1.0) * pc[k * n + j - 1];
      pc[(k + 1) * n + j] = v / (k + 1.0);
    }
  // invert the lower-triangular pc: x^a = Σ_k m[a][k] P_k  (pc[k][k] != 0)
  std::vector<double> m(n * n, 0.0);
  for (int a = 0; a < n; ++a) {
    // x^a = (1/pc[a][a]) (P_a - Σ_{j<a} pc[a][j] x^j)
    std::vector<double> row(n, 0.0);
    row[a] = 1.0 / pc[a * n + a];
    for (int j = 0; j < a; ++j) {
      const double c = -pc[a * n + j] / pc[a * n + a];
      for (int k = 0; k <= j; ++k) row[k] += c * m[j * n + k];
    }
    for (int k = 0; k < n; ++k) m[a * n + k] = row[k];
  }
  for (int a = 0; a < n; ++a)
    for (int k = 0; k < n; ++k) m[a * n + k] /= std::sqrt(2.0 * k + 1.0);  // basis s_k P_k
  return m;
}

}  // namespace

template <int P>
void unscoped_fit(const LevelCtx& c, cudaStream_t s) {
  constexpr int L = rank3(P), LA = L + 1;
  const int LDV = (LA + UT - 1) / UT * UT;
  const int nt_tiles = LDV / UT;
  const int ntile = nt_tiles * (nt_tiles + 1) / 2;
  static std::once_flag table_once;  // the constant table of this device (one process per GPU)
  std::call_once(table_once, [] {
    const std::vector<double> m = legendre_to_monomial_table();
    FMI_CK(cudaMemcpyToSymbol(c_ue, m.data(), m.size() * sizeof(double)));
  });
  // exponent tables (Algorithm-2 order)
  std::vector<uint8_t> ex(3 * L);
  {
    int i = 0;
    for (int l = 0; l <= P; ++l)
      for (int m = 0; m <= P - l; ++m)
        for (int n = 0; n <= P - l - m; ++n) { ex[i] = (uint8_t)l; ex[L + i] = (uint8_t)m; ex[2 * L + i] = (uint8_t)n; ++i; }
  }
  DBuf<uint8_t> dex(3 * L, s);
  FMI_CK(cudaMemcpyAsync(dex.p, ex.data(), 3 * L, cudaMemcpyHostToDevice, s));
  const uint8_t *el = dex.p, *em = dex.p + L, *en = dex.p + 2 * L;
  // the level's point ranges and cells (host copies drive the per-node Gram launches)
  const int64_t count = c.count;
  std::vector<int64_t> st(count), en_(count);
  std::vector<int4> cell(count);
  FMI_CK(cudaMemcpyAsync(st.data(), c.nt.start + c.first, count * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaMemcpyAsync(en_.data(), c.nt.end + c.first, count * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaMemcpyAsync(cell.data(), c.nt.cell + c.first, count * sizeof(int4), cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaStreamSynchronize(s));
  int64_t nmax = 0;
  for (int64_t b = 0; b < count; ++b) nmax = std::max(nmax, en_[b] - st[b]);
  // 1-2. per node: Legendre rows of the node frame over slabs of its rows, split-K DMMA SYRK; the
  // nodes' Grams are solved in batches (3-5: one CTA per node)
  const int64_t slab = std::min<int64_t>(std::max<int64_t>(nmax, 1),
                                         std::max<int64_t>(4096, ((int64_t)1 << 28) / LDV));  // <= 2 GB
  const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(count, ((int64_t)1 << 28) / ((int64_t)LDV * LDV)));
  const int nsplit_max = std::max(1, 148 * 3 / ntile);
  DBuf<double> V((size_t)slab * LDV, s), part((size_t)nsplit_max * LDV * LDV, s);
  DBuf<double> G((size_t)batch * LDV * LDV, s), diag0((size_t)batch * LDV, s);
  DBuf<double> A((size_t)batch * LA * LA, s), work((size_t)batch * 3 * L, s);
  DBuf<int> kept((size_t)batch * L, s), nonpd(1, s);
  FMI_CK(cudaMemsetAsync(nonpd.p, 0, sizeof(int), s));
  const size_t csmem = (size_t)CKB * chol_ldp(LA) * sizeof(double);
  // k_chol_bordered is shared by every degree: opt in once for the largest (p = 14) panel
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    const size_t most = (size_t)CKB * chol_ldp(rank3(UMAXP) + 1) * sizeof(double);
    FMI_CK(cudaFuncSetAttribute(k_chol_bordered, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)most));
  });
  // CholeskyQR2 (3b): FMI_CHOLQR2_RATIO overrides the relative-pivot trigger (0 disables the pass)
  static const double cholqr2_ratio = [] {
    const char* e = std::getenv("FMI_CHOLQR2_RATIO");
    return e ? std::atof(e) : kCholQR2Ratio;
  }();
  DBuf<double> minrat((size_t)batch, s), G2, Gc, diag2;
  std::vector<double> hrat(batch);
  const size_t tsmem = (size_t)QWARPS * QRB * LA * sizeof(double);
  static std::once_flag trsm_once;
  std::call_once(trsm_once, [] {
    const size_t most = (size_t)QWARPS * QRB * (rank3(UMAXP) + 1) * sizeof(double);
    FMI_CK(cudaFuncSetAttribute(k_rows_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)most));
  });
  int64_t n_cholqr2 = 0;
  for (int64_t b0 = 0; b0 < count; b0 += batch) {
    const int64_t nb = std::min(batch, count - b0);
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t node = b0 + b, s0 = st[node], n = en_[node] - s0;
      const double h = std::ldexp(1.0, -(cell[node].w + 1)), sc = std::ldexp(1.0, cell[node].w + 1);
      const double cx = (2.0 * cell[node].x + 1.0) * h, cy = (2.0 * cell[node].y + 1.0) * h,
                   cz = (2.0 * cell[node].z + 1.0) * h;
      const int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit_max, std::min(slab, n) / 512 + 1));
      for (int64_t r0 = 0; r0 < n; r0 += slab) {
        const int64_t nr = std::min(slab, n - r0);
        FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_leg_rows<P>, (unsigned)((nr + 31) / 32), UTHREADS, 0, c.ux + s0,
                   c.uy + s0, c.uz + s0, c.r + s0, r0, nr, el, em, en, L, LDV, V.p, cx, cy, cz, sc);
        FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_syrk_dmma, dim3((unsigned)ntile, (unsigned)nsplit), SYD_THREADS, 0, V.p, nr,
                   LDV, nsplit, r0 > 0, part.p);
      }
      FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_sum_splits, (unsigned)(((int64_t)LA * LA + 255) / 256), 256, 0, part.p,
                 nsplit, LDV, LA, G.p + b * LDV * LDV, diag0.p + b * LDV);
    }
    // 3-5
    FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_chol_bordered, (unsigned)nb, CTHREADS, csmem, G.p, LA, LDV, diag0.p, nonpd.p,
               minrat.p);
    // 3b. CholeskyQR2 pass for the nodes whose first factor may have lost digits (few points per unknown
    // or a small relative pivot) and whose rows fit one slab
    FMI_CK(cudaMemcpyAsync(hrat.data(), minrat.p, nb * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t node = b0 + b, s0 = st[node], n = en_[node] - s0;
      if (!(hrat[b] < cholqr2_ratio || (double)n < kCholQR2Fill * L) || cholqr2_ratio <= 0.0 || n > slab || n == 0)
        continue;
      if (!G2.p) {
        G2 = DBuf<double>((size_t)LDV * LDV, s);
        Gc = DBuf<double>((size_t)LDV * LDV, s);
        diag2 = DBuf<double>((size_t)LDV, s);
        FMI_CK(cudaMemsetAsync(Gc.p, 0, (size_t)LDV * LDV * sizeof(double), s));
      }
      const double h = std::ldexp(1.0, -(cell[node].w + 1)), sc = std::ldexp(1.0, cell[node].w + 1);
      const double cx = (2.0 * cell[node].x + 1.0) * h, cy = (2.0 * cell[node].y + 1.0) * h,
                   cz = (2.0 * cell[node].z + 1.0) * h;
      const int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit_max, n / 512 + 1));
      double* L1 = G.p + b * LDV * LDV;
      FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_leg_rows<P>, (unsigned)((n + 31) / 32), UTHREADS, 0, c.ux + s0, c.uy + s0,
                 c.uz + s0, c.r + s0, 0, n, el, em, en, L, LDV, V.p, cx, cy, cz, sc);
      FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_rows_trsm, (unsigned)((n + QWARPS * QRB - 1) / (QWARPS * QRB)), QWARPS * 32,
                 tsmem, V.p, n, LDV, LA, L1);
      FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_syrk_dmma, dim3((unsigned)ntile, (unsigned)nsplit), SYD_THREADS, 0, V.p, n,
                 LDV, nsplit, false, part.p);
      FMI_LAUNCH(KID_UNSCOPED_GRAM, s, k_sum_splits, (unsigned)(((int64_t)LA * LA + 255) / 256), 256, 0, part.p,
                 nsplit, LDV, LA, G2.p, diag2.p);
      FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_chol_bordered, 1u, CTHREADS, csmem, G2.p, LA, LDV, diag2.p, nonpd.p,
                 (double*)nullptr);
      FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_tri_product, (unsigned)(((int64_t)LA * LA + 255) / 256), 256, 0, L1, G2.p,
                 LA, LDV, Gc.p);
      FMI_CK(cudaMemcpyAsync(L1, Gc.p, (size_t)LDV * LDV * sizeof(double), cudaMemcpyDeviceToDevice, s));
      ++n_cholqr2;
    }
    FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_r_mono, dim3((unsigned)(((int64_t)LA * LA + 255) / 256), (unsigned)nb), 256, 0,
               G.p, L, LDV, el, em, en, P, A.p);
    FMI_LAUNCH(KID_UNSCOPED_SOLVE, s, k_unscoped_solve, (unsigned)nb, UTHREADS, 0, A.p, L, kDelta, work.p, kept.p,
               c.nt, c.first + b0);
  }
  V.release();
  part.release();
  prof_units(KID_UNSCOPED_SOLVE, n_cholqr2);
  // 6. residual and octant energies over the level's octant segments
  {
    int64_t points = 0;
    for (int64_t b = 0; b < count; ++b) points += en_[b] - st[b];
    const int64_t nseg = count * 8;
    DBuf<int64_t> counts(nseg, s), begin(nseg, s), nch(1, s);
    const int64_t ch = std::max<int64_t>(1024, (points + 148 * 4 - 1) / (148 * 4));
    const int64_t maxc = points / ch + nseg + 1;
    DBuf<Chunk> chunks(maxc, s);
    DBuf<double> partial(maxc, s);
    make_chunks(c.nt.child_start + c.first * 9, nullptr, nseg, ch, counts.p, begin.p, nch.p, chunks.p, maxc, s);
    FMI_LAUNCH(KID_RESIDUAL, s, k_unscoped_resid<P>, (unsigned)maxc, UTHREADS, 0, c.ux, c.uy, c.uz, c.r, c.nt,
               c.first, chunks.p, nch.p, partial.p);
    FMI_LAUNCH(KID_RESIDUAL_REDUCE, s, k_octant_ss, (unsigned)((nseg + 127) / 128), 128, 0, partial.p, begin.p, nch.p,
               c.nt, c.first, nseg);
    FMI_CK(cudaStreamSynchronize(s));
  }
}

#define FMI_INST(P) template void unscoped_fit<P>(const LevelCtx&, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5) FMI_INST(6) FMI_INST(7)
FMI_INST(8) FMI_INST(9) FMI_INST(10) FMI_INST(11) FMI_INST(12) FMI_INST(13) FMI_INST(14)
#undef FMI_INST

}  // namespace fmi
