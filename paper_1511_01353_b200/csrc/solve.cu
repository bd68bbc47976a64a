// solve.cu — K5: batched node solve (DESIGN.md §5 K5), one CTA per node.
//
// PAPER.md Algorithm 2 computes P_F = R⁻¹ Qᵀ f from the QR of Λ.  In Gram form, with the
// raw moments M and projection b of K4/K6:
//   D_α   = sqrt(G_αα) = sqrt(M_{2α}) / α!          (column norms of Λ)
//   G̃_αβ  = M_{α+β} / sqrt(M_{2α} M_{2β})           (Jacobi-equilibrated Gram; factorials cancel)
//   b̃_α   = b_α / sqrt(M_{2α})                     (= (Λᵀ r)_α / D_α)
//   G̃ c̃ = b̃  by Cholesky G̃ = R̃ᵀR̃  (R̃ = the R of the QR of Λ D⁻¹ up to row signs)
//   monomial coefficients a_α = c̃_α / sqrt(M_{2α}) = P_F,α / α!   (used by Horner in K6/K7)
// Rank rule (reading G9, identical to the oracle's QR column rejection): at step j the Schur
// complement diagonal s_jj equals the squared distance of equilibrated column j from the span of the
// kept columns; the column is dropped (coefficient 0) iff s_jj <= kDelta², or M_{2α} = 0.
//
// Layout and algorithm: the lower factor is kept per node in global memory (L2-resident while the
// node is processed; reused by the refinement solves), packed row-major, with b̃ appended as row 𝓛 —
// factoring the bordered matrix yields y = R̃⁻ᵀ b̃ in that row, so no forward substitution is needed.
// Right-looking blocked Cholesky: per block of KB columns the column panel (rows j0..𝓛, RHS row
// included) is factored in shared memory column by column (the same pivots, rejections and updates
// as the unblocked algorithm), written back, and the trailing triangle is updated once with 4x4
// register tiles.  The back substitution R̃ c̃ = y is blocked the same way (small triangular solve of
// the diagonal block, then a row-contiguous GEMV update of the rows above).
#include <mutex>
#include <algorithm>
#include <vector>

#include <cstdlib>
#include "fmi_internal.cuh"

namespace fmi {

namespace {

// threads per node: 128 for the small systems (more nodes per SM), 256 for 𝓛 >= 220 (p >= 9)
template <int P>
constexpr int k5_threads() { return rank3(P) >= 220 ? 256 : (rank3(P) >= 100 ? 128 : 64); }
constexpr int KB = 32;
#ifndef FMI_K5_PANEL_RB
#define FMI_K5_PANEL_RB 18
#endif

struct BasisTab {
  uint8_t l[286], m[286], n[286];
};

template <int P>
BasisTab make_basis() {
  BasisTab b{};
  int i = 0;
  for (int l = 0; l <= P; ++l)
    for (int m = 0; m <= P - l; ++m)
      for (int n = 0; n <= P - l - m; ++n) { b.l[i] = (uint8_t)l; b.m[i] = (uint8_t)m; b.n[i] = (uint8_t)n; ++i; }
  return b;
}

__host__ __device__ constexpr int64_t tri(int i) { return (int64_t)i * (i + 1) / 2; }

// optional phase timing (build with -DFMI_K5_TIMING): thread 0 of each CTA accumulates clock64 deltas
// between barriers; CTA 0 prints them at exit (tools/k5_timing.sh)
#ifdef FMI_K5_TIMING
#define K5T_DECL long long k5t_last = clock64(), k5t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define K5T(ph)                                  \
  if (tid == 0) {                                \
    const long long t_ = clock64();              \
    k5t_acc[ph] += t_ - k5t_last;                \
    k5t_last = t_;                               \
  }
#define K5T_PRINT                                                                                          \
  if (tid == 0 && blockIdx.x == 0)                                                                        \
    printf("k5 phases (cycles, CTA 0, L=%d): assemble %lld panel_load %lld diag %lld trsm %lld "          \
           "trailing %lld backsub %lld epilogue %lld\n", L, k5t_acc[0], k5t_acc[1], k5t_acc[2], k5t_acc[3], \
           k5t_acc[4], k5t_acc[5], k5t_acc[6]);
#else
#define K5T_DECL
#define K5T(ph)
#define K5T_PRINT
#endif

// 1/sqrt(x) for the Schur pivots (x in (delta², ~1]: no special operands): the hardware approximation
// and one third-order Newton step, branch-free (the library rsqrt carries a slow-path call)
__device__ __forceinline__ double rsqrt_pivot(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r * r, 1.0);
  return fma(fma(e, 0.375, 0.5), r * e, r);
}

// Cholesky with column rejection (G9) of a KR x KR diagonal block held one row per lane (row[c], c <= lane;
// rows >= bwd and entries c > lane are zero), software-pipelined: right after column c is scaled, column
// c+1 takes its update and its pivot (shuffle + reciprocal square root) is started, and the remaining
// columns' updates are issued behind it; no branches and no stores inside the loop.  Each lane keeps the
// pivot quantities of its own column (myinv: 1/p or 0; mys: the Schur pivot s_cc, for the minimum).
template <int KR>
__device__ __forceinline__ void chol_block(double (&row)[KR], int bwd, const double* __restrict__ dv, double delta2,
                                           int lane, double& myinv, double& mys) {
  auto pivot = [&](int c, double sjj, double& inv, double& p) {
    const bool keep = c < bwd && dv[c] > 0.0 && sjj > delta2;
    const double r = rsqrt_pivot(keep ? sjj : 1.0);
    inv = keep ? r : 0.0;
    p = keep ? sjj * r : 0.0;
  };
  double sjj = __shfl_sync(0xffffffffu, row[0], 0), inv, p;
  pivot(0, sjj, inv, p);
  myinv = 0.0;
  mys = INFINITY;
#pragma unroll
  for (int c = 0; c < KR; ++c) {
    if (lane == c) { myinv = inv; mys = sjj; }
    row[c] = lane == c ? p : row[c] * inv;
    double sjj_n = 0.0, inv_n = 0.0, p_n = 0.0;
    if (c + 1 < KR) {
      const double l = __shfl_sync(0xffffffffu, row[c], c + 1);
      row[c + 1] = fma(lane >= c + 1 ? -row[c] : 0.0, l, row[c + 1]);
      sjj_n = __shfl_sync(0xffffffffu, row[c + 1], c + 1);
      pivot(c + 1, sjj_n, inv_n, p_n);
    }
#pragma unroll
    for (int b0 = c + 2; b0 < KR; b0 += 8) {
      double l2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (b0 + k < KR) l2[k] = __shfl_sync(0xffffffffu, row[c], b0 + k);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (b0 + k < KR) row[b0 + k] = fma(lane >= b0 + k ? -row[c] : 0.0, l2[k], row[b0 + k]);
    }
    sjj = sjj_n;
    inv = inv_n;
    p = p_n;
  }
}

template <int P>
struct K5Shape {
  static constexpr int Q = 2 * P;
  static constexpr int K = rank3(Q);
  static constexpr int L = rank3(P);
  static constexpr int64_t NAB = tri(L) + L;  // packed lower factor + RHS row
  // panel column stride: rows padded to 4 (16-byte vectors of 4 rows), and not a multiple of 16 so that
  // consecutive columns of one row fall in different banks
  // (>= L + 8: the 8-row MMA tiles of the trailing update read up to 7 rows past the last one)
  static constexpr int LDP0 = (L + 8 + 1) & ~1;
  static constexpr int LDP = LDP0 % 16 == 0 ? LDP0 + 2 : LDP0;
  // shared: moments [K], dinv, piv, 1/piv, y/c [L], column-major panel [KB x LDP], exponents
  // the panel area also holds two 32x32 diagonal blocks in the back substitution
  static constexpr int PN = KB * LDP > 2 * KB * KB ? KB * LDP : 2 * KB * KB;
  static constexpr size_t SMEM = ((size_t)K + 4 * L + (size_t)PN + 8) * sizeof(double) + 3 * L + 16;
};

// NT = threads per node: k5_threads<P>() for full levels; 256 for levels with fewer nodes than CTA slots
// (the top levels of every build are latency-bound: one node per SM)
template <int P, int NT = k5_threads<P>()>
__global__ void __launch_bounds__(NT, NT == 512 ? 1 : (NT == 256 ? 2 : (NT == 128 ? 3 : 6)))
    k_solve(const double* __restrict__ mom, int mode, const double* __restrict__ segrhs, double* __restrict__ delta,
            NodeTable nt, int64_t first, int64_t count, double* __restrict__ fac,
            const __grid_constant__ BasisTab bt, double delta2, double refine2, double refine_fill,
            double mom_tol, int64_t n_root, double defer_tau, int64_t* __restrict__ nflag) {
  using S = K5Shape<P>;
  constexpr int Q = S::Q, K = S::K, L = S::L;
  constexpr int K5_THREADS = NT, K5_WARPS = K5_THREADS / 32;
  extern __shared__ __align__(16) double sm[];
  double* sM = sm;          // [K]
  double* dinv = sM + K;    // [L]
  double* piv = dinv + L;   // [L]
  double* pinv = piv + L;   // [L]  1/piv (0 for rejected columns)
  double* sy = pinv + L;    // [L]  b̃ -> y -> c̃
  constexpr int LDP = S::LDP;
  // column-major panel, 16-byte aligned: Pn[c * LDP + r] = row j0 + r, column j0 + c
  double* Pn = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sy + L) + 15) & ~uintptr_t(15));
  uint8_t* bl = reinterpret_cast<uint8_t*>(Pn + S::PN);
  uint8_t* bm = bl + L;
  uint8_t* bn = bm + L;
  __shared__ double smin_sh;
  __shared__ double ynorm_sh;
  __shared__ double errw[K5_WARPS];
  __shared__ double sinv[KB];  // inverse pivots of the current panel
  __shared__ double Dg[KB * KB];  // lookahead: the next panel's diagonal block (column-major, ld KB)
  // warp index broadcast from lane 0: provably warp-uniform for the compiler, so the warp-specialised
  // branches (diagonal block on warp 0) keep their shuffles and MMAs on the converged fast path
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  for (int i = tid; i < L; i += K5_THREADS) { bl[i] = bt.l[i]; bm[i] = bt.m[i]; bn[i] = bt.n[i]; }
  __syncthreads();

  K5T_DECL
  for (int64_t node = blockIdx.x; node < count; node += gridDim.x) {
    K5T(6)
    // mode 1 (refinement): bit-1 nodes only; mode 2 (direct-moment re-solve): bit-2 nodes only
    if (mode == 1 && !(nt.flag[first + node] & 2)) continue;
    if (mode == 2 && !(nt.flag[first + node] & 4)) continue;
    double* A = fac + node * S::NAB;
    const double* mp = mom + node * (int64_t)(2 * K + L);
    const double* bndg = mp + K + L;
    const double* bnd = Pn;  // the panel area is free until the factorisation: the bounds staged there
    if (tid == 0) smin_sh = INFINITY;
    for (int e = tid; e < K; e += K5_THREADS) {
      sM[e] = mp[e];
      if (mode == 0) Pn[e] = bndg[e];
    }
    static_assert(KB * S::LDP >= K, "the bound staging needs the panel area");
    __syncthreads();
    if (mode == 0 && !(sM[0] > 0.0)) {  // below the moment tree (M_000 = 0): accumulate directly
      if (tid == 0) {
        nt.flag[first + node] = 4;
        atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 1), 1ull);
      }
      __syncthreads();
      continue;
    }
    for (int i = tid; i < L; i += K5_THREADS) {
      const double m2 = sM[basis_index(Q, 2 * bl[i], 2 * bm[i], 2 * bn[i])];
      const double di = m2 > 0.0 ? 1.0 / sqrt(m2) : 0.0;
      dinv[i] = di;
      double b;
      if (mode == 1) {  // b1 = Λᵀ r1 over the node's 8 octant segments, fixed order
        b = 0.0;
        for (int o = 0; o < 8; ++o) b += segrhs[(node * 8 + o) * (L + 1) + i];
      } else {
        b = mp[K + i];
      }
      sy[i] = b * di;
    }
    __syncthreads();

    if (mode == 1) {
      // ---- refinement: forward substitution with the stored factor (blocked, rows contiguous) -----
      for (int i = tid; i < L; i += K5_THREADS) {
        piv[i] = A[tri(i) + i];
        pinv[i] = piv[i] > 0.0 ? 1.0 / piv[i] : 0.0;
      }
      __syncthreads();
      for (int j0 = 0; j0 < L; j0 += KB) {
        const int j1 = min(j0 + KB, L);
        // sy[i] -= Σ_{k<j0} L[i][k] y[k] for i in the block: one warp per row
        for (int i = j0 + warp; i < j1; i += K5_WARPS) {
          const double* Ai = A + tri(i);
          double v = 0.0;
          for (int k = lane; k < j0; k += 32) v = fma(Ai[k], sy[k], v);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) sy[i] -= v;
        }
        __syncthreads();
        if (warp == 0) {  // diagonal block, sequential rows
          for (int i = j0; i < j1; ++i) {
            const double* Ai = A + tri(i);
            double v = 0.0;
            for (int k = j0 + lane; k < i; k += 32) v = fma(Ai[k], sy[k], v);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sy[i] = piv[i] > 0.0 ? (sy[i] - v) / piv[i] : 0.0;
            __syncwarp();
          }
        }
        __syncthreads();
      }
    } else {
      // ---- assemble the equilibrated Gram + RHS row and check the moments' rounding bound -------
      double errl = 0.0;
      for (int i = warp; i <= L; i += K5_WARPS) {  // warp per packed row; row L = RHS
        double* Ai = A + tri(i);
        if (i == L) {
          for (int k = lane; k < L; k += 32) Ai[k] = sy[k];
          continue;
        }
        const int li = bl[i], mi = bm[i], ni = bn[i];
        const double di = dinv[i];
        for (int k = lane; k <= i; k += 32) {
          const int gi = basis_index(Q, li + bl[k], mi + bm[k], ni + bn[k]);
          const double dd = di * dinv[k];
          Ai[k] = sM[gi] * dd;
          if (mode == 0) errl = fmax(errl, bnd[gi] * dd);
        }
      }
      if (mode == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) errl = fmax(errl, __shfl_xor_sync(0xffffffffu, errl, o));
        if (lane == 0) errw[warp] = errl;
      }
      __syncthreads();
      if (mode == 0) {
        double em = 0.0;
        for (int w = 0; w < K5_WARPS; ++w) em = fmax(em, errw[w]);
        // translated moments lost their precision, or the node is below the moment tree (M_000 = 0:
        // no moments yet): accumulate them directly from the node's points
        if (!(em <= mom_tol) || !(sM[0] > 0.0)) {
          if (tid == 0) {
            nt.flag[first + node] = 4;
            atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 1), 1ull);
          }
          __syncthreads();
          continue;
        }
      }
      K5T(0)
      // ---- blocked right-looking Cholesky with column rejection, RHS row carried along ---------
      auto diag = [&](double* buf, int ld, int jb, int bwd) {
        // diagonal block: Cholesky with column rejection by warp 0, lane = row, the row in registers
        // (chol_block: software-pipelined pivots, shuffles, no shared-memory round trips)
        double row[KB];
#pragma unroll
        for (int c = 0; c < KB; ++c) row[c] = (c <= lane && lane < bwd) ? buf[c * ld + lane] : 0.0;
        double myinv, mys;
        chol_block<KB>(row, bwd, dinv + jb, delta2, lane, myinv, mys);
        double v = (lane < bwd && dinv[jb + lane] > 0.0) ? mys : INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double w = __shfl_xor_sync(0xffffffffu, v, o);
          v = (w < v || w != w) ? w : v;
        }
        if (lane == 0 && !(v >= smin_sh)) smin_sh = v;
        if (lane < bwd) {
#pragma unroll
          for (int c = 0; c < KB; ++c)
            if (c <= lane) buf[c * ld + lane] = row[c];
          sinv[lane] = myinv;
          pinv[jb + lane] = myinv;
          piv[jb + lane] = buf[lane * ld + lane];  // this lane's pivot p (its own store)
        }
      };
      bool dg_ready = false;  // Dg holds the factored diagonal block of the current panel
      for (int j0 = 0; j0 < L; j0 += KB) {
        const int bw = min(KB, L - j0), R = L - j0 + 1;  // panel rows j0..L (row L = RHS)
        // panel load: warp per row, lane = column (one coalesced 256-byte row segment per load), RB rows
        // per warp in flight (the rows were just written by the trailing update: L2 latency per round);
        // rows of the lookahead's diagonal block come from Dg
        constexpr int RB = K5_WARPS >= 16 ? 4 : FMI_K5_PANEL_RB;
        for (int r0 = warp * RB; r0 < R; r0 += K5_WARPS * RB) {
          double v[RB];
#pragma unroll
          for (int k = 0; k < RB; ++k) {
            const int r = r0 + k, i = j0 + r, c = lane;
            v[k] = 0.0;
            if (r < R && c < bw) {
              if (r < bw && dg_ready) {
                if (c <= r) v[k] = Dg[c * KB + r];
              } else if (i == L || c <= r) {
                v[k] = A[tri(i) + j0 + c];
              }
            }
          }
#pragma unroll
          for (int k = 0; k < RB; ++k)
            if (r0 + k < R && lane < bw) Pn[lane * LDP + r0 + k] = v[k];
        }
        __syncthreads();
        K5T(1)
        // (1) diagonal block (warp 0, lane = row, registers + shuffles) — already factored into Dg by
        // the lookahead of the previous panel, except for the first panel
        if (!dg_ready) {
          if (warp == 0) diag(Pn, LDP, j0, bw);
        }
        __syncthreads();
        K5T(2)
        // (2) rows below the diagonal block (RHS row included): L_r = A_r L_diag⁻ᵀ, thread per row,
        // the row in registers, the same updates in the same order as the unblocked algorithm
        for (int r = bw + tid; r < R; r += K5_THREADS) {
          double x[KB];
#pragma unroll
          for (int c = 0; c < KB; ++c) x[c] = c < bw ? Pn[c * LDP + r] : 0.0;
#pragma unroll
          for (int c = 0; c < KB; ++c) {
            if (c < bw) {
              const double inv = sinv[c];
              const double lc = x[c] * inv;
              x[c] = lc;
              if (inv > 0.0) {
#pragma unroll
                for (int c2 = c + 1; c2 < KB; ++c2)
                  if (c2 < bw) x[c2] -= lc * Pn[c * LDP + c2];
              }
            }
          }
#pragma unroll
          for (int c = 0; c < KB; ++c)
            if (c < bw) Pn[c * LDP + r] = x[c];
        }
        __syncthreads();
        K5T(3)
        for (int e = tid; e < R * bw; e += K5_THREADS) {
          const int r = e / bw, c = e % bw;
          const int i = j0 + r;
          if (i == L || c <= r) A[tri(i) + j0 + c] = Pn[c * LDP + r];
        }
        // trailing update A[i][k] -= Σ_c Pn[i-j0][c] Pn[k-j0][c], j1 <= k <= min(i, L-1), j1 <= i <= L:
        // a rank-bw SYRK on the FP64 tensor cores — warp = one 8x8 tile of the lower triangle at a time,
        // bw/4 DMMA (m8n8k4) steps with the fragments read from the column-major panel, the tile's old
        // values loaded first so their L2 latency overlaps the MMAs
        const int j1 = j0 + bw, R2 = L + 1 - j1;
        if (j1 < L) {
          // lookahead (8-warp CTAs, p >= 9): the next panel's diagonal block (updated by this panel)
          // into Dg, then warp 0 factors it while the other warps apply the rest of the trailing update;
          // smaller CTAs keep every warp on the trailing update
          constexpr bool kLook = K5_WARPS >= 8;
          const int bw2 = kLook ? min(KB, L - j1) : 0;
          for (int e = tid; e < bw2 * bw2; e += K5_THREADS) {
            const int r = e / bw2, c = e - r * bw2;
            if (c > r) continue;
            const double* pr = Pn + (j1 - j0 + r);
            const double* pc = Pn + (j1 - j0 + c);
            double acc = 0.0;
            for (int q = 0; q < bw; ++q) acc = fma(pr[q * LDP], pc[q * LDP], acc);
            Dg[c * KB + r] = A[tri(j1 + r) + j1 + c] - acc;
          }
          if constexpr (kLook) {
            __syncthreads();
            if (warp == 0) diag(Dg, KB, j1, bw2);
          }
          const int iend = j1 + bw2;  // rows j1..iend-1 (cols <= row): the next diagonal block (in Dg)
          const int nt8 = (R2 + 7) / 8;
          const int ntile = nt8 * (nt8 + 1) / 2;
          const int fr = lane & 3, fc = lane >> 2;  // fragment k-row and m/n-column of this lane
          constexpr int TPW = 4;  // tiles per warp in flight: independent MMA chains and old-value loads
          const int tw = kLook ? warp - 1 : warp, nw = kLook ? K5_WARPS - 1 : K5_WARPS;  // trailing warps
          for (int t0 = tw * TPW; tw >= 0 && t0 < ntile; t0 += nw * TPW) {
            int ci[TPW], ck0[TPW];
            bool v0[TPW], v1[TPW];
            double old0[TPW], old1[TPW], d0[TPW], d1[TPW];
            const double* pa[TPW];
            const double* pb[TPW];
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
              const int t = min(t0 + u, ntile - 1);  // a duplicate of the last tile is computed, not stored
              int ti = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
              while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
              while (ti * (ti + 1) / 2 > t) --ti;
              const int tk = t - ti * (ti + 1) / 2;
              const int i0 = j1 + 8 * ti, k0 = j1 + 8 * tk;
              // this lane's two C elements: row i0 + fc, columns k0 + 2 fr + {0, 1}
              ci[u] = i0 + fc;
              ck0[u] = k0 + 2 * fr;
              const bool own = t0 + u < ntile && i0 + 7 >= iend;  // not entirely in the next diagonal block
              v0[u] = own && ci[u] <= L && ck0[u] < L && (ck0[u] <= ci[u] || ci[u] == L);
              v1[u] = own && ci[u] <= L && ck0[u] + 1 < L && (ck0[u] + 1 <= ci[u] || ci[u] == L);
              old0[u] = v0[u] ? A[tri(ci[u]) + ck0[u]] : 0.0;
              old1[u] = v1[u] ? A[tri(ci[u]) + ck0[u] + 1] : 0.0;
              d0[u] = d1[u] = 0.0;
              pa[u] = Pn + (i0 - j0) + fc + fr * LDP;
              pb[u] = Pn + (k0 - j0) + fc + fr * LDP;
            }
#pragma unroll
            for (int c = 0; c < KB; c += 4) {  // columns past bw (last panel) enter as zeros
              const bool in = c + fr < bw;
#pragma unroll
              for (int u = 0; u < TPW; ++u) {
                const double a = in ? pa[u][c * LDP] : 0.0;
                const double b = in ? pb[u][c * LDP] : 0.0;
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(d0[u]), "+d"(d1[u]) : "d"(a), "d"(b));
              }
            }
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
              if (v0[u] && ci[u] >= iend) A[tri(ci[u]) + ck0[u]] = old0[u] - d0[u];
              if (v1[u] && ci[u] >= iend) A[tri(ci[u]) + ck0[u] + 1] = old1[u] - d1[u];
            }
          }
        }
        dg_ready = (K5_WARPS >= 8) && j1 < L;
        __syncthreads();
        K5T(4)
      }
      // y = row L of the factored bordered matrix; ‖y‖² = bᵀG⁻¹b = the residual energy the fit removes
      double yy = 0.0;
      for (int i = tid; i < L; i += K5_THREADS) {
        const double v = A[tri(L) + i];
        sy[i] = v;
        yy = fma(v, v, yy);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) yy += __shfl_xor_sync(0xffffffffu, yy, o);
      if (lane == 0) errw[warp] = yy;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < K5_WARPS; ++w) t += errw[w];
        ynorm_sh = t;
      }
    }

    // ---- back substitution R̃ c̃ = y (R̃ = factorᵀ), blocked from the bottom ----------------------
    // Lookahead: after a 32-row block is solved, the rows of the next block take its contribution and
    // the next diagonal block is staged; then warp 0 solves the next block while the other warps apply
    // the finished block to all rows above it (the GEMV runs off the critical path).
    {
      // diagonal block L[j0..j1)[j0..j1) -> buf (row-major bw x KB); the thread's loads issued together
      auto load_diag = [&](double* buf, int j0, int bw) {
        constexpr int NL = (KB * KB + K5_THREADS - 1) / K5_THREADS;
        double v[NL];
#pragma unroll
        for (int q = 0; q < NL; ++q) {
          const int e = tid + q * K5_THREADS;
          const int r = e / KB, c = e % KB;
          v[q] = (r < bw && c <= r) ? A[tri(j0 + r) + j0 + c] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NL; ++q) {
          const int e = tid + q * K5_THREADS;
          if (e < KB * KB && e / KB < bw) buf[e] = v[q];
        }
      };
      // c_j = (y_j - Σ_{j<i<j1} L[i][j] c_i) / L[j][j]: warp 0, lane t holds y_t, right-looking
      auto solve_diag = [&](const double* buf, int j0, int bw) {
        double yv = lane < bw ? sy[j0 + lane] : 0.0;
        const double pl = lane < bw ? pinv[j0 + lane] : 0.0;
        for (int j = bw - 1; j >= 0; --j) {
          const double cj = __shfl_sync(0xffffffffu, pl > 0.0 ? yv * pl : 0.0, j);
          if (lane < j) yv -= buf[j * KB + lane] * cj;
          if (lane == j) yv = cj;
        }
        if (lane < bw) sy[j0 + lane] = yv;
      };
      // y_k -= Σ_{i in [j0,j1)} L[i][k] c_i for k in [klo, khi), thread t of T (rows i contiguous in k)
      auto gemv = [&](int j0, int bw, int klo, int khi, int t, int T) {
        for (int k = klo + t; k < khi; k += T) {
          double a[KB];
#pragma unroll
          for (int q = 0; q < KB; ++q) a[q] = q < bw ? A[tri(j0 + q) + k] : 0.0;
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (q < bw) v = fma(a[q], sy[j0 + q], v);
          sy[k] -= v;
        }
      };
      int j1 = L, j0 = max(0, L - KB);
      load_diag(Pn, j0, j1 - j0);
      __syncthreads();
      if (warp == 0) solve_diag(Pn, j0, j1 - j0);
      __syncthreads();
      int cur = 0;
      while (j0 > 0) {
        const int bw = j1 - j0, jn0 = max(0, j0 - KB);
        double* nbuf = Pn + (cur ^ 1) * KB * KB;
        gemv(j0, bw, jn0, j0, tid, K5_THREADS);  // the next block's rows first
        load_diag(nbuf, jn0, j0 - jn0);
        __syncthreads();
        if (warp == 0) solve_diag(nbuf, jn0, j0 - jn0);
        else gemv(j0, bw, 0, jn0, tid - 32, K5_THREADS - 32);  // all rows above the next block
        __syncthreads();
        j1 = j0;
        j0 = jn0;
        cur ^= 1;
      }
    }

    K5T(5)
    double* out = nt.coef + (first + node) * (int64_t)L;
    if (mode == 1) {  // refinement correction δ (monomial form): delta[node] = δ, coef += δ
      for (int i = tid; i < L; i += K5_THREADS) {
        const double d = sy[i] * dinv[i];
        delta[node * (int64_t)L + i] = d;
        out[i] += d;
      }
      __syncthreads();
      continue;
    }
    for (int i = tid; i < L; i += K5_THREADS) out[i] = sy[i] * dinv[i];
    if (tid == 0) {
      int rk = 0;
      double mn = INFINITY;
      for (int i = 0; i < L; ++i)
        if (piv[i] > 0.0) { ++rk; mn = fmin(mn, piv[i]); }
      nt.rank[first + node] = rk;
      nt.minpiv[first + node] = rk ? mn : 0.0;
      // robust-path flag: a pivot of a non-zero column fell where fp64 Gram pivots stop tracking the
      // QR pivots (or the column was rejected) -> K5q re-fits the node by Householder QR;
      // semi-normal refinement flag (bit 1): small pivots, or few points per unknown, where the normal
      // equations lose digits (DESIGN.md §5 K5r)
      // the node's point count over all shards: the parent's octant count (root: n_root)
      const int32_t par = nt.parent[first + node];
      const int4 cc = nt.cell[first + node];
      const double npts = par < 0 ? (double)n_root
                                  : (double)nt.child_n[(int64_t)par * 8 + ((cc.x & 1) | ((cc.y & 1) << 1) | ((cc.z & 1) << 2))];
      const bool refine = refine2 > 0.0 && (smin_sh < refine2 || npts < refine_fill * L);
      const int fl = (smin_sh < kQrFlagPivot2) ? 1 : (refine ? 2 : 0);
      // defer this node's child projections when its predicted post-fit RMS — pre-fit block energy
      // (the parent's octant Σr²) minus the energy the fit removes (‖y‖²), over its points — is below
      // defer_tau: its children are then unlikely to be created (K6_PROJ runs for those that are)
      int defer = 0;
      if (isinf(defer_tau)) {  // split K6 (FMI_K6_SPLIT): every node's projections run in K6_PROJ
        defer = 8;
      } else if (par >= 0 && defer_tau > 0.0) {
        const int oc = (cc.x & 1) | ((cc.y & 1) << 1) | ((cc.z & 1) << 2);
        const double e_post2 = fmax(nt.child_ss[(int64_t)par * 8 + oc] - ynorm_sh, 0.0) / fmax(npts, 1.0);
        defer = e_post2 < defer_tau * defer_tau ? 8 : 0;
      }
      nt.flag[first + node] = fl | defer;
      if (fl == 2) atomicAdd(reinterpret_cast<unsigned long long*>(nflag), 1ull);
      if (defer) atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 2), 1ull);
    }
    __syncthreads();
  }
  K5T_PRINT
}

// ---- K5 resident variant (p <= 9): the whole bordered packed factor lives in shared memory ---------------
// Same arithmetic, order of updates, pivots and rejections as k_solve (so the same results up to the
// summation order of the DMMA tiles), but no panel copy and no global round trips: the diagonal block,
// the row solve and the DMMA trailing update all work in place on the packed rows in shared memory
// (𝓛 = 165: 111 KB -> 2 CTAs per SM; 𝓛 = 84: 29 KB -> 7).  The factor is copied to global memory once,
// coalesced, for the refinement solves (mode 1 copies it back).  To fit two 𝓛 = 165 factors per SM the
// moments are read through L1 (the node's K values are the only gather) and the pivots are read back
// from the factor's diagonal (a rejected column's diagonal entry is 0).
template <int P>
struct K5Res {
  using S = K5Shape<P>;
  static constexpr int L = S::L, K = S::K;
  static constexpr int64_t NAB = S::NAB;
  // dinv, sy [L each] | A[NAB] (16-byte aligned) | exponents
  static constexpr size_t A_OFF = ((2 * (size_t)L) + 1) & ~size_t(1);
  static constexpr size_t SMEM = (A_OFF + (size_t)NAB + 2) * sizeof(double) + 3 * L + 16;
  static constexpr bool fits = SMEM <= 227 * 1024;
};
#ifndef FMI_K5R_BLK2
#define FMI_K5R_BLK2 1
#endif
#ifndef FMI_K5R_MID
#define FMI_K5R_MID 64
#endif
template <int P>
constexpr int k5r_threads() { return rank3(P) >= 120 ? 256 : (rank3(P) >= 56 ? FMI_K5R_MID : 64); }
template <int P>
constexpr int k5r_minb() {
  constexpr size_t per = K5Res<P>::SMEM + 1024;
  constexpr int bys = (int)((228 * 1024) / per);
  constexpr int byt = 65536 / (k5r_threads<P>() * 128);  // >= 128 registers: the diagonal block row[32] unspilled
  constexpr int b = bys < byt ? bys : byt;
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

template <int P, int NT>
__global__ void __launch_bounds__(NT, k5r_minb<P>())
    k_solve_res(const double* __restrict__ mom, int mode, const double* __restrict__ segrhs,
                double* __restrict__ delta, NodeTable nt, int64_t first, int64_t count, double* __restrict__ fac,
                const __grid_constant__ BasisTab bt, double delta2, double refine2, double refine_fill,
                double mom_tol, int64_t n_root, double defer_tau, int64_t* __restrict__ nflag) {
  using R = K5Res<P>;
  constexpr int Q = 2 * P, K = R::K, L = R::L;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) double sm[];
  double* dinv = sm;
  double* sy = dinv + L;
  double* A = sm + R::A_OFF;  // packed lower rows 0..L-1 (row i at tri(i)), RHS row L at tri(L)
  uint8_t* bl = reinterpret_cast<uint8_t*>(A + R::NAB + 2);
  uint8_t* bm = bl + L;
  uint8_t* bn = bm + L;
  __shared__ double smin_sh, ynorm_sh;
  __shared__ double errw[NW];
  __shared__ double sinv[KB];
  // warp index broadcast from lane 0: provably warp-uniform for the compiler, so the warp-specialised
  // branches (diagonal block on warp 0) keep their shuffles and MMAs on the converged fast path
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  for (int i = tid; i < L; i += NT) { bl[i] = bt.l[i]; bm[i] = bt.m[i]; bn[i] = bt.n[i]; }
  __syncthreads();
  auto tri = [](int i) { return i * (i + 1) / 2; };  // 32-bit row offsets (NAB < 2^31)
  constexpr int K5_THREADS = NT;
  (void)K5_THREADS;
  K5T_DECL

  for (int64_t node = blockIdx.x; node < count; node += gridDim.x) {
    K5T(6)
    if (mode == 1 && !(nt.flag[first + node] & 2)) continue;
    if (mode == 2 && !(nt.flag[first + node] & 4)) continue;
    double* Ag = fac + node * R::NAB;
    const double* mp = mom + node * (int64_t)(2 * K + L);
    const double* bndg = mp + K + L;
    if (tid == 0) smin_sh = INFINITY;
    const double m000 = __ldg(mp);
    if (mode == 0 && !(m000 > 0.0)) {  // below the moment tree (M_000 = 0): accumulate directly
      if (tid == 0) {
        nt.flag[first + node] = 4;
        atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 1), 1ull);
      }
      __syncthreads();
      continue;
    }
    for (int i = tid; i < L; i += NT) {
      const double m2 = __ldg(mp + basis_index(Q, 2 * bl[i], 2 * bm[i], 2 * bn[i]));
      const double di = m2 > 0.0 ? 1.0 / sqrt(m2) : 0.0;
      dinv[i] = di;
      double b;
      if (mode == 1) {
        b = 0.0;
        for (int o = 0; o < 8; ++o) b += segrhs[(node * 8 + o) * (L + 1) + i];
      } else {
        b = mp[K + i];
      }
      sy[i] = b * di;
    }
    __syncthreads();

    if (mode == 1) {
      // ---- refinement: the stored factor back into shared memory, forward substitution ----------
      for (int64_t e = tid; e < R::NAB; e += NT) A[e] = Ag[e];
      __syncthreads();
      for (int j0 = 0; j0 < L; j0 += KB) {
        const int j1 = min(j0 + KB, L);
        for (int i = j0 + warp; i < j1; i += NW) {
          const double* Ai = A + tri(i);
          double v = 0.0;
          for (int k = lane; k < j0; k += 32) v = fma(Ai[k], sy[k], v);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) sy[i] -= v;
        }
        __syncthreads();
        if (warp == 0) {
          for (int i = j0; i < j1; ++i) {
            const double* Ai = A + tri(i);
            double v = 0.0;
            for (int k = j0 + lane; k < i; k += 32) v = fma(Ai[k], sy[k], v);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            const double pi = A[tri(i) + i];
            if (lane == 0) sy[i] = pi > 0.0 ? (sy[i] - v) / pi : 0.0;
            __syncwarp();
          }
        }
        __syncthreads();
      }
    } else {
      // ---- assemble the equilibrated Gram + RHS row in shared memory; moments' rounding bound -------
      double errl = 0.0;
      for (int i = warp; i <= L; i += NW) {
        double* Ai = A + tri(i);
        if (i == L) {
          for (int k = lane; k < L; k += 32) Ai[k] = sy[k];
          continue;
        }
        const int li = bl[i], mi = bm[i], ni = bn[i];
        const double di = dinv[i];
        for (int k = lane; k <= i; k += 32) {
          const int gi = basis_index(Q, li + bl[k], mi + bm[k], ni + bn[k]);
          const double dd = di * dinv[k];
          Ai[k] = __ldg(mp + gi) * dd;
          if (mode == 0) errl = fmax(errl, __ldg(bndg + gi) * dd);
        }
      }
      if (mode == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) errl = fmax(errl, __shfl_xor_sync(0xffffffffu, errl, o));
        if (lane == 0) errw[warp] = errl;
      }
      __syncthreads();
      if (mode == 0) {
        double em = 0.0;
        for (int w = 0; w < NW; ++w) em = fmax(em, errw[w]);
        if (!(em <= mom_tol)) {
          if (tid == 0) {
            nt.flag[first + node] = 4;
            atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 1), 1ull);
          }
          __syncthreads();
          continue;
        }
      }
      K5T(0)
      // ---- blocked right-looking Cholesky in place, column rejection, RHS row carried along --------
      // diagonal block of columns jb..jb+bwd-1: warp 0, lane = row, the row in registers (shuffles)
      auto diag = [&](int jb, int bwd) {
        double row[KB];
        const double* Ar = A + tri(jb + lane) + jb;
#pragma unroll
        for (int c = 0; c < KB; ++c) row[c] = (c <= lane && lane < bwd) ? Ar[c] : 0.0;
        double myinv, mys;
        chol_block<KB>(row, bwd, dinv + jb, delta2, lane, myinv, mys);
        // smallest Schur pivot of a non-zero column (NaN-propagating, as the unblocked rule)
        double v = (lane < bwd && dinv[jb + lane] > 0.0) ? mys : INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double w = __shfl_xor_sync(0xffffffffu, v, o);
          v = (w < v || w != w) ? w : v;
        }
        if (lane < bwd) sinv[lane] = myinv;
        if (lane == 0 && !(v >= smin_sh)) smin_sh = v;
        if (lane < bwd) {
          double* Aw = A + tri(jb + lane) + jb;
#pragma unroll
          for (int c = 0; c < KB; ++c)
            if (c <= lane) Aw[c] = row[c];
        }
      };
      // DMMA update of 8x8 tiles t in [t_lo, t_hi) of the trailing lower triangle rows/cols >= j1 by the
      // panel columns j0..j0+bw-1 (tile (ti, tk), tk <= ti, rows j1+8ti.., cols j1+8tk..)
#if FMI_K5R_BLK2
      // DMMA update of 16x16 blocks b in [b_lo, b_hi) of the trailing lower triangle (rows/cols >= j1) by
      // the panel columns j0..j0+bw-1: block (bi, bk), bk <= bi, rows j1+16bi.., cols j1+16bk.., as 2x2
      // 8x8 tiles that share their fragments (two A and two B fragment loads per four m8n8k4 steps, half
      // the shared-memory reads of independent tiles); the tile above the diagonal of a diagonal block is
      // skipped.  Blocks are numbered row-major, so the blocks of the next diagonal block are a prefix.
      const int fr = lane & 3, fc = lane >> 2;
      auto trailing = [&](int j0, int bw, int j1, int t_lo, int t_hi, int wid, int nwk, bool, int) {
        for (int t = t_lo + wid; t < t_hi; t += nwk) {
          int bi = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
          while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
          while (bi * (bi + 1) / 2 > t) --bi;
          const int bk = t - bi * (bi + 1) / 2;
          const bool dgb = bi == bk;
          const int i0 = j1 + 16 * bi, k0 = j1 + 16 * bk;
          // fragment rows (clamped into the matrix; rows past L are masked at the store)
          const double* pa0 = A + tri(min(i0 + fc, L)) + j0 + fr;
          const double* pa1 = A + tri(min(i0 + 8 + fc, L)) + j0 + fr;
          const double* pb0 = A + tri(min(k0 + fc, L)) + j0 + fr;
          const double* pb1 = A + tri(min(k0 + 8 + fc, L)) + j0 + fr;
          double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
          for (int c = 0; c < KB; c += 4) {  // columns past bw (last panel) enter as zeros
            const bool in = c + fr < bw;
            const double a0 = in ? pa0[c] : 0.0, a1 = in ? pa1[c] : 0.0;
            const double b0 = in ? pb0[c] : 0.0, b1 = in ? pb1[c] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[0][0]), "+d"(d[0][1]) : "d"(a0), "d"(b0));
            if (!dgb)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                           : "+d"(d[1][0]), "+d"(d[1][1]) : "d"(a0), "d"(b1));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[2][0]), "+d"(d[2][1]) : "d"(a1), "d"(b0));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[3][0]), "+d"(d[3][1]) : "d"(a1), "d"(b1));
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ci = i0 + 8 * (u >> 1) + fc, ck = k0 + 8 * (u & 1) + 2 * fr;
            if (ci > L || (u == 1 && dgb)) continue;
            double* Ar = A + tri(ci);
            if (ck < L && (ck <= ci || ci == L)) Ar[ck] -= d[u][0];
            if (ck + 1 < L && (ck + 1 <= ci || ci == L)) Ar[ck + 1] -= d[u][1];
          }
        }
      };
      constexpr int TB = 16;  // rows per trailing work item
#else
      constexpr int TPW = 4;
      constexpr int TB = 8;  // rows per trailing work item
      const int fr = lane & 3, fc = lane >> 2;
      auto trailing = [&](int j0, int bw, int j1, int t_lo, int t_hi, int wid, int nwk, bool skip_next, int iend) {
        for (int t0 = t_lo + wid * TPW; t0 < t_hi; t0 += nwk * TPW) {
          int ci[TPW], ck0[TPW];
          bool v0[TPW], v1[TPW];
          double d0[TPW], d1[TPW];
          const double* pa[TPW];
          const double* pb[TPW];
#pragma unroll
          for (int u = 0; u < TPW; ++u) {
            const int t = min(t0 + u, t_hi - 1);
            int ti = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
            while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
            while (ti * (ti + 1) / 2 > t) --ti;
            const int tk = t - ti * (ti + 1) / 2;
            const int i0 = j1 + 8 * ti, k0 = j1 + 8 * tk;
            ci[u] = i0 + fc;
            ck0[u] = k0 + 2 * fr;
            const bool own = t0 + u < t_hi && !(skip_next && i0 + 7 < iend);
            v0[u] = own && ci[u] <= L && ck0[u] < L && (ck0[u] <= ci[u] || ci[u] == L);
            v1[u] = own && ci[u] <= L && ck0[u] + 1 < L && (ck0[u] + 1 <= ci[u] || ci[u] == L);
            d0[u] = d1[u] = 0.0;
            // fragment rows (clamped into the matrix; rows past L are masked at the store)
            const int ra = min(i0 + fc, L), rb = min(k0 + fc, L);
            pa[u] = A + tri(ra) + j0 + fr;
            pb[u] = A + tri(rb) + j0 + fr;
          }
#pragma unroll
          for (int c = 0; c < KB; c += 4) {  // columns past bw (last panel) enter as zeros
            const bool in = c + fr < bw;
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
              const double a = in ? pa[u][c] : 0.0;
              const double b = in ? pb[u][c] : 0.0;
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                           : "+d"(d0[u]), "+d"(d1[u]) : "d"(a), "d"(b));
            }
          }
#pragma unroll
          for (int u = 0; u < TPW; ++u) {
            if (v0[u]) A[tri(ci[u]) + ck0[u]] -= d0[u];
            if (v1[u]) A[tri(ci[u]) + ck0[u] + 1] -= d1[u];
          }
        }
      };
#endif
      constexpr bool kLook = NW >= 4;
      bool dg_ready = false;
      for (int j0 = 0; j0 < L; j0 += KB) {
        const int bw = min(KB, L - j0), j1 = j0 + bw;
        if (!dg_ready && warp == 0) diag(j0, bw);  // else: factored by the lookahead (sinv set)
        __syncthreads();
        K5T(2)
        // rows below the diagonal block (RHS row included): x = A_r L_diag⁻ᵀ, thread per row
        for (int r = j1 + tid; r <= L; r += NT) {
          double* Ar = A + tri(r) + j0;
          double x[KB];
#pragma unroll
          for (int c = 0; c < KB; ++c) x[c] = c < bw ? Ar[c] : 0.0;
#pragma unroll
          for (int c2 = 0; c2 < KB; ++c2) {
            // left-looking order of the same updates: x[c2] -= x[c] L[c2][c] for c = 0..c2-1 (the order of
            // the right-looking loop), then the scaling; row c2 of the diagonal block is contiguous, so the
            // loads share one base register (no per-row address registers, no spills); branch-free: a
            // rejected column has inv = 0, x = 0
            const double* Lr = A + tri(min(j0 + c2, L)) + j0;
            double acc = x[c2];
#pragma unroll
            for (int c = 0; c < c2; ++c) acc = fma(-x[c], Lr[c], acc);
            x[c2] = c2 < bw ? acc * sinv[c2] : 0.0;
          }
#pragma unroll
          for (int c = 0; c < KB; ++c)
            if (c < bw) Ar[c] = x[c];
        }
        __syncthreads();
        K5T(3)
        if (j1 < L) {
          const int R2 = L + 1 - j1;
          const int nt8 = (R2 + TB - 1) / TB;
          const int ntile = nt8 * (nt8 + 1) / 2;
          const int bw2 = min(KB, L - j1);
          if (kLook) {
            // the next diagonal block's tiles first (rows j1..j1+bw2-1: tiles ti < 4), then warp 0
            // factors it while the other warps update the rest
            const int nd8 = (bw2 + TB - 1) / TB;
            const int ndt = nd8 * (nd8 + 1) / 2;
            trailing(j0, bw, j1, 0, ndt, warp, NW, false, 0);
            __syncthreads();
            if (warp == 0) diag(j1, bw2);
            else trailing(j0, bw, j1, ndt, ntile, warp - 1, NW - 1, false, 0);
          } else {
            trailing(j0, bw, j1, 0, ntile, warp, NW, false, 0);
          }
          dg_ready = kLook;
        }
        __syncthreads();
        K5T(4)
      }
      // y = row L of the factored bordered matrix; ‖y‖² = bᵀG⁻¹b
      double yy = 0.0;
      for (int i = tid; i < L; i += NT) {
        const double v = A[tri(L) + i];
        sy[i] = v;
        yy = fma(v, v, yy);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) yy += __shfl_xor_sync(0xffffffffu, yy, o);
      if (lane == 0) errw[warp] = yy;
      // the factor to global memory for the refinement solves (coalesced, off the critical path)
      for (int64_t e = tid; e < R::NAB; e += NT) Ag[e] = A[e];
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += errw[w];
        ynorm_sh = t;
      }
    }

    // ---- back substitution R̃ c̃ = y in place (R̃ = factorᵀ), blocked from the bottom ------------------
    {
      auto solve_diag = [&](int j0, int bw) {
        double yv = lane < bw ? sy[j0 + lane] : 0.0;
        const double pd = lane < bw ? A[tri(j0 + lane) + j0 + lane] : 0.0;
        const double pl = pd > 0.0 ? 1.0 / pd : 0.0;
        for (int j = bw - 1; j >= 0; --j) {
          const double cj = __shfl_sync(0xffffffffu, pl > 0.0 ? yv * pl : 0.0, j);
          if (lane < j) yv -= A[tri(j0 + j) + j0 + lane] * cj;
          if (lane == j) yv = cj;
        }
        if (lane < bw) sy[j0 + lane] = yv;
      };
      auto gemv = [&](int j0, int bw, int klo, int khi, int t, int T) {
        for (int k = klo + t; k < khi; k += T) {
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (q < bw) v = fma(A[tri(j0 + q) + k], sy[j0 + q], v);
          sy[k] -= v;
        }
      };
      int j1 = L, j0 = max(0, L - KB);
      if (warp == 0) solve_diag(j0, j1 - j0);
      __syncthreads();
      while (j0 > 0) {
        const int bw = j1 - j0, jn0 = max(0, j0 - KB);
        gemv(j0, bw, jn0, j0, tid, NT);  // the next block's rows first
        __syncthreads();
        if (NW > 1) {
          if (warp == 0) solve_diag(jn0, j0 - jn0);
          else gemv(j0, bw, 0, jn0, tid - 32, NT - 32);
        } else {
          solve_diag(jn0, j0 - jn0);
          gemv(j0, bw, 0, jn0, tid, NT);
        }
        __syncthreads();
        j1 = j0;
        j0 = jn0;
      }
    }

    K5T(5)
    double* out = nt.coef + (first + node) * (int64_t)L;
    if (mode == 1) {
      for (int i = tid; i < L; i += NT) {
        const double d = sy[i] * dinv[i];
        delta[node * (int64_t)L + i] = d;
        out[i] += d;
      }
      __syncthreads();
      continue;
    }
    for (int i = tid; i < L; i += NT) out[i] = sy[i] * dinv[i];
    if (tid == 0) {
      int rk = 0;
      double mn = INFINITY;
      for (int i = 0; i < L; ++i) {
        const double pi = A[tri(i) + i];
        if (pi > 0.0) { ++rk; mn = fmin(mn, pi); }
      }
      nt.rank[first + node] = rk;
      nt.minpiv[first + node] = rk ? mn : 0.0;
      const int32_t par = nt.parent[first + node];
      const int4 cc = nt.cell[first + node];
      const double npts = par < 0 ? (double)n_root
                                  : (double)nt.child_n[(int64_t)par * 8 + ((cc.x & 1) | ((cc.y & 1) << 1) | ((cc.z & 1) << 2))];
      const bool refine = refine2 > 0.0 && (smin_sh < refine2 || npts < refine_fill * L);
      const int fl = (smin_sh < kQrFlagPivot2) ? 1 : (refine ? 2 : 0);
      int defer = 0;
      if (isinf(defer_tau)) {
        defer = 8;
      } else if (par >= 0 && defer_tau > 0.0) {
        const int oc = (cc.x & 1) | ((cc.y & 1) << 1) | ((cc.z & 1) << 2);
        const double e_post2 = fmax(nt.child_ss[(int64_t)par * 8 + oc] - ynorm_sh, 0.0) / fmax(npts, 1.0);
        defer = e_post2 < defer_tau * defer_tau ? 8 : 0;
      }
      nt.flag[first + node] = fl | defer;
      if (fl == 2) atomicAdd(reinterpret_cast<unsigned long long*>(nflag), 1ull);
      if (defer) atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 2), 1ull);
    }
    __syncthreads();
  }
  K5T_PRINT
}

}  // namespace

template <int P>
void level_solve(const LevelCtx& c, const double* mom, int mode, const double* segrhs, double* delta, double refine2,
                 double refine_fill, int64_t n_root, int64_t* nflag, double* fac, cudaStream_t s, double defer_tau) {
  using S = K5Shape<P>;
  static const BasisTab bt = make_basis<P>();
  constexpr int NT = k5_threads<P>();
  static int small_max = 0;  // levels with <= small_max nodes run 256 threads per node (p <= 8)
  static int tiny_max = 0;   // levels with <= tiny_max nodes (at most one per SM) run 512 threads per node
  static int64_t grid_cap = 1 << 20;  // FMI_K5_CTAS_PER_SM (experiments): persistent CTAs per SM
  static std::once_flag attr_once;    // one opt-in per kernel instantiation (thread-safe)
  std::call_once(attr_once, [&] {
    int dev = 0, sms = 0;
    FMI_CK(cudaGetDevice(&dev));
    FMI_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FMI_CK(cudaFuncSetAttribute(k_solve<P, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    FMI_CK(cudaFuncSetAttribute(k_solve<P, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    if constexpr (NT < 256) {
      FMI_CK(cudaFuncSetAttribute(k_solve<P, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
      const char* e = std::getenv("FMI_K5_SMALL");
      small_max = e ? std::atoi(e) : 6 * sms;
    }
    const char* t = std::getenv("FMI_K5_TINY");
    tiny_max = t ? std::atoi(t) : sms;
    if (const char* e = std::getenv("FMI_K5_CTAS_PER_SM")) grid_cap = std::max<int64_t>(1, (int64_t)std::atoi(e) * sms);
  });
  const int64_t grid = std::min<int64_t>(c.count, grid_cap);
  if (grid <= 0) return;
  if (mode != 1) prof_units(KID_SOLVE, c.count);  // nodes factored (𝓛³/3 + 3𝓛² flop each)
  const int kid = mode == 1 ? KID_REFINE_SOLVE : KID_SOLVE;
  if constexpr (K5Res<P>::fits) {
    // shared-memory-resident factor (p <= 9); FMI_K5_RES=0 selects the global-memory kernel
    static const bool use_res = [] {
      const char* e = std::getenv("FMI_K5_RES");
      const bool on = !(e && std::atoi(e) == 0);
      if (on) FMI_CK(cudaFuncSetAttribute(k_solve_res<P, k5r_threads<P>()>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K5Res<P>::SMEM));
      return on;
    }();
    if (use_res) {
      FMI_LAUNCH(kid, s, (k_solve_res<P, k5r_threads<P>()>), (unsigned)grid, k5r_threads<P>(), K5Res<P>::SMEM, mom,
                 mode, segrhs, delta, c.nt, c.first, c.count, fac, bt, kDelta * kDelta, refine2, refine_fill,
                 kMomentTol, n_root, defer_tau, nflag);
      return;
    }
  }
#define K5_ARGS mom, mode, segrhs, delta, c.nt, c.first, c.count, fac, bt, kDelta * kDelta, refine2, refine_fill, \
                kMomentTol, n_root, defer_tau, nflag
  if (grid <= tiny_max) {  // latency-bound levels (the top of every tree): more warps per node
    FMI_LAUNCH(kid, s, (k_solve<P, 512>), (unsigned)grid, 512, S::SMEM, K5_ARGS);
  } else if (NT < 256 && grid <= small_max) {
    FMI_LAUNCH(kid, s, (k_solve<P, 256>), (unsigned)grid, 256, S::SMEM, K5_ARGS);
  } else {
    FMI_LAUNCH(kid, s, (k_solve<P, NT>), (unsigned)grid, NT, S::SMEM, K5_ARGS);
  }
#undef K5_ARGS
}

// doubles of per-node factor storage (bordered packed lower triangle)
size_t solve_factor_per_node(int p) {
  switch (p) {
#define C(P) case P: return (size_t)K5Shape<P>::NAB;
    C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10)
#undef C
  }
  return 0;
}

#define FMI_INST(P) \
  template void level_solve<P>(const LevelCtx&, const double*, int, const double*, double*, double, double, int64_t, \
                               int64_t*, double*, cudaStream_t, double);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
