// solve.cu — K5: batched node solve (DESIGN.md §3 K5), one CTA per node.
//
// PAPER.md Algorithm 2 computes P_F = R⁻¹ Qᵀ f from the QR of Λ.  In Gram form, with the
// raw moments M and projection b of K4:
//   D_α   = sqrt(G_αα) = sqrt(M_{2α}) / α!          (column norms of Λ)
//   G̃_αβ  = M_{α+β} / sqrt(M_{2α} M_{2β})           (Jacobi-equilibrated Gram; factorials cancel)
//   b̃_α   = b_α / sqrt(M_{2α})                     (= (Λᵀ r)_α / D_α)
//   G̃ c̃ = b̃  by Cholesky G̃ = R̃ᵀR̃  (R̃ = the R of the QR of Λ D⁻¹ up to row signs)
//   monomial coefficients a_α = c̃_α / sqrt(M_{2α}) = P_F,α / α!   (used by Horner in K6/K7)
// Rank rule (reading G9, identical to the oracle's QR column rejection): at step j the Schur
// complement diagonal s_jj equals the squared distance of equilibrated column j from the span of the
// kept columns; the column is dropped (coefficient 0) iff s_jj <= kDelta², or M_{2α} = 0.
#include <algorithm>
#include <vector>

#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int K5_THREADS = 256;

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

template <int P>
struct K5Shape {
  static constexpr int Q = 2 * P;
  static constexpr int K = rank3(Q);
  static constexpr int L = rank3(P);
  static constexpr int NA = L * (L + 1) / 2;
  static constexpr size_t VEC = (size_t)K + 5 * L;  // moments, b, dinv, col, piv, scratch
  static constexpr bool kSmemA = (VEC + NA) * sizeof(double) <= 220 * 1024;
  // global-matrix path: blocked right-looking Cholesky with a column panel of KB columns in smem
  static constexpr int KB = 32, PLD = KB + 1;
  static constexpr size_t PANEL = (size_t)L * PLD;
  static constexpr size_t SMEM = (kSmemA ? VEC + NA : VEC + PANEL) * sizeof(double);
};

__device__ __forceinline__ int64_t tri(int i) { return (int64_t)i * (i + 1) / 2; }

template <int P>
__global__ void __launch_bounds__(K5_THREADS)
    k_solve(const double* __restrict__ mom, int mode, const double* __restrict__ segrhs, double* __restrict__ delta,
            NodeTable nt, int64_t first, int64_t count, double* __restrict__ gscratch,
            const __grid_constant__ BasisTab bt, double delta2, double refine2, double refine_fill,
            double mom_tol, int64_t* __restrict__ nflag) {
  using S = K5Shape<P>;
  constexpr int Q = S::Q, K = S::K, L = S::L;
  extern __shared__ double sm[];
  double* sM = sm;          // [K]
  double* sb = sM + K;      // [L]  b̃ -> y -> c̃
  double* dinv = sb + L;    // [L]
  double* col = dinv + L;   // [L]
  double* piv = col + L;    // [L]
  double* red = piv + L;    // [L]
  double* A = S::kSmemA ? red + L : gscratch + (int64_t)blockIdx.x * S::NA;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = K5_THREADS / 32;
  __shared__ double smin_sh[1];
  __shared__ double errw[NWARP];
  // basis exponents in shared memory (thread-divergent lookups into the parameter bank serialise)
  __shared__ uint8_t bl[L], bm[L], bn[L];
  for (int i = tid; i < L; i += K5_THREADS) { bl[i] = bt.l[i]; bm[i] = bt.m[i]; bn[i] = bt.n[i]; }
  __syncthreads();

  for (int64_t node = blockIdx.x; node < count; node += gridDim.x) {
    // mode 1 (refinement): bit-1 nodes only; mode 2 (direct-moment re-solve): bit-2 nodes only
    if (mode == 1 && !(nt.flag[first + node] & 2)) continue;
    if (mode == 2 && !(nt.flag[first + node] & 4)) continue;
    if (tid == 0) smin_sh[0] = INFINITY;
    const double* mp = mom + node * (int64_t)(2 * K + L);
    const double* bnd = mp + K + L;
    for (int e = tid; e < K; e += K5_THREADS) sm[e] = mp[e];
    if (mode == 1) {  // b1 = Λᵀ r1 over the node's 8 octant segments, fixed order
      for (int e = tid; e < L; e += K5_THREADS) {
        double v = 0.0;
        for (int o = 0; o < 8; ++o) v += segrhs[(node * 8 + o) * (L + 1) + e];
        sb[e] = v;
      }
    } else {
      const double* bp = mp + K;
      for (int e = tid; e < L; e += K5_THREADS) sb[e] = bp[e];
    }
    __syncthreads();
    for (int i = tid; i < L; i += K5_THREADS) {
      const double m2 = sM[basis_index(Q, 2 * bl[i], 2 * bm[i], 2 * bn[i])];
      const double di = m2 > 0.0 ? 1.0 / sqrt(m2) : 0.0;
      dinv[i] = di;
      sb[i] *= di;
    }
    __syncthreads();
    double errl = 0.0;  // equilibrated rounding bound of the Gram (translated moments)
    for (int64_t e = tid; e < S::NA; e += K5_THREADS) {
      int i = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
      while (tri(i + 1) <= e) ++i;
      while (tri(i) > e) --i;
      const int k = (int)(e - tri(i));
      const int gi = basis_index(Q, bl[i] + bl[k], bm[i] + bm[k], bn[i] + bn[k]);
      const double dd = dinv[i] * dinv[k];
      A[e] = sM[gi] * dd;
      errl = fmax(errl, bnd[gi] * dd);
    }
    if (mode == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) errl = fmax(errl, __shfl_xor_sync(0xffffffffu, errl, o));
      if (lane == 0) errw[warp] = errl;
    }
    __syncthreads();
    if (mode == 0) {
      double em = 0.0;
      for (int w = 0; w < NWARP; ++w) em = fmax(em, errw[w]);
      if (!(em <= mom_tol)) {  // translated moments lost their precision: re-accumulate directly
        if (tid == 0) {
          nt.flag[first + node] = 4;
          atomicAdd(reinterpret_cast<unsigned long long*>(nflag + 1), 1ull);
        }
        __syncthreads();
        continue;
      }
    }

    if constexpr (S::kSmemA) {
      // right-looking Cholesky with column rejection (matrix in shared memory)
      for (int j = 0; j < L; ++j) {
        if (tid == 0) {
          const double s = A[tri(j) + j];
          const bool keep = dinv[j] > 0.0 && s > delta2;
          const double p = keep ? sqrt(s) : 0.0;
          piv[j] = p;
          A[tri(j) + j] = p;
          if (dinv[j] > 0.0 && !(s >= smin_sh[0])) smin_sh[0] = s;  // also catches NaN
        }
        __syncthreads();
        const double p = piv[j];
        if (p > 0.0) {
          const double inv = 1.0 / p;
          for (int i = j + 1 + tid; i < L; i += K5_THREADS) {
            const double v = A[tri(i) + j] * inv;
            A[tri(i) + j] = v;
            col[i] = v;
          }
          __syncthreads();
          for (int i = j + 1 + warp; i < L; i += NWARP) {
            const double ci = col[i];
            double* Ai = A + tri(i);
            for (int k = j + 1 + lane; k <= i; k += 32) Ai[k] -= ci * col[k];
          }
        } else {
          for (int i = j + 1 + tid; i < L; i += K5_THREADS) A[tri(i) + j] = 0.0;
        }
        __syncthreads();
      }
    } else {
      // Blocked right-looking Cholesky with column rejection, matrix in global scratch (L2-resident):
      // per block of KB columns, the column panel (rows j0..L-1) is factored in shared memory column by
      // column (the same pivots, rejections and updates as the unblocked algorithm), written back, and
      // the trailing triangle is updated once with 4x4 register tiles (SYRK against the panel).
      constexpr int KB = S::KB, PLD = S::PLD;
      double* Pn = red + L;  // panel [L - j0][PLD]
      for (int j0 = 0; j0 < L; j0 += KB) {
        const int bw = min(KB, L - j0), R = L - j0;
        for (int e = tid; e < R * bw; e += K5_THREADS) {
          const int r = e / bw, c = e % bw;
          Pn[r * PLD + c] = (c <= r) ? A[tri(j0 + r) + j0 + c] : 0.0;
        }
        __syncthreads();
        for (int c = 0; c < bw; ++c) {
          const int j = j0 + c;
          if (tid == 0) {
            const double sjj = Pn[c * PLD + c];
            const bool keep = dinv[j] > 0.0 && sjj > delta2;
            const double p = keep ? sqrt(sjj) : 0.0;
            piv[j] = p;
            Pn[c * PLD + c] = p;
            if (dinv[j] > 0.0 && !(sjj >= smin_sh[0])) smin_sh[0] = sjj;  // also catches NaN
          }
          __syncthreads();
          const double p = piv[j];
          const double inv = p > 0.0 ? 1.0 / p : 0.0;
          for (int r = c + 1 + tid; r < R; r += K5_THREADS) Pn[r * PLD + c] *= inv;
          __syncthreads();
          const int nc = bw - c - 1;
          if (p > 0.0 && nc > 0) {
            for (int e = tid; e < (R - c - 1) * nc; e += K5_THREADS) {
              const int r = c + 1 + e / nc, c2 = c + 1 + e % nc;
              if (c2 <= r) Pn[r * PLD + c2] -= Pn[r * PLD + c] * Pn[c2 * PLD + c];
            }
          }
          __syncthreads();
        }
        for (int e = tid; e < R * bw; e += K5_THREADS) {
          const int r = e / bw, c = e % bw;
          if (c <= r) A[tri(j0 + r) + j0 + c] = Pn[r * PLD + c];
        }
        // trailing update A[i][k] -= Σ_c Pn[i-j0][c] Pn[k-j0][c], j0+bw <= k <= i < L, 4x4 tiles
        const int j1 = j0 + bw, R2 = L - j1;
        if (R2 > 0) {
          const int nt = (R2 + 3) / 4;
          const int ntile = nt * (nt + 1) / 2;
          for (int t = tid; t < ntile; t += K5_THREADS) {
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
            const double* pi = Pn + (i0 - j0) * PLD;
            const double* pk = Pn + (k0 - j0) * PLD;
            for (int c = 0; c < bw; ++c) {
              double av[4], bv[4];
#pragma unroll
              for (int a = 0; a < 4; ++a) av[a] = (i0 + a < L) ? pi[a * PLD + c] : 0.0;
#pragma unroll
              for (int b = 0; b < 4; ++b) bv[b] = (k0 + b < L) ? pk[b * PLD + c] : 0.0;
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
                if (i < L && k <= i) A[tri(i) + k] -= acc[a][b];
              }
          }
        }
        __syncthreads();
      }
    }
    // forward substitution R̃ᵀ y = b̃
    for (int j = 0; j < L; ++j) {
      const double p = piv[j];
      const double yj = p > 0.0 ? sb[j] / p : 0.0;
      __syncthreads();
      for (int i = j + 1 + tid; i < L; i += K5_THREADS) sb[i] -= A[tri(i) + j] * yj;
      if (tid == 0) sb[j] = yj;
      __syncthreads();
    }
    // back substitution R̃ c̃ = y
    for (int j = L - 1; j >= 0; --j) {
      const double p = piv[j];
      const double cj = p > 0.0 ? sb[j] / p : 0.0;
      __syncthreads();
      const double* Aj = A + tri(j);
      for (int i = tid; i < j; i += K5_THREADS) sb[i] -= Aj[i] * cj;
      if (tid == 0) sb[j] = cj;
      __syncthreads();
    }
    double* out = nt.coef + (first + node) * (int64_t)L;
    if (mode == 1) {  // refinement correction δ (monomial form): delta[node] = δ, coef += δ
      for (int i = tid; i < L; i += K5_THREADS) {
        const double d = sb[i] * dinv[i];
        delta[node * (int64_t)L + i] = d;
        out[i] += d;
      }
      __syncthreads();
      continue;
    }
    for (int i = tid; i < L; i += K5_THREADS) out[i] = sb[i] * dinv[i];
    if (tid == 0) {
      int rk = 0;
      double mn = INFINITY;
      for (int i = 0; i < L; ++i)
        if (piv[i] > 0.0) { ++rk; mn = fmin(mn, piv[i]); }
      nt.rank[first + node] = rk;
      nt.minpiv[first + node] = rk ? mn : 0.0;
      // robust-path flag: a pivot of a non-zero column fell where fp64 Gram pivots stop tracking the
      // QR pivots (or the column was rejected) -> K5q re-fits the node by Householder QR
      // semi-normal refinement flag (bit 1): small pivots, or few points per unknown, where the normal
      // equations lose digits (DESIGN.md §5 K5r)
      const double npts = (double)(nt.end[first + node] - nt.start[first + node]);
      const bool refine = refine2 > 0.0 && (smin_sh[0] < refine2 || npts < refine_fill * L);
      const int fl = (smin_sh[0] < kQrFlagPivot2) ? 1 : (refine ? 2 : 0);
      nt.flag[first + node] = fl;
      if (fl == 2) atomicAdd(reinterpret_cast<unsigned long long*>(nflag), 1ull);
    }
    __syncthreads();
  }
}

}  // namespace

template <int P>
void level_solve(const LevelCtx& c, const double* mom, int mode, const double* segrhs, double* delta, double refine2,
                 int64_t* nflag, double* scratch, int64_t scratch_nodes, cudaStream_t s) {
  using S = K5Shape<P>;
  static const BasisTab bt = make_basis<P>();
  static bool attr = false;
  if (!attr) {
    FMI_CK(cudaFuncSetAttribute(k_solve<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    attr = true;
  }
  int64_t grid = c.count;
  if (!S::kSmemA) grid = std::min<int64_t>(grid, scratch_nodes);
  grid = std::min<int64_t>(grid, 1 << 20);
  FMI_LAUNCH(mode == 1 ? KID_REFINE_SOLVE : KID_SOLVE, s, k_solve<P>, (unsigned)grid, K5_THREADS, S::SMEM, mom, mode,
             segrhs, delta, c.nt, c.first, c.count, scratch, bt, kDelta * kDelta, refine2, kRefineFill, kMomentTol,
             nflag);
}

// bytes of global scratch the solve needs per concurrently processed node (0 if shared-memory resident)
size_t solve_scratch_per_node(int p) {
  switch (p) {
#define C(P) case P: return K5Shape<P>::kSmemA ? 0 : (size_t)K5Shape<P>::NA * sizeof(double);
    C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10)
#undef C
  }
  return 0;
}

#define FMI_INST(P) \
  template void level_solve<P>(const LevelCtx&, const double*, int, const double*, double*, double, int64_t*, \
                               double*, int64_t, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
