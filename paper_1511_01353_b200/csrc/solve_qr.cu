// solve_qr.cu — K5q: Householder-QR node solve for ill-conditioned nodes (DESIGN.md §3 K5q).
//
// The moment-Gram solve (K5) squares the condition number; its Schur-complement pivots stop tracking
// the QR pivots |R_jj|² once they fall below ~1e-10 (clustered or degenerate point sets), and the
// column-rejection decisions of reading G9 then become unreliable.  K5 flags such nodes; this kernel
// re-fits them exactly as PAPER.md Algorithm 2 does (QR of Λ, P_F = R⁻¹Qᵀf):
//   1. row-streamed Householder QR (TSQR) of the equilibrated [Λ D⁻¹ | r] over the node's points:
//      R <- qr([R; block]) for blocks of QB points (only the block rows and the diagonal carry
//      non-zeros below the diagonal, so each reflector touches 1 + QB rows);
//   2. column rejection on R (a column whose distance from the span of the kept columns is <= kDelta
//      is dropped), identical to the oracle's walk;
//   3. back substitution R_S c̃ = (Qᵀr)_S and a_α = c̃_α / sqrt(M_{2α}).
// One CTA per flagged node; the (𝓛+1) × (𝓛+1+QB) work matrix lives in a per-CTA global scratch slot
// (L2-resident).  Non-flagged nodes exit immediately.
#include <algorithm>
#include <mutex>

#include "horner.cuh"

namespace fmi {

namespace {

constexpr int KQ_THREADS = 256;
// points per TSQR block: 128 when the shared-memory work matrix still fits (fewer, longer reflector
// steps: the step cost is dominated by its reduction latency), else 64
__host__ __device__ constexpr int qb_of(int p) {
  return (size_t)(rank3(p) + 1) * (rank3(p) + 1 + 128) * sizeof(double) <= 200 * 1024 ? 128 : 64;
}

// dynamic shared memory of the work matrix (0: global scratch)
__host__ __device__ constexpr size_t qr_smem_bytes(int p) {
  return (size_t)(rank3(p) + 1) * (rank3(p) + 1 + qb_of(p)) * sizeof(double) <= 200 * 1024
             ? (size_t)(rank3(p) + 1) * (rank3(p) + 1 + qb_of(p)) * sizeof(double)
             : 0;
}

struct BasisTabQ {
  uint8_t l[286], m[286], n[286];
};

template <int P>
BasisTabQ make_basis_q() {
  BasisTabQ b{};
  int i = 0;
  for (int l = 0; l <= P; ++l)
    for (int m = 0; m <= P - l; ++m)
      for (int n = 0; n <= P - l - m; ++n) { b.l[i] = (uint8_t)l; b.m[i] = (uint8_t)m; b.n[i] = (uint8_t)n; ++i; }
  return b;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < KQ_THREADS / 32; ++w) s += red[w];
  return s;
}

template <int P>
__global__ void __launch_bounds__(KQ_THREADS)
    k_solve_qr(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
               const double* __restrict__ r, NodeTable nt, int64_t first, int64_t count,
               const double* __restrict__ mom, double* __restrict__ scratch, const __grid_constant__ BasisTabQ bt,
               double delta) {
  constexpr int Q = 2 * P, K = rank3(Q), L = rank3(P), LA = L + 1;
  constexpr int QB = qb_of(P);
  constexpr int LD = LA + QB;  // leading dimension (rows) of the column-major work matrix
  __shared__ double dinv[LA];
  __shared__ double v[LD];
  __shared__ double red[KQ_THREADS / 32];
  __shared__ int kept[L];
  __shared__ double piv[L];
  __shared__ double sol[L];
  // the work matrix in shared memory when it fits (p <= 7: 𝓛 = 84 -> 101 KB), else in the CTA's global
  // scratch slot (L2-resident): every reflector step is a chain of dependent accesses, so the on-chip copy
  // cuts its latency several-fold
  constexpr bool kSmem = qr_smem_bytes(P) > 0;
  extern __shared__ __align__(16) double qsm[];
  double* A = kSmem ? qsm : scratch + (int64_t)blockIdx.x * LA * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = KQ_THREADS / 32;
  __shared__ uint8_t bl[L], bm[L], bn[L];
  for (int i = tid; i < L; i += KQ_THREADS) { bl[i] = bt.l[i]; bm[i] = bt.m[i]; bn[i] = bt.n[i]; }
  __syncthreads();

  for (int64_t ln = blockIdx.x; ln < count; ln += gridDim.x) {
    const int64_t node = first + ln;
    if (!(nt.flag[node] & 1)) continue;
    const double* mp = mom + ln * (int64_t)(2 * K + L);
    for (int i = tid; i < L; i += KQ_THREADS) {
      const double m2 = mp[basis_index(Q, 2 * bl[i], 2 * bm[i], 2 * bn[i])];
      dinv[i] = m2 > 0.0 ? 1.0 / sqrt(m2) : 0.0;
    }
    if (tid == 0) dinv[L] = 1.0;  // the residual column is not scaled
    for (int e = tid; e < LA * LD; e += KQ_THREADS) A[e] = 0.0;
    __syncthreads();
    const int4 cc = nt.cell[node];
    const double h = ldexp(1.0, -(cc.w + 1)), scale = ldexp(1.0, cc.w + 1);
    const double cx = (2.0 * cc.x + 1.0) * h, cy = (2.0 * cc.y + 1.0) * h, cz = (2.0 * cc.z + 1.0) * h;
    const int64_t s0 = nt.start[node], s1 = nt.end[node];

    // ---- 1. TSQR over blocks of QB points --------------------------------------------------------
    for (int64_t b0 = s0; b0 < s1; b0 += QB) {
      const int nb = (int)min((int64_t)QB, s1 - b0);
      // block rows LA..LA+nb-1: equilibrated monomials and the residual
      for (int e = tid; e < QB * LA; e += KQ_THREADS) {
        const int row = e % QB, col = e / QB;
        double val = 0.0;
        if (row < nb) {
          const int64_t pi = b0 + row;
          if (col < L) {
            const double x = to_local(ux[pi], cx, scale);
            const double y = to_local(uy[pi], cy, scale);
            const double z = to_local(uz[pi], cz, scale);
            double m = 1.0;
            for (int k = 0; k < bl[col]; ++k) m *= x;
            for (int k = 0; k < bm[col]; ++k) m *= y;
            for (int k = 0; k < bn[col]; ++k) m *= z;
            val = m * dinv[col];
          } else {
            val = r[pi];
          }
        }
        A[(int64_t)col * LD + LA + row] = val;
      }
      __syncthreads();
      // structured Householder: column j has non-zeros at row j and rows LA.. only
      for (int j = 0; j < LA; ++j) {
        double* Aj = A + (int64_t)j * LD;
        double part = 0.0;
        for (int i = tid; i < QB; i += KQ_THREADS) { const double t = Aj[LA + i]; part += t * t; }
        const double sb = block_sum(part, red);
        if (sb == 0.0) { __syncthreads(); continue; }  // nothing below the diagonal: reflector = I
        const double d = Aj[j];
        const double nrm = sqrt(d * d + sb);
        const double alpha = d >= 0.0 ? -nrm : nrm;
        const double v0 = d - alpha;
        const double vtv = v0 * v0 + sb;
        const double beta = 2.0 / vtv;
        for (int i = tid; i < QB; i += KQ_THREADS) v[i] = Aj[LA + i];
        __syncthreads();
        // four columns per warp at a time: their dot products and shuffle reductions overlap
        for (int c0 = j + 1 + warp; c0 < LA; c0 += 4 * NWARP) {
          double w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * NWARP;
            w[u] = 0.0;
            if (c < LA) {
              const double* Ac = A + (int64_t)c * LD;
#pragma unroll
              for (int i = lane; i < QB; i += 32) w[u] += v[i] * Ac[LA + i];
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] += __shfl_xor_sync(0xffffffffu, w[u], o);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * NWARP;
            if (c < LA) {
              double* Ac = A + (int64_t)c * LD;
              const double bw = beta * (w[u] + v0 * Ac[j]);
#pragma unroll
              for (int i = lane; i < QB; i += 32) Ac[LA + i] -= bw * v[i];
              if (lane == 0) Ac[j] -= bw * v0;
            }
          }
        }
        __syncthreads();
        if (tid == 0) Aj[j] = alpha;
        for (int i = tid; i < QB; i += KQ_THREADS) Aj[LA + i] = 0.0;
        __syncthreads();
      }
    }

    // ---- 2. column rejection on R (rows 0..LA-1), rhs = column L ---------------------------------
    int k = 0;  // rows consumed by kept columns
    for (int j = 0; j < L; ++j) {
      double* Aj = A + (int64_t)j * LD;
      double part = 0.0;
      for (int i = k + tid; i < LA; i += KQ_THREADS) { const double t = Aj[i]; part += t * t; }
      const double nrm2 = block_sum(part, red);
      const double nrm = sqrt(nrm2);
      const bool keep = dinv[j] > 0.0 && nrm > delta;
      if (tid == 0) { kept[j] = keep ? k : -1; piv[j] = keep ? nrm : 0.0; }
      if (!keep) { __syncthreads(); continue; }
      const double d = Aj[k];
      const double alpha = d >= 0.0 ? -nrm : nrm;
      const double v0 = d - alpha;
      const double vtv = nrm2 - d * d + v0 * v0;
      const double beta = vtv > 0.0 ? 2.0 / vtv : 0.0;
      for (int i = k + tid; i < LA; i += KQ_THREADS) v[i] = (i == k) ? v0 : Aj[i];
      __syncthreads();
      for (int c = j + 1 + warp; c < LA; c += NWARP) {
        double* Ac = A + (int64_t)c * LD;
        double w = 0.0;
        for (int i = k + lane; i < LA; i += 32) w += v[i] * Ac[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        const double bw = beta * w;
        for (int i = k + lane; i < LA; i += 32) Ac[i] -= bw * v[i];
      }
      __syncthreads();
      if (tid == 0) Aj[k] = alpha;
      __syncthreads();
      ++k;
    }
    __syncthreads();

    // ---- 3. back substitution over the kept columns (row kept[j] holds column j's pivot) -----------
    const double* Ar = A + (int64_t)L * LD;  // Qᵀr
    for (int i = tid; i < L; i += KQ_THREADS) sol[i] = (kept[i] >= 0) ? Ar[kept[i]] : 0.0;
    __syncthreads();
    for (int j = L - 1; j >= 0; --j) {
      const int row = kept[j];
      if (row < 0) continue;  // uniform across the block
      const double* Aj = A + (int64_t)j * LD;
      const double cj = sol[j] / Aj[row];
      __syncthreads();
      // sol[i] -= R[row_i, j] * c_j for kept i < j, where R[row_i, j] = A[j][kept[i]]
      for (int i = tid; i < j; i += KQ_THREADS)
        if (kept[i] >= 0) sol[i] -= Aj[kept[i]] * cj;
      if (tid == 0) sol[j] = cj;
      __syncthreads();
    }
    double* out = nt.coef + node * (int64_t)L;
    for (int i = tid; i < L; i += KQ_THREADS) out[i] = sol[i] * dinv[i];
    if (tid == 0) {
      int rk = 0;
      double mn = INFINITY;
      for (int i = 0; i < L; ++i)
        if (kept[i] >= 0) { ++rk; mn = fmin(mn, fabs(piv[i])); }
      nt.rank[node] = rk;
      nt.minpiv[node] = rk ? mn : 0.0;
    }
    __syncthreads();
  }
}

}  // namespace

size_t solve_qr_scratch_per_cta(int p) {
  const int L = rank3(p), LA = L + 1;
  return (size_t)LA * (LA + qb_of(p)) * sizeof(double);
}

template <int P>
void level_solve_qr(const LevelCtx& c, const double* mom, double* scratch, int64_t slots, cudaStream_t s) {
  static const BasisTabQ bt = make_basis_q<P>();
  constexpr size_t smem = qr_smem_bytes(P);
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    if (smem > 0) FMI_CK(cudaFuncSetAttribute(k_solve_qr<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  const int64_t grid = std::min<int64_t>(c.count, slots);
  if (grid <= 0) return;
  FMI_LAUNCH(KID_SOLVE_QR, s, k_solve_qr<P>, (unsigned)grid, KQ_THREADS, smem, c.ux, c.uy, c.uz, c.r, c.nt, c.first,
             c.count, mom, scratch, bt, kDelta);
}

#define FMI_INST(P) template void level_solve_qr<P>(const LevelCtx&, const double*, double*, int64_t, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
