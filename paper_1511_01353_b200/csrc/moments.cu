// moments.cu — K4: per-node raw geometric moments and projection (DESIGN.md §3 K4).
//
// PAPER.md Algorithm 2 builds Λ(1:N, lmn) = x^l y^m z^n/(l!m!n!) and factors it (QR).  In
// Gram form every entry of ΛᵀΛ is a raw moment,  G_αβ = M_{α+β}/(α!β!),  M_γ = Σ_i u_i^γ, |γ| <= 2p,
// and the projection Λᵀr needs  b_α = Σ_i u_i^α r_i, |α| <= p  (the factorials are applied in the
// solve).  Per point that is C(2p+3,3) + 𝓛 multiply-adds instead of the dense Gram's 𝓛(𝓛+1)/2.
//
// The moments are computed as a masked outer-product contraction over the points of a chunk:
//   rows  (a,b), a+b <= 2p   X_i(a,b) = x_i^a y_i^b            (materialised per batch in smem)
//   cols  c = 0..2p          W_i(c)   = z_i^c                  moment entries a+b+c <= 2p
//         c' = 0..p          W_i(c')  = r_i z_i^c'             projection entries a+b+c' <= p
// Each thread owns a 4 rows × 4 cols register tile (16 fp64 accumulators) of the needed part of
// the (a,b) × c grid; rows are sorted by a+b so ragged tiles waste little.  Point batches are
// software-pipelined through shared memory (load/powers -> X -> accumulate, one barrier per batch).
// Several thread groups split the points of a chunk; their tiles are reduced in a fixed order, and
// chunk partials are reduced per node in chunk order (deterministic, no atomics).
#include <algorithm>
#include <vector>

#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int K4_THREADS = 512;
constexpr int K4_MAXROWP = 232;   // (2p+1)(2p+2)/2 rounded to 4 at p = 10
constexpr int K4_MAXTILE = 256;

// PROJ = false: moments (|γ| <= 2p) and projection; PROJ = true: projection only (refinement pass).
template <int P, bool PROJ = false>
struct K4Shape {
  static constexpr int Q = PROJ ? P : 2 * P;     // highest power generated
  static constexpr int NROW = (Q + 1) * (Q + 2) / 2;
  static constexpr int NROWP = (NROW + 3) / 4 * 4;
  static constexpr int CM = PROJ ? 0 : (Q + 1 + 3) / 4 * 4;
  static constexpr int CP = (P + 1 + 3) / 4 * 4;
  static constexpr int NW = CM + CP;
  static constexpr int NPW = 2 * (Q + 1);  // px[0..Q], py[0..Q]
  static constexpr int K = PROJ ? 0 : rank3(Q);   // moment entries written per chunk
  static constexpr int L = rank3(P);
};

struct K4Tab {
  int ntile;
  int groups;
  int batch;
  int pad;
  uint8_t rowA[K4_MAXROWP];
  uint8_t rowB[K4_MAXROWP];
  uint16_t tile[K4_MAXTILE];  // (row group << 8) | col block
};

template <int P, bool PROJ = false>
K4Tab make_tab() {
  using S = K4Shape<P, PROJ>;
  K4Tab t{};
  int row = 0;
  for (int s = 0; s <= S::Q; ++s)
    for (int a = 0; a <= s; ++a) { t.rowA[row] = (uint8_t)a; t.rowB[row] = (uint8_t)(s - a); ++row; }
  for (; row < S::NROWP; ++row) { t.rowA[row] = 255; t.rowB[row] = 255; }
  int nt = 0;
  for (int g = 0; g < S::NROWP / 4; ++g) {
    int smin = 1 << 20;
    for (int i = 0; i < 4; ++i) {
      int rr = 4 * g + i;
      if (rr < S::NROW) smin = std::min(smin, t.rowA[rr] + t.rowB[rr]);
    }
    int nm = PROJ ? 0 : (S::Q - smin + 1 + 3) / 4;
    for (int cb = 0; cb < nm; ++cb) t.tile[nt++] = (uint16_t)((g << 8) | cb);
    if (smin <= P) {
      int np = (P - smin + 1 + 3) / 4;
      for (int cb = 0; cb < np; ++cb) t.tile[nt++] = (uint16_t)((g << 8) | (S::CM / 4 + cb));
    }
  }
  t.ntile = nt;
  t.groups = std::max(1, K4_THREADS / nt);
  // points per batch: a multiple of the group count, ~32-48 points
  int per = std::max(1, (40 + t.groups - 1) / t.groups);
  t.batch = per * t.groups;
  if (t.batch > 64) t.batch = t.groups * std::max(1, 64 / t.groups);
  return t;
}

template <int P, bool PROJ = false>
size_t k4_smem_bytes(const K4Tab& t) {
  using S = K4Shape<P, PROJ>;
  size_t pipe = (size_t)t.batch * (2 * S::NROWP + 3 * S::NW + 2 * S::NPW);
  size_t red = (size_t)t.groups * t.ntile * 16;
  return std::max(pipe, red) * sizeof(double);
}

template <int P, bool PROJ>
__global__ void __launch_bounds__(K4_THREADS, 1)
    k_moments(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
              const double* __restrict__ r, const int4* __restrict__ cell, int64_t first,
              const Chunk* __restrict__ chunks, const int64_t* __restrict__ nchunks, const __grid_constant__ K4Tab tab,
              const int32_t* __restrict__ skip_flag, double* __restrict__ partial) {
  using S = K4Shape<P, PROJ>;
  constexpr int Q = S::Q;
  extern __shared__ double smem[];
  const int64_t cidx = blockIdx.x;
  if (cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  if (PROJ && (skip_flag[first + ck.owner] & 3)) return;  // QR-path or converged node: no refinement
  const int4 c = cell[first + ck.owner];
  const double h = ldexp(1.0, -(c.w + 1));
  const double scale = ldexp(1.0, c.w + 1);
  const double cx = (2.0 * c.x + 1.0) * h, cy = (2.0 * c.y + 1.0) * h, cz = (2.0 * c.z + 1.0) * h;

  const int B = tab.batch, G = tab.groups, NT = tab.ntile;
  double* sX = smem;                              // [2][B][NROWP]
  double* sW = sX + 2 * B * S::NROWP;             // [3][B][NW]
  double* sP = sW + 3 * B * S::NW;                // [2][B][NPW]
  const int tid = threadIdx.x;
  const int grp = tid / NT;
  const int t = tid - grp * NT;
  const bool worker = grp < G;
  int rg = 0, cb = 0;
  if (worker) { rg = tab.tile[t] >> 8; cb = tab.tile[t] & 255; }

  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;

  const int64_t n = ck.end - ck.start;
  const int nbatch = (int)((n + B - 1) / B);

  for (int it = -2; it < nbatch; ++it) {
    // stage A (batch it+2): local coordinates, powers, W row
    const int ia = it + 2;
    if (ia < nbatch && tid < B) {
      const int64_t pi = ck.start + (int64_t)ia * B + tid;
      double* Pp = sP + (ia & 1) * B * S::NPW + tid * S::NPW;
      double* Wp = sW + (ia % 3) * B * S::NW + tid * S::NW;
      if (pi < ck.end) {
        const double x = __dmul_rn(__dsub_rn(ux[pi], cx), scale);
        const double y = __dmul_rn(__dsub_rn(uy[pi], cy), scale);
        const double z = __dmul_rn(__dsub_rn(uz[pi], cz), scale);
        const double rv = r[pi];
        double px = 1.0, py = 1.0, pz = 1.0;
#pragma unroll
        for (int q = 0; q <= Q; ++q) {
          Pp[q] = px;
          Pp[Q + 1 + q] = py;
          Wp[q] = pz;
          if (q <= P) Wp[S::CM + q] = rv * pz;
          px *= x; py *= y; pz *= z;
        }
#pragma unroll
        for (int q = Q + 1; q < S::CM; ++q) Wp[q] = 0.0;
#pragma unroll
        for (int q = S::CM + P + 1; q < S::NW; ++q) Wp[q] = 0.0;
      } else {
#pragma unroll
        for (int q = 0; q < S::NPW; ++q) Pp[q] = 0.0;
#pragma unroll
        for (int q = 0; q < S::NW; ++q) Wp[q] = 0.0;
      }
    }
    // stage B (batch it+1): X(a,b) = x^a y^b
    const int ib = it + 1;
    if (ib >= 0 && ib < nbatch) {
      const double* Pp = sP + (ib & 1) * B * S::NPW;
      double* Xp = sX + (ib & 1) * B * S::NROWP;
      for (int e = tid; e < B * S::NROWP; e += K4_THREADS) {
        const int j = e / S::NROWP;
        const int row = e - j * S::NROWP;
        const int a = tab.rowA[row], b = tab.rowB[row];
        Xp[e] = (a <= Q) ? Pp[j * S::NPW + a] * Pp[j * S::NPW + Q + 1 + b] : 0.0;
      }
    }
    // stage C (batch it): 4×4 register-tile outer products
    if (it >= 0 && worker) {
      const double* Xp = sX + (it & 1) * B * S::NROWP + 4 * rg;
      const double* Wp = sW + (it % 3) * B * S::NW + 4 * cb;
      const int nb = (int)min((int64_t)B, n - (int64_t)it * B);
#pragma unroll 2
      for (int j = grp; j < nb; j += G) {
        const double2 x01 = *reinterpret_cast<const double2*>(Xp + j * S::NROWP);
        const double2 x23 = *reinterpret_cast<const double2*>(Xp + j * S::NROWP + 2);
        const double2 w01 = *reinterpret_cast<const double2*>(Wp + j * S::NW);
        const double2 w23 = *reinterpret_cast<const double2*>(Wp + j * S::NW + 2);
        const double xv[4] = {x01.x, x01.y, x23.x, x23.y};
        const double wv[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[i * 4 + k] = fma(xv[i], wv[k], acc[i * 4 + k]);
      }
    }
    __syncthreads();
  }

  // fixed-order reduction over the point groups, then scatter the needed entries to the partial
  double* red = smem;
  if (worker) {
#pragma unroll
    for (int k = 0; k < 16; ++k) red[(grp * NT + t) * 16 + k] = acc[k];
  }
  __syncthreads();
  if (grp == 0 && worker) {
    double* out = partial + cidx * (int64_t)(S::K + S::L);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = 4 * rg + i;
      const int a = tab.rowA[row], b = tab.rowB[row];
      if (a > Q) continue;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double v = 0.0;
        for (int g = 0; g < G; ++g) v += red[(g * NT + t) * 16 + i * 4 + k];
        const int col = 4 * cb + k;
        if (col < S::CM) {
          if (!PROJ && a + b + col <= Q) out[basis_index(Q, a, b, col)] = v;
        } else {
          const int cc = col - S::CM;
          if (a + b + cc <= P) out[S::K + basis_index(P, a, b, cc)] = v;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_moments_reduce(const double* __restrict__ partial,
                                                        const int64_t* __restrict__ chunk_begin,
                                                        const int64_t* __restrict__ nchunks, int64_t count, int KL,
                                                        double* __restrict__ mom) {
  const int64_t node = blockIdx.x;
  const int64_t c0 = chunk_begin[node];
  const int64_t c1 = node + 1 < count ? chunk_begin[node + 1] : *nchunks;
  for (int e = threadIdx.x; e < KL; e += blockDim.x) {
    double s = 0.0;
    for (int64_t ci = c0; ci < c1; ++ci) s += partial[ci * KL + e];
    mom[node * KL + e] = s;
  }
}

}  // namespace

template <int P, bool PROJ>
void launch_moments(const LevelCtx& c, const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks,
                    const int64_t* chunk_begin, const double* r, double* partial, double* mom, cudaStream_t s) {
  using S = K4Shape<P, PROJ>;
  static const K4Tab tab = make_tab<P, PROJ>();
  static const size_t smem = k4_smem_bytes<P, PROJ>(tab);
  static bool attr = false;
  if (!attr) {
    FMI_CK(cudaFuncSetAttribute(k_moments<P, PROJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (max_chunks <= 0) return;
  FMI_LAUNCH(PROJ ? KID_PROJECT : KID_MOMENTS, s, (k_moments<P, PROJ>), (unsigned)max_chunks, K4_THREADS, smem, c.ux,
             c.uy, c.uz, r, c.nt.cell, c.first, chunks, nchunks_dev, tab, c.nt.flag, partial);
  FMI_LAUNCH(KID_MOMENTS_REDUCE, s, k_moments_reduce, (unsigned)c.count, 256, 0, partial, chunk_begin, nchunks_dev,
             c.count, S::K + S::L, mom);
}

template <int P>
void level_moments(const LevelCtx& c, const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks,
                   const int64_t* chunk_begin, double* partial, double* mom, cudaStream_t s) {
  launch_moments<P, false>(c, chunks, nchunks_dev, max_chunks, chunk_begin, c.r, partial, mom, s);
}

template <int P>
void level_project(const LevelCtx& c, const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks,
                   const int64_t* chunk_begin, double* partial, double* proj, cudaStream_t s) {
  launch_moments<P, true>(c, chunks, nchunks_dev, max_chunks, chunk_begin, c.r, partial, proj, s);
}

#define FMI_INST(P)                                                                                           \
  template void level_moments<P>(const LevelCtx&, const Chunk*, const int64_t*, int64_t, const int64_t*, double*, \
                                 double*, cudaStream_t);                                                          \
  template void level_project<P>(const LevelCtx&, const Chunk*, const int64_t*, int64_t, const int64_t*, double*, \
                                 double*, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

// tile statistics for DESIGN.md / bench (useful fraction of the issued FMAs)
int k4_tile_count(int p) {
  switch (p) {
#define C(P) case P: return make_tab<P>().ntile;
    C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10)
#undef C
  }
  return 0;
}

}  // namespace fmi
