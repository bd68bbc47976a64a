// moments.cu — K4: per-node raw geometric moments and projection (DESIGN.md §3 K4).
//
// PAPER.md Algorithm 2 builds Λ(1:N, lmn) = x^l y^m z^n/(l!m!n!) and factors it (QR).  In
// Gram form every entry of ΛᵀΛ is a raw moment,  G_αβ = M_{α+β}/(α!β!),  M_γ = Σ_i u_i^γ, |γ| <= 2p,
// and the projection Λᵀr needs  b_α = Σ_i u_i^α r_i, |α| <= p  (the factorials are applied in the
// solve).  Per point that is C(2p+3,3) + 𝓛 multiply-adds instead of the dense Gram's 𝓛(𝓛+1)/2.
//
// The moments are a masked outer-product contraction over the points of a chunk:
//   rows  (a,b), a+b <= 2p   X_i(a,b) = x_i^a y_i^b
//   cols  c = 0..2p          W_i(c)   = z_i^c          -> moment entries a+b+c <= 2p
//         c' = 0..p          W_i(c')  = r_i z_i^c'     -> projection entries a+b+c' <= p
// Rows are ordered by s = a+b (then a) and cut into groups of 8; columns into blocks of 4.  Every
// consumer thread owns one needed 8×4 tile (32 fp64 accumulators).  Per batch of B points:
//   produce: warp-uniform tasks write whole rows X(a, ·) / W(·) for 32 consecutive points (lanes =
//            points, so stores are conflict-free); slot layouts are "row-in-tile major" so that the
//            16-byte loads of a warp whose lanes own different tiles spread over all banks;
//   consume: each thread walks point PAIRS (j, j+1): 8 + 4 LDS.128 feed 64 DFMA.
// Production of batch k+1 and consumption of batch k share one barrier interval (double buffer).
// Thread groups split a chunk's points; their tiles are reduced in a fixed order, and chunk
// partials per node in chunk order (deterministic, no atomics).
#include <algorithm>
#include <vector>

#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int K4_THREADS = 512;
constexpr int K4_WARPS = K4_THREADS / 32;
constexpr int K4_MAXTILE = 96;      // 84 at p = 10
constexpr int K4_MAXTASK = 64;
constexpr int K4_TASKS_PER_WARP = 8;
constexpr size_t K4_SMEM_LIMIT = 220 * 1024;

// PROJ = false: moments (|γ| <= 2p) and projection; PROJ = true: projection only (refinement pass).
template <int P, bool PROJ = false>
struct K4Shape {
  static constexpr int Q = PROJ ? P : 2 * P;     // highest power of x, y in the rows
  static constexpr int NROW = (Q + 1) * (Q + 2) / 2;
  static constexpr int NRG = (NROW + 7) / 8;      // 8-row groups
  static constexpr int NROWP = 8 * NRG;
  static constexpr int CM = PROJ ? 0 : (Q + 1 + 3) / 4 * 4;
  static constexpr int CP = (P + 1 + 3) / 4 * 4;
  static constexpr int NW = CM + CP;
  static constexpr int NCB = NW / 4;              // 4-column blocks
  static constexpr int K = PROJ ? 0 : rank3(Q);   // moment entries written per chunk
  static constexpr int L = rank3(P);
};

constexpr int row_s(int r) {
  int s = 0;
  while ((s + 1) * (s + 2) / 2 <= r) ++s;
  return s;
}

// compile-time geometry: tiles, point groups G, batch B, smem row stride SS = B + 2
template <int P, bool PROJ>
struct K4Geo {
  using S = K4Shape<P, PROJ>;
  static constexpr int ntile() {
    int nt = 0;
    for (int g = 0; g < S::NRG; ++g) {
      const int smin = row_s(8 * g);  // rows are sorted by s: the first row of a group has the least s
      nt += PROJ ? 0 : (S::Q - smin + 1 + 3) / 4;
      if (smin <= P) nt += (P - smin + 1 + 3) / 4;
    }
    return nt;
  }
  static constexpr int NT = ntile();
  static constexpr int GMAX = (K4_THREADS / NT) < 64 ? (K4_THREADS / NT) : 64;
  static constexpr long pick() {  // returns G * 1000 + B maximising thread use, then batch size
    long best = -1, arg = 1004;
    for (int G = (GMAX > 0 ? GMAX : 1); G >= 1; --G)
      for (int k = 1; k <= 64; ++k) {
        const int B = 2 * G * k;
        if (B % 4) continue;
        if (B > 128) break;
        const long pipe = 2L * (S::NROWP + S::NW) * (B + 2) * 8;
        if (pipe > (long)K4_SMEM_LIMIT) break;
        const long score = (long)(G * NT) * 1000 / K4_THREADS * 1000 + (B < 64 ? B : 64);
        if (score > best) { best = score; arg = (long)G * 1000 + B; }
      }
    return arg;
  }
  static constexpr int G = (int)(pick() / 1000);
  static constexpr int B = (int)(pick() % 1000);
  static constexpr int SS = B + 2;
  static constexpr int NLG = (B + 31) / 32;
  static constexpr int BUF = (S::NROWP + S::NW) * SS;  // doubles per pipeline buffer
};

struct K4Tab {
  int ntile;          // consumer tiles (needed 8×4 blocks)
  int groups;         // point groups (tile sets working on disjoint point pairs)
  int batch;          // points per batch B (multiple of 4)
  int stride;         // smem row stride S = B + 2 (S ≡ 2 mod 4: bank-spread 16-byte loads)
  int nlane_groups;   // ceil(B / 32)
  int ntask;
  uint16_t tile[K4_MAXTILE];                         // (row group << 8) | col block
  uint8_t task_a[K4_MAXTASK];                        // 255 = W task, else the x power a of an X task
  uint8_t task_h[K4_MAXTASK];                        // lane group
  uint8_t warp_task[K4_WARPS][K4_TASKS_PER_WARP];    // tasks of each warp (255 = none)
};

// exponents (a, b) of row r in the (s = a+b, a) order
__host__ __device__ __forceinline__ void row_exponents(int r, int& a, int& b) {
  int s = 0;
  while ((s + 1) * (s + 2) / 2 <= r) ++s;
  a = r - s * (s + 1) / 2;
  b = s - a;
}

template <int P, bool PROJ = false>
K4Tab make_tab() {
  using S = K4Shape<P, PROJ>;
  K4Tab t{};
  int nt = 0;
  for (int g = 0; g < S::NRG; ++g) {
    int smin = 1 << 20;
    for (int i = 0; i < 8; ++i) {
      const int rr = 8 * g + i;
      if (rr < S::NROW) { int a, b; row_exponents(rr, a, b); smin = std::min(smin, a + b); }
    }
    const int nm = PROJ ? 0 : (S::Q - smin + 1 + 3) / 4;
    for (int cb = 0; cb < nm; ++cb) t.tile[nt++] = (uint16_t)((g << 8) | cb);
    if (smin <= P) {
      const int np = (P - smin + 1 + 3) / 4;
      for (int cb = 0; cb < np; ++cb) t.tile[nt++] = (uint16_t)((g << 8) | (S::CM / 4 + cb));
    }
  }
  t.ntile = nt;
  using Geo = K4Geo<P, PROJ>;
  static_assert(Geo::NT <= K4_MAXTILE, "tile table too small");
  t.groups = Geo::G;
  t.batch = Geo::B;
  t.stride = Geo::SS;
  t.nlane_groups = Geo::NLG;
  // production tasks: X rows for every power a of x and lane group, one W task per lane group;
  // longest-processing-time assignment to the 16 warps
  struct Task { int a, h, len; };
  std::vector<Task> tasks;
  for (int h = 0; h < t.nlane_groups; ++h) {
    for (int a = 0; a <= S::Q; ++a) tasks.push_back({a, h, S::Q - a + 1 + 4});
    tasks.push_back({255, h, S::NW});
  }
  std::sort(tasks.begin(), tasks.end(), [](const Task& x, const Task& y) { return x.len > y.len; });
  t.ntask = (int)tasks.size();
  std::vector<int> load(K4_WARPS, 0), cnt(K4_WARPS, 0);
  for (int w = 0; w < K4_WARPS; ++w)
    for (int k = 0; k < K4_TASKS_PER_WARP; ++k) t.warp_task[w][k] = 255;
  for (int i = 0; i < t.ntask; ++i) {
    int w = 0;
    for (int v = 1; v < K4_WARPS; ++v)
      if (cnt[v] < K4_TASKS_PER_WARP && (load[v] < load[w] || cnt[w] >= K4_TASKS_PER_WARP)) w = v;
    t.task_a[i] = (uint8_t)tasks[i].a;
    t.task_h[i] = (uint8_t)tasks[i].h;
    t.warp_task[w][cnt[w]++] = (uint8_t)i;
    load[w] += tasks[i].len;
  }
  return t;
}

template <int P, bool PROJ = false>
size_t k4_smem_bytes(const K4Tab& t) {
  using S = K4Shape<P, PROJ>;
  const size_t pipe = (size_t)2 * (S::NROWP + S::NW) * K4Geo<P, PROJ>::SS;
  const size_t red = (size_t)t.groups * t.ntile * 32;
  return std::max(pipe, red) * sizeof(double);
}

// x^a by binary exponentiation (a <= 20)
__device__ __forceinline__ double ipow(double x, int a) {
  double r = 1.0, b = x;
  while (a) {
    if (a & 1) r *= b;
    b *= b;
    a >>= 1;
  }
  return r;
}

// rows (AA, b), b = 0..Q-AA, of one point: X(AA, b) = x^AA y^b at compile-time slots (row-in-tile major)
template <typename S, int SS, int AA>
__device__ __forceinline__ void xrow(double x, double y, double* Xj) {
  if constexpr (AA <= S::Q) {
    double v = 1.0;
#pragma unroll
    for (int e = 0; e < AA; ++e) v *= x;
#pragma unroll
    for (int b = 0; b <= S::Q - AA; ++b) {
      const int s = AA + b;
      const int row = s * (s + 1) / 2 + AA;
      Xj[((row & 7) * S::NRG + (row >> 3)) * SS] = v;
      v *= y;
    }
  }
}

template <int P, bool PROJ>
__global__ void __launch_bounds__(K4_THREADS, 1)
    k_moments(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
              const double* __restrict__ r, const int4* __restrict__ cell, int64_t first,
              const Chunk* __restrict__ chunks, const int64_t* __restrict__ nchunks,
              const __grid_constant__ K4Tab tab, const int32_t* __restrict__ skip_flag,
              double* __restrict__ partial) {
  using S = K4Shape<P, PROJ>;
  constexpr int Q = S::Q;
  extern __shared__ __align__(16) double smem[];
  const int64_t cidx = blockIdx.x;
  if (cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  if (PROJ && (skip_flag[first + ck.owner] & 3)) return;  // QR-path or converged node: no refinement
  const int4 c = cell[first + ck.owner];
  const double h = ldexp(1.0, -(c.w + 1));
  const double scale = ldexp(1.0, c.w + 1);
  const double cx = (2.0 * c.x + 1.0) * h, cy = (2.0 * c.y + 1.0) * h, cz = (2.0 * c.z + 1.0) * h;

  using Geo = K4Geo<P, PROJ>;
  constexpr int B = Geo::B, SS = Geo::SS, G = Geo::G, NT = Geo::NT, bufsz = Geo::BUF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / NT;
  const int t = tid - grp * NT;
  const bool worker = grp < G;
  int rg = 0, cb = 0;
  if (worker) { rg = tab.tile[t] >> 8; cb = tab.tile[t] & 255; }

  const int64_t n = ck.end - ck.start;
  const int nbatch = (int)((n + B - 1) / B);

  // producer: fill buffer `buf` with batch `bi` (every offset below is a compile-time constant)
  auto produce = [&](int bi, int buf) {
    double* X = smem + buf * bufsz;
    double* W = X + S::NROWP * SS;
    const int64_t base = ck.start + (int64_t)bi * B;
#pragma unroll 1
    for (int k = 0; k < K4_TASKS_PER_WARP; ++k) {
      const int ti = tab.warp_task[warp][k];
      if (ti == 255) break;
      const int a = tab.task_a[ti];
      const int j = 32 * tab.task_h[ti] + lane;
      const bool inb = j < B;
      const int64_t pi = base + j;
      const bool valid = inb && pi < ck.end;
      if (a != 255) {  // X task: rows (a, b), b = 0..Q-a, one fully unrolled walk per power a
        const double x = valid ? __dmul_rn(__dsub_rn(ux[pi], cx), scale) : 0.0;
        const double y = valid ? __dmul_rn(__dsub_rn(uy[pi], cy), scale) : 0.0;
        if (inb) {
          double* Xj = X + j;
          switch (a) {
#define FMI_XCASE(AA) case AA: xrow<S, SS, AA>(x, y, Xj); break;
            FMI_XCASE(0) FMI_XCASE(1) FMI_XCASE(2) FMI_XCASE(3) FMI_XCASE(4) FMI_XCASE(5) FMI_XCASE(6)
            FMI_XCASE(7) FMI_XCASE(8) FMI_XCASE(9) FMI_XCASE(10) FMI_XCASE(11) FMI_XCASE(12) FMI_XCASE(13)
            FMI_XCASE(14) FMI_XCASE(15) FMI_XCASE(16) FMI_XCASE(17) FMI_XCASE(18) FMI_XCASE(19) FMI_XCASE(20)
#undef FMI_XCASE
            default: break;
          }
        }
      } else if (inb) {  // W task: z^c (moments) and r z^c (projection); zero for padded points
        const double z = valid ? __dmul_rn(__dsub_rn(uz[pi], cz), scale) : 0.0;
        const double rv = valid ? r[pi] : 0.0;
        double* Wj = W + j;
        double v = valid ? 1.0 : 0.0;
#pragma unroll
        for (int col = 0; col < S::CM; ++col) {
          Wj[((col & 3) * S::NCB + (col >> 2)) * SS] = (col <= Q) ? v : 0.0;
          v *= z;
        }
        v = rv;
#pragma unroll
        for (int col = S::CM; col < S::NW; ++col) {
          Wj[((col & 3) * S::NCB + (col >> 2)) * SS] = (col - S::CM <= P) ? v : 0.0;
          v *= z;
        }
      }
    }
    // padded rows of the last 8-row group stay zero
    if (S::NROWP > S::NROW) {
      for (int row = S::NROW + warp; row < S::NROWP; row += K4_WARPS) {
        const int slot = (row & 7) * S::NRG + (row >> 3);
        for (int j = lane; j < B; j += 32) X[slot * SS + j] = 0.0;
      }
    }
  };

  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;

  produce(0, 0);
  __syncthreads();
  for (int it = 0; it < nbatch; ++it) {
    if (it + 1 < nbatch) produce(it + 1, (it + 1) & 1);
    if (worker) {
      const double* X = smem + (it & 1) * bufsz + rg * SS;            // slot (i, rg) = i*NRG + rg
      const double* W = smem + (it & 1) * bufsz + S::NROWP * SS + cb * SS;
      const int npairs = (int)((min((int64_t)B, n - (int64_t)it * B) + 1) >> 1);
#pragma unroll 1
      for (int pp = grp; pp < npairs; pp += G) {
        const int j = 2 * pp;
        double2 xv[8], wv[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = *reinterpret_cast<const double2*>(X + i * (S::NRG * SS) + j);
#pragma unroll
        for (int k = 0; k < 4; ++k) wv[k] = *reinterpret_cast<const double2*>(W + k * (S::NCB * SS) + j);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[i * 4 + k] = fma(xv[i].x, wv[k].x, acc[i * 4 + k]);
            acc[i * 4 + k] = fma(xv[i].y, wv[k].y, acc[i * 4 + k]);
          }
      }
    }
    __syncthreads();
  }

  // fixed-order reduction over the point groups, then scatter the needed entries to the partial
  double* red = smem;
  if (worker) {
#pragma unroll
    for (int k = 0; k < 32; ++k) red[(grp * NT + t) * 32 + k] = acc[k];
  }
  __syncthreads();
  if (grp == 0 && worker) {
    double* out = partial + cidx * (int64_t)(S::K + S::L);
    for (int i = 0; i < 8; ++i) {
      const int row = 8 * rg + i;
      if (row >= S::NROW) continue;
      int a, b;
      row_exponents(row, a, b);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double v = 0.0;
        for (int g = 0; g < G; ++g) v += red[(g * NT + t) * 32 + i * 4 + k];
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
