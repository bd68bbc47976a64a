// m2m.cu — upward translation of raw moments through the moment tree (DESIGN.md §5 M2M).
//
// The Gram of Algorithm 2 needs, for every fitted node, M_γ = Σ_i u_i^γ (|γ| <= 2p) in the
// node's own frame u = (x - c)/h.  A parent's points are the union of its children's, and
// a child's frame maps to the parent's by  u_p = (u_c + s)/2  per axis (s = +1 for the upper half,
// -1 for the lower; FMT_New_Octant).  Hence, per axis,
//     M_p[g] = Σ_{j<=g} C(g,j) s^(g-j) 2^-g M_c[j]      (binomial theorem; the other indices fixed),
// an exact identity; the coefficients C(g,j)·2^-g are exact in fp64 and every term is bounded by
// n·C(g,j)·2^-g, so the translation adds rounding of the same order as direct accumulation.
// Applying the three axis transforms to every child and adding the parent's directly accumulated
// owner segments (moments.cu) gives the parent's moments.  One CTA per parent; levels from the
// deepest up.  Deterministic (fixed child order, no atomics).
#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int M2M_THREADS = 256;

// Rounding bound of the moments (B >= |error of M|, entrywise): direct accumulation over n_own owner
// points with |u| <= 1 gives B = 64·eps·n_own; a translation adds (3Q+3)·eps·|M_c| per child and carries
// B_c, both through the all-positive transform T+ (s = +1):  B_p = B_own + Σ_c T+(B_c + (3Q+3)eps|M_c|).
// The solve rejects a translated Gram whose equilibrated bound exceeds kMomentTol (catastrophic
// cancellation, e.g. points clustered at the parent's centre) and the node is re-accumulated directly.
__global__ void k_bound_init(const NodeTable mt, int64_t n, int K, double* __restrict__ bnd) {
  const int64_t node = blockIdx.x;
  if (node >= n) return;
  int64_t own = mt.end[node] - mt.start[node];
  for (int o = 0; o < 8; ++o)
    if (mt.child[node * 8 + o] >= 0) own -= mt.child_start[node * 9 + o + 1] - mt.child_start[node * 9 + o];
  const double b = 64.0 * 1.1102230246251565e-16 * (double)own;
  for (int e = threadIdx.x; e < K; e += blockDim.x) bnd[node * K + e] = b;
}

template <int P>
__device__ __forceinline__ void translate3(const double* src, double* tmp, double* dst, bool add, double sx,
                                           double sy, double sz, const double* coef, const uint8_t* ea,
                                           const uint8_t* eb, const uint8_t* ec) {
  constexpr int Q = 2 * P, K = rank3(Q);
  const int tid = threadIdx.x;
  // z: src -> tmp
  for (int e = tid; e < K; e += M2M_THREADS) {
    const int a = ea[e], b = eb[e], g = ec[e];
    const double* cg = coef + g * (Q + 1);
    double v = 0.0, sg = 1.0;  // s^(g-j), j descending from g
    for (int j = g; j >= 0; --j) { v = fma(cg[j] * sg, src[basis_index(Q, a, b, j)], v); sg *= sz; }
    tmp[e] = v;
  }
  __syncthreads();
  // y: tmp -> src (src is consumed)
  double* t2 = const_cast<double*>(src);
  for (int e = tid; e < K; e += M2M_THREADS) {
    const int a = ea[e], g = eb[e], c = ec[e];
    const double* cg = coef + g * (Q + 1);
    double v = 0.0, sg = 1.0;
    for (int j = g; j >= 0; --j) { v = fma(cg[j] * sg, tmp[basis_index(Q, a, j, c)], v); sg *= sy; }
    t2[e] = v;
  }
  __syncthreads();
  // x: src -> dst (+=)
  for (int e = tid; e < K; e += M2M_THREADS) {
    const int g = ea[e], b = eb[e], c = ec[e];
    const double* cg = coef + g * (Q + 1);
    double v = 0.0, sg = 1.0;
    for (int j = g; j >= 0; --j) { v = fma(cg[j] * sg, t2[basis_index(Q, j, b, c)], v); sg *= sx; }
    dst[e] = add ? dst[e] + v : v;
  }
  __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(M2M_THREADS)
    k_m2m(double* __restrict__ mom, double* __restrict__ bnd, const int32_t* __restrict__ child, int64_t first,
          int64_t count) {
  constexpr int Q = 2 * P, K = rank3(Q);
  extern __shared__ double m2m_smem[];
  double* acc = m2m_smem;
  double* accb = acc + K;
  double* b0 = accb + K;
  double* b1 = b0 + K;
  double* coef = b1 + K;  // (Q+1)^2: C(g,j) 2^-g
  uint8_t* ea = reinterpret_cast<uint8_t*>(coef + (Q + 1) * (Q + 1));
  uint8_t* eb = ea + K;
  uint8_t* ec = eb + K;
  const int64_t node = first + blockIdx.x;
  const int tid = threadIdx.x;
  int nch = 0;
  for (int o = 0; o < 8; ++o) nch += child[node * 8 + o] >= 0;
  if (nch == 0) return;  // uniform over the CTA
  for (int e = tid; e < (Q + 1) * (Q + 1); e += M2M_THREADS) {
    const int g = e / (Q + 1), j = e % (Q + 1);
    double c = 0.0;
    if (j <= g) {
      double bin = 1.0;  // C(g, j), exact
      for (int t = 1; t <= j; ++t) bin = bin * (double)(g - j + t) / (double)t;
      c = ldexp(bin, -g);
    }
    coef[e] = c;
  }
  for (int e = tid; e < K; e += M2M_THREADS) {
    int l = 0;
    while (rank3(Q) - rank3(Q - l - 1) <= e) ++l;
    int rem = e - (rank3(Q) - rank3(Q - l));
    int m = 0;
    while (rem >= Q - l - m + 1) { rem -= Q - l - m + 1; ++m; }
    ea[e] = (uint8_t)l; eb[e] = (uint8_t)m; ec[e] = (uint8_t)rem;
    acc[e] = mom[node * K + e];
    accb[e] = bnd[node * K + e];
  }
  __syncthreads();
  constexpr double kT = (3.0 * Q + 3.0) * 1.1102230246251565e-16;
  for (int o = 0; o < 8; ++o) {
    const int32_t ch = child[node * 8 + o];
    if (ch < 0) continue;
    const double sx = (o & 1) ? 1.0 : -1.0, sy = (o & 2) ? 1.0 : -1.0, sz = (o & 4) ? 1.0 : -1.0;
    for (int e = tid; e < K; e += M2M_THREADS) b0[e] = mom[(int64_t)ch * K + e];
    __syncthreads();
    translate3<P>(b0, b1, acc, true, sx, sy, sz, coef, ea, eb, ec);
    for (int e = tid; e < K; e += M2M_THREADS) b0[e] = bnd[(int64_t)ch * K + e] + kT * fabs(mom[(int64_t)ch * K + e]);
    __syncthreads();
    translate3<P>(b0, b1, accb, true, 1.0, 1.0, 1.0, coef, ea, eb, ec);
  }
  for (int e = tid; e < K; e += M2M_THREADS) {
    mom[node * K + e] = acc[e];
    bnd[node * K + e] = accb[e];
  }
}

// next level's solve input: [moments (K) | projection (𝓛) | moment bound (K)] per node, gathered from
// the moment tree (mtid) and the parent's child-segment projections (srcseg) — or, for the root,
// segment 0.
__global__ void __launch_bounds__(256)
    k_gather_level(const double* __restrict__ mtmom, const double* __restrict__ mtbnd,
                   const int32_t* __restrict__ mtid, const double* __restrict__ segsum,
                   const int32_t* __restrict__ srcseg, int64_t first, int K, int L, double* __restrict__ out) {
  const int64_t ln = blockIdx.x;
  const int64_t m = mtid[first + ln];
  const int64_t sg = srcseg ? srcseg[ln] : 0;
  const int64_t st = 2 * K + L;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    out[ln * st + e] = mtmom[m * K + e];
    out[ln * st + K + L + e] = mtbnd[m * K + e];
  }
  for (int e = threadIdx.x; e < L; e += blockDim.x) out[ln * st + K + e] = segsum[sg * (L + 1) + e];
}

}  // namespace

void bound_init(const NodeTable& mt, int64_t n, int K, double* bnd, cudaStream_t s) {
  if (n <= 0) return;
  FMI_LAUNCH(KID_M2M, s, k_bound_init, (unsigned)n, 256, 0, mt, n, K, bnd);
}

template <int P>
void m2m_level(double* mom, double* bnd, const int32_t* child, int64_t first, int64_t count, cudaStream_t s) {
  constexpr int Q = 2 * P, K = rank3(Q);
  constexpr size_t smem = (4 * K + (Q + 1) * (Q + 1)) * sizeof(double) + 3 * K;
  static bool attr = false;
  if (!attr) {
    FMI_CK(cudaFuncSetAttribute(k_m2m<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (count <= 0) return;
  FMI_LAUNCH(KID_M2M, s, k_m2m<P>, (unsigned)count, M2M_THREADS, smem, mom, bnd, child, first, count);
}

void gather_level(const double* mtmom, const double* mtbnd, const int32_t* mtid, const double* segsum,
                  const int32_t* srcseg, int64_t first, int64_t count, int K, int L, double* out, cudaStream_t s) {
  if (count <= 0) return;
  FMI_LAUNCH(KID_LEVEL_GATHER, s, k_gather_level, (unsigned)count, 256, 0, mtmom, mtbnd, mtid, segsum, srcseg, first,
             K, L, out);
}

#define FMI_INST(P) template void m2m_level<P>(double*, double*, const int32_t*, int64_t, int64_t, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
