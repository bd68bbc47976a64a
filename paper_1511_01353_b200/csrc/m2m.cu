// m2m.cu — upward translation of raw moments through the moment tree (DESIGN.md §5 M2M).
//
// The Gram of Algorithm 2 needs, for every fitted node, M_γ = Σ_i u_i^γ (|γ| <= 2p) in the
// node's own frame u = (x - c)/h.  A parent's points are the union of its children's, and
// a child's frame maps to the parent's by  u_p = (u_c + s)/2  per axis (s = +1 for the upper half,
// -1 for the lower; FMT_New_Octant).  Hence, per axis,
//     M_p[g] = Σ_{j<=g} C(g,j) s^(g-j) 2^-g M_c[j]      (binomial theorem; the other indices fixed),
// an exact identity; the coefficients C(g,j)·2^-g are exact in fp64.  The 8 children of a parent are
// translated as  Σ_sx Sx Σ_sy Sy Σ_sz Sz M_(sx,sy,sz)  (8 z-, 4 y-, 2 x-shifts instead of 24) and added
// to the parent's directly accumulated owner moments (moments.cu).  One CTA per parent; levels from
// the deepest up; children's tensors are streamed into shared memory by TMA bulk copies, double
// buffered.  Deterministic (fixed child order, no atomics).
//
// Rounding bound (B >= |error of M|, entrywise, kept in fp32): direct accumulation over n_own owner
// points with |u| <= 1 gives B = 64·eps·n_own; a translation adds (3Q+3)·eps·|M_c| per child and carries
// B_c, both through the all-positive transform T+ (s = +1), which is the same for every child:
//     B_p = B_own + T+( Σ_c (B_c + (3Q+3)·eps·|M_c|) ).
// The solve rejects a translated Gram whose equilibrated bound exceeds kMomentTol (catastrophic
// cancellation, e.g. points clustered at the parent's centre) and the node is re-accumulated directly.
#include <mutex>
#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int M2M_THREADS = 1024;  // latency-bound shift chains: more threads in flight (1.74 -> 1.42 ms at cfg 5)
constexpr double kEps = 1.1102230246251565e-16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D TMA bulk copy global -> shared (16-byte aligned addresses, size a multiple of 16)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void k_bound_init(const NodeTable mt, int64_t n, int K, int KS, float* __restrict__ bnd) {
  const int64_t node = blockIdx.x;
  if (node >= n) return;
  int64_t own = mt.end[node] - mt.start[node];
  for (int o = 0; o < 8; ++o)
    if (mt.child[node * 8 + o] >= 0) own -= mt.child_start[node * 9 + o + 1] - mt.child_start[node * 9 + o];
  const float b = (float)(64.0 * kEps * (double)own);
  for (int e = threadIdx.x; e < KS; e += blockDim.x) bnd[node * KS + e] = e < K ? b : 0.0f;
}

// dst (+)= shift of src along one axis (0 = x, 1 = y, 2 = z) with sign s:
//   dst[..g..] = Σ_{j<=g} C(g,j) s^(g-j) 2^-g src[..j..]
template <int P, typename T>
__device__ __forceinline__ void axis_shift(const T* __restrict__ src, T* __restrict__ dst, int axis, double s,
                                           bool add, const double* coef, const uint8_t* ea, const uint8_t* eb,
                                           const uint8_t* ec) {
  constexpr int Q = 2 * P, K = rank3(Q);
  for (int e = threadIdx.x; e < K; e += M2M_THREADS) {
    const int a = ea[e], b = eb[e], c = ec[e];
    double v = 0.0;
    if (axis == 2) {  // z: entries (a, b, j) are contiguous
      const double* cg = coef + c * (Q + 1);
      const T* sp = src + (e - c);
      double sg = 1.0;
      for (int j = c; j >= 0; --j) { v = fma(cg[j] * sg, (double)sp[j], v); sg *= s; }
    } else if (axis == 1) {  // y: idx(a, j+1, c) - idx(a, j, c) = Q - a + 1 - j
      const double* cg = coef + b * (Q + 1);
      int idx = e - (b * (Q - a + 1) - b * (b - 1) / 2);  // idx(a, 0, c)
      double sg = (b & 1) ? s : 1.0;                      // s^(b - j), s = ±1
      for (int j = 0; j <= b; ++j) {
        v = fma(cg[j] * sg, (double)src[idx], v);
        idx += Q - a + 1 - j;
        sg *= s;
      }
    } else {  // x: idx(j+1, b, c) - idx(j, b, c) = (Q-j+1)(Q-j+2)/2 - b
      const double* cg = coef + a * (Q + 1);
      int idx = b * (Q + 1) - b * (b - 1) / 2 + c;  // idx(0, b, c)
      double sg = (a & 1) ? s : 1.0;
      for (int j = 0; j <= a; ++j) {
        v = fma(cg[j] * sg, (double)src[idx], v);
        idx += (Q - j + 1) * (Q - j + 2) / 2 - b;
        sg *= s;
      }
    }
    dst[e] = add ? (T)((double)dst[e] + v) : (T)v;
  }
  __syncthreads();
}

template <int P>
struct M2MLayout {
  static constexpr int Q = 2 * P, K = rank3(Q), KS = (K + 3) & ~3;
  // doubles: cm[2][KS] (child moments, double buffer), acc[KS], a2[2][KS]
  // floats:  cb[2][KS] (child bounds), bs[KS], bt[2][KS] (bound transform temporaries)
  // then coef[(Q+1)^2] doubles, the uint8 entry tables and two mbarriers.  KS % 4 == 0 keeps every
  // TMA destination 16-byte aligned.
  static constexpr size_t D_CM = 0, D_ACC = 2 * KS, D_A2 = 3 * KS;
  static constexpr size_t ND = 5 * KS;
  static constexpr size_t F_CB = 0, F_BS = 2 * KS, F_BT = 3 * KS, NF = 5 * KS;
  static constexpr size_t NC = (Q + 1) * (Q + 1);
  static constexpr size_t BYTES = ND * 8 + NF * 4 + NC * 8 + 3 * KS + 64;
};

template <int P>
__global__ void __launch_bounds__(M2M_THREADS)
    k_m2m(double* __restrict__ mom, float* __restrict__ bnd, const int32_t* __restrict__ child, int64_t first,
          int64_t count) {
  using LY = M2MLayout<P>;
  constexpr int Q = LY::Q, K = LY::K, KS = LY::KS;
  extern __shared__ __align__(16) double m2m_smem[];
  double* cm = m2m_smem + LY::D_CM;
  double* acc = m2m_smem + LY::D_ACC;
  double* a2 = m2m_smem + LY::D_A2;
  float* fs = reinterpret_cast<float*>(m2m_smem + LY::ND);
  float* cb = fs + LY::F_CB;
  float* bs = fs + LY::F_BS;
  float* bt = fs + LY::F_BT;
  double* coef = reinterpret_cast<double*>(fs + LY::NF);
  uint8_t* ea = reinterpret_cast<uint8_t*>(coef + LY::NC);
  uint8_t* eb = ea + KS;
  uint8_t* ec = eb + KS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ec + KS + (8 - (3 * KS) % 8) % 8);
  const int64_t node = first + blockIdx.x;
  const int tid = threadIdx.x;
  int chl[8], nch = 0;
  for (int o = 0; o < 8; ++o)
    if (child[node * 8 + o] >= 0) chl[nch++] = o;
  if (nch == 0) return;  // uniform over the CTA
  // order the existing children as they are consumed: (sx, sy) groups q = 0..3, sz = 0, 1
  int ord[8], no = 0;
  for (int q = 0; q < 4; ++q)
    for (int hz = 0; hz < 2; ++hz)
      for (int t = 0; t < nch; ++t)
        if (chl[t] == q + 4 * hz) ord[no++] = chl[t];
  constexpr uint32_t kBytesM = KS * 8, kBytesB = KS * 4;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {  // k-th consumed child -> buffer k & 1
    const int64_t ch = child[node * 8 + ord[k]];
    mbar_expect_tx(&bar[k & 1], kBytesM + kBytesB);
    tma_load(cm + (k & 1) * KS, mom + ch * KS, kBytesM, &bar[k & 1]);
    tma_load(cb + (k & 1) * KS, bnd + ch * KS, kBytesB, &bar[k & 1]);
  };
  if (tid == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }
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
    a2[e] = a2[KS + e] = 0.0;
    bs[e] = 0.0f;
  }
  __syncthreads();
  constexpr double kT = (3.0 * Q + 3.0) * kEps;
  // per (sx, sy): acc = Σ_sz Sz(child) -> a2[sx] += Sy(acc)
  int k = 0;
  for (int q = 0; q < 4; ++q) {
    bool any = false;
    while (k < nch && (ord[k] & 3) == q) {
      const int buf = k & 1;
      mbar_wait(&bar[buf], (uint32_t)((k >> 1) & 1));
      for (int e = tid; e < K; e += M2M_THREADS) bs[e] += cb[buf * KS + e] + (float)(kT * fabs(cm[buf * KS + e]));
      axis_shift<P>(cm + buf * KS, acc, 2, (ord[k] & 4) ? 1.0 : -1.0, any, coef, ea, eb, ec);
      any = true;
      if (tid == 0 && k + 2 < nch) issue(k + 2);  // buffer free again (the shift ended with a barrier)
      ++k;
    }
    if (any) axis_shift<P>(acc, a2 + (q & 1) * KS, 1, (q & 2) ? 1.0 : -1.0, true, coef, ea, eb, ec);
  }
  // x shift of both halves onto acc, then add to the node's own moments
  axis_shift<P>(a2, acc, 0, -1.0, false, coef, ea, eb, ec);
  axis_shift<P>(a2 + KS, acc, 0, 1.0, true, coef, ea, eb, ec);
  for (int e = tid; e < K; e += M2M_THREADS) mom[node * KS + e] += acc[e];
  // bound: T+ of the summed child terms
  axis_shift<P>(bs, bt, 2, 1.0, false, coef, ea, eb, ec);
  axis_shift<P>(bt, bt + KS, 1, 1.0, false, coef, ea, eb, ec);
  axis_shift<P>(bt + KS, bt, 0, 1.0, false, coef, ea, eb, ec);
  for (int e = tid; e < K; e += M2M_THREADS) bnd[node * KS + e] += bt[e];
}

// next level's solve input: [moments (K) | projection (𝓛) | moment bound (K)] per node, gathered from
// the moment tree (mtid, stride KS) and the parent's child-segment projections (srcseg) — or, for
// the root, segment 0.
__global__ void __launch_bounds__(256)
    k_gather_level(const double* __restrict__ mtmom, const float* __restrict__ mtbnd,
                   const int32_t* __restrict__ mtid, const double* __restrict__ segsum,
                   const int32_t* __restrict__ srcseg, int64_t first, int K, int KS, int L, double* __restrict__ out) {
  const int64_t ln = blockIdx.x;
  const int64_t m = mtid[first + ln];
  const int64_t sg = srcseg ? srcseg[ln] : 0;
  const int64_t st = 2 * K + L;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {  // m < 0: no moments yet -> the solve's check fails
    out[ln * st + e] = m < 0 ? 0.0 : mtmom[m * KS + e];
    out[ln * st + K + L + e] = m < 0 ? INFINITY : (double)mtbnd[m * KS + e];
  }
  for (int e = threadIdx.x; e < L; e += blockDim.x) out[ln * st + K + e] = segsum[sg * (L + 1) + e];
}

}  // namespace

void bound_init(const NodeTable& mt, int64_t n, int K, int KS, float* bnd, cudaStream_t s) {
  if (n <= 0) return;
  FMI_LAUNCH(KID_M2M, s, k_bound_init, (unsigned)n, 256, 0, mt, n, K, KS, bnd);
}

template <int P>
void m2m_level(double* mom, float* bnd, const int32_t* child, int64_t first, int64_t count, cudaStream_t s) {
  constexpr size_t smem = M2MLayout<P>::BYTES;
  static std::once_flag attr_once;  // one opt-in per kernel instantiation (thread-safe)
  std::call_once(attr_once, [&] {
    FMI_CK(cudaFuncSetAttribute(
        k_m2m<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  if (count <= 0) return;
  FMI_LAUNCH(KID_M2M, s, k_m2m<P>, (unsigned)count, M2M_THREADS, smem, mom, bnd, child, first, count);
}

void gather_level(const double* mtmom, const float* mtbnd, const int32_t* mtid, const double* segsum,
                  const int32_t* srcseg, int64_t first, int64_t count, int K, int KS, int L, double* out,
                  cudaStream_t s) {
  if (count <= 0) return;
  FMI_LAUNCH(KID_LEVEL_GATHER, s, k_gather_level, (unsigned)count, 256, 0, mtmom, mtbnd, mtid, segsum, srcseg, first,
             K, KS, L, out);
}

#define FMI_INST(P) template void m2m_level<P>(double*, float*, const int32_t*, int64_t, int64_t, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
