// eval.cu — K7: interpolant evaluation over Morton-sorted queries (DESIGN.md §5 K7) and the
// pre-summed node polynomials it uses.
//
// f(r) = Λ(r)·F_p (§2), accumulated over the nodes on the query's root-to-deepest-existing-node
// path ("only downward recursion to accumulate local polynomial representation of the residual",
// P:367-368 §4; reading G11).  After the build, every node's polynomial is pre-summed with all of its
// ancestors' — each ancestor polynomial translated into the node's frame, u_parent = (u_child + s)/2
// per axis (FMT_New_Octant), an exact change of variables — so a query evaluates ONE polynomial
// (the deepest node's) instead of one per level; the value equals the path sum up to rounding.
// Queries are processed in Morton order so that neighbouring threads use the same node (coefficient
// loads are warp-broadcast, L1-resident); results are scattered back to the caller's order.  A query
// outside the root cube gets the root polynomial only.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "horner.cuh"

namespace fmi {

namespace {

__device__ __forceinline__ double to_unit_e(double x, double lo, double w, bool unit) {
  return unit ? x : __ddiv_rn(__dsub_rn(x, lo), w);
}

// ---- pre-summed polynomials ----------------------------------------------------------------------
constexpr int PS_THREADS = 128;

// dst[..j..] = Σ_{g>=j} src[..g..] C(g,j) s^(g-j) 2^-g along one axis (Taylor shift of a polynomial
// from the parent frame to the child frame); entries in Algorithm-2 order of degree P.
template <int P>
__device__ __forceinline__ void poly_shift(const double* __restrict__ src, double* __restrict__ dst, int axis,
                                           double s, const double* coef, const uint8_t* ea, const uint8_t* eb,
                                           const uint8_t* ec) {
  constexpr int L = rank3(P);
  for (int e = threadIdx.x; e < L; e += PS_THREADS) {
    const int a = ea[e], b = eb[e], c = ec[e];
    double v = 0.0;
    if (axis == 2) {
      const double* sp = src + (e - c);
      double sg = 1.0;
      for (int g = c; g <= P - a - b; ++g) { v = fma(coef[g * (P + 1) + c] * sg, sp[g], v); sg *= s; }
    } else if (axis == 1) {
      double sg = 1.0;
      for (int g = b; g <= P - a - c; ++g) { v = fma(coef[g * (P + 1) + b] * sg, src[basis_index(P, a, g, c)], v); sg *= s; }
    } else {
      double sg = 1.0;
      for (int g = a; g <= P - b - c; ++g) { v = fma(coef[g * (P + 1) + a] * sg, src[basis_index(P, g, b, c)], v); sg *= s; }
    }
    dst[e] = v;
  }
  __syncthreads();
}

// pcoef[node] = coef[node] + shift(pcoef[parent]) for the nodes [first, first+count) of one level
template <int P>
__global__ void __launch_bounds__(PS_THREADS) k_presum(NodeTable nt, int64_t first, int64_t count) {
  constexpr int L = rank3(P);
  __shared__ double b0[L], b1[L];
  __shared__ double coef[(P + 1) * (P + 1)];
  __shared__ uint8_t ea[L], eb[L], ec[L];
  const int64_t node = first + blockIdx.x;
  const int tid = threadIdx.x;
  const int32_t par = nt.parent[node];
  if (par < 0) {
    for (int e = tid; e < L; e += PS_THREADS) nt.pcoef[node * L + e] = nt.coef[node * L + e];
    return;
  }
  for (int e = tid; e < (P + 1) * (P + 1); e += PS_THREADS) {
    const int g = e / (P + 1), j = e % (P + 1);
    double c = 0.0;
    if (j <= g) {
      double bin = 1.0;
      for (int t = 1; t <= j; ++t) bin = bin * (double)(g - j + t) / (double)t;
      c = ldexp(bin, -g);
    }
    coef[e] = c;
  }
  for (int e = tid; e < L; e += PS_THREADS) {
    int l = 0;
    while (rank3(P) - rank3(P - l - 1) <= e) ++l;
    int rem = e - (rank3(P) - rank3(P - l));
    int m = 0;
    while (rem >= P - l - m + 1) { rem -= P - l - m + 1; ++m; }
    ea[e] = (uint8_t)l; eb[e] = (uint8_t)m; ec[e] = (uint8_t)rem;
    b0[e] = nt.pcoef[(int64_t)par * L + e];
  }
  __syncthreads();
  const int4 c = nt.cell[node];  // octant bits = low bits of the cell (FMT_New_Octant)
  poly_shift<P>(b0, b1, 2, (c.z & 1) ? 1.0 : -1.0, coef, ea, eb, ec);
  poly_shift<P>(b1, b0, 1, (c.y & 1) ? 1.0 : -1.0, coef, ea, eb, ec);
  poly_shift<P>(b0, b1, 0, (c.x & 1) ? 1.0 : -1.0, coef, ea, eb, ec);
  for (int e = tid; e < L; e += PS_THREADS) nt.pcoef[node * L + e] = b1[e] + nt.coef[node * L + e];
}

// Two sorted queries per thread: warp w of a CTA takes 64 consecutive queries (lane l: base + l and
// base + 32 + l).  Sorted queries make the deepest node warp-uniform almost everywhere: the warp then
// stages that node's pre-summed coefficients in shared memory once (coalesced) and every lane
// evaluates its two queries with one coefficient read per two FMAs (horner3x2); otherwise each query
// reads its own node's coefficients through L1.
// query i: its root-cube coordinates (the 32-byte record written by the key kernel, or the raw point)
// and its key — issued for both of a thread's queries before either is used (independent loads in flight)
__device__ __forceinline__ void eval_fetch(const double* __restrict__ q, const double4* __restrict__ qpk,
                                           const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                           int64_t i, int64_t M, double lo0, double lo1, double lo2, double w,
                                           bool unit, int rec_idx, int64_t& qi, double& ux, double& uy, double& uz,
                                           uint64_t& key) {
  qi = 0;
  ux = uy = uz = 0.0;
  key = 0;
  if (i < M) {
    qi = idx ? (int64_t)idx[i] : i;
    if (keys) key = keys[i];
    if (qpk) {
      const double2* p = reinterpret_cast<const double2*>(qpk + qi);
      const double2 a = __ldg(p), b = __ldg(p + 1);
      ux = a.x; uy = a.y; uz = b.x;
      if (rec_idx) qi = (int64_t)b.y;  // bucketed records: idx is a bucket position, the input index is here
    } else {
      ux = to_unit_e(q[3 * qi + 0], lo0, w, unit);
      uy = to_unit_e(q[3 * qi + 1], lo1, w, unit);
      uz = to_unit_e(q[3 * qi + 2], lo2, w, unit);
    }
  }
}

// descend to the deepest existing node containing the query; local coordinates in its frame
__device__ __forceinline__ void eval_descend(int64_t i, int64_t M, bool have_keys, int Dk, const NodeTable& nt,
                                             double ux, double uy, double uz, uint64_t key, int64_t& node,
                                             double& x, double& y, double& z) {
  node = 0;
  const bool inside = ux >= 0.0 && ux <= 1.0 && uy >= 0.0 && uy <= 1.0 && uz >= 0.0 && uz <= 1.0;
  if (i < M && inside && have_keys) {
    for (int level = 0; level < Dk; ++level) {
      const int o = (int)((key >> (3 * (Dk - level - 1))) & 7ull);
      const int32_t ch = __ldg(nt.child + node * 8 + o);
      if (ch < 0) break;
      node = ch;
    }
  }
  const Frame fr = node_frame(nt.cell[node]);
  x = to_local(ux, fr.cx, fr.scale);
  y = to_local(uy, fr.cy, fr.scale);
  z = to_local(uz, fr.cz, fr.scale);
}

template <int P>
__global__ void __launch_bounds__(256) k_eval(const double* __restrict__ q, const double4* __restrict__ qpk,
                                              const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                              int64_t M, double lo0, double lo1, double lo2, double w, bool unit,
                                              int Dk, NodeTable nt, double* __restrict__ out, int rec_idx) {
  constexpr int L = rank3(P);
  constexpr int LA = (L + 1) & ~1;  // 16-byte aligned rows for pair loads
  __shared__ __align__(16) double cs[256 / 32][LA];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = ((int64_t)blockIdx.x * 8 + warp) * 64;
  const int64_t i0 = base + lane, i1 = base + 32 + lane;
  int64_t qi0, qi1, n0, n1;
  double x0, y0, z0, x1, y1, z1, ux0, uy0, uz0, ux1, uy1, uz1;
  uint64_t k0, k1;
  eval_fetch(q, qpk, keys, idx, i0, M, lo0, lo1, lo2, w, unit, rec_idx, qi0, ux0, uy0, uz0, k0);
  eval_fetch(q, qpk, keys, idx, i1, M, lo0, lo1, lo2, w, unit, rec_idx, qi1, ux1, uy1, uz1, k1);
  // sorted queries without a key array (the sort moved 32-bit keys): the key from the record's
  // root-cube coordinates, exactly as the key kernel formed it
  if (!keys && qpk) {
    k0 = morton_key(ux0, uy0, uz0, Dk);
    k1 = morton_key(ux1, uy1, uz1, Dk);
  }
  const bool have_keys = keys != nullptr || qpk != nullptr;
  eval_descend(i0, M, have_keys, Dk, nt, ux0, uy0, uz0, k0, n0, x0, y0, z0);
  eval_descend(i1, M, have_keys, Dk, nt, ux1, uy1, uz1, k1, n1, x1, y1, z1);
  const int64_t node0 = __shfl_sync(0xffffffffu, n0, 0);
  const bool uniform = __all_sync(0xffffffffu, (i0 >= M || n0 == node0) && (i1 >= M || n1 == node0));
  // CTA-wide node (the usual case: a node holds thousands of sorted queries): one coefficient copy for
  // all 8 warps, loaded by all 256 threads at once
  __shared__ long long cta_node[256 / 32];
  if (lane == 0) cta_node[warp] = uniform ? (long long)node0 : -1ll;
  __syncthreads();
  bool cta_uniform = true;
#pragma unroll
  for (int w8 = 0; w8 < 256 / 32; ++w8) cta_uniform = cta_uniform && cta_node[w8] == cta_node[0] && cta_node[w8] >= 0;
  double v0, v1;
  if (cta_uniform) {
    const double* a = nt.pcoef + node0 * L;
    for (int k = threadIdx.x; k < L; k += 256) cs[0][k] = __ldg(a + k);
    __syncthreads();
    const SmemCoef coef(cs[0]);
    horner3x2<P>(coef, x0, y0, z0, x1, y1, z1, v0, v1);
  } else if (uniform) {
    const double* a = nt.pcoef + node0 * L;
    for (int k = lane; k < L; k += 32) cs[warp][k] = __ldg(a + k);
    __syncwarp();
    const SmemCoef coef(cs[warp]);
    horner3x2<P>(coef, x0, y0, z0, x1, y1, z1, v0, v1);
  } else {
    const double* a0 = nt.pcoef + n0 * L;
    const double* a1 = nt.pcoef + n1 * L;
    auto c0 = [&](int k) { return __ldg(a0 + k); };
    auto c1 = [&](int k) { return __ldg(a1 + k); };
    v0 = horner3<P>(c0, x0, y0, z0);
    v1 = horner3<P>(c1, x1, y1, z1);
  }
  if (i0 < M) out[qi0] = v0;
  if (i1 < M) out[qi1] = v1;
}

// Pipelined persistent variant (the default for sorted queries with records): CTAs loop over tiles of
// 512 sorted queries; the random 32-byte query records of the tile two steps ahead are fetched into a
// shared-memory ring by cp.async while the current tile is evaluated, so the latency of the random
// reads overlaps the Horner work instead of stalling every CTA at its start (DESIGN.md §5 K7).
constexpr int EV_TILE = 512;
constexpr int EV_THREADS = 256;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int P>
__global__ void __launch_bounds__(EV_THREADS, 3)
    k_eval_pipe(const double4* __restrict__ qpk, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                int64_t M, int Dk, NodeTable nt, double* __restrict__ out, int rec_idx) {
  constexpr int L = rank3(P);
  constexpr int LA = (L + 1) & ~1;
  // dynamic shared memory: the record ring [2][EV_TILE] then the per-warp coefficient rows [8][LA]
  extern __shared__ __align__(16) double ev_smem[];
  double4 (*rec)[EV_TILE] = reinterpret_cast<double4 (*)[EV_TILE]>(ev_smem);
  double (*cs)[LA] = reinterpret_cast<double (*)[LA]>(ev_smem + 2 * EV_TILE * 4);
  __shared__ long long cta_node[EV_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (M + EV_TILE - 1) / EV_TILE;
  // thread tid owns tile positions tid and tid + 256 (the 64-query warp layout of k_eval below:
  // warp w takes positions 64w .. 64w+63, lane l the positions 64w + l and 64w + 32 + l)
  const int pos0 = warp * 64 + lane, pos1 = pos0 + 32;
  auto issue = [&](int64_t t, int slot) {
    if (t < ntiles) {
      const int64_t i0 = t * EV_TILE + pos0, i1 = t * EV_TILE + pos1;
      if (i0 < M) {
        const double4* src = qpk + idx[i0];
        cp_async16(&rec[slot][pos0], src);
        cp_async16(reinterpret_cast<double2*>(&rec[slot][pos0]) + 1, reinterpret_cast<const double2*>(src) + 1);
      }
      if (i1 < M) {
        const double4* src = qpk + idx[i1];
        cp_async16(&rec[slot][pos1], src);
        cp_async16(reinterpret_cast<double2*>(&rec[slot][pos1]) + 1, reinterpret_cast<const double2*>(src) + 1);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t t = blockIdx.x;
  issue(t, 0);
  issue(t + gridDim.x, 1);
  int slot = 0;
  for (; t < ntiles; t += gridDim.x, slot ^= 1) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's records (the next one in flight)
    const int64_t i0 = t * EV_TILE + pos0, i1 = t * EV_TILE + pos1;
    const double4 r0 = rec[slot][pos0], r1 = rec[slot][pos1];  // each thread reads only its own records
    const uint64_t k0 = i0 < M ? (keys ? keys[i0] : morton_key(r0.x, r0.y, r0.z, Dk)) : 0;
    const uint64_t k1 = i1 < M ? (keys ? keys[i1] : morton_key(r1.x, r1.y, r1.z, Dk)) : 0;
    const int64_t qi0 = i0 < M ? (rec_idx ? (int64_t)r0.w : (int64_t)idx[i0]) : 0;
    const int64_t qi1 = i1 < M ? (rec_idx ? (int64_t)r1.w : (int64_t)idx[i1]) : 0;
    int64_t n0, n1;
    double x0, y0, z0, x1, y1, z1;
    eval_descend(i0, M, true, Dk, nt, r0.x, r0.y, r0.z, k0, n0, x0, y0, z0);
    eval_descend(i1, M, true, Dk, nt, r1.x, r1.y, r1.z, k1, n1, x1, y1, z1);
    const int64_t node0 = __shfl_sync(0xffffffffu, n0, 0);
    const bool uniform = __all_sync(0xffffffffu, (i0 >= M || n0 == node0) && (i1 >= M || n1 == node0));
    if (lane == 0) cta_node[warp] = uniform ? (long long)node0 : -1ll;
    __syncthreads();
    bool cta_uniform = true;
#pragma unroll
    for (int w8 = 0; w8 < EV_THREADS / 32; ++w8)
      cta_uniform = cta_uniform && cta_node[w8] == cta_node[0] && cta_node[w8] >= 0;
    double v0, v1;
    if (cta_uniform) {
      const double* a = nt.pcoef + node0 * L;
      for (int k = tid; k < L; k += EV_THREADS) cs[0][k] = __ldg(a + k);
      __syncthreads();
      horner3x2<P>(SmemCoef(cs[0]), x0, y0, z0, x1, y1, z1, v0, v1);
    } else if (uniform) {
      const double* a = nt.pcoef + node0 * L;
      for (int k = lane; k < L; k += 32) cs[warp][k] = __ldg(a + k);
      __syncwarp();
      horner3x2<P>(SmemCoef(cs[warp]), x0, y0, z0, x1, y1, z1, v0, v1);
    } else {
      const double* a0 = nt.pcoef + n0 * L;
      const double* a1 = nt.pcoef + n1 * L;
      auto c0 = [&](int k) { return __ldg(a0 + k); };
      auto c1 = [&](int k) { return __ldg(a1 + k); };
      v0 = horner3<P>(c0, x0, y0, z0);
      v1 = horner3<P>(c1, x1, y1, z1);
    }
    if (i0 < M) out[qi0] = v0;
    if (i1 < M) out[qi1] = v1;
    __syncthreads();  // cs / cta_node reuse; this slot's records consumed
    issue(t + 2 * (int64_t)gridDim.x, slot);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace

template <int P>
void presum_level(const NodeTable& nt, int64_t first, int64_t count, cudaStream_t s) {
  if (count <= 0) return;
  FMI_LAUNCH(KID_PRESUM, s, k_presum<P>, (unsigned)count, PS_THREADS, 0, nt, first, count);
}

template <int P>
void eval_sorted(const double* q, const double4* qpk, const uint64_t* keys, const uint32_t* idx, int64_t M,
                 const double lo[3], double width, bool unit, int Dk, const NodeTable& nt, double* out,
                 cudaStream_t s, bool rec_idx) {
  if (M <= 0) return;
  static int pipe_ctas = -1;  // persistent CTAs of the pipelined kernel (FMI_EVAL_PIPE=0: the one-shot kernel)
  static std::once_flag once;
  constexpr size_t smem = ((size_t)2 * EV_TILE * 4 + (size_t)(EV_THREADS / 32) * ((rank3(P) + 1) & ~1)) * sizeof(double);
  std::call_once(once, [] {
    int dev = 0, sms = 0, per = 0;
    FMI_CK(cudaGetDevice(&dev));
    FMI_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FMI_CK(cudaFuncSetAttribute(k_eval_pipe<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FMI_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eval_pipe<P>, EV_THREADS, smem));
    const char* e = std::getenv("FMI_EVAL_PIPE");
    pipe_ctas = (e && std::atoi(e) > 0) ? sms * std::max(1, per) : 0;  // opt-in: measured slower (7.46 vs 6.83 ms, cfg 5)
  });
  if (qpk && idx && pipe_ctas > 0) {
    const int64_t ntiles = (M + EV_TILE - 1) / EV_TILE;
    FMI_LAUNCH(KID_EVAL, s, k_eval_pipe<P>, (unsigned)std::min<int64_t>(ntiles, pipe_ctas), EV_THREADS, smem, qpk, keys,
               idx, M, Dk, nt, out, rec_idx ? 1 : 0);
    return;
  }
  FMI_LAUNCH(KID_EVAL, s, k_eval<P>, (unsigned)((M + 511) / 512), 256, 0, q, qpk, keys, idx, M, lo[0], lo[1], lo[2],
             width, unit, Dk, nt, out, rec_idx ? 1 : 0);
}

#define FMI_INST(P)                                                                                            \
  template void eval_sorted<P>(const double*, const double4*, const uint64_t*, const uint32_t*, int64_t,          \
                               const double*, double, bool, int, const NodeTable&, double*, cudaStream_t, bool); \
  template void presum_level<P>(const NodeTable&, int64_t, int64_t, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
FMI_INST(11) FMI_INST(12) FMI_INST(13) FMI_INST(14)  // unscoped high-order trees (f2)
#undef FMI_INST

}  // namespace fmi
