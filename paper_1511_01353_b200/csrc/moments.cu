// moments.cu — K4: raw geometric moments by direct accumulation over points (DESIGN.md §5 K4).
//
// PAPER.md Algorithm 2 builds Λ(1:N, lmn) = x^l y^m z^n/(l!m!n!) and factors it (QR).  In
// Gram form every entry of ΛᵀΛ is a raw moment,  G_αβ = M_{α+β}/(α!β!),  M_γ = Σ_i u_i^γ, |γ| <= 2p,
// i.e. K = C(2p+3,3) multiply-adds per point instead of the dense Gram's 𝓛(𝓛+1)/2.  The moments depend
// on the geometry only: they are accumulated ONCE per build for every moment-tree node over its owner
// segments and translated upward by m2m.cu; a fit node whose translated moments fail the rounding
// check is re-accumulated here directly over its own points (fallback).
//
// Register-blocked, no shared-memory staging, no cross-lane reduction: the K outputs are cut into
// groups of <= 64 consecutive entries of the Algorithm-2 order (groups.cuh); a warp owns one group,
// each of its lanes one chunk (<= kMomentChunk points), so every output costs one FMA per point and the
// only extra work per point and group is z^0..z^cmax and one multiply per (a,b) pair.  Chunk partials
// are summed per node in chunk order (deterministic, no atomics).
#include "groups.cuh"
#include "horner.cuh"

#include <utility>

namespace fmi {

namespace {

// threads per CTA: p = 10 runs 128-thread CTAs, two per SM (254 registers), so that its 20 output
// groups fill 5 CTAs of 4 warps exactly (256-thread CTAs left 4 of every 24 warps idle)
#ifndef FMI_K4_THREADS_P10
#define FMI_K4_THREADS_P10 128
#endif
template <int P>
constexpr int k4_threads() { return P >= 10 ? FMI_K4_THREADS_P10 : 256; }
#ifndef FMI_K4_LIM
#define FMI_K4_LIM 64
#endif
#ifndef FMI_K4_PIPE
#define FMI_K4_PIPE 1
#endif
#ifndef FMI_K4_MINB
#define FMI_K4_MINB 1
#endif
// outputs per group (2·LIM accumulator registers): at p = 10 groups of <= 96 outputs (20 groups, 254
// registers, no spills) cut the per-point z-power and pair overhead (cfg 5: 43.4 -> 36.9 ms); smaller
// degrees keep 64 (more groups = more warps per chunk set: cfg 3/4 measured slower with 96)
#ifndef FMI_K4_LIM_P10
#define FMI_K4_LIM_P10 96
#endif
template <int P>
constexpr int k4_lim() { return P >= 10 ? FMI_K4_LIM_P10 : FMI_K4_LIM; }
constexpr int K4_RING = 8;  // per-lane point ring (cp.async prefetch distance K4_RING - 1)

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int P>
struct K4Plan {
  static constexpr int Q = 2 * P;
  static constexpr int K = rank3(Q);
  static constexpr int NG = grp::ngroups(Q, k4_lim<P>(), 0);
  static constexpr int THREADS = k4_threads<P>(), WARPS = THREADS / 32;
  static constexpr int NGB = (NG + WARPS - 1) / WARPS;  // CTAs per 32 chunks
  static constexpr int MG = grp::max_size(Q, k4_lim<P>(), 0);
};

// The point loop of one group g (compile-time): z powers, pair products and the group's FMAs, no
// per-point dispatch.  Points stream through a per-warp shared-memory ring filled by cp.async (8-byte
// LDGSTS): the load of point i+PD is in flight while points i..i+PD-1 are processed, without tying up
// registers.
template <int P, int g>
__device__ __forceinline__ void k4_loop(const double* __restrict__ ux, const double* __restrict__ uy,
                                        const double* __restrict__ uz, const Chunk& ck, const Frame& fr, double* rg,
                                        int lane, double* __restrict__ out) {
  constexpr int Q = 2 * P;
  constexpr int n = grp::group_size(Q, k4_lim<P>(), 0, g);
  double acc[n];
#pragma unroll
  for (int k = 0; k < n; ++k) acc[k] = 0.0;
  constexpr int R = K4_RING, PD = K4_RING - 1;
  auto issue = [&](int64_t j, int slot) {
    if (j < ck.end) {
      double* d = rg + slot * 96 + lane;
      cp_async8(d, ux + j);
      cp_async8(d + 32, uy + j);
      cp_async8(d + 64, uz + j);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < PD; ++k) issue(ck.start + k, k);
#if FMI_K4_PIPE
  // the next point's local coordinates are read while the current point is accumulated (the ring-load
  // and frame latency leave the FMA stream's critical path)
  asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");
  double x = to_local(rg[lane], fr.cx, fr.scale), y = to_local(rg[32 + lane], fr.cy, fr.scale),
         z = to_local(rg[64 + lane], fr.cz, fr.scale);
  int t = 0;
#pragma unroll 1
  for (int64_t i = ck.start; i < ck.end; ++i) {
    issue(i + PD, (t + PD) % R);
    t = (t + 1 == R) ? 0 : t + 1;
    asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");
    const double* sp = rg + t * 96 + lane;
    const double xn = sp[0], yn = sp[32], zn = sp[64];
    grp::accum<Q, k4_lim<P>(), 0, g>(x, y, z, 1.0, acc);
    x = to_local(xn, fr.cx, fr.scale);
    y = to_local(yn, fr.cy, fr.scale);
    z = to_local(zn, fr.cz, fr.scale);
  }
#else
  int t = 0;
#pragma unroll 1
  for (int64_t i = ck.start; i < ck.end; ++i, t = (t + 1 == R) ? 0 : t + 1) {
    asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");
    const double* sp = rg + t * 96 + lane;
    const double x = to_local(sp[0], fr.cx, fr.scale);
    const double y = to_local(sp[32], fr.cy, fr.scale);
    const double z = to_local(sp[64], fr.cz, fr.scale);
    issue(i + PD, (t + PD) % R);
    grp::accum<Q, k4_lim<P>(), 0, g>(x, y, z, 1.0, acc);
  }
#endif
  double* o = out + grp::out_begin(Q, k4_lim<P>(), 0, g);
#pragma unroll
  for (int k = 0; k < n; ++k) o[k] = acc[k];
}

template <int P, int... Gs>
__device__ __forceinline__ void k4_run(int gw, const double* __restrict__ ux, const double* __restrict__ uy,
                                       const double* __restrict__ uz, const Chunk& ck, const Frame& fr, double* rg,
                                       int lane, double* __restrict__ out, std::integer_sequence<int, Gs...>) {
  ((gw == Gs ? (k4_loop<P, Gs>(ux, uy, uz, ck, fr, rg, lane, out), 0) : 0), ...);
}

// Lane = chunk, warp = output group: lane l of warp w in CTA b accumulates group (b % NGB)·WARPS + w over
// the points of chunk 32·(b / NGB) + l (sequentially, in the frame of node cell[owner >> shift]) and writes
// its outputs to partial[chunk][..].  No cross-lane reduction; the 8 warps of a CTA read the same
// 32 chunks (L1 reuse).  Chunks are <= kMomentChunk points (make_chunks).
template <int P>
__global__ void __launch_bounds__(k4_threads<P>(), k4_threads<P>() < 256 ? 256 / k4_threads<P>() : FMI_K4_MINB)
    k_moments(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
              const int4* __restrict__ cell, int shift, const Chunk* __restrict__ chunks,
              const int64_t* __restrict__ nchunks, double* __restrict__ partial) {
  using PL = K4Plan<P>;
  constexpr int K = PL::K;
  __shared__ __align__(16) double ring[PL::WARPS * K4_RING * 3 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the NGB CTAs that read the same 32 chunks are adjacent in launch order (their re-reads hit L2)
  const int gw = (int)(blockIdx.x % PL::NGB) * PL::WARPS + warp;
  const int64_t cidx = (int64_t)(blockIdx.x / PL::NGB) * 32 + lane;
  if (gw >= PL::NG || cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  const Frame fr = node_frame(cell[ck.owner >> shift]);
  double* rg = ring + (size_t)warp * K4_RING * 3 * 32;
  k4_run<P>(gw, ux, uy, uz, ck, fr, rg, lane, partial + cidx * (int64_t)K,
            std::make_integer_sequence<int, PL::NG>{});
}

// out[node·stride + e] = Σ of the chunk partials of the node's ranges (rpn ranges per node: 8 owner
// segments, or 1 node range) in a fixed order, for nodes with (flag[node] & bit) when flag != nullptr.
// CTA = node, thread = entries; the chunk loop keeps 8 independent partial sums (chunks c ≡ k mod 8,
// combined k = 0..7) so nodes with many chunks have 8 loads in flight per thread; deterministic.
__global__ void __launch_bounds__(256) k_moments_reduce(const double* __restrict__ partial,
                                                        const int64_t* __restrict__ chunk_begin,
                                                        const int64_t* __restrict__ nchunks, int64_t nodes, int rpn,
                                                        int K, const int32_t* __restrict__ flag, int bit,
                                                        double* __restrict__ out, int64_t stride) {
  const int64_t node = blockIdx.x;
  if (flag && !(flag[node] & bit)) return;
  const int64_t c0 = chunk_begin[node * rpn];
  const int64_t c1 = node + 1 < nodes ? chunk_begin[(node + 1) * rpn] : *nchunks;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t ci = c0;
    for (; ci + 8 <= c1; ci += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) s[k] += partial[(ci + k) * K + e];
    }
    for (; ci < c1; ++ci) s[0] += partial[ci * K + e];
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += s[k];
    out[node * stride + e] = t;
  }
}

// Few nodes (a huge root re-accumulated directly): the chunk range of each node is cut into KR_SLICES
// fixed slices, CTA (node, slice, entry block) sums its slice in chunk order into slice partials, and
// k_slices_reduce adds the slices in order — the same fixed summation order every run.
constexpr int KR_SLICES = 64;
__global__ void __launch_bounds__(256) k_moments_reduce_sliced(const double* __restrict__ partial,
                                                               const int64_t* __restrict__ chunk_begin,
                                                               const int64_t* __restrict__ nchunks, int64_t nodes,
                                                               int rpn, int K, const int32_t* __restrict__ flag,
                                                               int bit, double* __restrict__ slices) {
  const int64_t node = blockIdx.x;
  const int sl = blockIdx.y;
  if (flag && !(flag[node] & bit)) return;
  const int64_t c0 = chunk_begin[node * rpn];
  const int64_t c1 = node + 1 < nodes ? chunk_begin[(node + 1) * rpn] : *nchunks;
  const int64_t n = c1 - c0;
  const int64_t a = c0 + n * sl / KR_SLICES, b = c0 + n * (sl + 1) / KR_SLICES;
  const int e = blockIdx.z * blockDim.x + threadIdx.x;
  if (e >= K) return;
  double s[4] = {0, 0, 0, 0};
  int64_t ci = a;
  for (; ci + 4 <= b; ci += 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) s[k] += partial[(ci + k) * K + e];
  }
  for (; ci < b; ++ci) s[0] += partial[ci * K + e];
  slices[(node * KR_SLICES + sl) * (int64_t)K + e] = (s[0] + s[1]) + (s[2] + s[3]);
}

__global__ void k_slices_reduce(const double* __restrict__ slices, int64_t nodes, int K,
                                const int32_t* __restrict__ flag, int bit, double* __restrict__ out, int64_t stride) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nodes * K) return;
  const int64_t node = g / K;
  const int e = (int)(g % K);
  if (flag && !(flag[node] & bit)) return;
  double t = 0.0;
  for (int sl = 0; sl < KR_SLICES; ++sl) t += slices[(node * KR_SLICES + sl) * (int64_t)K + e];
  out[node * stride + e] = t;
}

}  // namespace

template <int P>
void direct_moments(const double* ux, const double* uy, const double* uz, const int4* cell, int shift,
                    const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks, double* partial,
                    cudaStream_t s) {
  using PL = K4Plan<P>;
  if (max_chunks <= 0) return;
  FMI_LAUNCH(KID_MOMENTS, s, (k_moments<P>), (unsigned)((max_chunks + 31) / 32 * PL::NGB), PL::THREADS, 0, ux, uy,
             uz, cell, shift, chunks, nchunks_dev, partial);
}

void reduce_moments(const double* partial, const int64_t* chunk_begin, const int64_t* nchunks_dev, int64_t nodes,
                    int rpn, int K, const int32_t* flag, int bit, double* out, int64_t stride, cudaStream_t s) {
  if (nodes <= 0) return;
  if (nodes <= 16) {  // too few CTAs for the per-node reduction: slice the chunk ranges (cfg 4 root: 1.6 ms)
    DBuf<double> slices((size_t)nodes * KR_SLICES * K, s);
    FMI_LAUNCH(KID_MOMENTS_REDUCE, s, k_moments_reduce_sliced,
               dim3((unsigned)nodes, (unsigned)KR_SLICES, (unsigned)((K + 255) / 256)), 256, 0, partial, chunk_begin,
               nchunks_dev, nodes, rpn, K, flag, bit, slices.p);
    FMI_LAUNCH(KID_MOMENTS_REDUCE, s, k_slices_reduce, (unsigned)((nodes * K + 255) / 256), 256, 0, slices.p, nodes,
               K, flag, bit, out, stride);
    return;
  }
  FMI_LAUNCH(KID_MOMENTS_REDUCE, s, k_moments_reduce, (unsigned)nodes, 256, 0, partial, chunk_begin, nchunks_dev, nodes,
             rpn, K, flag, bit, out, stride);
}

#define FMI_INST(P)                                                                                          \
  template void direct_moments<P>(const double*, const double*, const double*, const int4*, int, const Chunk*, \
                                  const int64_t*, int64_t, double*, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

// K4 plan statistics for DESIGN.md / bench: groups and FP64 operations per point (useful FMAs = K)
int k4_groups(int p) {
  switch (p) {
#define C(P) case P: return K4Plan<P>::NG;
    C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10)
#undef C
  }
  return 0;
}

}  // namespace fmi
