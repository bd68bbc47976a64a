// groups.cuh — compile-time output groups for the register-blocked monomial accumulations of K4
// (raw moments, degree Q = 2p) and K6 (child projections, degree p).
//
// Outputs are the multi-indices (a,b,c), a+b+c <= Q, in the loop order of Algorithm 2 (P:322-324:
// a outer, b middle, c inner).  Pair q = (a,b) in a-major order owns the outputs c = 0..Q-a-b, which
// are CONTIGUOUS in that order, so a group of consecutive pairs is a contiguous range of outputs.
// A warp owns one group; each lane accumulates the group's outputs over its own points:
//     acc[(a,b,c)] += (x^a y^b w) · z^c        (w = 1 for moments, the residual for projections)
// with z^0..z^cmax formed once per point and one multiply per pair, so every output costs exactly one
// FMA and nothing outside the simplex is computed.  Everything below is constexpr: the accumulator
// indices of the unrolled code are compile-time constants (registers, no local memory).
#pragma once

#include "fmi_internal.cuh"

namespace fmi {
namespace grp {

__host__ __device__ constexpr int npairs(int Q) { return (Q + 1) * (Q + 2) / 2; }
__host__ __device__ constexpr int pair_a(int Q, int q) {
  int a = 0;
  while (q >= Q - a + 1) { q -= Q - a + 1; ++a; }
  return a;
}
__host__ __device__ constexpr int pair_b(int Q, int q) {
  int a = 0;
  while (q >= Q - a + 1) { q -= Q - a + 1; ++a; }
  return q;
}
__host__ __device__ constexpr int pair_out(int Q, int q) { return Q - pair_a(Q, q) - pair_b(Q, q) + 1; }
__host__ __device__ constexpr int pair_first(int Q, int q) { return basis_index(Q, pair_a(Q, q), pair_b(Q, q), 0); }

// Greedy partition: a group takes consecutive pairs while its output count stays <= LIM, and (if
// TARGET > 0) closes once it reaches TARGET outputs.
__host__ __device__ constexpr int next_cut(int Q, int LIM, int TARGET, int q) {
  int cum = 0;
  while (q < npairs(Q) && cum + pair_out(Q, q) <= LIM && (TARGET <= 0 || cum < TARGET)) { cum += pair_out(Q, q); ++q; }
  return q;
}
__host__ __device__ constexpr int ngroups(int Q, int LIM, int TARGET) {
  int g = 0, q = 0;
  while (q < npairs(Q)) { q = next_cut(Q, LIM, TARGET, q); ++g; }
  return g;
}
__host__ __device__ constexpr int pair_begin(int Q, int LIM, int TARGET, int g) {
  int q = 0;
  for (int k = 0; k < g && q < npairs(Q); ++k) q = next_cut(Q, LIM, TARGET, q);
  return q;
}
__host__ __device__ constexpr int out_begin(int Q, int LIM, int TARGET, int g) {
  const int q = pair_begin(Q, LIM, TARGET, g);
  return q >= npairs(Q) ? rank3(Q) : pair_first(Q, q);
}
__host__ __device__ constexpr int group_size(int Q, int LIM, int TARGET, int g) {
  return out_begin(Q, LIM, TARGET, g + 1) - out_begin(Q, LIM, TARGET, g);
}
__host__ __device__ constexpr int max_size(int Q, int LIM, int TARGET) {
  int m = 0;
  for (int g = 0; g < ngroups(Q, LIM, TARGET); ++g)
    m = group_size(Q, LIM, TARGET, g) > m ? group_size(Q, LIM, TARGET, g) : m;
  return m;
}
__host__ __device__ constexpr int group_cmax(int Q, int LIM, int TARGET, int g) {  // highest z power needed
  int smin = 1 << 20;
  for (int q = pair_begin(Q, LIM, TARGET, g); q < pair_begin(Q, LIM, TARGET, g + 1); ++q) {
    const int t = pair_a(Q, q) + pair_b(Q, q);
    smin = t < smin ? t : smin;
  }
  return smin > Q ? 0 : Q - smin;
}

// x^E by a compile-time square-and-multiply chain
template <int E>
__device__ __forceinline__ double cpow(double x) {
  if constexpr (E == 0) return 1.0;
  else if constexpr (E == 1) return x;
  else if constexpr (E % 2 == 0) { const double h = cpow<E / 2>(x); return h * h; }
  else return x * cpow<E - 1>(x);
}

// pairs q..q1-1 of a group: acc[pair_first(q) - o0 + c] += v z^c with v = x^a y^b w.  Along a row of
// equal a the pair values advance as two interleaved chains (v_{b+2} = v_b·y², one multiply per pair):
// half the dependent-multiply latency of a single chain; vn = the next pair's value.
template <int Q, int q, int q1, int o0>
__device__ __forceinline__ void pairs(double x, double y, double y2, const double* zp, double xw, double v, double vn,
                                      double* acc) {
  if constexpr (q < q1) {
    constexpr int base = pair_first(Q, q) - o0;
    constexpr int n = pair_out(Q, q);
#pragma unroll
    for (int c = 0; c < n; ++c) acc[base + c] = fma(v, zp[c], acc[base + c]);
    if constexpr (q + 1 < q1) {
      if constexpr (pair_a(Q, q + 1) == pair_a(Q, q)) {
        pairs<Q, q + 1, q1, o0>(x, y, y2, zp, xw, vn, v * y2, acc);
      } else {
        const double xn = xw * x;
        pairs<Q, q + 1, q1, o0>(x, y, y2, zp, xn, xn, xn * y, acc);
      }
    }
  }
}

// one point's contribution to group g
template <int Q, int LIM, int TARGET, int g>
__device__ __forceinline__ void accum(double x, double y, double z, double w, double* acc) {
  constexpr int q0 = pair_begin(Q, LIM, TARGET, g), q1 = pair_begin(Q, LIM, TARGET, g + 1);
  constexpr int o0 = out_begin(Q, LIM, TARGET, g);
  constexpr int CM = group_cmax(Q, LIM, TARGET, g);
  if constexpr (q0 < q1) {
    double zp[CM + 1];
    zp[0] = 1.0;
    if constexpr (CM >= 1) zp[1] = z;
    // log-depth power tree: z^c = z^(c/2) z^(c - c/2) (critical path ~log2(c) multiplies, not c)
#pragma unroll
    for (int c = 2; c <= CM; ++c) zp[c] = zp[c / 2] * zp[c - c / 2];
    const double xw = cpow<pair_a(Q, q0)>(x) * w;
    const double v0 = xw * cpow<pair_b(Q, q0)>(y);
    pairs<Q, q0, q1, o0>(x, y, y * y, zp, xw, v0, v0 * y, acc);
  }
}

// Butterfly reduce-scatter of N = 32·M values per lane over the 32 lanes of a warp: afterwards lane l
// holds the warp totals of entries M·l .. M·l+M-1 in v[0..M).  31·M shuffles instead of 5·N.
template <int N>
__device__ __forceinline__ void warp_reduce_scatter(double* v, int lane) {
  static_assert(N % 32 == 0, "N must be a multiple of 32");
#pragma unroll
  for (int half = N / 2, bit = 16; bit >= 1; half >>= 1, bit >>= 1) {
    const bool up = (lane & bit) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? v[i] : v[i + half];
      const double keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
}

}  // namespace grp
}  // namespace fmi
