// residual.cu — K6: fused residual update, octant-block energies and child projections
// (DESIGN.md §5 K6).
//
// For every octant block (segment = node*8 + o) of a level's nodes, one pass over its points does
//   1. r <- r - Σ_α a_α u^α  (Algorithm 2 last line; Horner in the node frame, 𝓛 FMA/point),
//   2. Σ r² over the block (Algorithm 1 line 7: E_RMS of the block after the parent's fit),
//   3. if the block may become a child (n_o >= 𝓛 and depth+1 <= max_depth, P:306 + G5), the child's
//      projection b_α = Σ_i u_i^α r_i in the CHILD frame (the Λᵀf of Algorithm 2 for the child,
//      P:331, with the factorials applied in the solve) — so the next level needs no pass of its own.
// Root mode (level -1): no polynomial is subtracted, the single segment is the root and the
// projection is taken in the root frame.
//
// Layout per CTA (one chunk of one segment): a producer phase (one thread per two points: Horner,
// store of r, child-frame coordinates to shared memory) and a projection phase in which warp w owns
// a fixed group of outputs (a contiguous range of the Algorithm-2 basis order) and its lanes walk the
// batch's points: per point, z^0..z^cmax are formed once and every output (a,b,c) of the group costs
// one FMA  acc += (x^a y^b r) · z^c.  Lane partials are reduced in a fixed order (deterministic).
#include <mutex>
#include <utility>

#include "groups.cuh"
#include "horner.cuh"

namespace fmi {

namespace {

#ifndef FMI_K6_PLIM
#define FMI_K6_PLIM 40
#endif
#ifndef FMI_K6_MINB
#define FMI_K6_MINB 2
#endif
constexpr int K6_THREADS = 256;
constexpr int K6_WARPS = K6_THREADS / 32;
// points per thread in the Horner phase: 2 in the fused kernel (register budget shared with the
// projection accumulators), 4 in the Horner-only variant (four independent Horner chains per thread)
__host__ __device__ constexpr int k6_ppt(int var) { return var == 1 ? 4 : 2; }
__host__ __device__ constexpr int k6_batch(int var) { return k6_ppt(var) * 256; }
// the next batch's points stream into a shared-memory stage (cp.async) while the current one is processed
__host__ __device__ constexpr size_t k6_stage_smem(int var) { return 2 * 4 * (size_t)k6_batch(var) * sizeof(double); }

__device__ __forceinline__ void k6_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// ---- compile-time output groups ------------------------------------------------------------------
// pairs (a,b), a+b <= P, in a-major order (= the (l,m) order of Algorithm 2); pair q owns
// the outputs c = 0..P-a-b, contiguous in the basis order.
__host__ __device__ constexpr int npairs(int P) { return (P + 1) * (P + 2) / 2; }
__host__ __device__ constexpr int pair_a(int P, int q) {
  int a = 0;
  while (q >= P - a + 1) { q -= P - a + 1; ++a; }
  return a;
}
__host__ __device__ constexpr int pair_b(int P, int q) {
  int a = 0;
  while (q >= P - a + 1) { q -= P - a + 1; ++a; }
  return q;
}
__host__ __device__ constexpr int pair_out(int P, int q) { return P - pair_a(P, q) - pair_b(P, q) + 1; }
__host__ __device__ constexpr int pair_first(int P, int q) {  // basis index of (a, b, 0)
  return basis_index(P, pair_a(P, q), pair_b(P, q), 0);
}
// number of output groups (a power of two dividing the warp count) with <= 40 outputs each
__host__ __device__ constexpr int proj_groups(int P) {
  int g = 1;
  while (g < K6_WARPS && (rank3(P) + g - 1) / g > FMI_K6_PLIM) g *= 2;
  return g;
}
// first pair of group g: greedy cut at cumulative outputs >= g * ceil(L/G)
__host__ __device__ constexpr int group_pair_begin(int P, int g) {
  const int G = proj_groups(P);
  if (g >= G) return npairs(P);
  const int target = (rank3(P) + G - 1) / G * g;
  int q = 0, cum = 0;
  while (q < npairs(P) && cum < target) { cum += pair_out(P, q); ++q; }
  return q;
}
__host__ __device__ constexpr int group_out_begin(int P, int g) {
  return group_pair_begin(P, g) >= npairs(P) ? rank3(P) : pair_first(P, group_pair_begin(P, g));
}
__host__ __device__ constexpr int group_size(int P, int g) { return group_out_begin(P, g + 1) - group_out_begin(P, g); }
__host__ __device__ constexpr int max_group(int P) {
  int m = 0;
  for (int g = 0; g < proj_groups(P); ++g) m = group_size(P, g) > m ? group_size(P, g) : m;
  return m;
}
__host__ __device__ constexpr int group_cmax(int P, int g) {  // highest z power the group needs
  int smin = 1 << 20;
  for (int q = group_pair_begin(P, g); q < group_pair_begin(P, g + 1); ++q) {
    const int t = pair_a(P, q) + pair_b(P, q);
    smin = t < smin ? t : smin;
  }
  return smin > P ? 0 : P - smin;
}

// pair q of a group: acc[pair_first(q) - o0 + c] += v z^c, c = 0..P-a-b, v = x^a y^b r; along a row of
// equal a the pair values advance as two interleaved chains (v_{b+2} = v_b·y²); vn = the next pair's
// value (compile-time recursion: every index is a constant)
template <int P, int q, int q1, int o0>
__device__ __forceinline__ void proj_pairs(double x, double y, double y2, const double* zp, double xr, double v,
                                           double vn, double* acc) {
  if constexpr (q < q1) {
    constexpr int base = pair_first(P, q) - o0;
    constexpr int n = pair_out(P, q);
#pragma unroll
    for (int c = 0; c < n; ++c) acc[base + c] = fma(v, zp[c], acc[base + c]);
    if constexpr (q + 1 < q1) {
      if constexpr (pair_a(P, q + 1) == pair_a(P, q)) {
        proj_pairs<P, q + 1, q1, o0>(x, y, y2, zp, xr, vn, v * y2, acc);
      } else {
        const double xn = xr * x;
        proj_pairs<P, q + 1, q1, o0>(x, y, y2, zp, xn, xn, xn * y, acc);
      }
    }
  }
}

template <int P, int g>
__device__ __forceinline__ void proj_accum(double x, double y, double z, double r, double* acc) {
  constexpr int q0 = group_pair_begin(P, g), q1 = group_pair_begin(P, g + 1);
  constexpr int o0 = group_out_begin(P, g);
  constexpr int CM = group_cmax(P, g);
  if constexpr (q0 < q1) {
    double zp[CM + 1];
    zp[0] = 1.0;
    if constexpr (CM >= 1) zp[1] = z;
#pragma unroll
    for (int c = 2; c <= CM; ++c) zp[c] = zp[c / 2] * zp[c - c / 2];  // log-depth power tree
    // first pair's x^a r and x^a y^b r by square-and-multiply (log-depth)
    const double xr = grp::cpow<pair_a(P, q0)>(x) * r;
    const double v = xr * grp::cpow<pair_b(P, q0)>(y);
    proj_pairs<P, q0, q1, o0>(x, y, y * y, zp, xr, v, v * y, acc);
  }
}

// the batch's points j = j0, j0 + step, ... < nb for the warp's group g (compile-time): no per-point
// dispatch
template <int P, int g>
__device__ __forceinline__ void proj_loop(const double* sx, const double* sy, const double* sz, const double* sr,
                                          int j0, int step, int nb, double* acc) {
#pragma unroll 1
  for (int j = j0; j < nb; j += step) proj_accum<P, g>(sx[j], sy[j], sz[j], sr[j], acc);
}

template <int P, int... Gs>
__device__ __forceinline__ void proj_run(int gw, const double* sx, const double* sy, const double* sz,
                                         const double* sr, int j0, int step, int nb, double* acc,
                                         std::integer_sequence<int, Gs...>) {
  ((gw == Gs ? (proj_loop<P, Gs>(sx, sy, sz, sr, j0, step, nb, acc), 0) : 0), ...);
}

// VAR: 0 = fused (Horner + Σr² + projections), 1 = Horner + Σr² only, 2 = projections only — the
// specialised variants carry no registers for the part they skip
template <int P, int VAR>
__global__ void __launch_bounds__(K6_THREADS, FMI_K6_MINB)
    k_residual(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
               double* __restrict__ r, NodeTable nt, int64_t first, const Chunk* __restrict__ chunks,
               const int64_t* __restrict__ nchunks, int depth, int D, int mode, int iter,
               const double* __restrict__ delta, double* __restrict__ partial) {
  constexpr int L = rank3(P);
  constexpr int G = proj_groups(P);
  constexpr int SUB = K6_WARPS / G;  // warps per output group (split the batch's points)
  constexpr int MG = max_group(P);
  constexpr int K6_PPT = k6_ppt(VAR), K6_BATCH = k6_batch(VAR);
  __shared__ __align__(16) double sa[L];
  __shared__ double sbuf[VAR == 1 ? 2 * L : 4 * K6_BATCH];  // batch coordinates in the child frame + residuals
  double* sx = sbuf;
  double* sy = sbuf + K6_BATCH;
  double* sz = sbuf + 2 * K6_BATCH;
  double* sr = sbuf + 3 * K6_BATCH;
  static_assert(VAR == 1 || SUB * L <= 4 * K6_BATCH, "reduction buffer");
  double (*red)[L] = reinterpret_cast<double (*)[L]>(sbuf);  // after the point loop
  __shared__ double redw[K6_WARPS];
  const int64_t cidx = blockIdx.x;
  if (cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  const int o = ck.owner & 7;
  const int64_t ln = ck.owner >> 3;
  const int64_t node = first + ln;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* out = partial + cidx * (int64_t)(L + 1);
  constexpr bool kHorner = VAR != 2, kProj = VAR != 1;
  const bool horner = kHorner && mode != K6_ROOT && mode != K6_PROJ;
  const bool refined = horner && (nt.flag[node] & 2);
  if (mode == K6_OWN && !refined) {  // refinement pass: this node takes no step
    for (int e = tid; e <= L; e += K6_THREADS) out[e] = 0.0;
    return;
  }
  bool project;
  Frame fn{}, fc{};
  if (mode == K6_ROOT) {
    project = kProj;
    fc = node_frame(nt.cell[node]);
  } else {
    const int4 c = nt.cell[node];
    fn = node_frame(c);
    if (mode == K6_OWN) {
      project = kProj;
      fc = fn;
    } else {
      const int64_t n_o = nt.child_start[node * 9 + o + 1] - nt.child_start[node * 9 + o];
      // potential child (P:306 integer guard + G5), unless deferred (flag bit 3: see K6_PROJ)
      project = kProj && (mode == K6_PROJ || (n_o >= L && depth + 1 <= D && !(nt.flag[node] & 8)));
      fc = node_frame(make_int4(2 * c.x + (o & 1), 2 * c.y + ((o >> 1) & 1), 2 * c.z + ((o >> 2) & 1), c.w + 1));
    }
    // polynomial to subtract: the fit, or (refined nodes) the last refinement correction
    const bool use_delta = (mode == K6_OWN) ? (iter > 0) : refined;
    const double* src = use_delta ? delta + ln * L : nt.coef + node * L;
    for (int i = tid; i < L; i += K6_THREADS) sa[i] = src[i];
  }
  __syncthreads();
  const SmemCoef coef(sa);
  const int gw = warp % G, sub = warp / G;
  double acc[(kProj && MG > 0) ? MG : 1];
#pragma unroll
  for (int k = 0; k < MG; ++k) acc[k] = 0.0;
  double ss = 0.0;
  // stage[b & 1][array][K6_BATCH]: thread tid copies (and later reads) elements tid + k·K6_THREADS
  extern __shared__ __align__(16) double stage[];
  auto issue = [&](int64_t base, int buf) {
    if (base < ck.end) {
      double* st = stage + (size_t)buf * 4 * K6_BATCH;
#pragma unroll
      for (int k = 0; k < K6_PPT; ++k) {
        const int64_t i = base + tid + k * K6_THREADS;
        const int64_t j = i < ck.end ? i : ck.start;
        const int e = tid + k * K6_THREADS;
        k6_cp8(st + e, ux + j);
        k6_cp8(st + K6_BATCH + e, uy + j);
        k6_cp8(st + 2 * K6_BATCH + e, uz + j);
        k6_cp8(st + 3 * K6_BATCH + e, r + j);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(ck.start, 0);
  int buf = 0;
  for (int64_t base = ck.start; base < ck.end; base += K6_BATCH, buf ^= 1) {
    issue(base + K6_BATCH, buf ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    double X[K6_PPT], Y[K6_PPT], Z[K6_PPT], R[K6_PPT];
    bool V[K6_PPT];
    {
      const double* st = stage + (size_t)buf * 4 * K6_BATCH;
#pragma unroll
      for (int k = 0; k < K6_PPT; ++k) {
        const int e = tid + k * K6_THREADS;
        V[k] = base + e < ck.end;
        X[k] = st[e]; Y[k] = st[K6_BATCH + e]; Z[k] = st[2 * K6_BATCH + e]; R[k] = st[3 * K6_BATCH + e];
      }
    }
    if (kHorner && horner) {
      double hx[K6_PPT], hy[K6_PPT], hz[K6_PPT], pv[K6_PPT];
#pragma unroll
      for (int k = 0; k < K6_PPT; ++k) {
        hx[k] = to_local(X[k], fn.cx, fn.scale);
        hy[k] = to_local(Y[k], fn.cy, fn.scale);
        hz[k] = to_local(Z[k], fn.cz, fn.scale);
      }
      if constexpr (K6_PPT == 4) {
        horner3x4<P>(coef, hx, hy, hz, pv);
      } else {
        static_assert(K6_PPT == 2 || P < 0, "points per thread");
        horner3x2<P>(coef, hx[0], hy[0], hz[0], hx[1], hy[1], hz[1], pv[0], pv[1]);
      }
#pragma unroll
      for (int k = 0; k < K6_PPT; ++k) {
        R[k] -= pv[k];
        if (V[k]) { r[base + tid + k * K6_THREADS] = R[k]; ss = fma(R[k], R[k], ss); }
      }
    }
    if constexpr (kProj) if (project) {
#pragma unroll
      for (int k = 0; k < K6_PPT; ++k) {
        const int j = tid + k * K6_THREADS;
        sx[j] = to_local(X[k], fc.cx, fc.scale);
        sy[j] = to_local(Y[k], fc.cy, fc.scale);
        sz[j] = to_local(Z[k], fc.cz, fc.scale);
        sr[j] = V[k] ? R[k] : 0.0;
      }
      __syncthreads();
      const int nb = (int)min((int64_t)K6_BATCH, ck.end - base);
      proj_run<P>(gw, sx, sy, sz, sr, sub * 32 + lane, 32 * SUB, nb, acc, std::make_integer_sequence<int, G>{});
      __syncthreads();
    }
  }
  // Σ r² (fixed-order CTA reduction)
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
  if (lane == 0) redw[warp] = ss;
  // projection: lane reduction per output, then over the SUB warps of a group in fixed order
  if constexpr (kProj) if (project) {
    const int ob = [&] {
      int v = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) if (g == gw) v = group_out_begin(P, g);
      return v;
    }();
    const int on = [&] {
      int v = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) if (g == gw) v = group_size(P, g);
      return v;
    }();
#pragma unroll
    for (int k = 0; k < MG; ++k) {
      double v = acc[k];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
      if (lane == 0 && k < on) red[sub][ob + k] = v;
    }
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < K6_WARPS; ++w) t += redw[w];
    out[L] = t;
  }
  for (int e = tid; e < L; e += K6_THREADS) {
    double v = 0.0;
    if (project)
      for (int s = 0; s < SUB; ++s) v += red[s][e];
    out[e] = v;
  }
}

// The gather of the sorted points fused with the root projection (b = Λᵀf in the root frame, which
// needs no tree): every batch's 32-byte records packed[perm[i]] are gathered by cp.async (per-thread
// random addresses, in flight while the previous batch is projected), written out as the SoA arrays
// ux, uy, uz, r of the later passes, and projected.  f (optional): values uploaded separately
// (late-value path), taken from f[perm[i]] with the finiteness flag *bad.
template <int P>
__global__ void __launch_bounds__(K6_THREADS, FMI_K6_MINB)
    k_gather_root(const double4* __restrict__ packed, uint32_t* __restrict__ perm, const uint32_t* __restrict__ orig,
                  const double* __restrict__ f, int* __restrict__ bad, double* __restrict__ ux,
                  double* __restrict__ uy, double* __restrict__ uz, double* __restrict__ r,
                  const Chunk* __restrict__ chunks, const int64_t* __restrict__ nchunks,
                  double* __restrict__ partial, uint64_t* __restrict__ keys, int D, int64_t r0, int64_t n_stride) {
  constexpr int L = rank3(P);
  constexpr int G = proj_groups(P);
  constexpr int SUB = K6_WARPS / G;
  constexpr int MG = max_group(P);
  constexpr int PPT = 2, BATCH = PPT * K6_THREADS;
  __shared__ double sbuf[4 * BATCH];  // batch coordinates in the root frame + values
  double* sx = sbuf;
  double* sy = sbuf + BATCH;
  double* sz = sbuf + 2 * BATCH;
  double* sr = sbuf + 3 * BATCH;
  static_assert(SUB * L <= 4 * BATCH, "reduction buffer");
  double (*red)[L] = reinterpret_cast<double (*)[L]>(sbuf);
  extern __shared__ __align__(16) double stage[];  // [2][BATCH] records (4 doubles) + [2][BATCH] values
  // chunk mode: CTA = one chunk of consecutive batches; stride mode (n_stride > 0, bucketed records):
  // CTA b takes batches b, b + grid, ... of [r0, n_stride), so the CTAs in flight gather from a window of
  // consecutive positions (a part of one bucket of records, L2-resident) instead of one chunk each
  const int64_t cidx = blockIdx.x;
  int64_t c0, c1, step;
  if (n_stride > 0) {
    c0 = r0 + cidx * BATCH;
    c1 = n_stride;
    step = (int64_t)gridDim.x * BATCH;
  } else {
    if (cidx >= *nchunks) return;
    const Chunk ck = chunks[cidx];
    c0 = ck.start;
    c1 = ck.end;
    step = BATCH;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = warp % G, sub = warp / G;
  double* out = partial + cidx * (int64_t)(L + 1);
  double acc[MG > 0 ? MG : 1];
#pragma unroll
  for (int k = 0; k < MG; ++k) acc[k] = 0.0;
  double* srec = stage;                    // [2][BATCH][4]
  double* sval = stage + 2 * BATCH * 4;    // [2][BATCH]
  uint32_t pn[PPT];                        // perm of the next batch (loaded one batch ahead)
  uint32_t pi[PPT];                        // its input indices (bucketed keys: orig[perm]; else perm)
  auto load_perm = [&](int64_t base) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int64_t i = base + tid + k * K6_THREADS;
      pn[k] = i < c1 ? perm[i] : 0u;
    }
    if (orig) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int64_t i = base + tid + k * K6_THREADS;
        pi[k] = orig[pn[k]];
        if (i < c1) perm[i] = pi[k];  // the tree keeps input indices
      }
    } else {
#pragma unroll
      for (int k = 0; k < PPT; ++k) pi[k] = pn[k];
    }
  };
  auto issue = [&](int64_t base, int buf) {
    if (base < c1) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int e = tid + k * K6_THREADS;
        double* d = srec + ((size_t)buf * BATCH + e) * 4;
        const double* src = reinterpret_cast<const double*>(packed + pn[k]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                     "l"(src) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d + 2)),
                     "l"(src + 2) : "memory");
        if (f) k6_cp8(sval + (size_t)buf * BATCH + e, f + pi[k]);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  load_perm(c0);
  issue(c0, 0);
  load_perm(c0 + step);
  int buf = 0;
  const Frame fc = node_frame(make_int4(0, 0, 0, 0));
  int nbad = 0;
  for (int64_t base = c0; base < c1; base += step, buf ^= 1) {
    issue(base + step, buf ^ 1);
    load_perm(base + 2 * step);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int e = tid + k * K6_THREADS;
      const int64_t i = base + e;
      const bool v = i < c1;
      const double* rec = srec + ((size_t)buf * BATCH + e) * 4;
      const double X = rec[0], Y = rec[1], Z = rec[2];
      const double R = f ? sval[(size_t)buf * BATCH + e] : rec[3];
      if (v) {
        ux[i] = X; uy[i] = Y; uz[i] = Z; r[i] = R;
        if (keys) keys[i] = morton_key(X, Y, Z, D);  // the full key, recomputed (the sort moved 32-bit keys)
        if (f && !isfinite(R)) nbad = 1;
      }
      sx[e] = to_local(X, fc.cx, fc.scale);
      sy[e] = to_local(Y, fc.cy, fc.scale);
      sz[e] = to_local(Z, fc.cz, fc.scale);
      sr[e] = v ? R : 0.0;
    }
    __syncthreads();
    const int nb = (int)min((int64_t)BATCH, c1 - base);
    proj_run<P>(gw, sx, sy, sz, sr, sub * 32 + lane, 32 * SUB, nb, acc, std::make_integer_sequence<int, G>{});
    __syncthreads();
  }
  if (nbad) *bad = 1;
  const int ob = [&] {
    int v = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) if (g == gw) v = group_out_begin(P, g);
    return v;
  }();
  const int on = [&] {
    int v = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) if (g == gw) v = group_size(P, g);
    return v;
  }();
#pragma unroll
  for (int k = 0; k < MG; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && k < on) red[sub][ob + k] = v;
  }
  __syncthreads();
  for (int e = tid; e < L; e += K6_THREADS) {
    double v = 0.0;
    for (int q = 0; q < SUB; ++q) v += red[q][e];
    out[e] = v;
  }
  if (tid == 0) out[L] = 0.0;
}

// segment sums: partial chunks of segment (node*8+o) -> segsum[seg][𝓛+1]; Σr² also to the node table
// (child_ss) for the decisions.  CTA per (segment, 32 consecutive entries): lane = entry, warp w
// sums the chunks c ≡ w (mod 8) with 2 independent accumulators, the 8 warp sums are then added in warp
// order (fixed order: deterministic).
__global__ void __launch_bounds__(256)
    k_residual_reduce(const double* __restrict__ partial, const int64_t* __restrict__ chunk_begin,
                      const int64_t* __restrict__ nchunks, int64_t nseg, NodeTable nt, int64_t first, int L,
                      bool write_ss, const int32_t* __restrict__ sel, double* __restrict__ segsum) {
  const int64_t sgi = blockIdx.x;
  if (sel && sel[sgi] < 0) return;  // K6_PROJ: only the selected segments are (re)written
  __shared__ double ws[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = chunk_begin[sgi];
  const int64_t c1 = sgi + 1 < nseg ? chunk_begin[sgi + 1] : *nchunks;
  {  // entry group blockIdx.y: entries 32·y .. 32·y + 31
    const int e = (int)blockIdx.y * 32 + lane;
    const int nw = (int)(blockDim.x >> 5);  // 1..8 warps, sized to the chunks per segment
    double a = 0.0, b = 0.0;
    if (e <= L) {
      int64_t c = c0 + warp;
      for (; c + nw < c1; c += 2 * nw) {
        a += partial[c * (L + 1) + e];
        b += partial[(c + nw) * (L + 1) + e];
      }
      if (c < c1) a += partial[c * (L + 1) + e];
    }
    ws[warp][lane] = a + b;
    __syncthreads();
    if (warp == 0 && e <= L) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += ws[w][lane];
      segsum[sgi * (L + 1) + e] = t;
      if (e == L && write_ss) nt.child_ss[first * 8 + sgi] = t;
    }
  }
}

}  // namespace

template <int P, int VAR>
void launch_residual(int kid, const LevelCtx& c, int mode, int iter, const double* delta, const Chunk* chunks,
                     const int64_t* nchunks_dev, int64_t max_chunks, double* partial, cudaStream_t s) {
  static std::once_flag attr_once;  // one opt-in per kernel instantiation (thread-safe)
  std::call_once(attr_once, [&] {
    FMI_CK(cudaFuncSetAttribute(
        k_residual<P, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k6_stage_smem(VAR)));
  });
  FMI_LAUNCH(kid, s, (k_residual<P, VAR>), (unsigned)max_chunks, K6_THREADS, k6_stage_smem(VAR), c.ux, c.uy, c.uz, c.r,
             c.nt, c.first, chunks, nchunks_dev, c.depth, c.D, mode, iter, delta, partial);
}

template <int P>
void level_residual(const LevelCtx& c, int mode, int iter, const double* delta, const Chunk* chunks,
                    const int64_t* nchunks_dev, int64_t max_chunks, const int64_t* chunk_begin, int64_t nseg,
                    double* partial, double* segsum, cudaStream_t s, const int32_t* sel, bool horner_only) {
  const int kid = mode == K6_ROOT ? KID_PROJECT : (mode == K6_OWN ? KID_REFINE : KID_RESIDUAL);
  if (max_chunks > 0) {
    if (mode == K6_ROOT || mode == K6_PROJ)
      launch_residual<P, 2>(kid, c, mode, iter, delta, chunks, nchunks_dev, max_chunks, partial, s);
    else if (mode == K6_CHILD && horner_only)
      launch_residual<P, 1>(kid, c, mode, iter, delta, chunks, nchunks_dev, max_chunks, partial, s);
    else
      launch_residual<P, 0>(kid, c, mode, iter, delta, chunks, nchunks_dev, max_chunks, partial, s);
  }
  // warps per segment CTA: about the chunks per segment (one warp for the many small segments of deep
  // adaptive levels, eight for the few huge ones of the top levels)
  int nw = 1;
  while (nw < 8 && (int64_t)nw * nseg < max_chunks) nw *= 2;
  FMI_LAUNCH(KID_RESIDUAL_REDUCE, s, k_residual_reduce, dim3((unsigned)nseg, (unsigned)((rank3(P) + 1 + 31) / 32)),
             32 * nw, 0, partial, chunk_begin, nchunks_dev, nseg, c.nt, c.first, rank3(P), mode == K6_CHILD, sel,
             segsum);
}

// resident CTAs of k_gather_root on the device (the stride-mode grid)
template <int P>
int gather_root_ctas() {
  static int ctas = [] {
    constexpr size_t smem = 2 * (size_t)(2 * K6_THREADS) * 5 * sizeof(double);
    int dev = 0, sms = 0, per = 0;
    FMI_CK(cudaGetDevice(&dev));
    FMI_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FMI_CK(cudaFuncSetAttribute(k_gather_root<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FMI_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gather_root<P>, K6_THREADS, smem));
    return sms * std::max(1, per);
  }();
  return ctas;
}

template <int P>
void gather_root_projection(const double4* packed, uint32_t* perm, const uint32_t* orig, const double* f, int* bad,
                            int64_t n,
                            double* ux, double* uy, double* uz, double* r, const Chunk* chunks,
                            const int64_t* nchunks_dev, int64_t max_chunks, const int64_t* chunk_begin,
                            double* partial, double* segsum, cudaStream_t s, uint64_t* keys, int D,
                            int64_t n_stride) {
  // stride mode: the range is cut into launches of <= kStrideSpan positions (a grid-wide step between
  // them bounds how far the persistent CTAs drift apart, i.e. the window of records in flight); launch
  // k writes partial rows [k·grid, (k+1)·grid)
  constexpr int64_t kStrideSpan = (int64_t)1 << 23;
  constexpr size_t smem = 2 * (size_t)(2 * K6_THREADS) * 5 * sizeof(double);
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    FMI_CK(cudaFuncSetAttribute(k_gather_root<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  if (n_stride > 0) {
    const int64_t nl = (n_stride + kStrideSpan - 1) / kStrideSpan;
    const int64_t grid = max_chunks / nl;  // CTAs per launch (max_chunks = nl · grid partial rows)
    for (int64_t k = 0; k < nl; ++k)
      FMI_LAUNCH(KID_PROJECT, s, k_gather_root<P>, (unsigned)grid, K6_THREADS, smem, packed, perm, orig, f, bad, ux,
                 uy, uz, r, chunks, nchunks_dev, partial + k * grid * (rank3(P) + 1), keys, D, k * kStrideSpan,
                 std::min(n_stride, (k + 1) * kStrideSpan));
  } else if (max_chunks > 0) {
    FMI_LAUNCH(KID_PROJECT, s, k_gather_root<P>, (unsigned)max_chunks, K6_THREADS, smem, packed, perm, orig, f, bad,
               ux, uy, uz, r, chunks, nchunks_dev, partial, keys, D, (int64_t)0, (int64_t)0);
  }
  FMI_LAUNCH(KID_RESIDUAL_REDUCE, s, k_residual_reduce, dim3(1u, (unsigned)((rank3(P) + 1 + 31) / 32)), 256, 0,
             partial, chunk_begin, nchunks_dev, (int64_t)1, NodeTable{}, (int64_t)0, rank3(P), false, nullptr, segsum);
  (void)n;
}

#define FMI_INST(P)                                                                                            \
  template void level_residual<P>(const LevelCtx&, int, int, const double*, const Chunk*, const int64_t*, int64_t, \
                                  const int64_t*, int64_t, double*, double*, cudaStream_t, const int32_t*, bool); \
  template void gather_root_projection<P>(const double4*, uint32_t*, const uint32_t*, const double*, int*, int64_t,   \
                                          double*,                                                                  \
                                          double*, double*, double*, const Chunk*, const int64_t*, int64_t,           \
                                          const int64_t*, double*, double*, cudaStream_t, uint64_t*, int,     \
                                          int64_t);                                                           \
  template int gather_root_ctas<P>();
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
