// horner.cuh — evaluation of a node polynomial Σ_α a_α u^α (monomial form, Algorithm-2 column order)
// by nested Horner in z, y, x: 𝓛 fused multiply-adds, coefficient offsets known at compile time.
// Used by K6 (residual update, "f <- f - Λ·P_F") and K7 (evaluation).
#pragma once

#include "fmi_internal.cuh"

namespace fmi {

// COEF(i) must yield coefficient i (e.g. a shared-memory read or an __ldg).  Every Horner chain starts
// at its highest coefficient (no fma(0, z, a) = a step: that product is not foldable by the compiler,
// z may be non-finite, and would cost one FP64 instruction per row).
template <int P, typename Coef>
__device__ __forceinline__ double horner3(const Coef& coef, double x, double y, double z) {
  double px = 0.0;
#pragma unroll
  for (int l = P; l >= 0; --l) {
    double py = 0.0;
#pragma unroll
    for (int m = P - l; m >= 0; --m) {
      // the row's coefficients are loaded back to back first (one latency per row, not per FMA)
      double cr[P + 1];
#pragma unroll
      for (int n = 0; n <= P - l - m; ++n) cr[n] = coef(basis_index(P, l, m, n));
      double pz = cr[P - l - m];
#pragma unroll
      for (int n = P - l - m - 1; n >= 0; --n) pz = fma(pz, z, cr[n]);
      py = (m == P - l) ? pz : fma(py, y, pz);
    }
    px = (l == P) ? py : fma(px, x, py);
  }
  return px;
}

// Loads coefficients i0 .. i0+n-1 into cr[]: 16-byte pair loads at even indices (one shared-memory
// wavefront per two coefficients when every lane reads the same address), if the reader offers them.
template <int P, typename Coef>
__device__ __forceinline__ void load_row(const Coef& coef, int i0, int n, double* cr) {
  if constexpr (Coef::kPairs) {
    int k = 0;
    if (i0 & 1) { cr[0] = coef(i0); k = 1; }
#pragma unroll
    for (; k + 1 < n; k += 2) {
      const double2 v = coef.pair(i0 + k);
      cr[k] = v.x;
      cr[k + 1] = v.y;
    }
    if (k < n) cr[k] = coef(i0 + k);
  } else {
#pragma unroll
    for (int k = 0; k < n; ++k) cr[k] = coef(i0 + k);
  }
}

// Two points per call: every coefficient load feeds two FMAs; each row's loads are issued back to back.
template <int P, typename Coef>
__device__ __forceinline__ void horner3x2(const Coef& coef, double x0, double y0, double z0, double x1, double y1,
                                          double z1, double& v0, double& v1) {
  double px0 = 0.0, px1 = 0.0;
#pragma unroll
  for (int l = P; l >= 0; --l) {
    double py0 = 0.0, py1 = 0.0;
#pragma unroll
    for (int m = P - l; m >= 0; --m) {
      double cr[P + 1];
      load_row<P>(coef, basis_index(P, l, m, 0), P - l - m + 1, cr);
      double pz0 = cr[P - l - m], pz1 = cr[P - l - m];
#pragma unroll
      for (int n = P - l - m - 1; n >= 0; --n) {
        pz0 = fma(pz0, z0, cr[n]);
        pz1 = fma(pz1, z1, cr[n]);
      }
      py0 = (m == P - l) ? pz0 : fma(py0, y0, pz0);
      py1 = (m == P - l) ? pz1 : fma(py1, y1, pz1);
    }
    px0 = (l == P) ? py0 : fma(px0, x0, py0);
    px1 = (l == P) ? py1 : fma(px1, x1, py1);
  }
  v0 = px0;
  v1 = px1;
}

// Four points per call: every coefficient load feeds four FMAs, four independent chains.
template <int P, typename Coef>
__device__ __forceinline__ void horner3x4(const Coef& coef, const double* x, const double* y, const double* z,
                                          double* v) {
  double px[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int l = P; l >= 0; --l) {
    double py[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int m = P - l; m >= 0; --m) {
      double cr[P + 1];
      load_row<P>(coef, basis_index(P, l, m, 0), P - l - m + 1, cr);
      double pz[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) pz[k] = cr[P - l - m];
#pragma unroll
      for (int n = P - l - m - 1; n >= 0; --n) {
#pragma unroll
        for (int k = 0; k < 4; ++k) pz[k] = fma(pz[k], z[k], cr[n]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) py[k] = (m == P - l) ? pz[k] : fma(py[k], y[k], pz[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) px[k] = (l == P) ? py[k] : fma(px[k], x[k], py[k]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = px[k];
}

// Shared-memory coefficient reader (plain loads: the callers' point loops contain a __syncthreads, so the
// compiler cannot hoist the 𝓛 coefficient loads out of them, but it may schedule them freely inside a
// Horner evaluation to overlap the row chains).
struct SmemCoef {
  static constexpr bool kPairs = true;  // coefficient 0 must be 16-byte aligned
  const double* p;
  __device__ __forceinline__ explicit SmemCoef(const double* q) : p(q) {}
  __device__ __forceinline__ double operator()(int i) const { return p[i]; }
  __device__ __forceinline__ double2 pair(int i) const {  // i even
    return *reinterpret_cast<const double2*>(p + i);
  }
};

// Volatile variant for point loops WITHOUT a barrier (the compiler must not hoist 𝓛 loads out of them).
struct SmemCoefVolatile {
  static constexpr bool kPairs = false;
  uint32_t base;  // shared-window address of coefficient 0
  __device__ __forceinline__ explicit SmemCoefVolatile(const double* p)
      : base((uint32_t)__cvta_generic_to_shared(p)) {}
  __device__ __forceinline__ double operator()(int i) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * (uint32_t)i));
    return v;
  }
};

// node frame: centre (2i+1)·2^-(d+1), scale 2^(d+1) (FMT_New_Octant; local map P:299)
struct Frame {
  double cx, cy, cz, scale;
};

// local coordinate (u - c)·s with one fused operation: s is a power of two and c·s = 2i+1 is an exact
// integer, so fma(u, s, -c·s) = RN((u - c)·s) = RN(u - c)·s — bit-identical to the two-step map of
// reading G18, at one FP64 instruction instead of two
__device__ __forceinline__ double to_local(double u, double c, double s) { return __fma_rn(u, s, -(c * s)); }
__device__ __forceinline__ Frame node_frame(int4 c) {
  const double h = ldexp(1.0, -(c.w + 1));
  Frame f;
  f.scale = ldexp(1.0, c.w + 1);
  f.cx = (2.0 * c.x + 1.0) * h;
  f.cy = (2.0 * c.y + 1.0) * h;
  f.cz = (2.0 * c.z + 1.0) * h;
  return f;
}

}  // namespace fmi
