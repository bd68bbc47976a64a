// eval.cu — K7: interpolant evaluation over Morton-sorted queries (DESIGN.md §3 K7).
//
// f(r) = Λ(r)·F_p (§2), accumulated over the nodes on the query's root-to-deepest-existing-node
// path ("only downward recursion to accumulate local polynomial representation of the residual",
// P:367-368 §4; reading G11).  Queries are processed in Morton order so that neighbouring threads walk
// the same nodes (coefficient loads are warp-broadcast, L1-resident); results are scattered back to the
// caller's order.  A query outside the root cube gets the root polynomial only.
#include "horner.cuh"

namespace fmi {

namespace {

__device__ __forceinline__ double to_unit_e(double x, double lo, double w, bool unit) {
  return unit ? x : __ddiv_rn(__dsub_rn(x, lo), w);
}

template <int P>
__global__ void __launch_bounds__(256) k_eval(const double* __restrict__ q, const uint64_t* __restrict__ keys,
                                              const uint32_t* __restrict__ idx, int64_t M, double lo0, double lo1,
                                              double lo2, double w, bool unit, int Dk, NodeTable nt,
                                              double* __restrict__ out) {
  constexpr int L = rank3(P);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int64_t qi = idx ? (int64_t)idx[i] : i;
  const double ux = to_unit_e(q[3 * qi + 0], lo0, w, unit);
  const double uy = to_unit_e(q[3 * qi + 1], lo1, w, unit);
  const double uz = to_unit_e(q[3 * qi + 2], lo2, w, unit);
  const bool inside = ux >= 0.0 && ux <= 1.0 && uy >= 0.0 && uy <= 1.0 && uz >= 0.0 && uz <= 1.0;
  int64_t node = 0;
  int4 cell = make_int4(0, 0, 0, 0);
  double acc = 0.0;
  const uint64_t key = keys ? keys[i] : 0;
  for (int level = 0;; ++level) {
    const Frame fr = node_frame(cell);
    const double x = __dmul_rn(__dsub_rn(ux, fr.cx), fr.scale);
    const double y = __dmul_rn(__dsub_rn(uy, fr.cy), fr.scale);
    const double z = __dmul_rn(__dsub_rn(uz, fr.cz), fr.scale);
    const double* a = nt.coef + node * L;
    auto coef = [&](int k) { return __ldg(a + k); };
    acc += horner3<P>(coef, x, y, z);
    if (!inside || level >= Dk) break;
    const int o = (int)((key >> (3 * (Dk - level - 1))) & 7ull);
    const int32_t ch = __ldg(nt.child + node * 8 + o);
    if (ch < 0) break;
    node = ch;
    cell = nt.cell[node];
  }
  out[qi] = acc;
}

}  // namespace

template <int P>
void eval_sorted(const double* q, const uint64_t* keys, const uint32_t* idx, int64_t M, const double lo[3],
                 double width, bool unit, int Dk, const NodeTable& nt, double* out, cudaStream_t s) {
  if (M <= 0) return;
  FMI_LAUNCH(KID_EVAL, s, k_eval<P>, (unsigned)((M + 255) / 256), 256, 0, q, keys, idx, M, lo[0], lo[1], lo[2],
             width, unit, Dk, nt, out);
}

#define FMI_INST(P)                                                                                            \
  template void eval_sorted<P>(const double*, const uint64_t*, const uint32_t*, int64_t, const double*, double, \
                               bool, int, const NodeTable&, double*, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
