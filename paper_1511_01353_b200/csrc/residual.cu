// residual.cu — K6: residual update and per-octant residual energy (DESIGN.md §3 K6).
//
// PAPER.md Algorithm 2 last line: f <- f - Λ·P_F over the node's points (here r <- r - Σ a_α u^α,
// Horner, 𝓛 FMA per point), then Algorithm 1 line 7: E_RMS of each octant block needs Σ r² over
// the block.  Work items are chunks of one octant block (segment node*8+o), so each CTA reduces one
// sum; segment sums are reduced in chunk order (deterministic).
#include "horner.cuh"

namespace fmi {

namespace {

constexpr int K6_THREADS = 256;

template <int P>
__global__ void __launch_bounds__(K6_THREADS)
    k_residual(const double* __restrict__ ux, const double* __restrict__ uy, const double* __restrict__ uz,
               double* __restrict__ r, NodeTable nt, int64_t first, const double* __restrict__ coefs,
               const Chunk* __restrict__ chunks, const int64_t* __restrict__ nchunks,
               const uint8_t* __restrict__ skip, double* __restrict__ seg_part) {
  constexpr int L = rank3(P);
  __shared__ double sa[L];
  __shared__ double red[K6_THREADS / 32];
  const int64_t cidx = blockIdx.x;
  if (cidx >= *nchunks) return;
  const Chunk ck = chunks[cidx];
  const int64_t lnode = ck.owner >> 3;
  const int64_t node = first + lnode;
  if (skip && skip[lnode]) return;  // refinement pass: node unchanged, keep its segment sums
  for (int i = threadIdx.x; i < L; i += K6_THREADS) sa[i] = coefs[lnode * L + i];
  const Frame fr = node_frame(nt.cell[node]);
  __syncthreads();
  const SmemCoef coef(sa);
  double acc = 0.0;
  const int64_t n = ck.end - ck.start;
  const int64_t half = (n + 1) / 2;  // thread t handles points t and t + half (two independent chains)
  for (int64_t k = threadIdx.x; k < half; k += K6_THREADS) {
    const int64_t i0 = ck.start + k;
    const int64_t i1 = i0 + half;
    const bool has1 = i1 < ck.end;
    const int64_t j1 = has1 ? i1 : i0;
    const double x0 = __dmul_rn(__dsub_rn(ux[i0], fr.cx), fr.scale);
    const double y0 = __dmul_rn(__dsub_rn(uy[i0], fr.cy), fr.scale);
    const double z0 = __dmul_rn(__dsub_rn(uz[i0], fr.cz), fr.scale);
    const double x1 = __dmul_rn(__dsub_rn(ux[j1], fr.cx), fr.scale);
    const double y1 = __dmul_rn(__dsub_rn(uy[j1], fr.cy), fr.scale);
    const double z1 = __dmul_rn(__dsub_rn(uz[j1], fr.cz), fr.scale);
    double v0, v1;
    horner3x2<P>(coef, x0, y0, z0, x1, y1, z1, v0, v1);
    const double r0 = r[i0] - v0;
    r[i0] = r0;
    acc = fma(r0, r0, acc);
    if (has1) {
      const double r1 = r[i1] - v1;
      r[i1] = r1;
      acc = fma(r1, r1, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < K6_THREADS / 32; ++w) s += red[w];
    seg_part[cidx] = s;
  }
}

__global__ void k_residual_reduce(const double* __restrict__ seg_part, const int64_t* __restrict__ chunk_begin,
                                  const int64_t* __restrict__ nchunks, int64_t nseg, NodeTable nt, int64_t first,
                                  const uint8_t* __restrict__ skip) {
  const int64_t sgi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sgi >= nseg) return;
  if (skip && skip[sgi >> 3]) return;
  const int64_t c0 = chunk_begin[sgi];
  const int64_t c1 = sgi + 1 < nseg ? chunk_begin[sgi + 1] : *nchunks;
  double s = 0.0;
  for (int64_t c = c0; c < c1; ++c) s += seg_part[c];
  nt.child_ss[first * 8 + sgi] = s;
}

}  // namespace

template <int P>
void level_residual(const LevelCtx& c, const double* coefs, const uint8_t* skip, const Chunk* chunks,
                    const int64_t* nchunks_dev, int64_t max_chunks, const int64_t* chunk_begin, double* seg_part,
                    cudaStream_t s) {
  if (max_chunks > 0)
    FMI_LAUNCH(KID_RESIDUAL, s, k_residual<P>, (unsigned)max_chunks, K6_THREADS, 0, c.ux, c.uy, c.uz, c.r, c.nt,
               c.first, coefs, chunks, nchunks_dev, skip, seg_part);
  const int64_t nseg = c.count * 8;
  FMI_LAUNCH(KID_RESIDUAL_REDUCE, s, k_residual_reduce, (unsigned)((nseg + 255) / 256), 256, 0, seg_part, chunk_begin,
             nchunks_dev, nseg, c.nt, c.first, skip);
}

#define FMI_INST(P)                                                                                         \
  template void level_residual<P>(const LevelCtx&, const double*, const uint8_t*, const Chunk*, const int64_t*,  \
                                  int64_t, const int64_t*, double*, cudaStream_t);
FMI_INST(0) FMI_INST(1) FMI_INST(2) FMI_INST(3) FMI_INST(4) FMI_INST(5)
FMI_INST(6) FMI_INST(7) FMI_INST(8) FMI_INST(9) FMI_INST(10)
#undef FMI_INST

}  // namespace fmi
