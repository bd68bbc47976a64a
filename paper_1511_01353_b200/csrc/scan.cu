// scan.cu — device exclusive prefix sums (int64) used for radix-sort offsets, chunk lists and node
// compaction.  Three phases: per-tile sums, one-CTA scan of the tile sums, per-tile scan + offset.
// Deterministic (no atomics).
#include "fmi_internal.cuh"

namespace fmi {

namespace {

constexpr int SC_THREADS = 512;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;  // 4096

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix, *total = block sum
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
  __shared__ int64_t wsum[SC_THREADS / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t inc = warp_incl_scan(v);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < SC_THREADS / 32) ? wsum[lane] : 0;
    int64_t wi = warp_incl_scan(w);
    if (lane < SC_THREADS / 32) wsum[lane] = wi - w;
    if (lane == SC_THREADS / 32 - 1) wsum[SC_THREADS / 32] = wi;  // slot after the warps: total
  }
  __syncthreads();
  int64_t res = inc - v + wsum[warp];
  *total = wsum[SC_THREADS / 32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(SC_THREADS) k_tile_sums(const int64_t* __restrict__ in, int64_t n,
                                                          int64_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * SC_TILE;
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    int64_t idx = base + (int64_t)i * SC_THREADS + threadIdx.x;
    if (idx < n) acc += in[idx];
  }
  int64_t tot;
  (void)block_excl_scan(acc, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// one CTA: exclusive scan of nb tile sums in place; writes grand total
__global__ void __launch_bounds__(SC_THREADS) k_scan_sums(int64_t* sums, int64_t nb, int64_t* total) {
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += SC_THREADS) {
    int64_t idx = base + threadIdx.x;
    int64_t v = idx < nb ? sums[idx] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan(v, &tot);
    if (idx < nb) sums[idx] = ex + carry;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_tiles(const int64_t* in, int64_t* out,
                                                           int64_t n, const int64_t* __restrict__ sums) {
  // each thread owns SC_ITEMS consecutive items (blocked arrangement via smem transpose for coalescing)
  __shared__ int64_t tile[SC_TILE];
  const int64_t base = (int64_t)blockIdx.x * SC_TILE;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    int64_t idx = base + (int64_t)i * SC_THREADS + threadIdx.x;
    tile[i * SC_THREADS + threadIdx.x] = idx < n ? in[idx] : 0;
  }
  __syncthreads();
  int64_t loc[SC_ITEMS];
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { loc[i] = tile[threadIdx.x * SC_ITEMS + i]; acc += loc[i]; }
  int64_t tot;
  int64_t ex = block_excl_scan(acc, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { tile[threadIdx.x * SC_ITEMS + i] = ex; ex += loc[i]; }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    int64_t idx = base + (int64_t)i * SC_THREADS + threadIdx.x;
    if (idx < n) out[idx] = tile[i * SC_THREADS + threadIdx.x];
  }
}

}  // namespace

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s) {
  if (n <= 0) {
    if (total) FMI_CK(cudaMemsetAsync(total, 0, sizeof(int64_t), s));
    return;
  }
  int64_t nb = (n + SC_TILE - 1) / SC_TILE;
  DBuf<int64_t> sums(nb, s);
  FMI_LAUNCH(KID_SCAN, s, k_tile_sums, (unsigned)nb, SC_THREADS, 0, in, n, sums.p);
  FMI_LAUNCH(KID_SCAN, s, k_scan_sums, 1, SC_THREADS, 0, sums.p, nb, total);
  FMI_LAUNCH(KID_SCAN, s, k_scan_tiles, (unsigned)nb, SC_THREADS, 0, in, out, n, sums.p);
}

}  // namespace fmi
