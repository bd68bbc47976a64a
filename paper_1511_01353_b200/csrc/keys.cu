// keys.cu — K1 Morton keys, K2 LSD radix sort of (key, index) pairs and the SoA gather.
//
// A recursive stable octant partition (FMT_Ordered_by_Octant, Alg. 1) applied level by
// level is exactly a stable sort by the interleaved cell key, so one global sort makes every octree
// node a contiguous point range (DESIGN.md §3 K1/K2).
//
// Octant digit of level t (1..D): o = bx + 2·by + 4·bz (x fastest), b* = bit (D-t) of
// q* = min(floor(u*·2^D), 2^D - 1).  u* is the root-cube unit coordinate; u* >= split plane <=> the
// bit is set (tie -> upper side) because u·2^D is an exact power-of-two scaling (G7, G18).
#include <mutex>
#include <algorithm>

#include "fmi_internal.cuh"

namespace fmi {

namespace {

// ------------------------------------------------------------------------------------------------
// bounding box + finiteness check (root frame, reading G6)
// ------------------------------------------------------------------------------------------------
constexpr int BB_THREADS = 256;

__global__ void __launch_bounds__(BB_THREADS) k_bbox_partial(const double* __restrict__ pts, int64_t n,
                                                             const double* __restrict__ f,
                                                             double* __restrict__ part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  double bad = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * BB_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * BB_THREADS) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double v = pts[3 * i + a];
      if (!isfinite(v)) bad = 1.0;
      mn[a] = fmin(mn[a], v);
      mx[a] = fmax(mx[a], v);
    }
    if (f && !isfinite(f[i])) bad = 1.0;
  }
  __shared__ double sm[7][BB_THREADS];
#pragma unroll
  for (int a = 0; a < 3; ++a) { sm[a][threadIdx.x] = mn[a]; sm[3 + a][threadIdx.x] = mx[a]; }
  sm[6][threadIdx.x] = bad;
  __syncthreads();
  for (int w = BB_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sm[a][threadIdx.x] = fmin(sm[a][threadIdx.x], sm[a][threadIdx.x + w]);
        sm[3 + a][threadIdx.x] = fmax(sm[3 + a][threadIdx.x], sm[3 + a][threadIdx.x + w]);
      }
      sm[6][threadIdx.x] = fmax(sm[6][threadIdx.x], sm[6][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 7) part[blockIdx.x * 8 + threadIdx.x] = sm[threadIdx.x][0];
}

__global__ void __launch_bounds__(BB_THREADS) k_bbox_final(const double* __restrict__ part, int nb,
                                                           double* __restrict__ out) {
  double r[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
  for (int b = threadIdx.x; b < nb; b += BB_THREADS) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      r[a] = fmin(r[a], part[b * 8 + a]);
      r[3 + a] = fmax(r[3 + a], part[b * 8 + 3 + a]);
    }
    r[6] = fmax(r[6], part[b * 8 + 6]);
  }
  __shared__ double sm[7][BB_THREADS];
#pragma unroll
  for (int a = 0; a < 7; ++a) sm[a][threadIdx.x] = r[a];
  __syncthreads();
  for (int w = BB_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sm[a][threadIdx.x] = fmin(sm[a][threadIdx.x], sm[a][threadIdx.x + w]);
        sm[3 + a][threadIdx.x] = fmax(sm[3 + a][threadIdx.x], sm[3 + a][threadIdx.x + w]);
      }
      sm[6][threadIdx.x] = fmax(sm[6][threadIdx.x], sm[6][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 7) out[threadIdx.x] = sm[threadIdx.x][0];
  if (threadIdx.x == 7) out[7] = 0.0;
}

// ------------------------------------------------------------------------------------------------
// K1 Morton keys
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t spread3(uint64_t v) { return morton_spread3(v); }
__device__ __forceinline__ uint64_t quantize(double u, int D) { return morton_quantize(u, D); }

// root-cube unit coordinate: (x - lo) / W, one IEEE subtraction and one division (same as the
// oracle's to_unit); identity for the unit cube.
__device__ __forceinline__ double to_unit(double x, double lo, double w, bool unit) {
  return unit ? x : __ddiv_rn(__dsub_rn(x, lo), w);
}

// packed != nullptr (fit points): also write (u_x, u_y, u_z, f) as one 32-byte record, so that the
// Morton-order gather reads ONE aligned sector per point instead of scattered pieces of pts and f.
// keys32 != nullptr: the 32-bit sort key (the key bits from bit_lo up) instead of the 64-bit key.
__global__ void __launch_bounds__(256) k_keys(const double* __restrict__ pts, int64_t n, double lo0, double lo1,
                                              double lo2, double w, bool unit, int D, uint64_t* __restrict__ keys,
                                              uint32_t* __restrict__ idx, const double* __restrict__ f,
                                              double4* __restrict__ packed, uint32_t* __restrict__ keys32,
                                              int bit_lo) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ux = to_unit(pts[3 * i + 0], lo0, w, unit);
  double uy = to_unit(pts[3 * i + 1], lo1, w, unit);
  double uz = to_unit(pts[3 * i + 2], lo2, w, unit);
  const uint64_t k = morton_key(ux, uy, uz, D);
  if (keys32) keys32[i] = (uint32_t)(k >> bit_lo);
  else keys[i] = k;
  idx[i] = (uint32_t)i;
  if (packed) packed[i] = make_double4(ux, uy, uz, f ? f[i] : 0.0);
}

// ------------------------------------------------------------------------------------------------
// K2 LSD radix sort, 8-bit digits, stable.  Upsweep histogram -> exclusive scan (digit-major) ->
// downsweep with warp-level stable ranking (match.any) and per-warp digit counters.
// ------------------------------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 12;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 3072 (12 items/thread: 64 registers, 4 CTAs/SM)
constexpr int RS_WARP_ITEMS = RS_TILE / RS_WARPS; // 384 (in-warp ranks fit 16 bits)
template <typename KT>
constexpr size_t scatter_smem() { return (size_t)RS_TILE * (sizeof(KT) + sizeof(uint32_t)); }

// KT = uint64_t (full Morton keys) or uint32_t (the sorted key bits only: less traffic per pass)
// Segmented passes (bucketed sort, seg != nullptr): every tile lies inside one segment (a top-digit
// bucket padded to whole tiles) and the counts are laid out segment-major, then digit, then tile, so that
// one exclusive scan gives each (tile, digit) its offset inside its own segment: the pass sorts every
// segment by the digit and keeps the segments in place.
struct SegTile {
  int32_t t0, nt;   // first tile and tile count of the tile's segment
  int64_t shift;    // padded -> dense position offset of the segment (the last pass compacts)
};
constexpr uint32_t kPadVal = 0xffffffffu;  // value of a padding slot (its key has every bit set: sorts last)

__device__ __forceinline__ int64_t count_index(const SegTile* seg, int64_t blk, int64_t nblk, int d, SegTile& sg) {
  if (!seg) return (int64_t)d * nblk + blk;
  sg = seg[blk];
  return (int64_t)sg.t0 * 256 + (int64_t)d * sg.nt + (blk - sg.t0);
}

template <typename KT>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const KT* __restrict__ keys, int64_t n, int shift,
                                                        int64_t nblk, int64_t* __restrict__ counts,
                                                        const SegTile* __restrict__ seg) {
  __shared__ int hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  // all 16 loads in flight before the first shared-memory atomic
  uint32_t d[RS_ITEMS];
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t idx = base + (int64_t)i * RS_THREADS + threadIdx.x;
    d[i] = idx < n ? (uint32_t)((__ldg(keys + idx) >> shift) & 255) : 256u;
  }
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i)
    if (d[i] < 256u) atomicAdd(&hist[d[i]], 1);
  __syncthreads();
  SegTile sg;
  counts[count_index(seg, blockIdx.x, nblk, threadIdx.x, sg)] = hist[threadIdx.x];
}

// Downsweep: stable rank of every item of the tile (per-warp match.any ranking + prefix over warps and
// digits), the tile is rearranged in shared memory in digit order, then written out so that
// consecutive threads store consecutive positions of each digit's global run (coalesced).
template <typename KT>
__global__ void __launch_bounds__(RS_THREADS, 4) k_rs_scatter(const KT* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin, int64_t n, int shift,
                                                           int64_t nblk, const int64_t* __restrict__ offs,
                                                           KT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           const SegTile* __restrict__ seg, int last,
                                                           const double4* __restrict__ rec_in,
                                                           double4* __restrict__ rec_out) {
  __shared__ int whist[RS_WARPS][257];
  __shared__ int tstart[257];           // exclusive prefix of the tile's digit counts
  __shared__ int64_t boff[256];
  extern __shared__ __align__(16) uint64_t rs_dyn[];
  KT* sk = reinterpret_cast<KT*>(rs_dyn);                           // [RS_TILE]
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + RS_TILE);         // [RS_TILE]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < RS_WARPS * 257; t += RS_THREADS) (&whist[0][0])[t] = 0;
  SegTile sg{0, 0, 0};
  boff[threadIdx.x] = offs[count_index(seg, blockIdx.x, nblk, threadIdx.x, sg)];
  __syncthreads();
  const int64_t tbase = (int64_t)blockIdx.x * RS_TILE;
  const int64_t base = tbase + (int64_t)warp * RS_WARP_ITEMS;
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool full = tbase + RS_TILE <= n;  // CTA-uniform: no past-the-end items in this tile
  KT k[RS_ITEMS];  // the values are read again (L2) when the tile is rearranged: fewer registers
  unsigned rank2[RS_ITEMS / 2];  // in-warp ranks (< RS_WARP_ITEMS), two 16-bit halves per register
  // digit of item it (256 = past the end); recomputed from the key instead of held in registers
  auto digit = [&](int it) { return base + it * 32 + lane < n ? (int)((k[it] >> shift) & 255) : 256; };
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    int64_t idx = base + it * 32 + lane;
    bool valid = idx < n;
    k[it] = valid ? kin[idx] : 0;
  }
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const int d = digit(it);
    // peers = lanes with the same digit, from one ballot per digit bit (VOTE on the ALU pipe instead of
    // MATCH on the address-divergence unit, which bounded this kernel); bit 8 marks past-the-end items
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
      peers &= ((d >> b) & 1) ? bb : ~bb;
    }
    if (!full) {
      const unsigned bb = __ballot_sync(0xffffffffu, d >> 8);
      peers &= (d >> 8) ? bb : ~bb;
    }
    int before = whist[warp][d];
    __syncwarp();
    int leader = __ffs(peers) - 1;
    if (lane == leader) whist[warp][d] = before + __popc(peers);
    __syncwarp();
    const unsigned rk = (unsigned)(before + __popc(peers & lt_mask));
    if (it % 2 == 0) rank2[it / 2] = rk;
    else rank2[it / 2] |= rk << 16;
  }
  __syncthreads();
  {  // exclusive prefix over warps for each digit; digit totals of the tile
    int d = threadIdx.x, run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      int t = whist[w][d];
      whist[w][d] = run;
      run += t;
    }
    tstart[d] = run;  // count for now
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 256 digit counts (8 per lane)
    int c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) { c[t] = tstart[lane * 8 + t]; sum += c[t]; }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - sum;
#pragma unroll
    for (int t = 0; t < 8; ++t) { tstart[lane * 8 + t] = run; run += c[t]; }
    if (lane == 31) tstart[256] = run;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const int d = digit(it);
    if (d < 256) {
      const int pos = tstart[d] + whist[warp][d] + (int)((rank2[it / 2] >> (16 * (it % 2))) & 0xffffu);
      sk[pos] = k[it];
      sv[pos] = vin[base + it * 32 + lane];
    }
  }
  __syncthreads();
  const int cnt = tstart[256];
  for (int pos = threadIdx.x; pos < cnt; pos += RS_THREADS) {
    const KT kk = sk[pos];
    const int d = (int)((kk >> shift) & 255);
    const int64_t g = boff[d] + (pos - tstart[d]);
    if (last) {  // last pass of a segmented sort: padding dropped, segments compacted, no keys
      const uint32_t v = sv[pos];
      // rec_out: the records themselves in sorted order (the value is a bucket position of rec_in; the
      // reads stay inside the tile's bucket, L2-resident), so the consumer reads them sequentially
      if (v != kPadVal) {
        if (rec_out) rec_out[g - sg.shift] = rec_in[v];
        else vout[g - sg.shift] = v;
      }
    } else {
      kout[g] = kk;
      vout[g] = sv[pos];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Bucketed keys (the sort's most significant digit first, fused with the record write): the 32-byte
// records (u_x, u_y, u_z, w) are written in top-digit (bucket) order, so that after the remaining
// digits are sorted inside each bucket the Morton-order gather reads records within one bucket at a
// time (L2-resident) instead of across the whole array; the (key, bucket position) pairs go to a
// layout with every bucket padded to whole sort tiles (segmented passes, no top-digit pass).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ int top_digit(uint32_t k, int nb) { return nb > 8 ? (int)(k >> (nb - 8)) : (int)k; }
#ifndef FMI_BK_ITEMS
#define FMI_BK_ITEMS 6
#endif
constexpr int BK_ITEMS = FMI_BK_ITEMS;
constexpr int BK_TILE = RS_THREADS * BK_ITEMS;      // 1536 points per top-digit tile
constexpr int BK_WARP_ITEMS = BK_TILE / RS_WARPS;   // 192
// staged coordinates + values, then the tile's keys and local indices in digit order: 66 KB (3 CTAs/SM)
constexpr size_t BK_SMEM = (size_t)BK_TILE * (4 * sizeof(double) + sizeof(uint32_t) + sizeof(uint16_t));

// the 32-bit sort key (key bits from bit_lo up) of point i and its root-cube unit coordinates (as k_keys)
__device__ __forceinline__ uint32_t sort_key32(const double* __restrict__ pts, int64_t i, double lo0, double lo1,
                                               double lo2, double w, bool unit, int D, int bit_lo, double& ux,
                                               double& uy, double& uz) {
  ux = to_unit(pts[3 * i + 0], lo0, w, unit);
  uy = to_unit(pts[3 * i + 1], lo1, w, unit);
  uz = to_unit(pts[3 * i + 2], lo2, w, unit);
  return (uint32_t)(morton_key(ux, uy, uz, D) >> bit_lo);
}

__global__ void __launch_bounds__(RS_THREADS) k_bk_hist(const double* __restrict__ pts, int64_t n, double lo0,
                                                        double lo1, double lo2, double w, bool unit, int D,
                                                        int bit_lo, int nb, int64_t nblk,
                                                        int64_t* __restrict__ counts) {
  __shared__ int hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * BK_TILE;
  uint32_t d[BK_ITEMS];
#pragma unroll
  for (int i = 0; i < BK_ITEMS; ++i) {
    const int64_t idx = base + (int64_t)i * RS_THREADS + threadIdx.x;
    double ux, uy, uz;
    d[i] = idx < n ? (uint32_t)top_digit(sort_key32(pts, idx, lo0, lo1, lo2, w, unit, D, bit_lo, ux, uy, uz), nb)
                   : 256u;
  }
#pragma unroll
  for (int i = 0; i < BK_ITEMS; ++i)
    if (d[i] < 256u) atomicAdd(&hist[d[i]], 1);
  __syncthreads();
  counts[(int64_t)threadIdx.x * nblk + blockIdx.x] = hist[threadIdx.x];
}

// bucket layout from the scanned top-digit counts (one CTA): bucket d holds cnt[d] points at dense
// start offs[d·nblk]; padded to whole tiles it starts at tile tile0[d]; pshift[d] = padded - dense start
__global__ void __launch_bounds__(256) k_bk_layout(const int64_t* __restrict__ offs, int64_t nblk, int64_t n,
                                                   int32_t* __restrict__ tile0, int64_t* __restrict__ cnt,
                                                   int64_t* __restrict__ pshift) {
  __shared__ int64_t sc[256];
  const int d = threadIdx.x;
  const int64_t s0 = offs[(int64_t)d * nblk];
  const int64_t s1 = d < 255 ? offs[(int64_t)(d + 1) * nblk] : n;
  const int64_t c = s1 - s0;
  const int64_t tiles = (c + RS_TILE - 1) / RS_TILE;
  sc[d] = tiles;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive scan of the tile counts
    const int64_t v = d >= o ? sc[d - o] : 0;
    __syncthreads();
    sc[d] += v;
    __syncthreads();
  }
  const int64_t t0 = sc[d] - tiles;
  tile0[d] = (int32_t)t0;
  if (d == 255) tile0[256] = (int32_t)sc[255];
  cnt[d] = c;
  pshift[d] = t0 * RS_TILE - s0;
}

// per-tile segment table and padding (one CTA per tile of the padded layout, nblk + 256 tiles): slots
// past the end of their bucket's points, and whole tiles past the last bucket, become padding
__global__ void __launch_bounds__(256) k_bk_tiles(const int32_t* __restrict__ tile0, const int64_t* __restrict__ cnt,
                                                  const int64_t* __restrict__ pshift, SegTile* __restrict__ seg,
                                                  uint32_t* __restrict__ kpad, uint32_t* __restrict__ vpad) {
  __shared__ int32_t st0[257];
  for (int t = threadIdx.x; t < 257; t += 256) st0[t] = tile0[t];
  __syncthreads();
  const int64_t blk = blockIdx.x;
  int64_t real_end;  // first padding slot of this tile's segment
  SegTile sg;
  if (blk >= st0[256]) {
    sg = SegTile{(int32_t)blk, 1, 0};
    real_end = blk * RS_TILE;
  } else {
    int lo = 0, hi = 255;  // last bucket b with tile0[b] <= blk (empty buckets share their tile0)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (st0[mid] <= blk) lo = mid; else hi = mid - 1;
    }
    sg = SegTile{st0[lo], st0[lo + 1] - st0[lo], pshift[lo]};
    real_end = (int64_t)st0[lo] * RS_TILE + cnt[lo];
  }
  if (threadIdx.x == 0) seg[blk] = sg;
  for (int e = threadIdx.x; e < RS_TILE; e += 256) {
    const int64_t pos = blk * RS_TILE + e;
    if (pos >= real_end) { kpad[pos] = 0xffffffffu; vpad[pos] = kPadVal; }
  }
}

// the top-digit scatter: every point's record to its bucket position dst (bucket order, input order
// inside a bucket), (key, dst) to the padded layout, orig[dst] = input index (or, rec_idx, the input
// index in the record's fourth slot).  Tile of BK_TILE points: the coordinates (and values) are staged
// in shared memory by coalesced loads, ranked by digit (warp ballots), their keys and local indices
// rearranged in shared memory in digit order, then the records are formed and written so that
// consecutive threads store consecutive positions of each digit's run (coalesced).
__global__ void __launch_bounds__(RS_THREADS, BK_ITEMS <= 4 ? 4 : 3) k_bk_scatter(const double* __restrict__ pts,
                                                              const double* __restrict__ f, int64_t n, double lo0,
                                                              double lo1, double lo2, double w, bool unit, int D,
                                                              int bit_lo, int nb, int64_t nblk,
                                                              const int64_t* __restrict__ offs,
                                                              const int64_t* __restrict__ pshift,
                                                              double4* __restrict__ packed,
                                                              uint32_t* __restrict__ orig, int rec_idx,
                                                              uint32_t* __restrict__ kpad,
                                                              uint32_t* __restrict__ vpad) {
  __shared__ int whist[RS_WARPS][257];
  __shared__ int tstart[257];
  __shared__ int64_t boff[256];
  __shared__ int64_t psh[256];
  extern __shared__ __align__(16) uint64_t bk_dyn[];
  double* sd = reinterpret_cast<double*>(bk_dyn);                       // xyz [3·BK_TILE], f [BK_TILE]
  uint32_t* skey = reinterpret_cast<uint32_t*>(sd + 4 * BK_TILE);       // [BK_TILE] digit order
  uint16_t* sidx = reinterpret_cast<uint16_t*>(skey + BK_TILE);         // [BK_TILE] digit order
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < RS_WARPS * 257; t += RS_THREADS) (&whist[0][0])[t] = 0;
  boff[tid] = offs[(int64_t)tid * nblk + blockIdx.x];
  psh[tid] = pshift[tid];
  const int64_t tb = (int64_t)blockIdx.x * BK_TILE;
  const int cnt = (int)min((int64_t)BK_TILE, n - tb);
  // (1) coalesced staging of the tile's coordinates and values: 16-byte cp.async (all of a thread's
  // copies in flight at once) for full tiles of aligned arrays, element copies otherwise
  const bool vec = cnt == BK_TILE && ((reinterpret_cast<uintptr_t>(pts) | reinterpret_cast<uintptr_t>(f)) & 15) == 0;
  if (vec) {
    const double* src = pts + 3 * tb;
#pragma unroll
    for (int e = tid; e < 3 * BK_TILE / 2; e += RS_THREADS)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sd + 2 * e)),
                   "l"(src + 2 * e) : "memory");
    if (f) {
#pragma unroll
      for (int e = tid; e < BK_TILE / 2; e += RS_THREADS)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sd + 3 * BK_TILE + 2 * e)), "l"(f + tb + 2 * e)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  } else {
    for (int e = tid; e < 3 * cnt; e += RS_THREADS) sd[e] = pts[3 * tb + e];
    if (f)
      for (int e = tid; e < cnt; e += RS_THREADS) sd[3 * BK_TILE + e] = f[tb + e];
  }
  __syncthreads();
  // (2) keys, digits and in-warp ranks
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool full = cnt == BK_TILE;
  uint32_t k[BK_ITEMS];
  unsigned rank2[(BK_ITEMS + 1) / 2];
  auto digit = [&](int it) {
    return warp * BK_WARP_ITEMS + it * 32 + lane < cnt ? top_digit(k[it], nb) : 256;
  };
#pragma unroll
  for (int it = 0; it < BK_ITEMS; ++it) {
    const int li = warp * BK_WARP_ITEMS + it * 32 + lane;
    k[it] = 0;
    if (li < cnt) {
      const double ux = to_unit(sd[3 * li + 0], lo0, w, unit);
      const double uy = to_unit(sd[3 * li + 1], lo1, w, unit);
      const double uz = to_unit(sd[3 * li + 2], lo2, w, unit);
      k[it] = (uint32_t)(morton_key(ux, uy, uz, D) >> bit_lo);
    }
  }
#pragma unroll
  for (int it = 0; it < BK_ITEMS; ++it) {
    const int d = digit(it);
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
      peers &= ((d >> b) & 1) ? bb : ~bb;
    }
    if (!full) {
      const unsigned bb = __ballot_sync(0xffffffffu, d >> 8);
      peers &= (d >> 8) ? bb : ~bb;
    }
    const int before = whist[warp][d];
    __syncwarp();
    const int leader = __ffs(peers) - 1;
    if (lane == leader) whist[warp][d] = before + __popc(peers);
    __syncwarp();
    const unsigned rk = (unsigned)(before + __popc(peers & lt_mask));
    if (it % 2 == 0) rank2[it / 2] = rk;
    else rank2[it / 2] |= rk << 16;
  }
  __syncthreads();
  {  // exclusive prefix over warps for each digit; digit totals of the tile
    const int d = tid;
    int run = 0;
#pragma unroll
    for (int w2 = 0; w2 < RS_WARPS; ++w2) {
      const int t = whist[w2][d];
      whist[w2][d] = run;
      run += t;
    }
    tstart[d] = run;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 256 digit counts (8 per lane)
    int c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) { c[t] = tstart[lane * 8 + t]; sum += c[t]; }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - sum;
#pragma unroll
    for (int t = 0; t < 8; ++t) { tstart[lane * 8 + t] = run; run += c[t]; }
  }
  __syncthreads();
  // (3) keys and local indices in digit order
#pragma unroll
  for (int it = 0; it < BK_ITEMS; ++it) {
    const int d = digit(it);
    if (d < 256) {
      const int pos = tstart[d] + whist[warp][d] + (int)((rank2[it / 2] >> (16 * (it % 2))) & 0xffffu);
      skey[pos] = k[it];
      sidx[pos] = (uint16_t)(warp * BK_WARP_ITEMS + it * 32 + lane);
    }
  }
  __syncthreads();
  // (4) coalesced write-out: position pos of the tile goes to its digit's run
  for (int pos = tid; pos < cnt; pos += RS_THREADS) {
    const uint32_t kk = skey[pos];
    const int li = sidx[pos];
    const int d = top_digit(kk, nb);
    const int64_t dst = boff[d] + (pos - tstart[d]);
    const double wv = f ? sd[3 * BK_TILE + li] : (rec_idx ? (double)(tb + li) : 0.0);
    packed[dst] = make_double4(to_unit(sd[3 * li + 0], lo0, w, unit), to_unit(sd[3 * li + 1], lo1, w, unit),
                               to_unit(sd[3 * li + 2], lo2, w, unit), wv);
    if (orig) orig[dst] = (uint32_t)(tb + li);
    kpad[dst + psh[d]] = kk;
    vpad[dst + psh[d]] = (uint32_t)dst;
  }
}

__global__ void k_iota32(uint32_t* __restrict__ v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

// ------------------------------------------------------------------------------------------------
// SoA gather in Morton order
// ------------------------------------------------------------------------------------------------
// orig (bucketed keys, optional): perm[i] is a bucket position, the input index is orig[perm[i]]; with
// compose, perm[i] is replaced by the input index once read (the tree keeps input indices)
__global__ void __launch_bounds__(256) k_gather(const double4* __restrict__ packed, uint32_t* __restrict__ perm,
                                                int64_t n, double* __restrict__ ux, double* __restrict__ uy,
                                                double* __restrict__ uz, double* __restrict__ r,
                                                uint64_t* __restrict__ keys, int D, const uint32_t* __restrict__ orig,
                                                int compose) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  const double2* p = reinterpret_cast<const double2*>(packed + j);  // one 32-byte sector
  const double2 a = __ldg(p), b = __ldg(p + 1);
  if (orig && compose) perm[i] = orig[j];
  ux[i] = a.x;
  uy[i] = a.y;
  uz[i] = b.x;
  r[i] = b.y;
  if (keys) keys[i] = morton_key(a.x, a.y, b.x, D);
}

// variant for values uploaded after the keys were built (fmi_build with page-locked host f): the value
// comes from f[input index]; a non-finite value raises *bad
__global__ void __launch_bounds__(256) k_gather_f(const double4* __restrict__ packed, uint32_t* __restrict__ perm,
                                                  const double* __restrict__ f, int64_t n, double* __restrict__ ux,
                                                  double* __restrict__ uy, double* __restrict__ uz,
                                                  double* __restrict__ r, int* __restrict__ bad,
                                                  uint64_t* __restrict__ keys, int D,
                                                  const uint32_t* __restrict__ orig, int compose) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  const uint32_t o = orig ? orig[j] : j;
  const double2* p = reinterpret_cast<const double2*>(packed + j);
  const double2 a = __ldg(p), b = __ldg(p + 1);
  const double v = __ldg(f + o);
  if (orig && compose) perm[i] = o;
  ux[i] = a.x;
  uy[i] = a.y;
  uz[i] = b.x;
  r[i] = v;
  if (keys) keys[i] = morton_key(a.x, a.y, b.x, D);
  if (!isfinite(v)) *bad = 1;
}

// sharded build helpers ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cell_label(double ux, double uy, double uz, int s) {
  return (uint32_t)(spread3(quantize(ux, s)) | (spread3(quantize(uy, s)) << 1) | (spread3(quantize(uz, s)) << 2));
}

__global__ void k_cell_counts(const double* __restrict__ pts, int64_t n, double lo0, double lo1, double lo2, double w,
                              bool unit, int s, unsigned long long* __restrict__ counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cell_label(to_unit(pts[3 * i], lo0, w, unit), to_unit(pts[3 * i + 1], lo1, w, unit),
                                to_unit(pts[3 * i + 2], lo2, w, unit), s);
  atomicAdd(&counts[c], 1ull);  // integer counts: order-independent
}

__global__ void k_dest(const double* __restrict__ pts, int64_t n, double lo0, double lo1, double lo2, double w,
                       bool unit, int s, const int32_t* __restrict__ owner, uint64_t* __restrict__ key,
                       uint32_t* __restrict__ idx, unsigned long long* __restrict__ counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cell_label(to_unit(pts[3 * i], lo0, w, unit), to_unit(pts[3 * i + 1], lo1, w, unit),
                                to_unit(pts[3 * i + 2], lo2, w, unit), s);
  const int r = owner[c];
  key[i] = (uint64_t)r;
  idx[i] = (uint32_t)i;
  atomicAdd(&counts[r], 1ull);
}

__global__ void k_part_gather(const double* __restrict__ pts, const double* __restrict__ f,
                              const uint32_t* __restrict__ idx, int64_t n, double* __restrict__ pts_out,
                              double* __restrict__ f_out, int64_t* __restrict__ idx_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = idx[i];
  pts_out[3 * i] = pts[3 * j];
  pts_out[3 * i + 1] = pts[3 * j + 1];
  pts_out[3 * i + 2] = pts[3 * j + 2];
  if (f_out) f_out[i] = f[j];
  if (idx_out) idx_out[i] = j;
}

__global__ void k_scatter_vals(const double* __restrict__ vals, const int64_t* __restrict__ idx, int64_t m,
                               double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[idx[i]] = vals[i];
}

}  // namespace

void cell_counts(const double* pts, int64_t n, const double lo[3], double width, bool unit, int s, int64_t* counts,
                 cudaStream_t st) {
  FMI_CK(cudaMemsetAsync(counts, 0, sizeof(int64_t) << (3 * s), st));
  if (n <= 0) return;
  FMI_LAUNCH(KID_MISC, st, k_cell_counts, (unsigned)((n + 255) / 256), 256, 0, pts, n, lo[0], lo[1], lo[2], width,
             unit, s, reinterpret_cast<unsigned long long*>(counts));
}

void partition_points(const double* pts, const double* f, int64_t n, const double lo[3], double width, bool unit,
                      int s, const int32_t* owner, int world, double* pts_out, double* f_out, int64_t* idx_out,
                      int64_t* send_counts, cudaStream_t st) {
  FMI_CK(cudaMemsetAsync(send_counts, 0, sizeof(int64_t) * world, st));
  if (n <= 0) return;
  DBuf<uint64_t> key(n, st), ktmp(n, st);
  DBuf<uint32_t> idx(n, st), itmp(n, st);
  FMI_LAUNCH(KID_MISC, st, k_dest, (unsigned)((n + 255) / 256), 256, 0, pts, n, lo[0], lo[1], lo[2], width, unit, s,
             owner, key.p, idx.p, reinterpret_cast<unsigned long long*>(send_counts));
  int bits = 1;
  while ((1 << bits) < world) ++bits;
  radix_sort_pairs(key.p, idx.p, ktmp.p, itmp.p, n, bits, st);  // stable: input order within a shard
  FMI_LAUNCH(KID_MISC, st, k_part_gather, (unsigned)((n + 255) / 256), 256, 0, pts, f, idx.p, n, pts_out, f_out,
             idx_out);
}

void scatter_values(const double* vals, const int64_t* idx, int64_t m, double* out, cudaStream_t st) {
  if (m <= 0) return;
  FMI_LAUNCH(KID_MISC, st, k_scatter_vals, (unsigned)((m + 255) / 256), 256, 0, vals, idx, m, out);
}

void bbox_and_check(const double* pts, int64_t n, double* out8, const double* f, cudaStream_t s) {
  int nb = (int)std::min<int64_t>((n + BB_THREADS - 1) / BB_THREADS, 1184);
  if (nb < 1) nb = 1;
  DBuf<double> part((size_t)nb * 8, s);
  FMI_LAUNCH(KID_MISC, s, k_bbox_partial, nb, BB_THREADS, 0, pts, n, f, part.p);
  FMI_LAUNCH(KID_MISC, s, k_bbox_final, 1, BB_THREADS, 0, part.p, nb, out8);
}

void morton_keys(const double* pts, int64_t n, const double lo[3], double width, bool unit, int D, uint64_t* keys,
                 uint32_t* idx, cudaStream_t s, const double* f, double4* packed, uint32_t* keys32, int bit_lo) {
  if (n <= 0) return;
  unsigned grid = (unsigned)((n + 255) / 256);
  // algorithmic bytes: coordinates read (24), key (8, or 4 for a sort key) + index (4) written, record
  // written (32), value read (8)
  prof_units(KID_KEYS, n * (24 + (keys32 ? 4 : 8) + 4 + (packed ? 32 : 0) + (f ? 8 : 0)));
  FMI_LAUNCH(KID_KEYS, s, k_keys, grid, 256, 0, pts, n, lo[0], lo[1], lo[2], width, unit, D, keys, idx, f, packed,
             keys32, bit_lo);
}

template <typename KT>
void radix_sort_impl(KT*& keys, uint32_t*& vals, KT*& keys_tmp, uint32_t*& vals_tmp, int64_t n, int nbits,
                     cudaStream_t s, int bit_lo) {
  if (n <= 1 || nbits <= 0) return;
  static std::once_flag attr_once;  // one opt-in per kernel instantiation (thread-safe)
  std::call_once(attr_once, [&] {
    FMI_CK(cudaFuncSetAttribute(k_rs_scatter<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)scatter_smem<KT>()));
  });
  const int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
  DBuf<int64_t> counts((size_t)nblk * 256, s);
  KT* ka = keys; uint32_t* va = vals; KT* kb = keys_tmp; uint32_t* vb = vals_tmp;
  for (int shift = bit_lo; shift < nbits; shift += 8) {
    // items of this pass: key read (histogram) + key and index read and written (scatter)
    prof_units(KID_SORT, n * (int64_t)(3 * sizeof(KT) + 8));
    FMI_LAUNCH(KID_SORT, s, k_rs_hist<KT>, (unsigned)nblk, RS_THREADS, 0, ka, n, shift, nblk, counts.p,
               (const SegTile*)nullptr);
    exclusive_scan_i64(counts.p, counts.p, nblk * 256, nullptr, s);
    FMI_LAUNCH(KID_SORT, s, k_rs_scatter<KT>, (unsigned)nblk, RS_THREADS, scatter_smem<KT>(), ka, va, n, shift, nblk,
               counts.p, kb, vb, (const SegTile*)nullptr, 0, (const double4*)nullptr, (double4*)nullptr);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // the sorted result is in (ka, va): hand the buffers back swapped instead of copying
  keys = ka; vals = va; keys_tmp = kb; vals_tmp = vb;
}

void radix_sort_pairs(uint64_t*& keys, uint32_t*& vals, uint64_t*& keys_tmp, uint32_t*& vals_tmp, int64_t n,
                      int nbits, cudaStream_t s, int bit_lo) {
  radix_sort_impl<uint64_t>(keys, vals, keys_tmp, vals_tmp, n, nbits, s, bit_lo);
}

void radix_sort_pairs32(uint32_t*& keys, uint32_t*& vals, uint32_t*& keys_tmp, uint32_t*& vals_tmp, int64_t n,
                        int nbits, cudaStream_t s) {
  radix_sort_impl<uint32_t>(keys, vals, keys_tmp, vals_tmp, n, nbits, s, 0);
}

const double4* bucket_sort_keys(const double* pts, const double* f, int64_t n, const double lo[3], double width,
                                bool unit, int D, int bit_lo, int nb, double4* packed, uint32_t* orig, bool rec_idx,
                                uint32_t* perm, cudaStream_t s, double4* rec_sorted) {
  if (n <= 0) return packed;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    FMI_CK(cudaFuncSetAttribute(k_rs_scatter<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)scatter_smem<uint32_t>()));
    FMI_CK(cudaFuncSetAttribute(k_bk_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK_SMEM));
  });
  const int64_t nblk = (n + BK_TILE - 1) / BK_TILE;                // top-digit tiles
  const int64_t nblk2 = (n + RS_TILE - 1) / RS_TILE + 256;  // padded layout: at most one partial tile per bucket
  const int64_t n2 = nblk2 * RS_TILE;
  DBuf<int64_t> counts((size_t)std::max(nblk, nblk2) * 256, s), cnt(256, s), pshift(256, s);
  DBuf<int32_t> tile0(257, s);
  DBuf<SegTile> seg((size_t)nblk2, s);
  DBuf<uint32_t> ka(n2, s), va(n2, s), kb(n2, s), vb(n2, s);
  // the top digit: histogram (coordinates 24 B), then the scatter (coordinates 24 B + value 8 B read; record
  // 32 B, orig 4 B, key and position 8 B written)
  prof_units(KID_KEYS, n * (24 + 24 + (f ? 8 : 0) + 32 + (orig ? 4 : 0) + 8));
  FMI_LAUNCH(KID_KEYS, s, k_bk_hist, (unsigned)nblk, RS_THREADS, 0, pts, n, lo[0], lo[1], lo[2], width, unit, D,
             bit_lo, nb, nblk, counts.p);
  exclusive_scan_i64(counts.p, counts.p, nblk * 256, nullptr, s);
  FMI_LAUNCH(KID_KEYS, s, k_bk_layout, 1, 256, 0, counts.p, nblk, n, tile0.p, cnt.p, pshift.p);
  FMI_LAUNCH(KID_KEYS, s, k_bk_tiles, (unsigned)nblk2, 256, 0, tile0.p, cnt.p, pshift.p, seg.p, ka.p, va.p);
  FMI_LAUNCH(KID_KEYS, s, k_bk_scatter, (unsigned)nblk, RS_THREADS, BK_SMEM, pts, f, n, lo[0], lo[1], lo[2], width, unit,
             D, bit_lo, nb, nblk, counts.p, pshift.p, packed, orig, rec_idx ? 1 : 0, ka.p, va.p);
  // the remaining digits inside each bucket: segmented LSD passes over bits [0, nb - 8), the last one
  // writing the dense permutation (bucket positions in Morton order)
  const int npass = nb > 8 ? (nb - 8 + 7) / 8 : 0;
  if (npass == 0) {  // the bucket order is the sorted order
    if (!rec_sorted) FMI_LAUNCH(KID_MISC, s, k_iota32, (unsigned)((n + 255) / 256), 256, 0, perm, n);
    return packed;
  }
  uint32_t *k0 = ka.p, *v0 = va.p, *k1 = kb.p, *v1 = vb.p;
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    const bool last = pass + 1 == npass;
    // key read (histogram) + key and value read, key and value written (the last pass: value only, or
    // with rec_sorted the 32-byte record read and written instead)
    prof_units(KID_SORT, n * (int64_t)(last ? (rec_sorted ? 76 : 16) : 20));
    FMI_LAUNCH(KID_SORT, s, k_rs_hist<uint32_t>, (unsigned)nblk2, RS_THREADS, 0, k0, n2, shift, nblk2, counts.p,
               (const SegTile*)seg.p);
    exclusive_scan_i64(counts.p, counts.p, nblk2 * 256, nullptr, s);
    FMI_LAUNCH(KID_SORT, s, k_rs_scatter<uint32_t>, (unsigned)nblk2, RS_THREADS, scatter_smem<uint32_t>(), k0, v0, n2,
               shift, nblk2, counts.p, last ? nullptr : k1, last ? perm : v1, (const SegTile*)seg.p, last ? 1 : 0,
               (const double4*)packed, last ? rec_sorted : nullptr);
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  return rec_sorted ? rec_sorted : packed;
}

void gather_points(const double4* packed, uint32_t* perm, int64_t n, double* ux, double* uy, double* uz, double* r,
                   cudaStream_t s, const double* f, int* bad, uint64_t* keys, int D, const uint32_t* orig,
                   bool compose) {
  if (n <= 0) return;
  unsigned grid = (unsigned)((n + 255) / 256);
  if (f)
    FMI_LAUNCH(KID_GATHER, s, k_gather_f, grid, 256, 0, packed, perm, f, n, ux, uy, uz, r, bad, keys, D, orig,
               compose ? 1 : 0);
  else
    FMI_LAUNCH(KID_GATHER, s, k_gather, grid, 256, 0, packed, perm, n, ux, uy, uz, r, keys, D, orig, compose ? 1 : 0);
}

}  // namespace fmi
