// level.cu — per-level octree bookkeeping (K3 of DESIGN.md §3): octant block bounds of every active
// node from the sorted Morton keys, chunk lists, child decisions and compaction of the next level.
//
// PAPER.md Algorithm 1:
//   line 4  FMT_Ordered_by_Octant -> the octant blocks of a node are contiguous sub-ranges of the
//           Morton-sorted points; their bounds come from a binary search on the level-(d+1) digit.
//   lines 5-11 block bounds (running start j, end j+n_o: reading G2), E_RMS = sqrt(Σ r²/n_o) on the
//           post-fit residual (G3), child iff E_RMS > τ and n_o >= 𝓛 (G4) and
//           depth+1 <= max_depth (G5).  FMT_New_Octant: child cell = 2·cell + octant bits.
#include "fmi_internal.cuh"

namespace fmi {

namespace {

__device__ __forceinline__ int digit_at(uint64_t key, int level, int D) {
  return (int)((key >> (3 * (D - level))) & 7ull);
}

// K3: child_start[node*9 + o], o = 0..8, via lower_bound on the digit of level depth+1
__global__ void k_children(const uint64_t* __restrict__ keys, NodeTable nt, int64_t first, int64_t count,
                           int depth, int D) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 9) return;
  const int64_t node = first + t / 9;
  const int o = (int)(t % 9);
  const int64_t s = nt.start[node], e = nt.end[node];
  int64_t res;
  if (o == 0) {
    res = s;
  } else if (o == 8 || depth >= D) {
    res = e;  // beyond the key depth no split exists: all points in block 0
  } else {
    int64_t lo = s, hi = e;  // first index with digit >= o
    while (lo < hi) {
      int64_t mid = lo + ((hi - lo) >> 1);
      if (digit_at(keys[mid], depth + 1, D) < o) lo = mid + 1; else hi = mid;
    }
    res = lo;
  }
  nt.child_start[node * 9 + o] = res;
}

// range accessor for chunk lists: mode 0 = node ranges, mode 1 = octant segments (node*8 + o)
struct RangeSrc {
  const int64_t* a;     // mode 0: start[]; mode 1: child_start[] (9 per node)
  const int64_t* b;     // mode 0: end[]
  const int32_t* mask;  // mode 1 (optional): child[] — a segment whose child node exists is empty
  int mode;
  const int32_t* flag;  // mode 0 (optional): a range i with !(flag[i] & bit) is empty
  int bit;
  const int32_t* sel;   // mode 1 (optional): a segment i with sel[i] < 0 is empty
  __device__ __forceinline__ void get(int64_t i, int64_t& s, int64_t& e) const {
    if (mode == 0) {
      s = a[i]; e = b[i];
      if (flag && !(flag[i] & bit)) e = s;
    } else {
      int64_t nd = i >> 3; int o = (int)(i & 7); s = a[nd * 9 + o]; e = a[nd * 9 + o + 1];
      if (sel && sel[i] < 0) e = s;
      if (mask) {
        // owner runs: consecutive segments without a child node are one range, attributed to the
        // first segment of the run (so a leaf's points form a single range)
        if (mask[i] >= 0 || (o > 0 && mask[i - 1] < 0)) {
          e = s;
        } else {
          int oe = o + 1;
          while (oe < 8 && mask[nd * 8 + oe] < 0) ++oe;
          e = a[nd * 9 + oe];
        }
      }
    }
  }
};

__global__ void k_chunk_counts(RangeSrc src, int64_t nr, int64_t ch, int64_t* __restrict__ counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  int64_t s, e;
  src.get(i, s, e);
  int64_t n = e - s;
  counts[i] = n > 0 ? (n + ch - 1) / ch : 0;
}

// thread per chunk slot: locate the owning range by binary search on chunk_begin; balanced split
__global__ void k_chunk_fill(RangeSrc src, int64_t nr, const int64_t* __restrict__ chunk_begin,
                             const int64_t* __restrict__ nchunks, Chunk* __restrict__ chunks, int64_t max_chunks) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = *nchunks;
  if (c >= total || c >= max_chunks) return;
  int64_t lo = 0, hi = nr - 1;  // last i with chunk_begin[i] <= c
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo + 1) >> 1);
    if (chunk_begin[mid] <= c) lo = mid; else hi = mid - 1;
  }
  const int64_t i = lo;
  int64_t s, e;
  src.get(i, s, e);
  const int64_t n = e - s;
  const int64_t cnt = (i + 1 < nr ? chunk_begin[i + 1] : total) - chunk_begin[i];
  const int64_t k = c - chunk_begin[i];
  Chunk ck;
  ck.owner = (int32_t)i;
  ck.pad = 0;
  ck.start = s + (n * k) / cnt;
  ck.end = s + (n * (k + 1)) / cnt;
  chunks[c] = ck;
}

// decisions: flags[node*8+o] for the level; child_rms/child counts are kept in the node table.
// geo (moment tree): the integer guards only — every cell that COULD become a node.
// Sharded build (fmi_build_dist): gcnt = global octant counts of the level (summed over shards) for
// the global levels; owned_only = the children are the shard's own subtree roots (depth = shard
// depth): a child is created only where this shard holds its points.
__global__ void k_decide(NodeTable nt, int64_t first, int64_t count, int depth, int D, int L, double tau, bool geo,
                         const int64_t* __restrict__ gcnt, bool owned_only, int64_t geo_min,
                         int64_t* __restrict__ flags) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 8) return;
  const int64_t node = first + t / 8;
  const int o = (int)(t % 8);
  const int64_t n_loc = nt.child_start[node * 9 + o + 1] - nt.child_start[node * 9 + o];
  const int64_t n_o = gcnt ? gcnt[t] : n_loc;
  const bool owned = !owned_only || n_loc > 0;
  if (geo) {
    flags[t] = (n_o > 0 && n_o >= L && n_o >= geo_min && depth + 1 <= D && owned) ? 1 : 0;
    return;
  }
  nt.child_n[node * 8 + o] = n_o;
  const double ss = nt.child_ss[node * 8 + o];
  const double e = n_o > 0 ? sqrt(ss / (double)n_o) : 0.0;       // E_RMS
  const bool make = n_o > 0 && e > tau && n_o >= L && depth + 1 <= D;  // P:306 (+ G5)
  flags[t] = (make && owned) ? 1 : 0;
  if (o == 0) {  // node post-fit RMS over all its points, fixed octant order
    double tot = 0.0;
    int64_t n = 0;
    for (int k = 0; k < 8; ++k) {
      tot += nt.child_ss[node * 8 + k];
      n += gcnt ? gcnt[(t / 8) * 8 + k] : nt.child_start[node * 9 + k + 1] - nt.child_start[node * 9 + k];
    }
    nt.rms[node] = n > 0 ? sqrt(tot / (double)n) : 0.0;
  }
}

// segments of children created under a deferred parent (the deferred projection pass)
__global__ void k_defer_sel(NodeTable nt, int64_t first, int64_t count, int32_t* __restrict__ sel) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 8) return;
  const int64_t node = first + t / 8;
  sel[t] = ((nt.flag[node] & 8) && nt.child[node * 8 + (t % 8)] >= 0) ? 1 : -1;
}

// local octant counts of the level's nodes (for the global-level sums of a sharded build)
__global__ void k_octant_counts(NodeTable nt, int64_t first, int64_t count, int64_t* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 8) return;
  const int64_t node = first + t / 8;
  const int o = (int)(t % 8);
  out[t] = nt.child_start[node * 9 + o + 1] - nt.child_start[node * 9 + o];
}

// compaction: emit the children of the level in (parent, octant) order = canonical (depth, prefix) order
// mt_child (fit tree only): child table of the moment tree; the new node's moment-tree id is its
// parent's moment-tree child o.  srcseg[k] = level-local segment of new node k (its projection).
__global__ void k_emit(NodeTable nt, int64_t first, int64_t count, int depth, const int64_t* __restrict__ flags,
                       const int64_t* __restrict__ pos, const int32_t* __restrict__ mt_child,
                       int32_t* __restrict__ srcseg, int64_t* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 8) return;
  const int64_t node = first + t / 8;
  const int o = (int)(t % 8);
  const int64_t next_first = first + count;
  if (flags[t]) {
    const int64_t id = next_first + pos[t];
    nt.start[id] = nt.child_start[node * 9 + o];
    nt.end[id] = nt.child_start[node * 9 + o + 1];
    int4 c = nt.cell[node];
    nt.cell[id] = make_int4(2 * c.x + (o & 1), 2 * c.y + ((o >> 1) & 1), 2 * c.z + ((o >> 2) & 1), depth + 1);
    nt.parent[id] = (int32_t)node;
    nt.child[node * 8 + o] = (int32_t)id;
    if (mt_child) {
      const int32_t pm = nt.mtid[node];  // -1: deeper than the moment tree (moments accumulated on demand)
      nt.mtid[id] = pm < 0 ? -1 : mt_child[(int64_t)pm * 8 + o];
      srcseg[pos[t]] = (int32_t)t;
    }
    for (int k = 0; k < 8; ++k) nt.child[id * 8 + k] = -1;
  } else {
    nt.child[node * 8 + o] = -1;
  }
  if (t == count * 8 - 1) {
    out[0] = pos[t] + flags[t];
  }
  // children of parents whose child projections were deferred (flag bit 3): their projection pass
  if (mt_child && flags[t] && (nt.flag[node] & 8)) atomicAdd(reinterpret_cast<unsigned long long*>(out + 2), 1ull);
}

// total points of the emitted nodes (single CTA, fixed order)
__global__ void k_points_of(const NodeTable nt, const int64_t* __restrict__ out_count, int64_t first,
                            int64_t* __restrict__ out_points) {
  __shared__ int64_t sm[256];
  const int64_t cnt = *out_count;
  int64_t acc = 0;
  for (int64_t i = threadIdx.x; i < cnt; i += 256) acc += nt.end[first + i] - nt.start[first + i];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_points = sm[0];
}

}  // namespace

void level_children(const LevelCtx& c, cudaStream_t s) {
  int64_t work = c.count * 9;
  FMI_LAUNCH(KID_CHILDREN, s, k_children, (unsigned)((work + 255) / 256), 256, 0, c.keys, c.nt, c.first, c.count,
             c.depth, c.Dk);
}

void make_chunks_impl(RangeSrc src, int64_t nr, int64_t ch, int64_t* counts_tmp, int64_t* chunk_begin,
                      int64_t* nchunks_dev, Chunk* chunks, int64_t max_chunks, cudaStream_t s) {
  FMI_LAUNCH(KID_CHUNKS, s, k_chunk_counts, (unsigned)((nr + 255) / 256), 256, 0, src, nr, ch, counts_tmp);
  exclusive_scan_i64(counts_tmp, chunk_begin, nr, nchunks_dev, s);
  if (max_chunks > 0)
    FMI_LAUNCH(KID_CHUNKS, s, k_chunk_fill, (unsigned)((max_chunks + 255) / 256), 256, 0, src, nr, chunk_begin,
               nchunks_dev, chunks, max_chunks);
}

void make_chunks(const int64_t* rstart, const int64_t* rend, int64_t nr, int64_t ch, int64_t* counts_tmp,
                 int64_t* chunk_begin, int64_t* nchunks_dev, Chunk* chunks, int64_t max_chunks, cudaStream_t s,
                 const int32_t* seg_mask, const int32_t* range_flag, int flag_bit, const int32_t* seg_sel) {
  RangeSrc src{rstart, rend, seg_mask, rend ? 0 : 1, range_flag, flag_bit, seg_sel};
  make_chunks_impl(src, nr, ch, counts_tmp, chunk_begin, nchunks_dev, chunks, max_chunks, s);
}

void defer_select(const LevelCtx& c, int32_t* sel, cudaStream_t s) {
  const int64_t work = c.count * 8;
  if (work <= 0) return;
  FMI_LAUNCH(KID_DECIDE, s, k_defer_sel, (unsigned)((work + 255) / 256), 256, 0, c.nt, c.first, c.count, sel);
}

void octant_counts(const LevelCtx& c, int64_t* out, cudaStream_t s) {
  const int64_t work = c.count * 8;
  if (work <= 0) return;
  FMI_LAUNCH(KID_DECIDE, s, k_octant_counts, (unsigned)((work + 255) / 256), 256, 0, c.nt, c.first, c.count, out);
}

void level_decide(const LevelCtx& c, bool geo, const int32_t* mt_child, int32_t* srcseg, int64_t* flags_tmp,
                  int64_t* scan_tmp, int64_t* dev_out, cudaStream_t s, const int64_t* gcnt, bool owned_only,
                  int64_t geo_min) {
  int64_t work = c.count * 8;
  unsigned grid = (unsigned)((work + 255) / 256);
  FMI_LAUNCH(KID_DECIDE, s, k_decide, grid, 256, 0, c.nt, c.first, c.count, c.depth, c.D, c.L, c.tau, geo, gcnt,
             owned_only, geo_min, flags_tmp);
  exclusive_scan_i64(flags_tmp, scan_tmp, work, nullptr, s);
  FMI_LAUNCH(KID_DECIDE, s, k_emit, grid, 256, 0, c.nt, c.first, c.count, c.depth, flags_tmp, scan_tmp, mt_child,
             srcseg, dev_out);
  FMI_LAUNCH(KID_DECIDE, s, k_points_of, 1, 256, 0, c.nt, dev_out, c.first + c.count, dev_out + 1);
}

}  // namespace fmi
