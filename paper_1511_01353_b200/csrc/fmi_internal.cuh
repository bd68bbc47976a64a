// fmi_internal.cuh — internal declarations of the B200 free-mesh interpolator (not part of the ABI).
//
// Data layout in HBM:
//   points, Morton order, SoA fp64: ux[N], uy[N], uz[N] (root-cube unit coordinates), r[N] (residual)
//   keys[N] uint64 Morton keys (3·D bits), perm[N] uint32 (Morton position -> input index)
//   node table (all levels, level-contiguous): NodeTable below
//   per-level scratch: chunk lists, moment partials [chunks][K+𝓛], node moments [nodes][K+𝓛]
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace fmi {

constexpr int kMaxDegree = 10;
constexpr int kMaxDepth = 20;  // keys carry max_depth + 1 <= 21 levels (63 bits)
// Column-rejection threshold of the node solve (reading G9): a column whose Schur
// complement diagonal of the equilibrated Gram is <= kDelta^2 is dropped.
constexpr double kDelta = 1e-6;

// ---------------------------------------------------------------------------------------------
// multi-index arithmetic (Algorithm-2 loop order: l outer, m middle, n inner)
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr int rank3(int k) { return k < 0 ? 0 : (k + 1) * (k + 2) * (k + 3) / 6; }
// position of (l, m, n), l+m+n <= Q, in the Algorithm-2 order of total degree Q
__host__ __device__ constexpr int basis_index(int Q, int l, int m, int n) {
  return rank3(Q) - rank3(Q - l) + m * (Q - l + 1) - m * (m - 1) / 2 + n;
}

// ---------------------------------------------------------------------------------------------
// error handling (C++ exceptions internally, converted to codes at the C ABI)
// ---------------------------------------------------------------------------------------------
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);
#define FMI_CK(x) ::fmi::check_cuda((x), #x, __FILE__, __LINE__)

// ---------------------------------------------------------------------------------------------
// launch bookkeeping and optional per-kernel event timing (fmi_profile_*)
// ---------------------------------------------------------------------------------------------
enum KernelId {
  KID_KEYS = 0, KID_SORT, KID_GATHER, KID_MOMENTS, KID_MOMENTS_REDUCE, KID_SOLVE, KID_CHILDREN,
  KID_RESIDUAL, KID_RESIDUAL_REDUCE, KID_DECIDE, KID_CHUNKS, KID_SCAN, KID_EVAL, KID_MISC, KID_PROJECT,
  KID_M2M, KID_LEVEL_GATHER, KID_REFINE_SOLVE, KID_REFINE, KID_PRESUM, KID_UNSCOPED_GRAM, KID_UNSCOPED_SOLVE,
  KID_SOLVE_QR,
  KID_COUNT
};
const char* kernel_name(int kid);
void prof_begin(int kid, cudaStream_t s);
void prof_end(int kid, cudaStream_t s, unsigned grid = 0);
inline unsigned launch_blocks(dim3 g) { return g.x * g.y * g.z; }
void prof_collect();  // after a stream sync: accumulate elapsed times of completed launches
// algorithmic work units processed by the launches of a kernel (items per sort pass, keyed points,
// solved nodes, ...), summed while profiling is on; bench.py turns them into bytes / flops
void prof_units(int kid, int64_t units);

// dist.cu: the library-owned NCCL communicator (fmi_dist_init); fail(FMI_ENCCL) on errors
void dist_nccl_unique_id(void* out128);
void dist_nccl_init(int rank, int world, const void* id128);
void dist_nccl_finalize();
bool dist_comm_ready(int world);
void dist_comm_allreduce(void* dev, int64_t n, int dtype, cudaStream_t s);  // in place, SUM

#define FMI_LAUNCH(kid, stream, kernel, grid, block, smem, ...)                          \
  do {                                                                                   \
    ::fmi::prof_begin((kid), (stream));                                                  \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                          \
    FMI_CK(cudaGetLastError());                                                          \
    ::fmi::prof_end((kid), (stream), ::fmi::launch_blocks(dim3(grid)));                   \
  } while (0)

// ---------------------------------------------------------------------------------------------
// Morton key of a root-cube unit coordinate (K1): q* = min(floor(u*·2^D), 2^D - 1) with an
// exact power-of-two scaling (reading G7/G18), bits interleaved x fastest (octant o = bx + 2by + 4bz).
// Shared by the key kernel and by the kernels that recompute keys from gathered coordinates.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t morton_spread3(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint64_t morton_quantize(double u, int D) {
  const double scale = (double)(1ull << D);
  double t = floor(__dmul_rn(u, scale));  // exact power-of-two scaling, no contraction
  t = fmin(fmax(t, 0.0), scale - 1.0);    // u = 1 -> top cell; outside queries are clamped
  return (uint64_t)t;
}
__device__ __forceinline__ uint64_t morton_key(double ux, double uy, double uz, int D) {
  return morton_spread3(morton_quantize(ux, D)) | (morton_spread3(morton_quantize(uy, D)) << 1) |
         (morton_spread3(morton_quantize(uz, D)) << 2);
}

// ---------------------------------------------------------------------------------------------
// stream-ordered device buffers
// ---------------------------------------------------------------------------------------------
void* dmalloc(size_t bytes, cudaStream_t s);
int64_t guard_violations();  // FMI_GUARD diagnostics (fmi_guard_violations)
void dfree(void* p, cudaStream_t s);

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    p = count ? static_cast<T*>(dmalloc(count * sizeof(T), st)) : nullptr;
  }
  void ensure(size_t count, cudaStream_t st) { if (count > n) alloc(count, st); }
  void release() { if (p) dfree(p, s); p = nullptr; n = 0; }
  ~DBuf() { release(); }
};

// ---------------------------------------------------------------------------------------------
// shared structures
// ---------------------------------------------------------------------------------------------
struct Chunk {
  int32_t owner;   // node (level-local) or segment (node*8 + octant) index
  int32_t pad;
  int64_t start;   // [start, end) in Morton order
  int64_t end;
};

// node table (all levels; nodes of one level are contiguous, in canonical (depth, prefix) order)
struct NodeTable {
  int64_t* start = nullptr;      // [cap]
  int64_t* end = nullptr;        // [cap]
  int4* cell = nullptr;          // [cap] (i, j, k, depth)
  int32_t* parent = nullptr;     // [cap]
  int32_t* child = nullptr;      // [cap*8]
  int64_t* child_start = nullptr;// [cap*9] octant block bounds (G2)
  double* child_ss = nullptr;    // [cap*8] Σ r² of each octant block after the node's fit
  double* coef = nullptr;        // [cap*L] monomial-form coefficients a_lmn = P_F,lmn / (l!m!n!)
  double* rms = nullptr;         // [cap]
  double* minpiv = nullptr;      // [cap]
  int32_t* rank = nullptr;       // [cap]
  int32_t* flag = nullptr;       // [cap] bit0: re-fitted by the QR path (K5q)
  int32_t* mtid = nullptr;       // [cap] node of the moment tree holding this node's moments
  double* pcoef = nullptr;       // [cap*L] pre-summed polynomial: own + ancestors' in this node's frame
  int64_t* child_n = nullptr;    // [cap*8] octant counts n_o (global ones for the global levels of a sharded build)
};

// ---------------------------------------------------------------------------------------------
// kernels / launchers (defined in the .cu files)
// ---------------------------------------------------------------------------------------------
// scan.cu: exclusive prefix sum of int64 (in place allowed); returns nothing, total via `total` (device)
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, cudaStream_t s);

// keys.cu
void bbox_and_check(const double* pts, int64_t n, double* out8 /*device: min3,max3,nonfinite,unused*/,
                    const double* f, cudaStream_t s);
// f/packed (fit points): also write the 32-byte records (u_x, u_y, u_z, f) read by gather_points
// keys32 (optional): write the sort key (key >> bit_lo, < 2^32) instead of the 64-bit key (keys unused)
void morton_keys(const double* pts, int64_t n, const double lo[3], double width, bool unit, int D, uint64_t* keys,
                 uint32_t* idx, cudaStream_t s, const double* f = nullptr, double4* packed = nullptr,
                 uint32_t* keys32 = nullptr, int bit_lo = 0);
// LSD radix sort of (keys, vals) by key bits [bit_lo, nbits), stable.  On return keys/vals point at the
// sorted data and keys_tmp/vals_tmp at the scratch (the pointers may have been swapped).
void radix_sort_pairs(uint64_t*& keys, uint32_t*& vals, uint64_t*& keys_tmp, uint32_t*& vals_tmp, int64_t n,
                      int nbits, cudaStream_t s, int bit_lo = 0);
// the same over 32-bit sort keys (bits [0, nbits)): 20 B per item and pass instead of 32
void radix_sort_pairs32(uint32_t*& keys, uint32_t*& vals, uint32_t*& keys_tmp, uint32_t*& vals_tmp, int64_t n,
                        int nbits, cudaStream_t s);
// f (optional): take the values from f[perm[i]] instead of the records (values uploaded after the keys
// were built); *bad is set if one is non-finite
// keys (optional): also write the 64-bit Morton keys (D levels) recomputed from the gathered coordinates
// orig (bucketed keys): perm holds bucket positions and orig the input index of each; compose: replace
// perm[i] by the input index once read
void gather_points(const double4* packed, uint32_t* perm, int64_t n, double* ux, double* uy, double* uz,
                   double* r, cudaStream_t s, const double* f = nullptr, int* bad = nullptr,
                   uint64_t* keys = nullptr, int D = 0, const uint32_t* orig = nullptr, bool compose = false);
// Bucketed keys + sort (single-GPU 32-bit sort keys of nb = 3·levels bits): the top 8 key bits first,
// fused with the record write (records in bucket order, orig[pos] = input index, or the input index in
// the record's fourth slot with rec_idx), then the remaining bits sorted inside each bucket; perm[i] =
// the bucket position of the i-th point in Morton order.  pts/f device pointers, n < 2^32.  rec_sorted
// (optional, n records): the last pass writes the records themselves in Morton order there instead of
// perm.  Returns the array holding the records in Morton order when perm is not written (packed when the
// top digit was the whole key, else rec_sorted), packed otherwise.
const double4* bucket_sort_keys(const double* pts, const double* f, int64_t n, const double lo[3], double width,
                                bool unit, int D, int bit_lo, int nb, double4* packed, uint32_t* orig, bool rec_idx,
                                uint32_t* perm, cudaStream_t s, double4* rec_sorted = nullptr);

// sharded build helpers (keys.cu): depth-s cell histogram, partition by owner shard, scatter
void cell_counts(const double* pts, int64_t n, const double lo[3], double width, bool unit, int s, int64_t* counts,
                 cudaStream_t st);
void partition_points(const double* pts, const double* f, int64_t n, const double lo[3], double width, bool unit,
                      int s, const int32_t* owner, int world, double* pts_out, double* f_out, int64_t* idx_out,
                      int64_t* send_counts, cudaStream_t st);
void scatter_values(const double* vals, const int64_t* idx, int64_t m, double* out, cudaStream_t st);

// chunks.cu (level bookkeeping)
// Build a chunk list over `nr` ranges with at most `ch` points per chunk: rend != nullptr: ranges
// [rstart[i], rend[i]); rend == nullptr: octant segments i = node*8+o of a child_start table (rstart),
// with seg_mask (a child table): owner runs only — maximal runs of consecutive segments whose child
// does not exist, each attributed to its first segment (the other segments are empty);
// node ranges: range i is empty unless (range_flag[i] & flag_bit) when range_flag != nullptr.
// chunk_begin[i] (exclusive scan of per-range chunk counts) and *nchunks (device) are written.
void make_chunks(const int64_t* rstart, const int64_t* rend, int64_t nr, int64_t ch, int64_t* counts_tmp,
                 int64_t* chunk_begin, int64_t* nchunks_dev, Chunk* chunks, int64_t max_chunks, cudaStream_t s,
                 const int32_t* seg_mask = nullptr, const int32_t* range_flag = nullptr, int flag_bit = 0,
                 const int32_t* seg_sel = nullptr);

// level ops (level.cu)
struct LevelCtx {
  const uint64_t* keys;
  const double* ux; const double* uy; const double* uz;
  double* r;
  NodeTable nt;
  int64_t first;      // global index of the level's first node
  int64_t count;      // active nodes at this level
  int depth;          // depth of the level
  int D;              // max_depth (depth guard, G5)
  int Dk;             // key depth (bits per axis of the Morton keys) = max_depth + 1
  int p, L, K;
  double tau;
};
void level_children(const LevelCtx& c, cudaStream_t s);  // child_start for the level's nodes
// moments.cu: raw moments (|γ| <= 2p, K per node) of every moment-tree node over its owner segments
// (chunks over segments node*8+o whose child does not exist), reduced per node in chunk order.
// (moments.cu) direct accumulation: partial[chunk][K] over each chunk's points in the frame of node
// cell[chunk.owner >> shift]; reduce_moments sums the chunks of each node's rpn ranges in chunk order
// into out[node*stride ..], for nodes with (flag[node] & bit) when flag != nullptr.
template <int P> void direct_moments(const double* ux, const double* uy, const double* uz, const int4* cell,
                                     int shift, const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks,
                                     double* partial, cudaStream_t s);
void reduce_moments(const double* partial, const int64_t* chunk_begin, const int64_t* nchunks_dev, int64_t nodes,
                    int rpn, int K, const int32_t* flag, int bit, double* out, int64_t stride, cudaStream_t s);
// (m2m.cu) direct-accumulation rounding bound of every moment-tree node (64·eps·owner points);
// moment-tree tensors use the padded stride KS = K rounded up to a multiple of 4 (16-byte rows for TMA, fp64 and fp32)
void bound_init(const NodeTable& mt, int64_t n, int K, int KS, float* bnd, cudaStream_t s);
// m2m.cu: mom[node] += Σ_children translate(mom[child]) for the nodes [first, first+count) (one level)
template <int P> void m2m_level(double* mom, float* bnd, const int32_t* child, int64_t first, int64_t count,
                                cudaStream_t s);
// m2m.cu: out[k] = [mtmom[m] (K) | segsum[srcseg[k]][0..𝓛) | mtbnd[m] (K)], m = mtid[first+k]
// (srcseg null: segment 0)
void gather_level(const double* mtmom, const float* mtbnd, const int32_t* mtid, const double* segsum,
                  const int32_t* srcseg, int64_t first, int64_t count, int K, int KS, int L, double* out,
                  cudaStream_t s);
// solve.cu: mom = [moments (K) | projection b (𝓛) | moment rounding bound (K)] per level-local node
// -> nt.coef (monomial form).  mode 0: flag bit0 -> K5q (pivot < kQrFlagPivot2), bit1 -> semi-normal
// refinement (pivot < refine2 or n < kRefineFill·𝓛; counted in nflag[0]), bit2 (value 4, exclusive) ->
// translated moments failed the rounding check (counted in nflag[1]; no solve).  mode 1: refinement
// step for bit-1 nodes, b1 = Σ_o segrhs[node*8+o][0..𝓛), δ -> delta[node][𝓛], coef += δ.  mode 2:
// re-solve of bit-2 nodes after direct accumulation (no rounding check).
template <int P> void level_solve(const LevelCtx& c, const double* mom, int mode, const double* segrhs,
                                  double* delta, double refine2, double refine_fill, int64_t n_root,
                                  int64_t* nflag, double* fac, cudaStream_t s, double defer_tau = 0.0);
// fac: per level-local node solve_factor_per_node(p) doubles (bordered packed lower factor, kept for
// the refinement solves)
size_t solve_factor_per_node(int p);
// refinement gate (DESIGN.md §5 K5r)
constexpr double kRefinePivot2 = 1e-6;
constexpr double kRefineFill = 2.0;
constexpr int kRefineSteps = 2;
// largest accepted equilibrated rounding bound of a translated Gram (DESIGN.md §5 M2M)
constexpr double kMomentTol = 1e-11;
// moment-tree cells need >= kMomentTreeFill·𝓛 points: smaller (deeper) fit nodes, which are few, get
// their moments accumulated on demand (the fallback path), and the costly last M2M level disappears
constexpr double kMomentTreeFill = 8.0;
// points per K4 work item (one lane accumulates one chunk)
constexpr int64_t kMomentChunk = 1024;
// residual.cu (fused K6): over the chunks of the level's octant segments:
//   K6_CHILD: r -= node polynomial (nt.coef, or delta[node] for refined nodes), Σ r² per segment
//             (-> nt.child_ss) and the projection onto every potential child's frame;
//   K6_ROOT:  one segment (the root range), no subtraction, projection in the root frame;
//   K6_OWN:   refinement step `iter` of bit-1 nodes only: r -= (iter ? delta : coef), projection in
//             the node's own frame.
// segsum[seg][0..𝓛) = projection, segsum[seg][𝓛] = Σ r².
//   K6_PROJ:  child-frame projections only (residual already updated) for the segments selected by
//             sel (children created under a parent whose projections were deferred, flag bit 3).
enum K6Mode { K6_CHILD = 0, K6_ROOT = 1, K6_OWN = 2, K6_PROJ = 3 };
template <int P> void level_residual(const LevelCtx& c, int mode, int iter, const double* delta, const Chunk* chunks,
                                     const int64_t* nchunks_dev, int64_t max_chunks, const int64_t* chunk_begin,
                                     int64_t nseg, double* partial, double* segsum, cudaStream_t s,
                                     const int32_t* sel = nullptr, bool horner_only = false);
// the gather of the sorted points (ux, uy, uz, r from packed[perm]) fused with the root projection
// b = Λᵀf in the root frame -> segsum[0..𝓛] (chunks over [0, n)); f (optional): separately uploaded
// values with the finiteness flag *bad
template <int P> void gather_root_projection(const double4* packed, uint32_t* perm, const uint32_t* orig,
                                             const double* f, int* bad,
                                             int64_t n, double* ux, double* uy, double* uz, double* r,
                                             const Chunk* chunks, const int64_t* nchunks_dev, int64_t max_chunks,
                                             const int64_t* chunk_begin, double* partial, double* segsum,
                                             cudaStream_t s, uint64_t* keys = nullptr, int D = 0,
                                             int64_t n_stride = 0);
// n_stride > 0: max_chunks persistent CTAs stride over batches of [0, n_stride) (chunks unused; one
// partial per CTA); gather_root_ctas = the resident CTA count for that grid
template <int P> int gather_root_ctas();
// child projections of a node are deferred (flag bit 3) when its predicted post-fit RMS (pre-fit energy
// minus the energy the fit removes) is below kDeferTheta·τ: its children are then unlikely to be
// created, and the projection pass runs only for those that are
constexpr double kDeferTheta = 1.0;
// decisions + compaction: writes the next level's nodes at [first+count, ...), returns via dev_out[0] the
// number of new nodes and dev_out[1] their total points.  geo: moment tree (integer guards only).
// mt_child/srcseg (fit tree): moment-tree ids and source segments of the new nodes.
// gcnt (sharded build, global levels): global octant counts [count*8]; owned_only: create only the
// children whose points this shard holds (the shard's subtree roots).
// geo_min (moment tree): a cell needs at least this many points to get a moment-tree node.
void level_decide(const LevelCtx& c, bool geo, const int32_t* mt_child, int32_t* srcseg, int64_t* flags_tmp,
                  int64_t* scan_tmp, int64_t* dev_out, cudaStream_t s, const int64_t* gcnt = nullptr,
                  bool owned_only = false, int64_t geo_min = 0);
// local octant counts [count*8] of the level's nodes
void octant_counts(const LevelCtx& c, int64_t* out, cudaStream_t s);
// sel[node*8+o] = 1 for children created under a parent with deferred projections (flag bit 3), else -1
void defer_select(const LevelCtx& c, int32_t* sel, cudaStream_t s);

// solve_qr.cu (robust path for ill-conditioned nodes)
size_t solve_qr_scratch_per_cta(int p);
template <int P> void level_solve_qr(const LevelCtx& c, const double* mom, double* scratch, int64_t slots,
                                     cudaStream_t s);
// Gram pivot below which a node is re-fitted by K5q (DESIGN.md §2 G9, §3 K5q)
constexpr double kQrFlagPivot2 = 1e-9;

// eval.cu
// eval.cu: pcoef of the nodes [first, first+count) of one level (parents' pcoef must be final)
template <int P> void presum_level(const NodeTable& nt, int64_t first, int64_t count, cudaStream_t s);
// unscoped.cu: the single-node fit up to degree 14 by QR through the Legendre basis;
// c = the root level (count 1, child_start set); writes coef/pcoef/rank/minpiv/flag of the root, the
// residual r (in place) and the root's octant energies child_ss.
template <int P> void unscoped_fit(const LevelCtx& c, cudaStream_t s);
// qpk (optional): the queries' root-cube coordinates as 32-byte records (from morton_keys); rec_idx: the
// records are in bucket order (bucket_sort_keys), idx holds bucket positions and each record's fourth slot
// the query's input index (the output position)
template <int P> void eval_sorted(const double* q, const double4* qpk, const uint64_t* keys, const uint32_t* idx,
                                  int64_t M, const double lo[3], double width, bool unit, int Dk, const NodeTable& nt,
                                  double* out, cudaStream_t s, bool rec_idx = false);

}  // namespace fmi
