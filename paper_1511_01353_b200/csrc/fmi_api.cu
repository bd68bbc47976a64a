// fmi_api.cu — the C ABI (include/fmi.h) and the host orchestration of the level-synchronous build.
//
// fmi_build runs PAPER.md Algorithm 1 breadth-first: all nodes of one depth form a level,
// and every step of the level runs as a device kernel over all of its nodes at once (run_levels):
//   moment tree + raw moments once per build (K4 + M2M: the Gram of Alg. 2)
//   per level: K5 node solve -> fused K6 residual update + block energies + child
//   projections (Qᵀf of the children) -> decisions + compaction.
// Host synchronisations per fit level: two small counter reads (after K5: refinement / direct-moment /
// deferral counts; after the decisions: the next level's size), plus two more on the rare levels with
// nodes whose translated moments fail the rounding check; one per moment-tree level.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/fmi.h"
#include "fmi_internal.cuh"

namespace fmi {

__global__ void k_scatter_residual(const double* __restrict__ r, const uint32_t* __restrict__ perm, int64_t n,
                                   double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = r[i];
}

__global__ void k_ss_from_segsum(NodeTable nt, int64_t first, int64_t nseg, int L, const double* __restrict__ segsum) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nseg) nt.child_ss[first * 8 + t] = segsum[t * (L + 1) + L];
}

// rows of src [count][K] into dst rows (stride) for nodes with (flag & bit)
__global__ void k_copy_flagged(const double* __restrict__ src, int K, double* __restrict__ dst, int64_t stride,
                               const int32_t* __restrict__ flag, int bit) {
  const int64_t node = blockIdx.x;
  if (!(flag[node] & bit)) return;
  for (int e = threadIdx.x; e < K; e += blockDim.x) dst[node * stride + e] = src[node * (int64_t)K + e];
}

// QR-flagged global nodes of a sharded build are refined instead (K5q needs all the node's points)
__global__ void k_qr_to_refine(NodeTable nt, int64_t first, int64_t count, int64_t* __restrict__ nref) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count && (nt.flag[first + t] & 3) == 1) {
    nt.flag[first + t] = (nt.flag[first + t] & ~3) | 2;
    atomicAdd(reinterpret_cast<unsigned long long*>(nref), 1ull);
  }
}


// the root node's table entries, written by a one-thread kernel (no host->device copy: a copy would
// queue behind a large upload on the copy engine, e.g. fmi_transfer's overlapped query upload)
__global__ void k_set_root(NodeTable t, int64_t N, bool fit) {
  t.start[0] = 0;
  t.end[0] = N;
  t.cell[0] = make_int4(0, 0, 0, 0);
  t.parent[0] = -1;
  for (int k = 0; k < 8; ++k) t.child[k] = -1;
  if (fit) t.mtid[0] = 0;
}

// mark every node of a level as deferred (flag bit 3): its child projections run in K6_PROJ
__global__ void k_defer_all(NodeTable nt, int64_t first, int64_t count) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) nt.flag[first + t] |= 8;
}

// the range [0, n) of the root segment (a kernel: no host->device copy behind an upload)
__global__ void k_fill_range(int64_t* se, int64_t n) {
  se[0] = 0;
  se[1] = n;
}

}  // namespace fmi

using namespace fmi;

// ------------------------------------------------------------------------------------------------
// thread-local state, errors
// ------------------------------------------------------------------------------------------------
namespace {
thread_local int tl_err = 0;
thread_local std::string tl_msg;
thread_local cudaStream_t tl_stream = 0;

void set_error(int code, const std::string& msg) {
  tl_err = code;
  tl_msg = msg;
}
}  // namespace

namespace fmi {

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  std::string m = std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" + std::to_string(line) + ")";
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(FMI_ENOMEM, m);
  }
  fail(FMI_ECUDA, m);
}

// ------------------------------------------------------------------------------------------------
// memory: stream-ordered pool allocations; the pool keeps freed memory for reuse across calls
// ------------------------------------------------------------------------------------------------
namespace {
std::once_flag g_pool_once;
}

// FMI_GUARD=1 (diagnostics; compute-sanitizer is closed on the GPU pool): every library buffer gets
// 4 KiB guard bands filled with 0xA5 before and after it; dfree checks them (an out-of-bounds write of
// any kernel into a neighbouring allocation shows up there) and counts violations (fmi_guard_violations)
namespace {
constexpr size_t kGuardBytes = 4096;
constexpr int kGuardByte = 0xA5;
const bool g_guard = [] { const char* e = std::getenv("FMI_GUARD"); return e && std::atoi(e) > 0; }();
std::mutex g_guard_mu;
std::unordered_map<void*, size_t> g_guard_map;
std::atomic<int64_t> g_guard_violations{0};
}  // namespace
int64_t guard_violations() { return g_guard_violations.load(); }

void* dmalloc(size_t bytes, cudaStream_t s) {
  std::call_once(g_pool_once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  });
  void* p = nullptr;
  const size_t g = g_guard ? kGuardBytes : 0;
  cudaError_t e = cudaMallocAsync(&p, bytes + 2 * g, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(FMI_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
  }
  if (!g) return p;
  // FMI_GUARD: guard bands before and after every library buffer, checked when it is freed
  FMI_CK(cudaMemsetAsync(p, kGuardByte, g, s));
  FMI_CK(cudaMemsetAsync(static_cast<char*>(p) + g + bytes, kGuardByte, g, s));
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guard_map[static_cast<char*>(p) + g] = bytes;
  return static_cast<char*>(p) + g;
}

void dfree(void* p, cudaStream_t s) {
  if (!p) return;
  if (!g_guard) {
    cudaFreeAsync(p, s);
    return;
  }
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guard_map.find(p);
    if (it == g_guard_map.end()) return;  // not ours (cannot happen): leak rather than corrupt
    bytes = it->second;
    g_guard_map.erase(it);
  }
  char* base = static_cast<char*>(p) - kGuardBytes;
  std::vector<unsigned char> h(2 * kGuardBytes);
  cudaMemcpyAsync(h.data(), base, kGuardBytes, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h.data() + kGuardBytes, static_cast<char*>(p) + bytes, kGuardBytes, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  for (size_t i = 0; i < h.size(); ++i)
    if (h[i] != (unsigned char)kGuardByte) {
      g_guard_violations.fetch_add(1);
      fprintf(stderr, "[fmi guard] %s guard of a %zu-byte buffer overwritten at byte %zd\n",
              i < kGuardBytes ? "front" : "back", bytes,
              i < kGuardBytes ? (ssize_t)i - (ssize_t)kGuardBytes : (ssize_t)(i - kGuardBytes));
      break;
    }
  cudaFreeAsync(base, s);
}

// ------------------------------------------------------------------------------------------------
// launch counting and profiling
// ------------------------------------------------------------------------------------------------
namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<bool> g_prof{false};
std::atomic<uint32_t> g_prof_mask{~0u};  // kernel ids whose launches are timed (fmi_profile_select)
static_assert(KID_COUNT <= 32, "g_prof_mask holds one bit per kernel id");
std::mutex g_prof_mu;
struct Pending {
  int kid;
  unsigned grid;
  cudaEvent_t a, b;
};
// FMI_PROF_LOG=1 (with profiling on): every timed launch (kernel, grid, ms) to stderr — diagnostics
const bool g_prof_log = [] { const char* e = std::getenv("FMI_PROF_LOG"); return e && std::atoi(e) > 0; }();
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_event_pool;
double g_prof_ms[KID_COUNT];
int64_t g_prof_n[KID_COUNT];
int64_t g_prof_units[KID_COUNT];
thread_local cudaEvent_t tl_open = nullptr;

cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  FMI_CK(cudaEventCreate(&e));
  return e;
}
const char* kNames[KID_COUNT] = {"keys",     "sort",     "gather", "moments", "moments_reduce",
                                 "solve",    "children", "residual", "residual_reduce",
                                 "decide",   "chunks",   "scan",   "eval",    "misc",
                                 "project",  "m2m",      "level_gather", "refine_solve", "refine", "presum",
                                 "unscoped_gram", "unscoped_solve", "solve_qr"};
}  // namespace

const char* kernel_name(int kid) { return (kid >= 0 && kid < KID_COUNT) ? kNames[kid] : "?"; }

void prof_begin(int kid, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof.load(std::memory_order_relaxed)) return;
  if (!((g_prof_mask.load(std::memory_order_relaxed) >> kid) & 1u)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  tl_open = get_event();
  FMI_CK(cudaEventRecord(tl_open, s));
}

void prof_end(int kid, cudaStream_t s, unsigned grid) {
  if (!g_prof.load(std::memory_order_relaxed) || !tl_open) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t b = get_event();
  FMI_CK(cudaEventRecord(b, s));
  g_pending.push_back({kid, grid, tl_open, b});
  tl_open = nullptr;
}

void prof_units(int kid, int64_t units) {
  if (!g_prof.load(std::memory_order_relaxed) || kid < 0 || kid >= KID_COUNT) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_units[kid] += units;
}

void prof_collect() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      g_prof_ms[p.kid] += ms;
      g_prof_n[p.kid] += 1;
      if (g_prof_log) fprintf(stderr, "[fmi launch] %s grid=%u %.4f ms\n", kNames[p.kid], p.grid, ms);
    }
    cudaGetLastError();
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  g_pending.clear();
}

}  // namespace fmi

// ------------------------------------------------------------------------------------------------
// the tree
// ------------------------------------------------------------------------------------------------
struct fmi_tree {
  int p = 0, L = 0, K = 0, D = 0, Dk = 0, depth_max = 0;
  int Dsorted = 0;  // key levels sorted (octant digits valid down to this depth)
  int refine_steps = kRefineSteps;   // env FMI_REFINE_STEPS
  double refine2 = kRefinePivot2;    // env FMI_REFINE_PIVOT2
  double refine_fill = kRefineFill;  // env FMI_REFINE_FILL
  int64_t mt_min = 0;                // moment-tree cell minimum (points); env FMI_MT_FILL (multiple of 𝓛)
  double defer_theta = kDeferTheta;  // env FMI_DEFER_THETA (0: never defer)
  bool k6_split = true;              // env FMI_K6_SPLIT=0: fused K6 (Horner + projections in one pass)
  int64_t split_min = 0;             // levels with at least this many points run the split K6
  int64_t deferred_children = 0;     // children whose projections ran in a K6_PROJ pass
  double tau = 0;
  double lo[3] = {0, 0, 0};
  double width = 1;
  bool unit = true;
  int64_t N = 0;     // points on this shard
  int64_t Ntot = 0;  // points over all shards (= N unless sharded)
  int64_t nodes = 0;
  int64_t cap = 0;
  NodeTable nt;
  std::vector<int64_t> lvl_first, lvl_count, lvl_points;
  const fmi_dist* dist = nullptr;  // sharded build: collectives (valid during fmi_build_dist only)
  int shard_depth = 0;             // nodes of depth < shard_depth are global (summed over shards)
  int64_t mt_nodes = 0;       // moment-tree size (introspection)
  int64_t direct_nodes = 0;   // fit nodes whose moments were re-accumulated directly (M2M check)
  int64_t refined_nodes = 0;  // fit nodes that took semi-normal refinement steps
  double* residual = nullptr;  // Morton order
  uint32_t* perm = nullptr;    // Morton position -> input index
  cudaStream_t stream = 0;
};

namespace {

// FMI_TRACE=1: host wall time of the build phases to stderr; FMI_TRACE=2: the stream is synchronised
// at every mark (device + host time per phase).  Diagnostics only.
struct Trace {
  int level = 0;
  std::chrono::steady_clock::time_point t0, last;
  std::string out;
  explicit Trace() {
    if (const char* e = std::getenv("FMI_TRACE")) level = std::atoi(e);
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what, cudaStream_t s) {
    if (!level) return;
    if (level >= 2) cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    char buf[96];
    snprintf(buf, sizeof buf, " %s=%.2f", what, std::chrono::duration<double, std::milli>(now - last).count());
    out += buf;
    last = now;
  }
  void flush(const char* tag) {
    if (!level) return;
    const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    // the stream-ordered pool's reserved bytes: growth between two identical builds = fresh physical memory
    // mapped inside the build (a host-side stall of tens of ms)
    int dev = 0;
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &used);
    }
    cudaGetLastError();
    fprintf(stderr, "[fmi trace] %s total=%.2f ms pool_reserved=%.1f MB pool_used_high=%.1f MB:%s\n", tag, tot,
            reserved / 1048576.0, used / 1048576.0, out.c_str());
  }
};

thread_local Trace* tl_trace = nullptr;
inline void tmark(const char* what, cudaStream_t s) {
  if (tl_trace) tl_trace->mark(what, s);
}

// pinned 64-byte staging area for the small per-level device->host reads (allocated once per thread)
int64_t* host_staging() {
  thread_local int64_t* p = nullptr;
  if (!p) FMI_CK(cudaMallocHost(&p, 8 * sizeof(int64_t)));
  return p;
}

void free_table(NodeTable& t, cudaStream_t s) {
  dfree(t.start, s); dfree(t.end, s); dfree(t.cell, s); dfree(t.parent, s); dfree(t.child, s);
  dfree(t.child_start, s); dfree(t.child_ss, s); dfree(t.coef, s); dfree(t.rms, s); dfree(t.minpiv, s);
  dfree(t.rank, s); dfree(t.flag, s); dfree(t.mtid, s); dfree(t.pcoef, s); dfree(t.child_n, s);
  t = NodeTable{};
}

template <typename T>
void grow_array(T*& p, int64_t old_n, int64_t new_n, cudaStream_t s) {
  T* q = static_cast<T*>(dmalloc((size_t)new_n * sizeof(T), s));
  if (p && old_n > 0) FMI_CK(cudaMemcpyAsync(q, p, (size_t)old_n * sizeof(T), cudaMemcpyDeviceToDevice, s));
  dfree(p, s);
  p = q;
}

// grow a node table to hold `need` nodes; fit = false: geometry fields only (moment tree)
void ensure_table(NodeTable& t, int64_t& cap, int64_t need, int L, bool fit, cudaStream_t s) {
  if (need <= cap) return;
  int64_t nc = std::max<int64_t>(need, std::max<int64_t>(1024, cap * 2));
  const int64_t keep = cap;  // copy every existing slot (children of the current level included)
  grow_array(t.start, keep, nc, s);
  grow_array(t.end, keep, nc, s);
  grow_array(t.cell, keep, nc, s);
  grow_array(t.parent, keep, nc, s);
  grow_array(t.child, keep * 8, nc * 8, s);
  grow_array(t.child_start, keep * 9, nc * 9, s);
  if (fit) {
    grow_array(t.child_ss, keep * 8, nc * 8, s);
    grow_array(t.coef, keep * L, nc * L, s);
    grow_array(t.rms, keep, nc, s);
    grow_array(t.minpiv, keep, nc, s);
    grow_array(t.rank, keep, nc, s);
    grow_array(t.flag, keep, nc, s);
    grow_array(t.mtid, keep, nc, s);
    grow_array(t.pcoef, keep * L, nc * L, s);
    grow_array(t.child_n, keep * 8, nc * 8, s);
  }
  cap = nc;
}

void set_root(NodeTable& t, int64_t N, bool fit, cudaStream_t s) {
  FMI_LAUNCH(KID_MISC, s, k_set_root, 1, 1, 0, t, N, fit);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// host-buffer overlaps (late value upload, query upload during the fit) only pay off on large inputs;
// FMI_NO_OVERLAP=1 disables them (diagnostics)
constexpr int64_t kOverlapMin = (int64_t)1 << 20;
// K6 split (Horner-only pass + projections of created children) from this many points per level on
// (env FMI_K6_SPLIT_MIN overrides: the parity tests force the split at small sizes)
constexpr int64_t kSplitMinPointsDefault = (int64_t)1 << 25;
bool no_overlap() {
  static const bool v = std::getenv("FMI_NO_OVERLAP") != nullptr;
  return v;
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// chunk size for a pass over `points` points in `nseg` contiguous segments, aiming at per_sm_chunks
// chunks per SM (whole waves of the 2-CTA/SM K6 kernels): every segment adds at most one partial chunk,
// so the size is taken for per_sm_chunks·148 − nseg full chunks — the total then stays within the whole
// waves instead of spilling a few CTAs into an extra, nearly empty wave (segments >= half the target:
// many waves anyway, the plain size)
int64_t choose_chunk(int64_t points, int64_t min_ch, int64_t per_sm_chunks, int64_t nseg) {
  const int64_t tgt = 148 * per_sm_chunks;
  const int64_t avail = 2 * nseg < tgt ? tgt - nseg : tgt;
  return std::max(min_ch, (points + avail - 1) / avail);
}

// thrown by run_levels when the moment tree needs key digits below the sorted depth
struct KeysShort {};

// back to an empty tree (before a rebuild)
void reset_tree(fmi_tree* T, cudaStream_t s) {
  free_table(T->nt, s);
  T->cap = 0;
  T->nodes = 0;
  T->mt_nodes = T->direct_nodes = T->refined_nodes = T->deferred_children = 0;
  T->lvl_first.clear();
  T->lvl_count.clear();
  T->lvl_points.clear();
  T->depth_max = 0;
}

// Collective SUM over the shards of a sharded build (fmi_dist): stage through the caller's exchange
// buffer, synchronise, call the caller's collective, copy back (stream-ordered).
void dist_sum_raw(const fmi_dist* d, void* dev, int64_t n, int dtype, cudaStream_t s) {
  if (!d || n <= 0) return;
  if (!d->allreduce) {  // the library-owned NCCL communicator: in place, on the stream, no host round trip
    dist_comm_allreduce(dev, n, dtype, s);
    return;
  }
  const int64_t bytes = n * (dtype == 2 ? 4 : 8);
  if (bytes > d->xbuf_bytes)
    fail(FMI_EINPUT, "fmi_dist exchange buffer too small: need " + std::to_string(bytes) + " bytes");
  FMI_CK(cudaMemcpyAsync(d->xbuf, dev, bytes, cudaMemcpyDeviceToDevice, s));
  FMI_CK(cudaStreamSynchronize(s));
  if (d->allreduce(d->ctx, n, dtype) != 0) fail(FMI_ENCCL, "sharded build: the allreduce callback failed");
  FMI_CK(cudaMemcpyAsync(dev, d->xbuf, bytes, cudaMemcpyDeviceToDevice, s));
}

void dist_sum(const fmi_tree* T, void* dev, int64_t n, int dtype, cudaStream_t s) {
  dist_sum_raw(T->dist, dev, n, dtype, s);
}

// values still uploading when the level build starts (fmi_build with page-locked host f): the moment
// tree, K4 and M2M need only the coordinates; the values are gathered (with the root projection) once
// the upload event has completed
struct LateValues {
  const double4* packed;
  uint32_t* perm;
  const uint32_t* orig;  // bucketed keys: input index of each bucket position (else nullptr)
  const double* f;
  int* bad;
  cudaEvent_t ready;
};

template <int P>
void fused_gather_root(const double4* packed, uint32_t* perm, const uint32_t* orig, const double* f, int* bad,
                       int64_t N, double* ux, double* uy, double* uz, double* r, double* root_b, cudaStream_t s,
                       uint64_t* keys = nullptr, int D = 0);

// Level-synchronous build:
//  A. moment tree: every cell with >= 𝓛 points down to max_depth (integer guards of P:306 + G5,
//     ignoring τ) — the fit tree is a subtree of it;
//  B. raw moments of every moment-tree node: one pass over all points (owner segments), then the
//     upward translation (M2M), deepest level first;
//  C. root projection (one pass), then per fit level: gather [moments | projection] -> K5 solve
//     (+ K5q QR re-fit of flagged nodes) -> fused K6 (residual, block energies, child projections)
//     -> decisions + compaction.  Small counter read-backs: after K5 and after the decisions.
template <int P>
void run_levels(fmi_tree* T, const uint64_t* keys, double* ux, double* uy, double* uz, double* r, cudaStream_t s,
                const double* root_b, const LateValues* late) {
  constexpr int L = rank3(P), K = rank3(2 * P);
  DBuf<int64_t> counts, begin, flags, scan, dev_small(8, s), nflag(3, s), gcnt;
  DBuf<int32_t> dsel;
  DBuf<Chunk> chunks;
  DBuf<double> partial, mtmom, segsum, lvlmom, scratch, delta;
  DBuf<float> mtbnd;
  constexpr int KS = (K + 3) & ~3;  // padded moment-tree stride (16-byte rows for TMA)
  DBuf<int32_t> srcseg;
  int64_t* host_small = host_staging();
  NodeTable mt;
  int64_t mt_cap = 0;
  try {
    // ---- A. moment tree --------------------------------------------------------------------------
    std::vector<int64_t> mfirst, mcount;
    ensure_table(mt, mt_cap, 16, L, false, s);
    set_root(mt, T->N, false, s);
    {
      int64_t first = 0, count = 1;
      bool short_keys = false;  // this shard's moment tree reaches below the sorted key levels
      for (int depth = 0; count > 0; ++depth) {
        if (depth >= T->Dsorted) {  // octant digits below this depth are not sorted
          short_keys = true;
          break;
        }
        mfirst.push_back(first);
        mcount.push_back(count);
        ensure_table(mt, mt_cap, first + count + 8 * count, L, false, s);
        LevelCtx c{keys, ux, uy, uz, r, mt, first, count, depth, T->D, T->Dk, P, L, K, T->tau};
        level_children(c, s);
        flags.ensure(count * 8, s);
        scan.ensure(count * 8, s);
        const bool global = T->dist && depth < T->shard_depth;
        if (global) {  // global level of a sharded build: decisions on the summed octant counts
          gcnt.ensure(count * 8, s);
          octant_counts(c, gcnt.p, s);
          dist_sum(T, gcnt.p, count * 8, 1, s);
        }
        level_decide(c, true, nullptr, nullptr, flags.p, scan.p, dev_small.p + 2, s, global ? gcnt.p : nullptr,
                     global && depth + 1 == T->shard_depth, T->mt_min);
        FMI_CK(cudaMemcpyAsync(host_small, dev_small.p + 2, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
        first += count;
        count = host_small[0];
      }
      if (T->dist) {
        // sharded: every shard re-sorts if any shard is short (the retry repeats the global levels'
        // collectives, so all shards must take it together); Dsorted > shard_depth, so every shard has
        // completed the same global-level collectives when it gets here
        DBuf<int64_t> flag(1, s);
        const int64_t one = short_keys ? 1 : 0;
        FMI_CK(cudaMemcpyAsync(flag.p, &one, sizeof one, cudaMemcpyHostToDevice, s));
        dist_sum(T, flag.p, 1, 1, s);
        int64_t any = 0;
        FMI_CK(cudaMemcpyAsync(&any, flag.p, sizeof any, cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
        short_keys = any != 0;
      }
      if (short_keys) throw KeysShort{};
      T->mt_nodes = first;
    }
    tmark("mtree", s);
    const int64_t MT = T->mt_nodes;
    // ---- B. owner-segment moments + M2M (with rounding bounds) ------------------------------------
    {
      const int64_t ch = kMomentChunk;
      const int64_t maxc = T->N / ch + 8 * MT + 1;
      counts.ensure(MT * 8, s);
      begin.ensure(MT * 8, s);
      chunks.ensure(maxc, s);
      make_chunks(mt.child_start, nullptr, MT * 8, ch, counts.p, begin.p, dev_small.p, chunks.p, maxc, s, mt.child);
      FMI_CK(cudaMemcpyAsync(host_small, dev_small.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      FMI_CK(cudaStreamSynchronize(s));
      const int64_t nch = std::min(host_small[0], maxc);
      partial.ensure((size_t)nch * K, s);
      mtmom.alloc((size_t)MT * KS, s);
      mtbnd.alloc((size_t)MT * KS, s);
      tmark("chunks", s);
      direct_moments<P>(ux, uy, uz, mt.cell, 3, chunks.p, dev_small.p, nch, partial.p, s);
      reduce_moments(partial.p, begin.p, dev_small.p, MT, 8, K, nullptr, 0, mtmom.p, KS, s);
      bound_init(mt, MT, K, KS, mtbnd.p, s);
      tmark("moments", s);
      for (int d = (int)mfirst.size() - 2; d >= 0; --d)
        m2m_level<P>(mtmom.p, mtbnd.p, mt.child, mfirst[d], mcount[d], s);
      if (T->dist) {  // global moment-tree nodes (depth < s, a prefix of the table): sum the partials
        const int64_t nglob = T->shard_depth < (int)mfirst.size() ? mfirst[T->shard_depth] : MT;
        dist_sum(T, mtmom.p, nglob * KS, 0, s);
        dist_sum(T, mtbnd.p, nglob * KS, 2, s);
      }
      tmark("m2m", s);
    }
    // ---- C. fit levels ---------------------------------------------------------------------------
    ensure_table(T->nt, T->cap, 16, L, true, s);
    set_root(T->nt, T->N, true, s);
    T->nodes = 1;
    int64_t first = 0, count = 1, points = T->N;
    if (late) {  // values uploaded meanwhile: gather them with the root projection, check finiteness
      FMI_CK(cudaStreamWaitEvent(s, late->ready, 0));
      segsum.ensure((size_t)(L + 1), s);
      fused_gather_root<P>(late->packed, late->perm, late->orig, late->f, late->bad, T->N, ux, uy, uz, r, segsum.p,
                           s);
      FMI_CK(cudaMemcpyAsync(host_small, late->bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      FMI_CK(cudaStreamSynchronize(s));
      if (*reinterpret_cast<int*>(host_small)) fail(FMI_EINPUT, "non-finite coordinate or value");
      lvlmom.ensure((size_t)(2 * K + L), s);
      gather_level(mtmom.p, mtbnd.p, T->nt.mtid, segsum.p, nullptr, 0, 1, K, KS, L, lvlmom.p, s);
    } else if (root_b) {  // root projection already taken by the fused gather (fused_gather_root)
      segsum.ensure((size_t)(L + 1), s);
      FMI_CK(cudaMemcpyAsync(segsum.p, root_b, (size_t)(L + 1) * sizeof(double), cudaMemcpyDeviceToDevice, s));
      lvlmom.ensure((size_t)(2 * K + L), s);
      gather_level(mtmom.p, mtbnd.p, T->nt.mtid, segsum.p, nullptr, 0, 1, K, KS, L, lvlmom.p, s);
    } else {  // root projection b = Λᵀf in the root frame
      LevelCtx c{keys, ux, uy, uz, r, T->nt, 0, 1, 0, T->D, T->Dk, P, L, K, T->tau};
      const int64_t ch = choose_chunk(T->N, 1024, 32, 1);
      const int64_t maxc = T->N / ch + 2;
      counts.ensure(8, s);
      begin.ensure(8, s);
      chunks.ensure(maxc, s);
      make_chunks(T->nt.start, T->nt.end, 1, ch, counts.p, begin.p, dev_small.p, chunks.p, maxc, s);
      partial.ensure((size_t)maxc * (L + 1), s);
      segsum.ensure((size_t)(L + 1), s);
      level_residual<P>(c, K6_ROOT, 0, nullptr, chunks.p, dev_small.p, maxc, begin.p, 1, partial.p, segsum.p, s);
      if (T->dist && T->shard_depth > 0) dist_sum(T, segsum.p, L + 1, 0, s);
      lvlmom.ensure((size_t)(2 * K + L), s);
      gather_level(mtmom.p, mtbnd.p, T->nt.mtid, segsum.p, nullptr, 0, 1, K, KS, L, lvlmom.p, s);
    }
    tmark("rootproj", s);
    const size_t fac_per_node = solve_factor_per_node(P);
    const int64_t qr_slots = 148;
    DBuf<double> qr_scratch((size_t)qr_slots * solve_qr_scratch_per_cta(P) / sizeof(double), s);
    bool short_fit = false;  // a fit node below the sorted key levels (fit nodes need only >= 𝓛 points)
    for (int depth = 0; count > 0; ++depth) {
      if (depth >= T->Dsorted) {  // octant digits below this depth are not sorted
        short_fit = true;
        break;
      }
      T->lvl_first.push_back(first);
      T->lvl_count.push_back(count);
      T->lvl_points.push_back(points);
      T->depth_max = depth;
      ensure_table(T->nt, T->cap, first + count + 8 * count, L, true, s);
      tmark("table", s);
      LevelCtx c{keys, ux, uy, uz, r, T->nt, first, count, depth, T->D, T->Dk, P, L, K, T->tau};
      level_children(c, s);
      tmark("children", s);
      const bool global = T->dist && depth < T->shard_depth;  // nodes summed over the shards
      // K5: solve; nodes whose translated moments fail the rounding check are re-accumulated directly
      FMI_CK(cudaMemsetAsync(nflag.p, 0, 3 * sizeof(int64_t), s));
      scratch.ensure((size_t)count * fac_per_node, s);
      tmark("scratch", s);
      // deferral: single shard only; split mode defers every node (Horner-only K6 + K6_PROJ)
      // split-K6 threshold on the whole-job level size (a shard holds ~1/world of it)
      const bool big_level = points * (T->dist ? T->dist->world : 1) >= T->split_min;
      const double defer_tau =
          global ? 0.0 : ((T->k6_split && big_level) ? INFINITY : T->defer_theta * T->tau);
      level_solve<P>(c, lvlmom.p, 0, nullptr, nullptr, T->refine2, T->refine_fill, T->Ntot, nflag.p, scratch.p, s,
                     defer_tau);
      tmark("k5", s);
      FMI_CK(cudaMemcpyAsync(&host_small[2], nflag.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      FMI_CK(cudaStreamSynchronize(s));
      tmark("k5sync", s);
      if (host_small[3] > 0) {
        // few flagged nodes, possibly huge (a root): longer chunks keep the chunk count (and the
        // per-node partial sums) bounded
        const int64_t chd = std::max<int64_t>(kMomentChunk, points / (148 * 64));
        const int64_t maxd = points / chd + count + 1;
        counts.ensure(count, s);
        begin.ensure(count, s);
        chunks.ensure(maxd, s);
        make_chunks(T->nt.start + first, T->nt.end + first, count, chd, counts.p, begin.p, dev_small.p, chunks.p,
                    maxd, s, nullptr, T->nt.flag + first, 4);
        FMI_CK(cudaMemcpyAsync(host_small, dev_small.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
        const int64_t nchd = std::min(host_small[0], maxd);
        partial.ensure((size_t)nchd * K, s);
        direct_moments<P>(ux, uy, uz, T->nt.cell + first, 0, chunks.p, dev_small.p, nchd, partial.p, s);
        if (global) {  // partial direct moments of the flagged global nodes -> summed over the shards
          DBuf<double> tmp((size_t)count * K, s);
          FMI_CK(cudaMemsetAsync(tmp.p, 0, (size_t)count * K * sizeof(double), s));
          reduce_moments(partial.p, begin.p, dev_small.p, count, 1, K, T->nt.flag + first, 4, tmp.p, K, s);
          dist_sum(T, tmp.p, count * K, 0, s);
          FMI_LAUNCH(KID_MISC, s, k_copy_flagged, (unsigned)count, 256, 0, tmp.p, K, lvlmom.p, 2 * K + L,
                     T->nt.flag + first, 4);
        } else {
          reduce_moments(partial.p, begin.p, dev_small.p, count, 1, K, T->nt.flag + first, 4, lvlmom.p, 2 * K + L, s);
        }
        level_solve<P>(c, lvlmom.p, 2, nullptr, nullptr, T->refine2, T->refine_fill, T->Ntot, nflag.p, scratch.p, s,
                       defer_tau);
        T->direct_nodes += host_small[3];
        FMI_CK(cudaMemcpyAsync(&host_small[2], nflag.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
      }
      if (global) {  // K5q needs all of a node's points: global nodes take refinement steps instead
        FMI_LAUNCH(KID_MISC, s, k_qr_to_refine, (unsigned)((count + 255) / 256), 256, 0, T->nt, first, count, nflag.p);
        FMI_CK(cudaMemcpyAsync(&host_small[2], nflag.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
      }
      const int64_t nref = host_small[2], ndefer_nodes = host_small[4];
      tmark("solve", s);
      // K6 form of this level: fused (Horner + Σr² + child projections) when most nodes may have
      // children; when at least half of the nodes deferred their projections (predicted leaves), all are
      // deferred and the level runs the Horner-only K6 (more points in flight per thread, no projection
      // registers) followed by K6_PROJ for the children actually created
      // the split pays on big levels (cfg 5: 2e8 points); small adaptive levels keep the fused pass
      bool horner_only = T->k6_split && !global && big_level;
      if (!global && !horner_only && big_level && ndefer_nodes * 2 >= count && ndefer_nodes > 0) {
        if (ndefer_nodes < count)
          FMI_LAUNCH(KID_MISC, s, k_defer_all, (unsigned)((count + 255) / 256), 256, 0, T->nt, first, count);
        horner_only = true;
      }
      if (!global) level_solve_qr<P>(c, lvlmom.p, qr_scratch.p, qr_slots, s);
      // fused K6 over the level's octant segments
      const int64_t ch6 = choose_chunk(points, 1024, 32, count * 8);
      const int64_t max6 = points / ch6 + 8 * count + 1;
      counts.ensure(count * 8, s);
      begin.ensure(count * 8, s);
      chunks.ensure(max6, s);
      make_chunks(T->nt.child_start + first * 9, nullptr, count * 8, ch6, counts.p, begin.p, dev_small.p + 1,
                  chunks.p, max6, s);
      partial.ensure((size_t)max6 * (L + 1), s);
      segsum.ensure((size_t)count * 8 * (L + 1), s);
      // semi-normal refinement of small-pivot nodes (DESIGN.md §5 K5r): r1 = r - Λc, b1 = Λᵀr1 (own
      // frame), δ = G⁻¹b1 with the same Gram, c += δ; the fused pass below then subtracts the last δ.
      if (nref > 0) {
        T->refined_nodes += nref;
        delta.ensure((size_t)count * L, s);
        // FMI_REFINE_STEPS=0: the K6_CHILD pass still reads δ of the flagged nodes — make it zero
        if (T->refine_steps == 0) FMI_CK(cudaMemsetAsync(delta.p, 0, (size_t)count * L * sizeof(double), s));
        for (int it = 0; it < T->refine_steps; ++it) {
          level_residual<P>(c, K6_OWN, it, delta.p, chunks.p, dev_small.p + 1, max6, begin.p, count * 8, partial.p,
                            segsum.p, s);
          if (global) dist_sum(T, segsum.p, count * 8 * (L + 1), 0, s);
          level_solve<P>(c, lvlmom.p, 1, segsum.p, delta.p, T->refine2, T->refine_fill, T->Ntot, nflag.p, scratch.p, s);
        }
      }
      tmark("qr+refine", s);
      level_residual<P>(c, K6_CHILD, 0, delta.p, chunks.p, dev_small.p + 1, max6, begin.p, count * 8, partial.p,
                        segsum.p, s, nullptr, horner_only);
      tmark("residual", s);
      flags.ensure(count * 8, s);
      scan.ensure(count * 8, s);
      srcseg.ensure(count * 8, s);
      if (global) {  // child projections, block energies and octant counts summed over the shards
        dist_sum(T, segsum.p, count * 8 * (L + 1), 0, s);
        FMI_LAUNCH(KID_MISC, s, k_ss_from_segsum, (unsigned)((count * 8 + 255) / 256), 256, 0, T->nt, first,
                   count * 8, L, segsum.p);
        gcnt.ensure(count * 8, s);
        octant_counts(c, gcnt.p, s);
        dist_sum(T, gcnt.p, count * 8, 1, s);
      }
      FMI_CK(cudaMemsetAsync(dev_small.p + 4, 0, sizeof(int64_t), s));
      level_decide(c, false, mt.child, srcseg.p, flags.p, scan.p, dev_small.p + 2, s, global ? gcnt.p : nullptr,
                   global && depth + 1 == T->shard_depth);
      FMI_CK(cudaMemcpyAsync(host_small, dev_small.p + 2, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      FMI_CK(cudaStreamSynchronize(s));
      const int64_t nnew = host_small[0], npts = host_small[1], ndefer = host_small[2];
      tmark("decide", s);
      if (ndefer > 0) {  // children created under deferred parents: their projections now (K6_PROJ)
        dsel.ensure(count * 8, s);
        defer_select(c, dsel.p, s);
        make_chunks(T->nt.child_start + first * 9, nullptr, count * 8, ch6, counts.p, begin.p, dev_small.p + 1,
                    chunks.p, max6, s, nullptr, nullptr, 0, dsel.p);
        level_residual<P>(c, K6_PROJ, 0, nullptr, chunks.p, dev_small.p + 1, max6, begin.p, count * 8, partial.p,
                          segsum.p, s, dsel.p);
        T->deferred_children += ndefer;
      }
      if (nnew > 0) {
        lvlmom.ensure((size_t)nnew * (2 * K + L), s);
        gather_level(mtmom.p, mtbnd.p, T->nt.mtid, segsum.p, srcseg.p, first + count, nnew, K, KS, L, lvlmom.p, s);
      }
      first += count;
      T->nodes = first + nnew;
      count = nnew;
      points = npts;
    }
    if (T->dist) {  // sharded: the re-sort is collective (see the moment tree)
      DBuf<int64_t> flag(1, s);
      const int64_t one = short_fit ? 1 : 0;
      FMI_CK(cudaMemcpyAsync(flag.p, &one, sizeof one, cudaMemcpyHostToDevice, s));
      dist_sum(T, flag.p, 1, 1, s);
      int64_t any = 0;
      FMI_CK(cudaMemcpyAsync(&any, flag.p, sizeof any, cudaMemcpyDeviceToHost, s));
      FMI_CK(cudaStreamSynchronize(s));
      short_fit = any != 0;
    }
    if (short_fit) throw KeysShort{};
    // pre-summed polynomials for the evaluation (f1), level by level from the root
    for (size_t d = 0; d < T->lvl_first.size(); ++d) presum_level<P>(T->nt, T->lvl_first[d], T->lvl_count[d], s);
    tmark("presum", s);
  } catch (...) {
    free_table(mt, s);
    throw;
  }
  free_table(mt, s);
}

// the gather of the sorted points fused with the root projection (single-GPU builds): chunks over [0, N)
template <int P>
void fused_gather_root(const double4* packed, uint32_t* perm, const uint32_t* orig, const double* f, int* bad,
                       int64_t N, double* ux, double* uy, double* uz, double* r, double* root_b, cudaStream_t s,
                       uint64_t* keys, int D) {
  constexpr int L = rank3(P);
  if (orig) {
    // bucketed records: persistent CTAs striding over the batches in order (the window of positions in
    // flight stays inside one bucket of records, L2-resident); one partial per CTA
    constexpr int64_t kSpan = (int64_t)1 << 23;  // = kStrideSpan of gather_root_projection
    const int64_t nl = (N + kSpan - 1) / kSpan;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((std::min(N, kSpan) + 511) / 512, gather_root_ctas<P>()));
    DBuf<int64_t> bn(2, s);
    FMI_LAUNCH(KID_MISC, s, k_fill_range, 1, 1, 0, bn.p, nl * grid);  // chunk_begin = 0, nchunks = partial rows
    DBuf<double> partial((size_t)(nl * grid) * (L + 1), s);
    gather_root_projection<P>(packed, perm, orig, f, bad, N, ux, uy, uz, r, nullptr, bn.p + 1, nl * grid, bn.p,
                              partial.p, root_b, s, keys, D, N);
    return;
  }
  DBuf<int64_t> se(2, s), counts(1, s), begin(1, s), nch(1, s);
  FMI_LAUNCH(KID_MISC, s, k_fill_range, 1, 1, 0, se.p, N);
  const int64_t ch = choose_chunk(N, 1024, 32, 1);
  const int64_t maxc = N / ch + 2;
  DBuf<Chunk> chunks(maxc, s);
  DBuf<double> partial((size_t)maxc * (L + 1), s);
  make_chunks(se.p, se.p + 1, 1, ch, counts.p, begin.p, nch.p, chunks.p, maxc, s);
  gather_root_projection<P>(packed, perm, orig, f, bad, N, ux, uy, uz, r, chunks.p, nch.p, maxc, begin.p, partial.p,
                            root_b, s, keys, D);
}

// the QR path (unscoped.cu) — every node fitted by the paper's QR through
// the Legendre basis, level by level (Alg. 1): degrees 11..14 (beyond the fp64 moment Gram),
// any max_depth; the unscoped fit of Fig. 1 is its max_depth = 0 case (one level, the root)
template <int P>
void run_unscoped(fmi_tree* T, const uint64_t* keys, double* ux, double* uy, double* uz, double* r, cudaStream_t s) {
  constexpr int L = rank3(P);
  DBuf<int64_t> dev_small(8, s), flags, scan;
  int64_t* host_small = host_staging();
  ensure_table(T->nt, T->cap, 16, L, true, s);
  set_root(T->nt, T->N, true, s);
  T->nodes = 1;
  int64_t first = 0, count = 1, points = T->N;
  for (int depth = 0; count > 0; ++depth) {
    if (depth >= T->Dsorted) throw KeysShort{};  // octant digits below this depth are not sorted
    T->lvl_first.push_back(first);
    T->lvl_count.push_back(count);
    T->lvl_points.push_back(points);
    T->depth_max = depth;
    ensure_table(T->nt, T->cap, first + count + 8 * count, L, true, s);
    LevelCtx c{keys, ux, uy, uz, r, T->nt, first, count, depth, T->D, T->Dk, P, L, rank3(2 * P), T->tau};
    level_children(c, s);
    unscoped_fit<P>(c, s);
    flags.ensure(count * 8, s);
    scan.ensure(count * 8, s);
    FMI_CK(cudaMemsetAsync(dev_small.p + 4, 0, sizeof(int64_t), s));
    level_decide(c, false, nullptr, nullptr, flags.p, scan.p, dev_small.p + 2, s);
    FMI_CK(cudaMemcpyAsync(host_small, dev_small.p + 2, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    const int64_t nnew = host_small[0], npts = host_small[1];
    first += count;
    T->nodes = first + nnew;
    count = nnew;
    points = npts;
  }
  for (size_t d = 0; d < T->lvl_first.size(); ++d) presum_level<P>(T->nt, T->lvl_first[d], T->lvl_count[d], s);
  tmark("qr levels", s);
}

template <int P>
void run_eval(const fmi_tree* T, const double* q, const double4* qpk, const uint64_t* keys, const uint32_t* idx,
              int64_t M, int Dk, double* out, cudaStream_t s, bool rec_idx = false) {
  eval_sorted<P>(q, qpk, keys, idx, M, T->lo, T->width, T->unit, Dk, T->nt, out, s, rec_idx);
}

#define FMI_DISPATCH(p, FN, ...)                      \
  switch (p) {                                        \
    case 0: FN<0>(__VA_ARGS__); break;                \
    case 1: FN<1>(__VA_ARGS__); break;                \
    case 2: FN<2>(__VA_ARGS__); break;                \
    case 3: FN<3>(__VA_ARGS__); break;                \
    case 4: FN<4>(__VA_ARGS__); break;                \
    case 5: FN<5>(__VA_ARGS__); break;                \
    case 6: FN<6>(__VA_ARGS__); break;                \
    case 7: FN<7>(__VA_ARGS__); break;                \
    case 8: FN<8>(__VA_ARGS__); break;                \
    case 9: FN<9>(__VA_ARGS__); break;                \
    case 10: FN<10>(__VA_ARGS__); break;              \
    default: fail(FMI_EPRECOND, "degree out of range"); \
  }

// degrees 0..14 (the evaluation, pre-summing and unscoped-fit instantiations)
#define FMI_DISPATCH14(p, FN, ...)                    \
  switch (p) {                                        \
    case 11: FN<11>(__VA_ARGS__); break;              \
    case 12: FN<12>(__VA_ARGS__); break;              \
    case 13: FN<13>(__VA_ARGS__); break;              \
    case 14: FN<14>(__VA_ARGS__); break;              \
    default: FMI_DISPATCH(p, FN, __VA_ARGS__);        \
  }

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(FMI_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  }
}

// after_inputs (optional): called once the host->device copies of the inputs are enqueued, with the
// stream that carries the last of them (fmi_transfer chains its query upload after it, overlapping the
// fit)
fmi_tree* build_impl(const double* pts, const double* f, int64_t N, int degree, double tol, int max_depth,
                     const fmi_dist* dist, const std::function<void(cudaStream_t)>& after_inputs = nullptr) {
  if ((!pts || !f) && !(dist && N == 0)) fail(FMI_EINPUT, "null pointer argument");
  if (N < 0) fail(FMI_EINPUT, "N < 0");
  if (degree < 0 || degree > FMI_MAX_DEGREE) fail(FMI_EPRECOND, "degree outside 0..14");
  if (degree > FMI_MAX_LEVEL_DEGREE && dist)
    fail(FMI_EPRECOND, "degree > 10 (the QR path) is single-GPU only");
  if (max_depth < 0 || max_depth > FMI_MAX_DEPTH) fail(FMI_EPRECOND, "max_depth outside 0..20");
  if (!(tol >= 0.0)) fail(FMI_EPRECOND, "tol must be >= 0 (and not NaN)");
  const int L = rank3(degree);
  if (dist) {
    if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || (dist->allreduce && !dist->xbuf))
      fail(FMI_EINPUT, "invalid fmi_dist");
    // no callback: the library-owned NCCL communicator (fmi_dist_init) must span the same ranks
    if (!dist->allreduce && !dist_comm_ready(dist->world))
      fail(FMI_ENCCL, "fmi_dist without an allreduce callback needs fmi_dist_init over the same world");
    if (dist->shard_depth < 0 || dist->shard_depth > 6) fail(FMI_EPRECOND, "shard_depth outside 0..6");
    if (!(dist->width > 0.0)) fail(FMI_EINPUT, "fmi_dist: root cube width must be > 0");
  } else if (N < L) {
    fail(FMI_EPRECOND, "N < rank: the root fit is underdetermined (S:348)");
  }
  if (N > (int64_t)UINT32_MAX) fail(FMI_EPRECOND, "N exceeds 2^32 - 1");
  require_device();
  cudaStream_t s = tl_stream;
  Trace trace;
  tl_trace = trace.level ? &trace : nullptr;

  // inputs on the device
  DBuf<double> dpts_own, df_own;
  const double* dpts = pts;
  const double* df = f;
  if (N > 0 && !is_device_ptr(pts)) {
    dpts_own.alloc((size_t)N * 3, s);
    FMI_CK(cudaMemcpyAsync(dpts_own.p, pts, (size_t)N * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    dpts = dpts_own.p;
  }
  // Page-locked host values (single-GPU build): uploaded on a side stream after the points, while the
  // bounding box, keys and sort run; the gather takes them then (and checks their finiteness).
  struct SideStream {
    cudaStream_t st = nullptr;
    cudaEvent_t e_pts = nullptr, e_f = nullptr;
    ~SideStream() {
      if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
      if (e_pts) cudaEventDestroy(e_pts);
      if (e_f) cudaEventDestroy(e_f);
    }
  } side;
  // (large inputs only: the side stream costs more than it hides on small builds)
  const bool late_f = !dist && N >= kOverlapMin && !is_device_ptr(f) && is_pinned_host(f) && !no_overlap();
  if (N > 0 && !is_device_ptr(f)) {
    df_own.alloc((size_t)N, s);
    df = df_own.p;
    if (late_f) {
      FMI_CK(cudaStreamCreateWithFlags(&side.st, cudaStreamNonBlocking));
      FMI_CK(cudaEventCreateWithFlags(&side.e_pts, cudaEventDisableTiming));
      FMI_CK(cudaEventCreateWithFlags(&side.e_f, cudaEventDisableTiming));
      FMI_CK(cudaEventRecord(side.e_pts, s));  // after the point upload and the allocation
      FMI_CK(cudaStreamWaitEvent(side.st, side.e_pts, 0));
      FMI_CK(cudaMemcpyAsync(df_own.p, f, (size_t)N * sizeof(double), cudaMemcpyHostToDevice, side.st));
      FMI_CK(cudaEventRecord(side.e_f, side.st));
    } else {
      FMI_CK(cudaMemcpyAsync(df_own.p, f, (size_t)N * sizeof(double), cudaMemcpyHostToDevice, s));
    }
  }
  if (after_inputs) after_inputs(late_f ? side.st : s);

  // root frame (G6) + finiteness
  DBuf<double> bb(8, s);
  bbox_and_check(dpts, N, bb.p, late_f ? nullptr : df, s);
  double hb[8];
  FMI_CK(cudaMemcpyAsync(hb, bb.p, sizeof hb, cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaStreamSynchronize(s));
  tmark("inputs+bbox", s);
  int64_t Ntot = N;
  if (dist) {  // global point count and finiteness: every shard takes the same decision
    int64_t* hs = host_staging();
    hs[0] = N;
    hs[1] = hb[6] != 0.0 ? 1 : 0;
    DBuf<int64_t> two(2, s);
    FMI_CK(cudaMemcpyAsync(two.p, hs, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    dist_sum_raw(dist, two.p, 2, 1, s);
    FMI_CK(cudaMemcpyAsync(hs, two.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    Ntot = hs[0];
    if (hs[1] != 0) fail(FMI_EINPUT, "non-finite coordinate or value (on some shard)");
    if (Ntot < L) fail(FMI_EPRECOND, "N < rank: the root fit is underdetermined (S:348)");
  } else if (hb[6] != 0.0) {
    fail(FMI_EINPUT, "non-finite coordinate or value");
  }

  fmi_tree* T = new fmi_tree();
  try {
    T->p = degree;
    T->L = L;
    T->K = rank3(2 * degree);
    T->D = max_depth;
    T->Dk = max_depth + 1;
    T->tau = tol;
    T->N = N;
    T->Ntot = Ntot;
    T->stream = s;
    T->dist = dist;
    T->shard_depth = dist ? dist->shard_depth : 0;
    if (const char* e = std::getenv("FMI_REFINE_STEPS")) T->refine_steps = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("FMI_REFINE_PIVOT2")) T->refine2 = std::atof(e);
    if (const char* e = std::getenv("FMI_REFINE_FILL")) T->refine_fill = std::atof(e);
    if (const char* e = std::getenv("FMI_DEFER_THETA")) T->defer_theta = std::atof(e);
    if (const char* e = std::getenv("FMI_K6_SPLIT")) T->k6_split = std::atoi(e) != 0;
    T->split_min = kSplitMinPointsDefault;
    if (const char* e = std::getenv("FMI_K6_SPLIT_MIN")) T->split_min = std::atoll(e);
    {
      double mf = kMomentTreeFill;
      if (const char* e = std::getenv("FMI_MT_FILL")) mf = std::atof(e);
      T->mt_min = (int64_t)std::ceil(mf * L);
    }
    if (T->refine_steps == 0) T->refine2 = 0.0;  // no node is flagged for refinement
    bool unit = hb[0] >= 0.0 && hb[1] >= 0.0 && hb[2] >= 0.0 && hb[3] <= 1.0 && hb[4] <= 1.0 && hb[5] <= 1.0;
    if (dist) {  // the common root cube of the shards
      T->unit = dist->lo[0] == 0.0 && dist->lo[1] == 0.0 && dist->lo[2] == 0.0 && dist->width == 1.0;
      for (int a = 0; a < 3; ++a) T->lo[a] = dist->lo[a];
      T->width = dist->width;
    } else if (unit) {
      T->unit = true;
      T->lo[0] = T->lo[1] = T->lo[2] = 0.0;
      T->width = 1.0;
    } else {
      T->unit = false;
      for (int a = 0; a < 3; ++a) T->lo[a] = hb[a];
      double w = std::max(hb[3] - hb[0], std::max(hb[4] - hb[1], hb[5] - hb[2]));
      T->width = w > 0.0 ? w : 1.0;
    }
    // K1 keys + K2 sort + gather.  Only the top Dsort levels of the keys are sorted: no node is deeper
    // than the moment tree, whose depth is ~log8(N/𝓛) for space-filling data.  If the moment tree does
    // reach depth Dsort (clustered data), run_levels throws KeysShort and the sort is redone over all
    // levels.  Sharded builds take Dsort from the global point count, at least one level below the
    // shard depth, and agree on the retry collectively (run_levels).
    DBuf<uint64_t> keys(N, s), ktmp;  // ktmp: the 64-bit sort only
    DBuf<uint32_t> perm(N, s), ptmp(N, s);
    DBuf<double4> packed(N, s);
    DBuf<uint32_t> orig;  // bucketed keys: input index of every bucket position
    DBuf<double> ux(N, s), uy(N, s), uz(N, s), r(N, s);
    // the unscoped QR path (f2): degrees 11..14, or any degree at max_depth = 0 with FMI_UNSCOPED_QR=1
    // the QR path (unscoped.cu): degrees 11..14, or any degree with FMI_QR_PATH=1 (FMI_UNSCOPED_QR=1:
    // the same, max_depth = 0 only)
    const bool unscoped = !dist && (degree > FMI_MAX_LEVEL_DEGREE || std::getenv("FMI_QR_PATH") ||
                                    (max_depth == 0 && std::getenv("FMI_UNSCOPED_QR")));
    int Dsort = T->Dk;
    if (!std::getenv("FMI_FULL_SORT")) {
      const double fill = std::max(1.0, (double)std::max<int64_t>(Ntot, 1) / (double)L);
      Dsort = std::min(T->Dk, (int)std::ceil(std::log(fill) / std::log(8.0)) + 1);
      if (dist) Dsort = std::min(T->Dk, std::max(Dsort, dist->shard_depth + 1));
    }
    DBuf<int> fbad;
    DBuf<double> rootb;  // the root projection from the fused gather
    if (late_f) {
      fbad.alloc(1, s);
      FMI_CK(cudaMemsetAsync(fbad.p, 0, sizeof(int), s));
    }
    for (;;) {
      // the sorted key bits fit 32 bits (3·Dsort <= 32; every single-GPU and space-filling case): sort
      // 32-bit keys (20 B per item and pass instead of 32) in the two halves of the key buffer, and let
      // the gather recompute the full 64-bit keys from the gathered coordinates
      const bool key32 = 3 * Dsort <= 32;
      uint64_t* kout = key32 ? keys.p : nullptr;  // gathers write the full keys (sorted order)
      // bucketed keys (FMI_BUCKET_SORT=2; measured slower for the build, whose gather is bound by the
      // fused root projection): the top digit first, fused with the record write, so the gather reads
      // the records bucket by bucket
      const bool bucket_env = [] {  // FMI_BUCKET_SORT=2: also for the build's points
        const char* e = std::getenv("FMI_BUCKET_SORT");
        return e && std::atoi(e) >= 2;
      }();
      const bool bucket = key32 && bucket_env;
      if (bucket) {
        orig.ensure(N, s);
        bucket_sort_keys(dpts, late_f ? nullptr : df, N, T->lo, T->width, T->unit, T->Dk, 3 * (T->Dk - Dsort),
                         3 * Dsort, packed.p, orig.p, false, perm.p, s);
        tmark("keys", s);
      } else if (key32) {
        uint32_t* k32 = reinterpret_cast<uint32_t*>(keys.p);
        uint32_t* k32tmp = k32 + N;
        morton_keys(dpts, N, T->lo, T->width, T->unit, T->Dk, nullptr, perm.p, s, late_f ? nullptr : df, packed.p,
                    k32, 3 * (T->Dk - Dsort));
        tmark("keys", s);
        radix_sort_pairs32(k32, perm.p, k32tmp, ptmp.p, N, 3 * Dsort, s);
      } else {
        morton_keys(dpts, N, T->lo, T->width, T->unit, T->Dk, keys.p, perm.p, s, late_f ? nullptr : df, packed.p);
        tmark("keys", s);
        ktmp.ensure(N, s);
        radix_sort_pairs(keys.p, perm.p, ktmp.p, ptmp.p, N, 3 * T->Dk, s, 3 * (T->Dk - Dsort));
      }
      T->Dsorted = Dsort;
      tmark("sort", s);
      // single-GPU level path: the gather fused with the root projection (it needs no tree)
      const bool fuse_root = !unscoped && !dist;
      if (fuse_root) rootb.ensure((size_t)L + 1, s);
      const uint32_t* op = bucket ? orig.p : nullptr;  // bucket position -> input index
      LateValues late{packed.p, perm.p, op, df, fbad.p, side.e_f};
      const bool late_levels = late_f && fuse_root;  // values join inside run_levels (after K4/M2M)
      if (late_levels) {
        gather_points(packed.p, perm.p, N, ux.p, uy.p, uz.p, r.p, s, nullptr, nullptr, kout, T->Dk, op,
                      false);  // coordinates now (r: placeholder; perm still bucket positions)
      } else if (late_f) {
        FMI_CK(cudaStreamWaitEvent(s, side.e_f, 0));
        gather_points(packed.p, perm.p, N, ux.p, uy.p, uz.p, r.p, s, df, fbad.p, kout, T->Dk, op, true);
        int hbad = 0;
        FMI_CK(cudaMemcpyAsync(&hbad, fbad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        FMI_CK(cudaStreamSynchronize(s));
        if (hbad) fail(FMI_EINPUT, "non-finite coordinate or value");
      } else if (fuse_root) {
        FMI_DISPATCH(degree, fused_gather_root, packed.p, perm.p, op, nullptr, nullptr, N, ux.p, uy.p, uz.p, r.p,
                     rootb.p, s, kout, T->Dk);
      } else {
        gather_points(packed.p, perm.p, N, ux.p, uy.p, uz.p, r.p, s, nullptr, nullptr, kout, T->Dk, op, true);
      }
      tmark("gather", s);
      try {
        if (unscoped) {
          FMI_DISPATCH14(degree, run_unscoped, T, keys.p, ux.p, uy.p, uz.p, r.p, s);
        } else {
          FMI_DISPATCH(degree, run_levels, T, keys.p, ux.p, uy.p, uz.p, r.p, s,
                       (fuse_root && !late_levels) ? rootb.p : nullptr, late_levels ? &late : nullptr);
        }
        break;
      } catch (const KeysShort&) {
        reset_tree(T, s);
        Dsort = T->Dk;
      }
    }
    ktmp.release();
    ptmp.release();
    orig.release();
    packed.release();
    dpts_own.release();
    df_own.release();
    T->dist = nullptr;
    T->residual = r.p;
    r.p = nullptr;
    T->perm = perm.p;
    perm.p = nullptr;
    FMI_CK(cudaStreamSynchronize(s));
  } catch (...) {
    free_table(T->nt, s);
    dfree(T->residual, s);
    dfree(T->perm, s);
    delete T;
    throw;
  }
  prof_collect();
  tmark("end", s);
  trace.flush("build");
  tl_trace = nullptr;
  return T;
}

// one evaluation pass over device queries dq[0..m) -> dout[0..m) on stream s (K1 + K2 + K7)
void eval_device(const fmi_tree* T, const double* dq, int64_t m, double* dout, cudaStream_t s) {
  const int Dk = T->depth_max;
  if (Dk == 0) {
    FMI_DISPATCH14(T->p, run_eval, T, dq, nullptr, nullptr, nullptr, m, 0, dout, s);
  } else {
    DBuf<uint32_t> idx(m, s), itmp(m, s);
    DBuf<double4> qpk(m, s);
    const bool bucket = [] {  // FMI_BUCKET_SORT=0: the plain LSD sort of the queries
      const char* e = std::getenv("FMI_BUCKET_SORT");
      return !(e && std::atoi(e) == 0);
    }();
    if (3 * Dk <= 32 && bucket) {
      // bucketed records (top key digit first, the input index in each record): K7 reads the records of
      // one bucket at a time; the keys are recomputed from the records
      // the last sort pass writes the records themselves in Morton order: K7 reads them sequentially
      // (no index array, no dependent gather), the input index rides in each record
      idx.release();
      itmp.release();
      DBuf<double4> qsorted(m, s);
      const double4* rec = bucket_sort_keys(dq, nullptr, m, T->lo, T->width, T->unit, Dk, 0, 3 * Dk, qpk.p, nullptr,
                                            true, nullptr, s, qsorted.p);
      FMI_DISPATCH14(T->p, run_eval, T, dq, rec, nullptr, nullptr, m, Dk, dout, s, true);
    } else if (3 * Dk <= 32) {  // 32-bit sort keys; K7 recomputes each key from the query's record
      DBuf<uint32_t> k32(m, s), k32tmp(m, s);
      morton_keys(dq, m, T->lo, T->width, T->unit, Dk, nullptr, idx.p, s, nullptr, qpk.p, k32.p, 0);
      radix_sort_pairs32(k32.p, idx.p, k32tmp.p, itmp.p, m, 3 * Dk, s);
      k32.release();
      k32tmp.release();
      FMI_DISPATCH14(T->p, run_eval, T, dq, qpk.p, nullptr, idx.p, m, Dk, dout, s);
    } else {
      DBuf<uint64_t> keys(m, s), ktmp(m, s);
      morton_keys(dq, m, T->lo, T->width, T->unit, Dk, keys.p, idx.p, s, nullptr, qpk.p);
      radix_sort_pairs(keys.p, idx.p, ktmp.p, itmp.p, m, 3 * Dk, s);
      FMI_DISPATCH14(T->p, run_eval, T, dq, qpk.p, keys.p, idx.p, m, Dk, dout, s);
    }
  }
}

constexpr int64_t kEvalChunk = (int64_t)1 << 24;  // queries per pipelined chunk (host buffers)

int eval_impl(const fmi_tree* T, const double* q, int64_t M, double* out) {
  if (!T) fail(FMI_EINPUT, "null tree");
  if (M < 0) fail(FMI_EINPUT, "M < 0");
  if (M == 0) return 0;
  if (!q || !out) fail(FMI_EINPUT, "null pointer argument");
  if (M > (int64_t)UINT32_MAX) fail(FMI_EPRECOND, "M exceeds 2^32 - 1");
  cudaStream_t s = tl_stream;
  const bool host_q = !is_device_ptr(q), host_out = !is_device_ptr(out);
  if (M > kEvalChunk && ((host_q && is_pinned_host(q)) || (host_out && is_pinned_host(out))) &&
      !(host_q && !is_pinned_host(q)) && !(host_out && !is_pinned_host(out))) {
    // Page-locked host buffers: chunks of queries flow H2D (copy stream) -> keys/sort/eval (compute
    // stream) -> D2H (second copy stream), so the PCIe transfers of one chunk overlap the compute of
    // its neighbours.  Query and output buffers are double-buffered.
    const int64_t CH = kEvalChunk, nck = (M + CH - 1) / CH;
    cudaStream_t sin = nullptr, sout = nullptr;
    cudaEvent_t e_h2d[2] = {nullptr, nullptr}, e_comp[2] = {nullptr, nullptr}, e_d2h[2] = {nullptr, nullptr};
    auto release = [&] {
      for (int b = 0; b < 2; ++b) {
        if (e_h2d[b]) cudaEventDestroy(e_h2d[b]);
        if (e_comp[b]) cudaEventDestroy(e_comp[b]);
        if (e_d2h[b]) cudaEventDestroy(e_d2h[b]);
      }
      if (sin) cudaStreamDestroy(sin);
      if (sout) cudaStreamDestroy(sout);
    };
    DBuf<double> dqb[2], doutb[2];
    try {
      FMI_CK(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking));
      FMI_CK(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        FMI_CK(cudaEventCreateWithFlags(&e_h2d[b], cudaEventDisableTiming));
        FMI_CK(cudaEventCreateWithFlags(&e_comp[b], cudaEventDisableTiming));
        FMI_CK(cudaEventCreateWithFlags(&e_d2h[b], cudaEventDisableTiming));
        if (host_q) dqb[b].alloc((size_t)CH * 3, s);
        if (host_out) doutb[b].alloc((size_t)CH, s);
      }
      FMI_CK(cudaEventRecord(e_comp[0], s));  // allocations visible to the copy streams
      FMI_CK(cudaStreamWaitEvent(sin, e_comp[0], 0));
      FMI_CK(cudaStreamWaitEvent(sout, e_comp[0], 0));
      for (int64_t k = 0; k < nck; ++k) {
        const int b = (int)(k & 1);
        const int64_t c0 = k * CH, m = std::min(CH, M - c0);
        const double* qk = q + 3 * c0;
        if (host_q) {
          if (k >= 2) FMI_CK(cudaStreamWaitEvent(sin, e_comp[b], 0));  // chunk k-2 done with dqb[b]
          FMI_CK(cudaMemcpyAsync(dqb[b].p, qk, (size_t)m * 3 * sizeof(double), cudaMemcpyHostToDevice, sin));
          FMI_CK(cudaEventRecord(e_h2d[b], sin));
          FMI_CK(cudaStreamWaitEvent(s, e_h2d[b], 0));
          qk = dqb[b].p;
        }
        double* ok = out + c0;
        if (host_out) {
          if (k >= 2) FMI_CK(cudaStreamWaitEvent(s, e_d2h[b], 0));  // chunk k-2's values copied out
          ok = doutb[b].p;
        }
        eval_device(T, qk, m, ok, s);
        FMI_CK(cudaEventRecord(e_comp[b], s));
        if (host_out) {
          FMI_CK(cudaStreamWaitEvent(sout, e_comp[b], 0));
          FMI_CK(cudaMemcpyAsync(out + c0, doutb[b].p, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, sout));
          FMI_CK(cudaEventRecord(e_d2h[b], sout));
        }
      }
      FMI_CK(cudaStreamSynchronize(sin));
      FMI_CK(cudaStreamSynchronize(sout));
      FMI_CK(cudaStreamSynchronize(s));
    } catch (...) {
      if (sin) cudaStreamSynchronize(sin);
      if (sout) cudaStreamSynchronize(sout);
      cudaStreamSynchronize(s);
      release();
      throw;
    }
    for (int b = 0; b < 2; ++b) {
      dqb[b].release();
      doutb[b].release();
    }
    FMI_CK(cudaStreamSynchronize(s));
    release();
    prof_collect();
    return 0;
  }
  DBuf<double> dq_own, dout_own;
  const double* dq = q;
  double* dout = out;
  if (host_q) {
    dq_own.alloc((size_t)M * 3, s);
    FMI_CK(cudaMemcpyAsync(dq_own.p, q, (size_t)M * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    dq = dq_own.p;
  }
  if (host_out) {
    dout_own.alloc((size_t)M, s);
    dout = dout_own.p;
  }
  eval_device(T, dq, M, dout, s);
  if (host_out) FMI_CK(cudaMemcpyAsync(out, dout, (size_t)M * sizeof(double), cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaStreamSynchronize(s));
  prof_collect();
  return 0;
}

uint64_t morton_label(int depth, int i, int j, int k) {
  uint64_t out = 0;
  for (int t = 0; t < depth; ++t) {
    int b = depth - 1 - t;
    uint64_t o = ((i >> b) & 1) | (((j >> b) & 1) << 1) | (((k >> b) & 1) << 2);
    out = (out << 3) | o;
  }
  return out;
}

template <typename F>
int guard(F&& fn) {
  try {
    tl_err = 0;
    return fn();
  } catch (const Error& e) {
    tl_trace = nullptr;
    set_error(e.code, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    tl_trace = nullptr;
    set_error(FMI_ECUDA, e.what());
    return FMI_ECUDA;
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------------
// ---- tree files (SPEC FMT1-like record layout) ------------------------------------------
namespace {
constexpr char kMagic[8] = {'F', 'M', 'I', 'T', 'R', 'E', 'E', '1'};
constexpr int32_t kFileVersion = 1;
struct FileHeader {
  char magic[8];
  int32_t version, p, depth_max, unit;
  int64_t nodes, N;
  double lo[3], width, tau;
  int32_t D, pad;
};
template <typename T>
void dump(FILE* fp, const T* dev, int64_t n, cudaStream_t s) {
  std::vector<T> h((size_t)n);
  if (n) FMI_CK(cudaMemcpyAsync(h.data(), dev, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, s));
  FMI_CK(cudaStreamSynchronize(s));
  if (n && fwrite(h.data(), sizeof(T), (size_t)n, fp) != (size_t)n) fail(FMI_EINPUT, "short write");
}
template <typename T>
std::vector<T> undump(FILE* fp, T* dev, int64_t n, cudaStream_t s) {
  std::vector<T> h((size_t)n);
  if (n && fread(h.data(), sizeof(T), (size_t)n, fp) != (size_t)n) fail(FMI_EVERSION, "truncated tree file");
  if (n) FMI_CK(cudaMemcpyAsync(dev, h.data(), (size_t)n * sizeof(T), cudaMemcpyHostToDevice, s));
  FMI_CK(cudaStreamSynchronize(s));
  return h;
}

// A loaded file is untrusted input: the evaluation kernels follow child indices and the level
// tables are indexed by depth, so every node record is checked before the tree is handed out
// (FMI_EVERSION with the offending node index).
void validate_nodes(const std::vector<int4>& cell, const std::vector<int32_t>& parent,
                    const std::vector<int32_t>& child, const std::vector<int32_t>& rank, int depth_max, int D, int L) {
  const int64_t n = (int64_t)cell.size();
  auto bad = [](int64_t i, const char* what) {
    fail(FMI_EVERSION, "corrupt tree file: node " + std::to_string(i) + ": " + what);
  };
  for (int64_t i = 0; i < n; ++i) {
    const int d = cell[i].w;
    if (d < 0 || d > depth_max || d > D) bad(i, "depth out of range");
    if (i == 0 ? d != 0 : (d != cell[i - 1].w && d != cell[i - 1].w + 1)) bad(i, "depths not level-contiguous");
    const int64_t side = int64_t(1) << d;
    if (cell[i].x < 0 || cell[i].y < 0 || cell[i].z < 0 || cell[i].x >= side || cell[i].y >= side || cell[i].z >= side)
      bad(i, "cell outside its level");
    if (rank[i] < 0 || rank[i] > L) bad(i, "rank out of range");
    const int32_t pa = parent[i];
    if (i == 0) {
      if (pa != -1) bad(i, "root has a parent");
    } else if (pa < 0 || pa >= i || cell[pa].w != d - 1) {
      bad(i, "parent index");
    }
    for (int o = 0; o < 8; ++o) {
      const int32_t c = child[(size_t)i * 8 + o];
      if (c == -1) continue;
      if (c <= i || c >= n || parent[c] != i || cell[c].w != d + 1 || cell[c].x != 2 * cell[i].x + (o & 1) ||
          cell[c].y != 2 * cell[i].y + ((o >> 1) & 1) || cell[c].z != 2 * cell[i].z + ((o >> 2) & 1))
        bad(i, "child index");
    }
  }
  if (n > 0 && cell[n - 1].w != depth_max) bad(n - 1, "deepest level differs from the header");
}
}  // namespace

extern "C" {

fmi_tree* fmi_build(const double* pts, const double* f, int64_t N, int degree, double tol, int max_depth) {
  fmi_tree* out = nullptr;
  guard([&] {
    out = build_impl(pts, f, N, degree, tol, max_depth, nullptr);
    return 0;
  });
  return out;
}

fmi_tree* fmi_build_dist(const double* pts, const double* f, int64_t N, int degree, double tol, int max_depth,
                         const fmi_dist* dist) {
  fmi_tree* out = nullptr;
  guard([&] {
    if (!dist) fail(FMI_EINPUT, "null fmi_dist");
    out = build_impl(pts, f, N, degree, tol, max_depth, dist);
    return 0;
  });
  return out;
}

int fmi_get_unique_id(void* out128) {
  return guard([&] {
    if (!out128) fail(FMI_EINPUT, "null id buffer");
    dist_nccl_unique_id(out128);
    return 0;
  });
}

int fmi_dist_init(int rank, int world, const void* id128) {
  return guard([&] {
    if (!id128 || world < 1 || rank < 0 || rank >= world) fail(FMI_EINPUT, "invalid rank / world / id");
    require_device();
    dist_nccl_init(rank, world, id128);
    return 0;
  });
}

int fmi_dist_finalize(void) {
  return guard([&] {
    dist_nccl_finalize();
    return 0;
  });
}

int fmi_dist_allreduce(void* dev, int64_t n, int dtype) {
  return guard([&] {
    if (n < 0 || (n > 0 && !dev) || dtype < 0 || dtype > 2) fail(FMI_EINPUT, "invalid argument");
    if (n > 0 && !is_device_ptr(dev)) fail(FMI_EINPUT, "fmi_dist_allreduce needs a device pointer");
    cudaStream_t s = tl_stream;
    dist_comm_allreduce(dev, n, dtype, s);
    FMI_CK(cudaStreamSynchronize(s));
    return 0;
  });
}

int64_t fmi_dist_xbuf_bytes(int degree, int shard_depth) {
  if (degree < 0 || degree > FMI_MAX_LEVEL_DEGREE || shard_depth < 0 || shard_depth > 6) {
    set_error(FMI_EPRECOND, "degree or shard_depth out of range");
    return FMI_EPRECOND;
  }
  const int64_t L = rank3(degree), K = rank3(2 * degree), KS = (K + 3) & ~3;
  const int64_t cells = (int64_t)1 << (3 * shard_depth);           // nodes of depth shard_depth - 1, x 8
  const int64_t nglob = (cells * 8 - 1) / 7;                         // nodes of depth < shard_depth (+1 slack)
  int64_t words = std::max<int64_t>(16, nglob * KS);                 // moment-tree prefix (fp64; fp32 bound smaller)
  words = std::max(words, cells * (L + 1));                          // segment sums of the last global level
  words = std::max(words, (cells / 8 + 1) * K);                      // direct-moment fallback of one level
  return words * 8;
}

int fmi_bbox(const double* pts, int64_t N, double* out6) {
  return guard([&] {
    if (!pts || !out6 || N <= 0) fail(FMI_EINPUT, "invalid argument");
    require_device();
    cudaStream_t s = tl_stream;
    DBuf<double> own;
    const double* d = pts;
    if (!is_device_ptr(pts)) {
      own.alloc((size_t)N * 3, s);
      FMI_CK(cudaMemcpyAsync(own.p, pts, (size_t)N * 24, cudaMemcpyHostToDevice, s));
      d = own.p;
    }
    DBuf<double> bb(8, s);
    bbox_and_check(d, N, bb.p, nullptr, s);
    double hb[8];
    FMI_CK(cudaMemcpyAsync(hb, bb.p, sizeof hb, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    for (int a = 0; a < 6; ++a) out6[a] = hb[a];
    return 0;
  });
}

int fmi_cell_counts(const double* pts, int64_t N, const double* lo3, double width, int s_depth, int64_t* counts) {
  return guard([&] {
    if ((!pts && N > 0) || !lo3 || !counts || N < 0 || !(width > 0.0)) fail(FMI_EINPUT, "invalid argument");
    if (s_depth < 0 || s_depth > 6) fail(FMI_EPRECOND, "cell depth outside 0..6");
    require_device();
    cudaStream_t s = tl_stream;
    const bool unit = lo3[0] == 0.0 && lo3[1] == 0.0 && lo3[2] == 0.0 && width == 1.0;
    const int64_t nc = (int64_t)1 << (3 * s_depth);
    DBuf<double> own;
    const double* d = pts;
    if (N > 0 && !is_device_ptr(pts)) {
      own.alloc((size_t)N * 3, s);
      FMI_CK(cudaMemcpyAsync(own.p, pts, (size_t)N * 24, cudaMemcpyHostToDevice, s));
      d = own.p;
    }
    DBuf<int64_t> dc(nc, s);
    cell_counts(d, N, lo3, width, unit, s_depth, dc.p, s);
    FMI_CK(cudaMemcpyAsync(counts, dc.p, nc * 8, is_device_ptr(counts) ? cudaMemcpyDeviceToDevice
                                                                      : cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    return 0;
  });
}

int fmi_partition(const double* pts, const double* f, int64_t N, const double* lo3, double width, int s_depth,
                  const int32_t* owner, int world, double* pts_out, double* f_out, int64_t* idx_out,
                  int64_t* send_counts) {
  return guard([&] {
    if (!lo3 || !owner || !send_counts || N < 0 || world < 1 || world > 256 || !(width > 0.0) ||
        (N > 0 && (!pts || !pts_out)))
      fail(FMI_EINPUT, "invalid argument");
    if (s_depth < 0 || s_depth > 6) fail(FMI_EPRECOND, "cell depth outside 0..6");
    for (const void* p : {(const void*)pts, (const void*)f, (const void*)pts_out, (const void*)f_out,
                          (const void*)idx_out, (const void*)owner, (const void*)send_counts})
      if (p && !is_device_ptr(p)) fail(FMI_EINPUT, "fmi_partition needs device pointers");
    if (f_out && !f) fail(FMI_EINPUT, "f_out without f");
    require_device();
    cudaStream_t s = tl_stream;
    const bool unit = lo3[0] == 0.0 && lo3[1] == 0.0 && lo3[2] == 0.0 && width == 1.0;
    partition_points(pts, f, N, lo3, width, unit, s_depth, owner, world, pts_out, f_out, idx_out, send_counts, s);
    FMI_CK(cudaStreamSynchronize(s));
    return 0;
  });
}

int fmi_scatter(const double* vals, const int64_t* idx, int64_t M, double* out) {
  return guard([&] {
    if (M < 0 || (M > 0 && (!vals || !idx || !out))) fail(FMI_EINPUT, "invalid argument");
    for (const void* p : {(const void*)vals, (const void*)idx, (const void*)out})
      if (M > 0 && !is_device_ptr(p)) fail(FMI_EINPUT, "fmi_scatter needs device pointers");
    cudaStream_t s = tl_stream;
    scatter_values(vals, idx, M, out, s);
    FMI_CK(cudaStreamSynchronize(s));
    return 0;
  });
}

int fmi_eval(const fmi_tree* tree, const double* q, int64_t M, double* out) {
  return guard([&] { return eval_impl(tree, q, M, out); });
}

int fmi_transfer(const double* pts, const double* f, int64_t N, const double* q, int64_t M, double* out, int degree,
                 double tol, int max_depth) {
  return guard([&] {
    // Queries in page-locked host memory are uploaded on a side stream while the build computes (the
    // PCIe copy overlaps the fit instead of following it); other queries are copied by eval_impl.
    cudaPointerAttributes qa{};
    const bool q_pinned = q && M >= kOverlapMin && !no_overlap() && cudaPointerGetAttributes(&qa, q) == cudaSuccess &&
                          qa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    cudaStream_t s2 = nullptr;
    cudaEvent_t e_in = nullptr, e_q = nullptr;
    double* dq = nullptr;
    auto cleanup = [&] {
      if (e_in) cudaEventDestroy(e_in);
      if (e_q) cudaEventDestroy(e_q);
      if (s2) cudaStreamDestroy(s2);
    };
    std::function<void(cudaStream_t)> upload;
    if (q_pinned) {
      FMI_CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
      FMI_CK(cudaEventCreateWithFlags(&e_in, cudaEventDisableTiming));
      FMI_CK(cudaEventCreateWithFlags(&e_q, cudaEventDisableTiming));
      upload = [&](cudaStream_t cs) {
        dq = static_cast<double*>(dmalloc((size_t)M * 3 * sizeof(double), s2));
        FMI_CK(cudaEventRecord(e_in, cs));        // the input uploads are enqueued before this
        FMI_CK(cudaStreamWaitEvent(s2, e_in, 0));  // one PCIe transfer at a time
        FMI_CK(cudaMemcpyAsync(dq, q, (size_t)M * 3 * sizeof(double), cudaMemcpyHostToDevice, s2));
        FMI_CK(cudaEventRecord(e_q, s2));
      };
    }
    fmi_tree* T = nullptr;
    int rc = 0;
    try {
      T = build_impl(pts, f, N, degree, tol, max_depth, nullptr, upload);
      if (dq) {
        FMI_CK(cudaStreamWaitEvent(tl_stream, e_q, 0));
        rc = eval_impl(T, dq, M, out);
      } else {
        rc = eval_impl(T, q, M, out);
      }
    } catch (...) {
      if (T) fmi_free(T);
      if (dq) { cudaStreamSynchronize(s2); dfree(dq, tl_stream); }
      cleanup();
      throw;
    }
    fmi_free(T);
    if (dq) dfree(dq, tl_stream);
    FMI_CK(cudaStreamSynchronize(tl_stream));
    cleanup();
    return rc;
  });
}


int fmi_save(const fmi_tree* T, const char* path) {
  return guard([&] {
    if (!T || !path) fail(FMI_EINPUT, "null argument");
    FILE* fp = fopen(path, "wb");
    if (!fp) fail(FMI_EINPUT, std::string("cannot open ") + path);
    try {
      FileHeader h{};
      std::memcpy(h.magic, kMagic, 8);
      h.version = kFileVersion;
      h.p = T->p;
      h.depth_max = T->depth_max;
      h.unit = T->unit;
      h.nodes = T->nodes;
      h.N = T->Ntot;
      for (int a = 0; a < 3; ++a) h.lo[a] = T->lo[a];
      h.width = T->width;
      h.tau = T->tau;
      h.D = T->D;
      if (fwrite(&h, sizeof h, 1, fp) != 1) fail(FMI_EINPUT, "short write");
      const int64_t n = T->nodes, L = T->L;
      cudaStream_t s = tl_stream;
      dump(fp, T->nt.cell, n, s);
      dump(fp, T->nt.parent, n, s);
      dump(fp, T->nt.child, n * 8, s);
      dump(fp, T->nt.child_n, n * 8, s);
      dump(fp, T->nt.child_ss, n * 8, s);
      dump(fp, T->nt.coef, n * L, s);
      dump(fp, T->nt.pcoef, n * L, s);
      dump(fp, T->nt.rms, n, s);
      dump(fp, T->nt.minpiv, n, s);
      dump(fp, T->nt.rank, n, s);
      dump(fp, T->nt.flag, n, s);
    } catch (...) {
      fclose(fp);
      throw;
    }
    fclose(fp);
    return 0;
  });
}

fmi_tree* fmi_load(const char* path) {
  fmi_tree* out = nullptr;
  guard([&] {
    if (!path) fail(FMI_EINPUT, "null path");
    require_device();
    FILE* fp = fopen(path, "rb");
    if (!fp) fail(FMI_EINPUT, std::string("cannot open ") + path);
    fmi_tree* T = nullptr;
    cudaStream_t s = tl_stream;
    try {
      FileHeader h{};
      if (fread(&h, sizeof h, 1, fp) != 1 || std::memcmp(h.magic, kMagic, 8) != 0)
        fail(FMI_EVERSION, "not an fmi tree file");
      if (h.version != kFileVersion) fail(FMI_EVERSION, "unsupported tree file version");
      if (h.p < 0 || h.p > FMI_MAX_DEGREE || h.nodes < 1 || h.nodes > (int64_t(1) << 31) - 1 || h.depth_max < 0 ||
          h.depth_max > FMI_MAX_DEPTH || h.D < 0 || h.D > FMI_MAX_DEPTH || h.depth_max > h.D ||
          !(h.width > 0) || !std::isfinite(h.width) ||
          !std::isfinite(h.lo[0]) || !std::isfinite(h.lo[1]) || !std::isfinite(h.lo[2]) || !(h.tau >= 0) || h.N < 0)
        fail(FMI_EVERSION, "corrupt tree file header");
      T = new fmi_tree();
      T->p = h.p;
      T->L = rank3(h.p);
      T->K = rank3(2 * h.p);
      T->D = h.D;
      T->Dk = h.D + 1;
      T->depth_max = h.depth_max;
      T->unit = h.unit != 0;
      T->N = 0;  // no fit points: fmi_residual is unavailable
      T->Ntot = h.N;
      for (int a = 0; a < 3; ++a) T->lo[a] = h.lo[a];
      T->width = h.width;
      T->tau = h.tau;
      T->stream = s;
      ensure_table(T->nt, T->cap, h.nodes, T->L, true, s);
      T->nodes = h.nodes;
      const int64_t n = h.nodes, L = T->L;
      const std::vector<int4> cell = undump(fp, T->nt.cell, n, s);
      const std::vector<int32_t> parent = undump(fp, T->nt.parent, n, s);
      const std::vector<int32_t> child = undump(fp, T->nt.child, n * 8, s);
      undump(fp, T->nt.child_n, n * 8, s);
      undump(fp, T->nt.child_ss, n * 8, s);
      undump(fp, T->nt.coef, n * L, s);
      undump(fp, T->nt.pcoef, n * L, s);
      undump(fp, T->nt.rms, n, s);
      undump(fp, T->nt.minpiv, n, s);
      const std::vector<int32_t> rank = undump(fp, T->nt.rank, n, s);
      undump(fp, T->nt.flag, n, s);
      validate_nodes(cell, parent, child, rank, h.depth_max, h.D, (int)L);
      // level bookkeeping from the (canonical, level-contiguous) depths
      for (int64_t i = 0; i < n; ++i) {
        const int d = cell[i].w;
        if (d >= (int)T->lvl_first.size()) {
          T->lvl_first.push_back(i);
          T->lvl_count.push_back(0);
          T->lvl_points.push_back(0);
        }
        T->lvl_count[d]++;
      }
      // start/end are not stored (no fit points); zero them for the export
      FMI_CK(cudaMemsetAsync(T->nt.start, 0, (size_t)n * 8, s));
      FMI_CK(cudaMemsetAsync(T->nt.end, 0, (size_t)n * 8, s));
      FMI_CK(cudaMemsetAsync(T->nt.child_start, 0, (size_t)n * 9 * 8, s));
      FMI_CK(cudaStreamSynchronize(s));
    } catch (...) {
      fclose(fp);
      if (T) {
        free_table(T->nt, s);
        delete T;
      }
      throw;
    }
    fclose(fp);
    out = T;
    return 0;
  });
  return out;
}

void fmi_free(fmi_tree* T) {
  if (!T) return;
  cudaStream_t s = tl_stream;
  free_table(T->nt, s);
  dfree(T->residual, s);
  dfree(T->perm, s);
  cudaStreamSynchronize(s);
  cudaGetLastError();
  delete T;
}

int fmi_last_error(const char** msg) {
  if (msg) *msg = tl_msg.c_str();
  return tl_err;
}

int fmi_set_stream(void* stream) {
  tl_stream = static_cast<cudaStream_t>(stream);
  return 0;
}

int64_t fmi_node_count(const fmi_tree* T) {
  if (!T) { set_error(FMI_EINPUT, "null tree"); return FMI_EINPUT; }
  return T->nodes;
}

int fmi_rank(const fmi_tree* T) {
  if (!T) { set_error(FMI_EINPUT, "null tree"); return FMI_EINPUT; }
  return T->L;
}

int64_t fmi_export_nodes(const fmi_tree* T, fmi_node* out, double* coeffs, int64_t cap) {
  int64_t written = 0;
  int rc = guard([&] {
    if (!T || !out) fail(FMI_EINPUT, "null argument");
    const int64_t n = std::min<int64_t>(cap, T->nodes);
    if (n <= 0) return 0;
    const int L = T->L;
    const int64_t nn = T->nodes;
    std::vector<int64_t> st(nn), en(nn), cs(nn * 9), cn(nn * 8);
    std::vector<int4> cell(nn);
    std::vector<int32_t> par(nn), child(nn * 8), rank(nn), flag(nn);
    std::vector<double> ss(nn * 8), rms(nn), mp(nn), coef((size_t)nn * L);
    cudaStream_t s = tl_stream;
    FMI_CK(cudaMemcpyAsync(st.data(), T->nt.start, nn * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(en.data(), T->nt.end, nn * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(cs.data(), T->nt.child_start, nn * 9 * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(cn.data(), T->nt.child_n, nn * 8 * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(cell.data(), T->nt.cell, nn * sizeof(int4), cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(par.data(), T->nt.parent, nn * 4, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(child.data(), T->nt.child, nn * 8 * 4, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(rank.data(), T->nt.rank, nn * 4, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(flag.data(), T->nt.flag, nn * 4, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(ss.data(), T->nt.child_ss, nn * 8 * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(rms.data(), T->nt.rms, nn * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(mp.data(), T->nt.minpiv, nn * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaMemcpyAsync(coef.data(), T->nt.coef, (size_t)nn * L * 8, cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    // factorials of the basis (P_F = a_lmn · l! m! n!)
    std::vector<double> fac(L);
    {
      double f1[32];
      f1[0] = 1.0;
      for (int i = 1; i < 32; ++i) f1[i] = f1[i - 1] * i;
      int i = 0;
      for (int l = 0; l <= T->p; ++l)
        for (int m = 0; m <= T->p - l; ++m)
          for (int k = 0; k <= T->p - l - m; ++k) fac[i++] = f1[l] * f1[m] * f1[k];
    }
    for (int64_t i = 0; i < n; ++i) {
      fmi_node& o = out[i];
      std::memset(&o, 0, sizeof o);
      o.depth = cell[i].w;
      o.cell[0] = cell[i].x; o.cell[1] = cell[i].y; o.cell[2] = cell[i].z;
      o.prefix = morton_label(cell[i].w, cell[i].x, cell[i].y, cell[i].z);
      o.n_points = 0;
      for (int k = 0; k < 8; ++k) o.n_points += cn[i * 8 + k];
      o.rank = rank[i];
      o.parent = par[i];
      o.flags = flag[i];
      o.residual_rms = rms[i];
      o.min_pivot = mp[i];
      for (int k = 0; k < 8; ++k) {
        const int64_t no = cn[i * 8 + k];  // global counts for the global nodes of a sharded build
        o.child_count[k] = no;
        o.child_rms[k] = no > 0 ? std::sqrt(ss[i * 8 + k] / (double)no) : NAN;
        o.child[k] = child[i * 8 + k];
      }
      if (coeffs)
        for (int j = 0; j < L; ++j) coeffs[i * L + j] = coef[(size_t)i * L + j] * fac[j];
    }
    written = n;
    return 0;
  });
  return rc ? rc : written;
}

int fmi_root_cube(const fmi_tree* T, double* lo3, double* width) {
  if (!T || !lo3 || !width) { set_error(FMI_EINPUT, "null argument"); return FMI_EINPUT; }
  for (int a = 0; a < 3; ++a) lo3[a] = T->lo[a];
  *width = T->width;
  return 0;
}

int fmi_residual(const fmi_tree* T, double* out) {
  return guard([&] {
    if (!T || !out) fail(FMI_EINPUT, "null argument");
    if (!T->residual) fail(FMI_EINPUT, "the tree has no fit points (loaded from a file)");
    cudaStream_t s = tl_stream;
    DBuf<double> tmp;
    double* d = out;
    const bool host = !is_device_ptr(out);
    if (host) { tmp.alloc(T->N, s); d = tmp.p; }
    FMI_LAUNCH(KID_MISC, s, k_scatter_residual, (unsigned)((T->N + 255) / 256), 256, 0, T->residual, T->perm, T->N, d);
    if (host) FMI_CK(cudaMemcpyAsync(out, d, T->N * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMI_CK(cudaStreamSynchronize(s));
    return 0;
  });
}

int fmi_level_stats(const fmi_tree* T, int64_t* nodes, int64_t* points, int cap) {
  if (!T) { set_error(FMI_EINPUT, "null tree"); return FMI_EINPUT; }
  int n = (int)T->lvl_count.size();
  for (int i = 0; i < std::min(n, cap); ++i) {
    if (nodes) nodes[i] = T->lvl_count[i];
    if (points) points[i] = T->lvl_points[i];
  }
  return n;
}

int fmi_build_stats(const fmi_tree* T, int64_t* out, int cap) {
  if (!T || !out) { set_error(FMI_EINPUT, "null argument"); return FMI_EINPUT; }
  const int64_t v[4] = {T->mt_nodes, T->direct_nodes, T->refined_nodes, T->deferred_children};
  const int n = std::min(cap, 4);
  for (int i = 0; i < n; ++i) out[i] = v[i];
  return 4;
}

int fmi_profile_enable(int on) {
  g_prof.store(on != 0);
  return 0;
}

int fmi_profile_select(const char* kernels) {
  if (!kernels || !*kernels) {
    g_prof_mask.store(~0u);
    return 0;
  }
  uint32_t mask = 0;
  const char* b = kernels;
  while (*b) {
    const char* e = b;
    while (*e && *e != ',') ++e;
    int hit = -1;
    for (int k = 0; k < KID_COUNT; ++k)
      if (std::strlen(kNames[k]) == (size_t)(e - b) && std::strncmp(kNames[k], b, (size_t)(e - b)) == 0) hit = k;
    if (hit < 0) {
      set_error(FMI_EINPUT, "fmi_profile_select: unknown kernel name in '" + std::string(kernels) + "'");
      return FMI_EINPUT;
    }
    mask |= 1u << hit;
    b = *e ? e + 1 : e;
  }
  g_prof_mask.store(mask);
  return 0;
}

int fmi_profile_reset(void) {
  prof_collect();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int k = 0; k < KID_COUNT; ++k) { g_prof_ms[k] = 0.0; g_prof_n[k] = 0; g_prof_units[k] = 0; }
  g_launches.store(0);
  return 0;
}

int fmi_profile_get(const char* kernel, double* total_ms, int64_t* launches) {
  prof_collect();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int k = 0; k < KID_COUNT; ++k) {
    if (kernel && std::strcmp(kernel, kNames[k]) == 0) {
      if (total_ms) *total_ms = g_prof_ms[k];
      if (launches) *launches = g_prof_n[k];
      return 0;
    }
  }
  set_error(FMI_EINPUT, "unknown kernel name");
  return FMI_EINPUT;
}

int fmi_profile_units(const char* kernel, int64_t* units) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int k = 0; k < KID_COUNT; ++k) {
    if (kernel && std::strcmp(kernel, kNames[k]) == 0) {
      if (units) *units = g_prof_units[k];
      return 0;
    }
  }
  set_error(FMI_EINPUT, "unknown kernel name");
  return FMI_EINPUT;
}

int64_t fmi_launch_count(void) { return g_launches.load(); }

int64_t fmi_guard_violations(void) { return fmi::guard_violations(); }

}  // extern "C"
