/*
 * fmi.h — C ABI of the B200-native free-mesh interpolator (arXiv 1511.01353, Challacombe,
 * "A N-Body Solver for Free Mesh Interpolation").
 *
 * The library implements the data-parallel hot path of the paper's Free Mesh Transform:
 *   fmi_build — the top-down octree residual fit, Algorithm 1 (FMT_Mesh_to_Tree,
 *               P:294-314) with Algorithm 2 (FMT_Mesh_to_Moments) at every node;
 *   fmi_eval  — the interpolant f(r) = Λ(r)·F_p summed over each query's root-to-deepest-node
 *               path (§2; "only downward recursion to accumulate local polynomial
 *               representation of the residual", §4).
 * Citations: P:<line> = PAPER.md line; G<k> = reading k of the paper-gap ledger.
 *
 * Every step runs in hand-written CUDA kernels for sm_100a; there is no CPU fallback.  All
 * arithmetic is IEEE fp64.
 *
 * Conventions shared by all calls
 *   - Pointers may be host or device pointers (detected with cudaPointerGetAttributes).  Host
 *     inputs are copied to the device inside the call; host outputs are copied back.
 *   - The caller owns every array it passes; the library never keeps or frees them and never
 *     writes to input arrays (the paper overwrites x and f in place; we copy).
 *   - Work is issued on the stream set with fmi_set_stream (default: the legacy default stream)
 *     and every call returns after that stream is synchronised.
 *   - Errors: functions returning int return 0 on success or a negative FMI_E* code; functions
 *     returning a pointer return NULL.  fmi_last_error() returns the code and a message of the
 *     last failure on the calling thread.
 *   - Not thread-safe for concurrent calls on the same tree handle; distinct handles may be used
 *     from distinct threads if each thread sets its own stream.
 */
#ifndef FMI_H_
#define FMI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMI_OK 0
#define FMI_EINPUT (-1)      /* null pointer, N < 0, M < 0, non-finite coordinate or value      */
#define FMI_EPRECOND (-2)    /* N < 𝓛 (root underdetermined), degree/max_depth/tol range */
#define FMI_EVERSION (-3)    /* reserved (tree import)                                           */
#define FMI_ENUMERIC (-4)    /* non-finite coefficients (unreachable with the pivot guard)       */
#define FMI_ECUDA (-5)       /* CUDA runtime error or no CUDA device                            */
#define FMI_ENCCL (-6)       /* a collective of a sharded build failed (the fmi_dist callback)     */
#define FMI_ENOMEM (-7)      /* device allocation failed                                         */

#define FMI_MAX_DEGREE 14        /* degrees p = 0..14 (𝓛 up to 680); p > 10 only unscoped (below)  */
#define FMI_MAX_LEVEL_DEGREE 10  /* the octree (level) path and sharded builds: p = 0..10 (𝓛 <= 286)  */
#define FMI_MAX_DEPTH 20     /* keys carry max_depth+1 <= 21 levels (63-bit Morton keys)           */

typedef struct fmi_tree fmi_tree; /* opaque; owned by the library until fmi_free */

/*
 * fmi_build — fit the octree interpolant to N scattered samples.
 *   pts        N×3 row-major fp64 (x0,y0,z0,x1,...), host or device.
 *   f          N fp64 sample values, host or device.
 *   N          number of points, N >= 𝓛 = (p+1)(p+2)(p+3)/6 (G1).
 *   degree     total degree p of the local polynomials, 0 <= p <= FMI_MAX_DEGREE.  The basis is the
 *              geometric moments Λ_lmn(u) = u1^l u2^m u3^n/(l!m!n!) in Algorithm-2 loop order
 *              (P:185-189).  Degrees 11..14 (𝓛 up to 680) are the paper's unscoped
 *              experiment (§3, Fig. 1) and need max_depth = 0:
 *              FMI_EPRECOND otherwise.  Such a fit (and any max_depth = 0 fit when the environment
 *              sets FMI_UNSCOPED_QR=1) is computed by the QR path of DESIGN.md §5 "f2": the R of the
 *              monomial Vandermonde as R_V·C through the Legendre basis, then the same rejection walk.
 *   tol        τ >= 0: an octant block becomes a child iff E_RMS > τ and n_o >= 𝓛
 *              and depth+1 <= max_depth (G5).  E_RMS = sqrt(Σ r²/n_o) over the post-fit residual.
 *   max_depth  0..FMI_MAX_DEPTH, root depth 0.
 * Root frame (G6): the cube [0,1]^3 if every point lies in it, else the isotropic bounding cube.
 * Node fit (G9): the least-squares fit of Algorithm 2 computed from the column-equilibrated
 * moment Gram with a column-rejection Cholesky (a column whose residual norm against the kept
 * columns is <= 1e-6 of its own norm is dropped, coefficient 0).
 * Returns a tree handle or NULL (see fmi_last_error).
 */
fmi_tree* fmi_build(const double* pts, const double* f, int64_t N, int degree, double tol, int max_depth);

/*
 * Sharded (multi-GPU) build — SURVEY.md §8(e), DESIGN.md §6.  One process (or thread) per shard, each
 * with its own device/stream.  The shards' points are partitioned by the cells of depth shard_depth
 * (s) of the common root cube: all points of a depth-s cell must be on one shard (fmi_cell_counts +
 * fmi_partition + an all-to-all exchange do that).  Nodes of depth < s ("global" nodes) are built from
 * sums over all shards: moments, projections, octant counts and residual energies are summed by the
 * caller-provided collective; every shard then holds identical global nodes (same solve, same
 * decisions).  Nodes of depth >= s are local to the shard holding their cell: no communication.
 * With s > max_depth every node is global and the points may be partitioned arbitrarily.
 *   allreduce        NULL: the library-owned NCCL communicator (fmi_dist_init over the same world) sums
 *                    in place on the device buffers, on the library stream — the multi-GPU path.
 *                    Otherwise a caller collective (the single-GPU virtual-shard tests):
 *   xbuf/xbuf_bytes  device exchange buffer owned by the caller (>= fmi_dist_xbuf_bytes())
 *   allreduce        collective in-place SUM over all shards of the first n elements of xbuf
 *                    (dtype 0 = fp64, 1 = int64, 2 = fp32); called from the building thread, after
 *                    the library stream was synchronised; must complete before returning; returns 0
 *                    or non-zero on failure (-> FMI_ENCCL).  Every shard makes the same sequence of
 *                    calls with the same n.
 *   lo, width        the common root cube (G6) — every shard must pass the same.
 * N may be 0 on a shard.  The tree a shard returns holds the global nodes and its local subtrees;
 * fmi_eval on it is correct for queries in the cells it owns and for any query whose deepest node is
 * global.
 */
typedef struct {
  int rank, world;
  int shard_depth;
  double lo[3], width;
  void* xbuf;
  int64_t xbuf_bytes;
  int (*allreduce)(void* ctx, int64_t n, int dtype);
  void* ctx;
} fmi_dist;

fmi_tree* fmi_build_dist(const double* pts, const double* f, int64_t N, int degree, double tol, int max_depth,
                         const fmi_dist* dist);

/*
 * Library-owned NCCL communicator (one per process, one process per GPU).
 *   fmi_get_unique_id   rank 0: write the 128-byte NCCL unique id to out128 (host memory); the caller
 *                       broadcasts it to the other ranks (e.g. torch.distributed).
 *   fmi_dist_init       collective over the world ranks (current CUDA device): creates the communicator
 *                       (replacing a previous one).  A sharded build whose fmi_dist has allreduce == NULL
 *                       then sums its global-level quantities with ncclAllReduce in place on the device
 *                       buffers, on the library stream (no exchange buffer, no host round trip).
 *   fmi_dist_finalize   destroy the communicator (idempotent).
 *   fmi_dist_allreduce  in-place SUM over the ranks of n elements at the DEVICE pointer dev (dtype 0 fp64,
 *                       1 int64, 2 fp32) on the library stream; returns after it completed.
 * NCCL is loaded at run time (libnccl.so.2, the one the process already has when torch is imported).
 * All return 0, FMI_EINPUT (bad argument), FMI_ECUDA (no device) or FMI_ENCCL (NCCL missing / failed,
 * or no communicator).
 */
int fmi_get_unique_id(void* out128);
int fmi_dist_init(int rank, int world, const void* id128);
int fmi_dist_finalize(void);
int fmi_dist_allreduce(void* dev, int64_t n, int dtype);

/* Exchange-buffer size (bytes) a sharded build needs for this degree and shard depth. */
int64_t fmi_dist_xbuf_bytes(int degree, int shard_depth);

/* Helpers of the sharded build and of query routing (device kernels; pointers host or device).
 *   fmi_bbox         out6 = min x,y,z, max x,y,z of the N points (host out); 0 or a code.
 *   fmi_cell_counts  counts[8^s] (int64) of points per depth-s cell of the root cube (lo, width),
 *                    cells numbered by Morton label; s in 0..6.
 *   fmi_partition    stable partition of the points by the owner shard of their depth-s cell
 *                    (owner[8^s] int32 in 0..world-1): pts_out/f_out/idx_out (any may be NULL except
 *                    pts_out) receive the points grouped by destination shard, idx_out their original
 *                    indices; send_counts[world] (int64) the group sizes.
 *   fmi_scatter      out[idx[i]] = vals[i], i < M (returns results to the caller's order). */
int fmi_bbox(const double* pts, int64_t N, double* out6);
int fmi_cell_counts(const double* pts, int64_t N, const double* lo3, double width, int s, int64_t* counts);
int fmi_partition(const double* pts, const double* f, int64_t N, const double* lo3, double width, int s,
                  const int32_t* owner, int world, double* pts_out, double* f_out, int64_t* idx_out,
                  int64_t* send_counts);
int fmi_scatter(const double* vals, const int64_t* idx, int64_t M, double* out);

/*
 * fmi_eval — evaluate the interpolant at M query points.
 *   q    M×3 row-major fp64, host or device.
 *   out  M fp64, host or device, caller-allocated; written in q's order.
 * A query outside the root cube receives the root polynomial only (extrapolation).
 * Returns 0 or a negative FMI_E* code.
 */
int fmi_eval(const fmi_tree* tree, const double* q, int64_t M, double* out);

/*
 * fmi_transfer — the paper's mesh-to-mesh transfer f_p -> f_q (§2: f'_q = Λ'·F_p):
 * fmi_build over (pts, f, N) + fmi_eval at (q, M) into out + fmi_free, in one call.  Arguments and
 * errors as fmi_build / fmi_eval.  Returns 0 or a negative FMI_E* code.
 */
int fmi_transfer(const double* pts, const double* f, int64_t N, const double* q, int64_t M, double* out, int degree,
                 double tol, int max_depth);

/*
 * Tree files (layout after SPEC's FMT1 node records): header (magic "FMITREE1", version,
 * degree, depth, root cube, τ, point count) + per-node cell, parent, children, octant counts and
 * energies, coefficients P_F (monomial form) and the pre-summed polynomials, rms, pivots, ranks, flags.
 * fmi_save returns 0 or a code; fmi_load returns a tree (NULL on error: FMI_EVERSION for a foreign or
 * corrupt file).  A loaded tree evaluates and exports like a built one; fmi_residual is unavailable.
 */
int fmi_save(const fmi_tree* tree, const char* path);
fmi_tree* fmi_load(const char* path);

/* fmi_free — release the tree and its device memory.  NULL-safe. */
void fmi_free(fmi_tree* tree);

/* fmi_last_error — code of the last failure on this thread (0 if none); *msg (optional) points to a
 * thread-local message valid until the next library call on this thread. */
int fmi_last_error(const char** msg);

/* fmi_set_stream — CUDA stream (cudaStream_t passed as void*) for subsequent calls on this thread;
 * NULL = legacy default stream. */
int fmi_set_stream(void* stream);

/* ------------------------------------------------------------------------------------------------
 * Introspection (parity harness and benchmark; not on the timed path).
 * ------------------------------------------------------------------------------------------------ */

typedef struct {
  int32_t depth;          /* root = 0                                                          */
  int32_t cell[3];        /* integer cell (i,j,k) at this depth; centre (2i+1)/2^(d+1) in the   */
                          /* root cube's unit coordinates, half-width 1/2^(d+1)  */
  uint64_t prefix;        /* Morton label: level digits o = bx + 2by + 4bz, most significant    */
                          /* first (G7)                                                  */
  int64_t n_points;       /* points of the node                                                */
  int32_t rank;           /* kept columns (𝓛 unless truncated, G9)                             */
  int32_t parent;         /* index in the exported order of the parent, -1 for the root       */
  int32_t flags;          /* bit 0: fitted by the Householder-QR path (ill-conditioned node)   */
  int32_t reserved;
  double residual_rms;    /* sqrt(Σ r²/n) over the node's points after its own fit            */
  double min_pivot;       /* smallest kept Cholesky pivot sqrt(s_jj) of the equilibrated Gram */
  int64_t child_count[8]; /* n_o of each octant block                                 */
  double child_rms[8];    /* E_RMS of each octant block; NaN if n_o == 0              */
  int32_t child[8];       /* exported index of the child node or -1                           */
} fmi_node;

/* Number of nodes of the tree (or a negative code). */
int64_t fmi_node_count(const fmi_tree* tree);

/* Coefficient count 𝓛 of the tree (or a negative code). */
int fmi_rank(const fmi_tree* tree);

/* Export up to cap nodes in canonical (depth, prefix) order.  coeffs (may be NULL) receives
 * cap×𝓛 doubles: P_F of each node in the Λ basis and Algorithm-2 column order.
 * Returns the number of nodes written or a negative code. */
int64_t fmi_export_nodes(const fmi_tree* tree, fmi_node* out, double* coeffs, int64_t cap);

/* Root cube of the tree: lo[3] and edge width (G6). */
int fmi_root_cube(const fmi_tree* tree, double* lo3, double* width);

/* Final residual r_i (after the deepest fit containing point i) in INPUT order; out is N fp64,
 * host or device.  Bookkeeping identity: interpolant(x_i) + r_i = f_i. */
int fmi_residual(const fmi_tree* tree, double* out);

/* Build statistics: levels, and per level (up to cap entries) the active node count and the
 * number of points in active nodes (point-levels). Returns the number of levels. */
int fmi_level_stats(const fmi_tree* tree, int64_t* nodes, int64_t* points, int cap);

/* Build statistics: out[0] = moment-tree nodes (cells with >= 8𝓛 points down to max_depth),
 * out[1] = fit nodes whose moments were accumulated directly (below the moment tree, or the translated
 * moments failed the rounding check), out[2] = fit nodes that took semi-normal refinement steps,
 * out[3] = children whose projections ran in a deferred pass.  Returns the number of statistics (4)
 * or a negative code; writes min(cap, 4) entries. */
int fmi_build_stats(const fmi_tree* tree, int64_t* out, int cap);

/* ------------------------------------------------------------------------------------------------
 * Profiling (bench.py).  When enabled, every kernel launch of the library is bracketed by CUDA
 * events on the library stream; fmi_profile_get returns, per kernel name, the summed device time
 * in ms and the launch count since the last fmi_profile_reset.
 * ------------------------------------------------------------------------------------------------ */
int fmi_profile_enable(int on);
int fmi_profile_reset(void);
/* kernel names: "keys", "sort", "gather", "moments", "moments_reduce", "solve", "children",
 * "residual", "residual_reduce", "decide", "chunks", "scan", "eval", "misc", "project", "m2m",
 * "level_gather", "refine_solve", "refine", "presum", "unscoped_gram", "unscoped_solve", "solve_qr" */
int fmi_profile_get(const char* kernel, double* total_ms, int64_t* launches);
/* Algorithmic work units the kernel's launches processed since the last reset (while enabled):
 * "keys" keyed points + queries, "sort" items summed over the 8-bit passes actually executed,
 * "solve" nodes factored by the Gram solve (K5), "refine_solve" node substitutions (K5r).
 * bench.py multiplies them by the per-unit bytes / flops of DESIGN.md §5.  0 / FMI_EINPUT. */
int fmi_profile_units(const char* kernel, int64_t* units);
/* Restrict the event timing to the named kernels (comma-separated names from the list above, no spaces;
 * NULL or "" = every kernel, the default).  bench.py times only the kernels it reports rooflines for
 * inside its timed region: bracketing every one of the ~200 small launches of a step with events costs
 * ~1.9 ms per cfg-5 step on the host launch path.  Launch and unit counters are not
 * affected.  0 / FMI_EINPUT (unknown name; the selection is left unchanged). */
int fmi_profile_select(const char* kernels);
/* Total kernel launches issued by the library since load (or since fmi_profile_reset). */
int64_t fmi_launch_count(void);
/* Diagnostics (a stand-in for compute-sanitizer memcheck, which is closed on the GPU pool): with the
 * environment variable FMI_GUARD=1 set before the first build, every library-owned device buffer gets
 * 4 KiB guard bands (0xA5) before and after it, checked when the buffer is freed; returns the number of
 * overwritten guard bands seen since load (each also reported on stderr).  0 when FMI_GUARD is off. */
int64_t fmi_guard_violations(void);

#ifdef __cplusplus
}
#endif

#endif /* FMI_H_ */
