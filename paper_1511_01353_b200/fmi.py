"""Thin ctypes binding of ``libfmi.so`` (include/fmi.h).  Argument marshalling only: every step of the
fit and the evaluation runs in the library's CUDA kernels.  There is no CPU fallback: importing this
module without the built library, or calling it without a CUDA device, raises.

Arrays may be numpy arrays (host memory; copied inside the call) or CUDA torch tensors (device
memory; used in place).  All arrays are float64, C-contiguous; points are (N, 3) row-major.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfmi.so")

FMI_OK = 0
FMI_EINPUT = -1
FMI_EPRECOND = -2
FMI_EVERSION = -3
FMI_ENUMERIC = -4
FMI_ECUDA = -5
FMI_ENCCL = -6
FMI_ENOMEM = -7
MAX_DEGREE = 14        # p > MAX_LEVEL_DEGREE only with max_depth = 0 (unscoped fit, f2)
MAX_LEVEL_DEGREE = 10
MAX_DEPTH = 20

# every symbol include/fmi.h declares (tests check the library exports all of them)
EXPORTED = (
    "fmi_build", "fmi_eval", "fmi_free", "fmi_last_error", "fmi_set_stream", "fmi_node_count", "fmi_rank",
    "fmi_export_nodes", "fmi_root_cube", "fmi_residual", "fmi_level_stats", "fmi_profile_enable",
    "fmi_profile_reset", "fmi_profile_get", "fmi_launch_count", "fmi_guard_violations", "fmi_build_stats", "fmi_build_dist",
    "fmi_dist_xbuf_bytes", "fmi_bbox", "fmi_cell_counts", "fmi_partition", "fmi_scatter", "fmi_transfer",
    "fmi_save", "fmi_load", "fmi_profile_units", "fmi_profile_select",
    "fmi_get_unique_id", "fmi_dist_init", "fmi_dist_finalize", "fmi_dist_allreduce",
)

# allreduce(ctx, n, dtype) -> int: in-place SUM of the first n elements of the exchange buffer
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int)


class FmiDist(ctypes.Structure):
    """struct fmi_dist (include/fmi.h): shard rank/world, shard depth, common root cube, exchange buffer
    and the collective-sum callback of a sharded build."""
    _fields_ = [
        ("rank", ctypes.c_int), ("world", ctypes.c_int), ("shard_depth", ctypes.c_int),
        ("lo", ctypes.c_double * 3), ("width", ctypes.c_double),
        ("xbuf", ctypes.c_void_p), ("xbuf_bytes", ctypes.c_int64),
        ("allreduce", ALLREDUCE_FN), ("ctx", ctypes.c_void_p),
    ]

KERNELS = ("keys", "sort", "gather", "moments", "moments_reduce", "solve", "children", "residual",
           "residual_reduce", "decide", "chunks", "scan", "eval", "misc", "project", "m2m", "level_gather",
           "refine_solve", "refine", "presum", "unscoped_gram", "unscoped_solve", "solve_qr")


class FmiNode(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_int32), ("cell", ctypes.c_int32 * 3), ("prefix", ctypes.c_uint64),
        ("n_points", ctypes.c_int64), ("rank", ctypes.c_int32), ("parent", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("residual_rms", ctypes.c_double), ("min_pivot", ctypes.c_double),
        ("child_count", ctypes.c_int64 * 8), ("child_rms", ctypes.c_double * 8), ("child", ctypes.c_int32 * 8),
    ]


class FmiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fmi error {code}: {msg}")
        self.code = code


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfmi.so (raises if it is missing: build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, D, I64, I32, VP = ctypes.POINTER, ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.fmi_build.restype = VP
    lib.fmi_build.argtypes = [VP, VP, I64, I32, D, I32]
    lib.fmi_eval.restype = I32
    lib.fmi_eval.argtypes = [VP, VP, I64, VP]
    lib.fmi_free.restype = None
    lib.fmi_free.argtypes = [VP]
    lib.fmi_last_error.restype = I32
    lib.fmi_last_error.argtypes = [P(ctypes.c_char_p)]
    lib.fmi_set_stream.restype = I32
    lib.fmi_set_stream.argtypes = [VP]
    lib.fmi_node_count.restype = I64
    lib.fmi_node_count.argtypes = [VP]
    lib.fmi_rank.restype = I32
    lib.fmi_rank.argtypes = [VP]
    lib.fmi_export_nodes.restype = I64
    lib.fmi_export_nodes.argtypes = [VP, P(FmiNode), VP, I64]
    lib.fmi_root_cube.restype = I32
    lib.fmi_root_cube.argtypes = [VP, P(D), P(D)]
    lib.fmi_residual.restype = I32
    lib.fmi_residual.argtypes = [VP, VP]
    lib.fmi_level_stats.restype = I32
    lib.fmi_level_stats.argtypes = [VP, P(I64), P(I64), I32]
    lib.fmi_profile_enable.restype = I32
    lib.fmi_profile_enable.argtypes = [I32]
    lib.fmi_profile_reset.restype = I32
    lib.fmi_profile_reset.argtypes = []
    lib.fmi_profile_select.restype = I32
    lib.fmi_profile_select.argtypes = [ctypes.c_char_p]
    lib.fmi_profile_get.restype = I32
    lib.fmi_profile_get.argtypes = [ctypes.c_char_p, P(D), P(I64)]
    lib.fmi_get_unique_id.restype = I32
    lib.fmi_get_unique_id.argtypes = [VP]
    lib.fmi_dist_init.restype = I32
    lib.fmi_dist_init.argtypes = [I32, I32, VP]
    lib.fmi_dist_finalize.restype = I32
    lib.fmi_dist_finalize.argtypes = []
    lib.fmi_dist_allreduce.restype = I32
    lib.fmi_dist_allreduce.argtypes = [VP, I64, I32]
    lib.fmi_profile_units.restype = I32
    lib.fmi_profile_units.argtypes = [ctypes.c_char_p, P(I64)]
    lib.fmi_build_dist.restype = VP
    lib.fmi_build_dist.argtypes = [VP, VP, I64, I32, D, I32, P(FmiDist)]
    lib.fmi_dist_xbuf_bytes.restype = I64
    lib.fmi_dist_xbuf_bytes.argtypes = [I32, I32]
    lib.fmi_bbox.restype = I32
    lib.fmi_bbox.argtypes = [VP, I64, P(D)]
    lib.fmi_cell_counts.restype = I32
    lib.fmi_cell_counts.argtypes = [VP, I64, P(D), D, I32, VP]
    lib.fmi_partition.restype = I32
    lib.fmi_partition.argtypes = [VP, VP, I64, P(D), D, I32, VP, I32, VP, VP, VP, VP]
    lib.fmi_scatter.restype = I32
    lib.fmi_scatter.argtypes = [VP, VP, I64, VP]
    lib.fmi_transfer.restype = I32
    lib.fmi_transfer.argtypes = [VP, VP, I64, VP, I64, VP, I32, D, I32]
    lib.fmi_save.restype = I32
    lib.fmi_save.argtypes = [VP, ctypes.c_char_p]
    lib.fmi_load.restype = VP
    lib.fmi_load.argtypes = [ctypes.c_char_p]
    lib.fmi_build_stats.restype = I32
    lib.fmi_build_stats.argtypes = [VP, P(I64), I32]
    lib.fmi_launch_count.restype = I64
    lib.fmi_launch_count.argtypes = []
    lib.fmi_guard_violations.restype = I64
    lib.fmi_guard_violations.argtypes = []
    _lib = lib
    return lib


def last_error() -> tuple[int, str]:
    lib = load_library()
    msg = ctypes.c_char_p()
    code = lib.fmi_last_error(ctypes.byref(msg))
    return code, (msg.value.decode() if msg.value else "")


def _raise_last(default_code: int = FMI_ECUDA):
    code, msg = last_error()
    raise FmiError(code or default_code, msg)


def _ptr(a, ncols: int | None, name: str):
    """(pointer, length, keepalive) of a float64 C-contiguous host array or CUDA tensor."""
    if hasattr(a, "is_cuda") and hasattr(a, "data_ptr"):  # torch tensor
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError(f"{name}: CUDA tensors must be float64 and contiguous")
        n = a.shape[0] if a.dim() else 0
        if ncols is not None and (a.dim() != 2 or a.shape[1] != ncols):
            raise ValueError(f"{name}: expected shape (n, {ncols})")
        return ctypes.c_void_p(a.data_ptr()), n, a
    arr = np.asarray(a)
    if arr.dtype != np.float64 or not arr.flags.c_contiguous:
        arr = np.ascontiguousarray(arr, dtype=np.float64)
    if ncols is not None:
        if arr.ndim != 2 or arr.shape[1] != ncols:
            raise ValueError(f"{name}: expected shape (n, {ncols})")
    n = arr.shape[0] if arr.ndim else 0
    return ctypes.c_void_p(arr.ctypes.data), n, arr


def _out_ptr(out, m: int):
    """(pointer, keepalive) of a caller-provided result buffer of M doubles.  The library writes M
    doubles through the pointer, so nothing may be converted (a converted copy would swallow the
    result) and the length must be exactly M (a shorter buffer would be overrun)."""
    if hasattr(out, "is_cuda") and hasattr(out, "data_ptr"):
        import torch
        if out.dtype != torch.float64 or not out.is_contiguous():
            raise TypeError("out: tensors must be float64 and contiguous")
    elif not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
              and out.flags.writeable):
        raise TypeError("out must be a writeable float64 C-contiguous numpy array or a float64 contiguous tensor")
    if out.ndim != 1 or out.shape[0] != m:
        raise ValueError(f"out must have shape ({m},)")
    op, _, keep = _ptr(out, None, "out")
    return op, keep


def set_stream(stream) -> None:
    """Use a CUDA stream (torch.cuda.Stream, raw handle int, or None) for subsequent calls."""
    lib = load_library()
    handle = getattr(stream, "cuda_stream", stream)
    lib.fmi_set_stream(ctypes.c_void_p(handle or 0))


class Tree:
    """Handle of a fitted octree (fmi_tree*).  Freed by ``free()`` or on garbage collection."""

    def __init__(self, handle: int, n: int, degree: int, tol: float, max_depth: int):
        self._h = handle
        self.n = n
        self.degree = degree
        self.tol = tol
        self.max_depth = max_depth

    @property
    def handle(self) -> int:
        if not self._h:
            raise FmiError(FMI_EINPUT, "tree already freed")
        return self._h

    def free(self) -> None:
        if self._h:
            load_library().fmi_free(ctypes.c_void_p(self._h))
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    # -- evaluation ---------------------------------------------------------------------------
    def eval(self, q, out=None):
        """Interpolant at the M query points q (M, 3); returns ``out`` (numpy if q is host memory)."""
        lib = load_library()
        qp, m, qk = _ptr(q, 3, "q")
        if out is None:
            if hasattr(q, "is_cuda"):
                import torch
                out = torch.empty(m, dtype=torch.float64, device=q.device)
            else:
                out = np.empty(m, dtype=np.float64)
        op, ok = _out_ptr(out, m)
        rc = lib.fmi_eval(ctypes.c_void_p(self.handle), qp, m, op)
        if rc != 0:
            _raise_last(rc)
        return out

    # -- introspection ------------------------------------------------------------------------
    @property
    def node_count(self) -> int:
        return int(load_library().fmi_node_count(ctypes.c_void_p(self.handle)))

    @property
    def rank(self) -> int:
        return int(load_library().fmi_rank(ctypes.c_void_p(self.handle)))

    def root_cube(self):
        lo = (ctypes.c_double * 3)()
        w = ctypes.c_double()
        load_library().fmi_root_cube(ctypes.c_void_p(self.handle), lo, ctypes.byref(w))
        return np.array(lo[:]), float(w.value)

    def export(self) -> dict:
        """All nodes in canonical (depth, prefix) order as numpy arrays; coeffs = P_F (Λ basis)."""
        lib = load_library()
        n = self.node_count
        L = self.rank
        nodes = (FmiNode * n)()
        coeffs = np.zeros((n, L), dtype=np.float64)
        got = lib.fmi_export_nodes(ctypes.c_void_p(self.handle), nodes, coeffs.ctypes.data_as(ctypes.c_void_p), n)
        if got < 0:
            _raise_last(int(got))
        return {
            "depth": np.array([nd.depth for nd in nodes], dtype=np.int64),
            "cell": np.array([list(nd.cell) for nd in nodes], dtype=np.int64).reshape(n, 3),
            "prefix": np.array([nd.prefix for nd in nodes], dtype=np.uint64),
            "n_points": np.array([nd.n_points for nd in nodes], dtype=np.int64),
            "rank": np.array([nd.rank for nd in nodes], dtype=np.int64),
            "parent": np.array([nd.parent for nd in nodes], dtype=np.int64),
            "flags": np.array([nd.flags for nd in nodes], dtype=np.int64),
            "residual_rms": np.array([nd.residual_rms for nd in nodes]),
            "min_pivot": np.array([nd.min_pivot for nd in nodes]),
            "child_count": np.array([list(nd.child_count) for nd in nodes], dtype=np.int64).reshape(n, 8),
            "child_rms": np.array([list(nd.child_rms) for nd in nodes]).reshape(n, 8),
            "child": np.array([list(nd.child) for nd in nodes], dtype=np.int64).reshape(n, 8),
            "coeffs": coeffs,
        }

    def residual(self, out=None):
        """Final residual at the fit points, in input order."""
        lib = load_library()
        if out is None:
            out = np.empty(self.n, dtype=np.float64)
        op, _ = _out_ptr(out, self.n)
        rc = lib.fmi_residual(ctypes.c_void_p(self.handle), op)
        if rc != 0:
            _raise_last(rc)
        return out

    def save(self, path: str) -> None:
        """Write the tree to a file (fmi_save)."""
        rc = load_library().fmi_save(ctypes.c_void_p(self.handle), str(path).encode())
        if rc != 0:
            _raise_last(rc)

    def level_stats(self):
        lib = load_library()
        nodes = (ctypes.c_int64 * 64)()
        pts = (ctypes.c_int64 * 64)()
        k = lib.fmi_level_stats(ctypes.c_void_p(self.handle), nodes, pts, 64)
        return np.array(nodes[:k], dtype=np.int64), np.array(pts[:k], dtype=np.int64)

    def build_stats(self) -> dict:
        """Moment-tree size, fit nodes re-accumulated directly (M2M rounding check), refined nodes."""
        lib = load_library()
        out = (ctypes.c_int64 * 4)()
        lib.fmi_build_stats(ctypes.c_void_p(self.handle), out, 4)
        return {"moment_tree_nodes": int(out[0]), "direct_moment_nodes": int(out[1]), "refined_nodes": int(out[2]),
                "deferred_children": int(out[3])}


def build(pts, f, degree: int, tol: float, max_depth: int) -> Tree:
    """Fit the octree interpolant (fmi_build).  pts (N, 3), f (N,): numpy (host) or CUDA tensors."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    fp, nf, fk = _ptr(f, None, "f")
    if nf != n:
        raise ValueError("pts and f disagree in length")
    h = lib.fmi_build(pp, fp, n, int(degree), float(tol), int(max_depth))
    if not h:
        _raise_last()
    return Tree(h, n, degree, tol, max_depth)


def transfer(pts, f, q, degree: int, tol: float, max_depth: int, out=None):
    """Mesh-to-mesh transfer f_p -> f_q (fmi_transfer): build over (pts, f), evaluate at q, free."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    fp, nf, fk = _ptr(f, None, "f")
    qp, m, qk = _ptr(q, 3, "q")
    if nf != n:
        raise ValueError("pts and f disagree in length")
    if out is None:
        if hasattr(q, "is_cuda"):
            import torch
            out = torch.empty(m, dtype=torch.float64, device=q.device)
        else:
            out = np.empty(m, dtype=np.float64)
    op, ok = _out_ptr(out, m)
    rc = lib.fmi_transfer(pp, fp, n, qp, m, op, int(degree), float(tol), int(max_depth))
    if rc != 0:
        _raise_last(rc)
    return out


def load(path: str) -> Tree:
    """A tree saved with Tree.save (fmi_load)."""
    lib = load_library()
    h = lib.fmi_load(str(path).encode())
    if not h:
        _raise_last()
    t = Tree(h, 0, None, None, None)
    return t


def build_dist(pts, f, degree: int, tol: float, max_depth: int, dist: FmiDist) -> Tree:
    """Sharded build (fmi_build_dist): this shard's points (already partitioned by depth-s cell)."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    fp, nf, fk = _ptr(f, None, "f")
    if nf != n:
        raise ValueError("pts and f disagree in length")
    h = lib.fmi_build_dist(pp, fp, n, int(degree), float(tol), int(max_depth), ctypes.byref(dist))
    if not h:
        _raise_last()
    return Tree(h, n, degree, tol, max_depth)


def dist_xbuf_bytes(degree: int, shard_depth: int) -> int:
    return int(load_library().fmi_dist_xbuf_bytes(int(degree), int(shard_depth)))


def bbox(pts) -> np.ndarray:
    """min x,y,z and max x,y,z of the points (fmi_bbox)."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    out = (ctypes.c_double * 6)()
    rc = lib.fmi_bbox(pp, n, out)
    if rc != 0:
        _raise_last(rc)
    return np.array(out[:])


def cell_counts(pts, lo, width: float, depth: int, out):
    """Points per depth-``depth`` cell of the root cube (fmi_cell_counts) into ``out`` (int64, 8^depth)."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    lo3 = (ctypes.c_double * 3)(*[float(v) for v in lo])
    rc = lib.fmi_cell_counts(pp, n, lo3, float(width), int(depth), ctypes.c_void_p(_data_ptr(out)))
    if rc != 0:
        _raise_last(rc)
    return out


def partition(pts, f, lo, width: float, depth: int, owner, world: int, pts_out, f_out=None, idx_out=None,
              send_counts=None):
    """Group points by the owner shard of their depth-``depth`` cell (fmi_partition; device tensors)."""
    lib = load_library()
    pp, n, pk = _ptr(pts, 3, "pts")
    fp = ctypes.c_void_p(_data_ptr(f)) if f is not None else None
    lo3 = (ctypes.c_double * 3)(*[float(v) for v in lo])
    rc = lib.fmi_partition(pp, fp, n, lo3, float(width), int(depth), ctypes.c_void_p(_data_ptr(owner)), int(world),
                           ctypes.c_void_p(_data_ptr(pts_out)),
                           ctypes.c_void_p(_data_ptr(f_out)) if f_out is not None else None,
                           ctypes.c_void_p(_data_ptr(idx_out)) if idx_out is not None else None,
                           ctypes.c_void_p(_data_ptr(send_counts)))
    if rc != 0:
        _raise_last(rc)


def scatter(vals, idx, out):
    """out[idx[i]] = vals[i] (fmi_scatter; device tensors)."""
    lib = load_library()
    m = int(vals.shape[0])
    rc = lib.fmi_scatter(ctypes.c_void_p(_data_ptr(vals)), ctypes.c_void_p(_data_ptr(idx)), m,
                         ctypes.c_void_p(_data_ptr(out)))
    if rc != 0:
        _raise_last(rc)


def _data_ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    return int(np.asarray(a).ctypes.data)


def profile_enable(on: bool = True) -> None:
    load_library().fmi_profile_enable(1 if on else 0)


def profile_select(kernels=None) -> None:
    """Time only the named kernels (an iterable of names from KERNELS); None = every kernel."""
    arg = ",".join(kernels).encode() if kernels else None
    if load_library().fmi_profile_select(arg) != 0:
        _raise_last(FMI_EINPUT)


def profile_reset() -> None:
    load_library().fmi_profile_reset()


def profile_get() -> dict:
    lib = load_library()
    out = {}
    for k in KERNELS:
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        if lib.fmi_profile_get(k.encode(), ctypes.byref(ms), ctypes.byref(n)) == 0:
            out[k] = (float(ms.value), int(n.value))
    return out


def get_unique_id() -> bytes:
    """rank 0: a fresh 128-byte NCCL unique id for fmi_dist_init (fmi_get_unique_id)."""
    buf = ctypes.create_string_buffer(128)
    rc = load_library().fmi_get_unique_id(buf)
    if rc != 0:
        _raise_last(rc)
    return buf.raw


def dist_init(rank: int, world: int, uid: bytes) -> None:
    """Create the library-owned NCCL communicator (collective over the ranks; fmi_dist_init)."""
    if len(uid) != 128:
        raise ValueError("the NCCL unique id is 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    rc = load_library().fmi_dist_init(int(rank), int(world), buf)
    if rc != 0:
        _raise_last(rc)


def dist_finalize() -> None:
    rc = load_library().fmi_dist_finalize()
    if rc != 0:
        _raise_last(rc)


def dist_allreduce(t) -> None:
    """In-place SUM over the ranks of a contiguous CUDA tensor (float64, int64 or float32) through the
    library communicator (fmi_dist_allreduce)."""
    import torch
    codes = {torch.float64: 0, torch.int64: 1, torch.float32: 2}
    if not (t.is_cuda and t.is_contiguous() and t.dtype in codes):
        raise TypeError("dist_allreduce needs a contiguous CUDA float64/int64/float32 tensor")
    rc = load_library().fmi_dist_allreduce(ctypes.c_void_p(t.data_ptr()), t.numel(), codes[t.dtype])
    if rc != 0:
        _raise_last(rc)


def profile_units() -> dict:
    """Algorithmic work units per kernel since the last reset (include/fmi.h fmi_profile_units)."""
    lib = load_library()
    out = {}
    for k in KERNELS:
        u = ctypes.c_int64()
        if lib.fmi_profile_units(k.encode(), ctypes.byref(u)) == 0:
            out[k] = int(u.value)
    return out


def launch_count() -> int:
    return int(load_library().fmi_launch_count())


def guard_violations() -> int:
    """Overwritten guard bands seen under FMI_GUARD=1 (include/fmi.h fmi_guard_violations)."""
    return int(load_library().fmi_guard_violations())


def rank_of(degree: int) -> int:
    """𝓛 = (p+1)(p+2)(p+3)/6 — host-side argument check helper."""
    return (degree + 1) * (degree + 2) * (degree + 3) // 6
