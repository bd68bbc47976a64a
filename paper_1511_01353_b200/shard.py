"""Sharded (multi-GPU) build and evaluation — SURVEY.md §8(e), DESIGN.md §6.

One process per GPU (torchrun; torch.distributed with NCCL over NVLink is the plumbing), or — for the
single-GPU "virtual shard" tests — one thread per shard with an in-process communicator.

Scheme (B200-first, "global top + local subtrees"): the points are partitioned by the cells of a
shard depth s of the common root cube, each shard owning a contiguous Morton range of depth-s cells
(balanced by point count).  Nodes of depth < s are *global*: every shard accumulates its partial
moments / projections / octant counts / residual energies and one SUM collective per quantity and
level makes them identical everywhere (the library calls back into ``Comm.allreduce_sum``).  Nodes of
depth >= s live on the shard owning their cell and need no communication.  Queries are routed to the
owner of their depth-s cell (all-to-all), evaluated locally and returned (all-to-all).

This module holds only host logic (shard choice, exchanges, routing); every point-wise step runs in
the library's kernels (fmi_cell_counts, fmi_partition, fmi_build_dist, fmi_eval, fmi_scatter).
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

MAX_SHARD_DEPTH = 4          # cell histogram depth (8^4 = 4096 cells)
BALANCE = 1.15               # accepted max shard load / mean


# ------------------------------------------------------------------------------------------------
# communicators
# ------------------------------------------------------------------------------------------------
class TorchComm:
    """torch.distributed process group: NCCL on GPUs (device tensors, NVLink/NVSwitch), gloo on CPU
    (device tensors are staged through host memory for gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host_staged = dist.get_backend(group) == "gloo"
        # NCCL process group: the sharded build's in-build sums go through the library-owned NCCL
        # communicator (fmi_dist_init), created once from a unique id broadcast over this group
        self.library_nccl = not self.host_staged
        self._lib_ready = False

    def ensure_library_comm(self, kernels):
        if self._lib_ready:
            return
        import torch
        uid = kernels.get_unique_id() if self.rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        self.dist.broadcast(t, src=0, group=self.group)
        kernels.dist_init(self.rank, self.world, bytes(t.cpu().tolist()))
        self._lib_ready = True

    def _op(self, t, fn):
        if self.host_staged and t.is_cuda:
            h = t.cpu()
            fn(h)
            t.copy_(h)
        else:
            fn(t)
            if t.is_cuda:  # the library reads the result on its own stream: complete the collective first
                import torch
                torch.cuda.current_stream(t.device).synchronize()

    def allreduce_sum(self, t):
        self._op(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group))

    def allreduce_min(self, t):
        self._op(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.MIN, group=self.group))

    def allreduce_max(self, t):
        self._op(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group))

    def all_to_all(self, out, inp, out_splits, in_splits):
        if self.host_staged and (out.is_cuda or inp.is_cuda):
            ho = out.cpu()
            self.dist.all_to_all_single(ho, inp.cpu(), output_split_sizes=out_splits, input_split_sizes=in_splits,
                                        group=self.group)
            out.copy_(ho)
            return
        self.dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                    group=self.group)


class LocalComm:
    """In-process communicator for shards run as threads (virtual shards on one device).  Reductions
    are taken on host copies, summed in rank order (deterministic)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.shared = shared
        self.rank = rank
        self.world = shared.world

    @classmethod
    def group(cls, world):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _gather(self, arr):
        sh = self.shared
        sh.barrier.wait()
        sh.slots[self.rank] = arr
        sh.barrier.wait()
        vals = list(sh.slots)
        sh.barrier.wait()
        return vals

    def _reduce(self, t, op):
        import torch
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        host = t.detach().cpu().numpy().copy()
        vals = self._gather(host)
        acc = vals[0].copy()
        for v in vals[1:]:
            acc = op(acc, v)
        t.copy_(torch.from_numpy(acc).to(t.device))
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()

    def allreduce_sum(self, t):
        self._reduce(t, np.add)

    def allreduce_min(self, t):
        self._reduce(t, np.minimum)

    def allreduce_max(self, t):
        self._reduce(t, np.maximum)

    def all_to_all(self, out, inp, out_splits, in_splits):
        import torch
        if inp.is_cuda:
            torch.cuda.current_stream().synchronize()
        host = inp.detach().cpu().numpy()
        offs = np.concatenate([[0], np.cumsum(in_splits)])
        pieces = [host[offs[d]:offs[d + 1]] for d in range(self.world)]
        allp = self._gather(pieces)
        mine = np.concatenate([allp[src][self.rank] for src in range(self.world)]) if self.world else host[:0]
        out.copy_(torch.from_numpy(mine.reshape(out.shape)).to(out.device))


# ------------------------------------------------------------------------------------------------
# host logic (pure; unit-tested on CPU)
# ------------------------------------------------------------------------------------------------
def root_cube_from_bbox(lo, hi):
    """Root cube rule (reading G6): the unit cube if every point lies in [0,1]^3, else the isotropic
    bounding cube of the data.  lo/hi are the GLOBAL min/max over all shards."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if np.all(lo >= 0.0) and np.all(hi <= 1.0):
        return np.zeros(3), 1.0
    w = float(np.max(hi - lo))
    return lo.copy(), (w if w > 0 else 1.0)


def coarsen_counts(counts: np.ndarray, from_depth: int, to_depth: int) -> np.ndarray:
    """Cell counts at a coarser depth: Morton labels nest, so a depth-t cell is a run of 8^(d-t) cells."""
    k = 8 ** (from_depth - to_depth)
    return counts.reshape(-1, k).sum(axis=1)


def assign_cells(counts: np.ndarray, world: int) -> np.ndarray:
    """Owner shard of every cell: contiguous Morton ranges with balanced point counts (greedy cut at
    the cumulative count nearest to (r+1)·total/world).  Deterministic: every shard computes the same
    array from the same (summed) counts."""
    counts = np.asarray(counts, dtype=np.int64)
    n = counts.shape[0]
    cum = np.cumsum(counts)
    total = int(cum[-1]) if n else 0
    owner = np.zeros(n, dtype=np.int32)
    start = 0
    for r in range(world - 1):
        target = total * (r + 1) / world
        # first cell index c >= start such that cum[c] is nearest to target (at least one cell left per shard)
        c = int(np.searchsorted(cum, target, side="left"))
        if c < n and c > 0 and abs(cum[c - 1] - target) <= abs(cum[c] - target):
            c -= 1
        c = max(c, start)
        c = min(c, n - (world - 1 - r))
        owner[start:c + 1] = r
        start = c + 1
    owner[start:] = world - 1
    return owner


def shard_loads(counts: np.ndarray, owner: np.ndarray, world: int) -> np.ndarray:
    return np.bincount(owner, weights=counts, minlength=world)


def choose_shard_depth(counts_max: np.ndarray, world: int, max_depth: int, smax: int = MAX_SHARD_DEPTH):
    """Smallest shard depth s in 1..smax whose balanced assignment keeps the largest shard within
    BALANCE of the mean (else smax); s = max_depth + 1 (every node global, no exchange) when that is
    not deeper.  Returns (s, owner at depth s)."""
    if world == 1:
        return 0, np.zeros(1, dtype=np.int32)
    if max_depth + 1 <= 1:
        return max_depth + 1, None
    best = None
    total = float(counts_max.sum())
    for s in range(1, smax + 1):
        if s >= max_depth + 1:
            return max_depth + 1, None
        c = coarsen_counts(counts_max, smax, s)
        owner = assign_cells(c, world)
        load = shard_loads(c, owner, world)
        best = (s, owner)
        if total == 0 or load.max() <= BALANCE * total / world:
            return best
    return best


# ------------------------------------------------------------------------------------------------
# the sharded interpolator
# ------------------------------------------------------------------------------------------------
class ShardedTree:
    """A shard's part of a sharded build plus what is needed to route queries."""

    def __init__(self, tree, comm, lo, width, shard_depth, owner, kernels=None):
        from . import fmi
        self.k = kernels or fmi
        self.tree = tree
        self.comm = comm
        self.lo = lo
        self.width = width
        self.shard_depth = shard_depth
        self.owner = owner  # np.int32[8^s] or None (every node global)

    def free(self):
        self.tree.free()

    def eval(self, q, out=None):
        """Evaluate this shard's queries q (M_local, 3) (CUDA tensor): route by owner cell, evaluate on
        the owning shard, return the values in q's order."""
        import torch
        fmi = self.k
        comm = self.comm
        m = int(q.shape[0])
        dev = q.device
        if out is None:
            out = torch.empty(m, dtype=torch.float64, device=dev)
        if self.owner is None or comm.world == 1:  # every node global: evaluate locally
            return self.tree.eval(q, out=out)
        owner_t = torch.from_numpy(self.owner).to(dev)
        q_sorted = torch.empty_like(q)
        idx = torch.empty(m, dtype=torch.int64, device=dev)
        send = torch.empty(comm.world, dtype=torch.int64, device=dev)
        fmi.partition(q, None, self.lo, self.width, self.shard_depth, owner_t, comm.world, q_sorted, None, idx, send)
        recv = torch.empty_like(send)
        comm.all_to_all(recv, send, [1] * comm.world, [1] * comm.world)
        s_list, r_list = send.cpu().tolist(), recv.cpu().tolist()
        q_recv = torch.empty((sum(r_list), 3), dtype=torch.float64, device=dev)
        comm.all_to_all(q_recv.view(-1), q_sorted.view(-1), [3 * v for v in r_list], [3 * v for v in s_list])
        vals = self.tree.eval(q_recv)
        back = torch.empty(m, dtype=torch.float64, device=dev)
        comm.all_to_all(back, vals, s_list, r_list)
        fmi.scatter(back, idx, out)
        return out


def build_sharded(pts, f, degree: int, tol: float, max_depth: int, comm, smax: int = MAX_SHARD_DEPTH,
                  kernels=None):
    """Collective sharded build over ``comm``: pts (N_local, 3), f (N_local,) CUDA tensors of this shard
    (any initial distribution).  Returns a ShardedTree.  ``kernels`` (default: the fmi binding) provides
    bbox / cell_counts / partition / scatter / dist_xbuf_bytes / build_dist / FmiDist / ALLREDUCE_FN."""
    import torch
    from . import fmi as _fmi
    fmi = kernels or _fmi
    dev = pts.device
    world, rank = comm.world, comm.rank
    n = int(pts.shape[0])
    # 1. common root cube (G6)
    bb = torch.tensor(fmi.bbox(pts) if n else [np.inf] * 3 + [-np.inf] * 3, dtype=torch.float64, device=dev)
    lo_t, hi_t = bb[:3].clone(), bb[3:].clone()
    comm.allreduce_min(lo_t)
    comm.allreduce_max(hi_t)
    lo, width = root_cube_from_bbox(lo_t.cpu().numpy(), hi_t.cpu().numpy())
    # 2. shard depth and cell ownership from the summed cell histogram
    counts = torch.zeros(8 ** smax, dtype=torch.int64, device=dev)
    fmi.cell_counts(pts, lo, width, smax, counts)
    comm.allreduce_sum(counts)
    s, owner = choose_shard_depth(counts.cpu().numpy(), world, max_depth, smax)
    # 3. exchange the points so that every depth-s cell lives on its owner shard
    if owner is not None and world > 1:
        owner_t = torch.from_numpy(owner).to(dev)
        p_sorted = torch.empty_like(pts)
        f_sorted = torch.empty_like(f)
        send = torch.empty(world, dtype=torch.int64, device=dev)
        fmi.partition(pts, f, lo, width, s, owner_t, world, p_sorted, f_sorted, None, send)
        recv = torch.empty_like(send)
        comm.all_to_all(recv, send, [1] * world, [1] * world)
        s_list, r_list = send.cpu().tolist(), recv.cpu().tolist()
        nr = sum(r_list)
        p_loc = torch.empty((nr, 3), dtype=torch.float64, device=dev)
        f_loc = torch.empty(nr, dtype=torch.float64, device=dev)
        comm.all_to_all(p_loc.view(-1), p_sorted.view(-1), [3 * v for v in r_list], [3 * v for v in s_list])
        comm.all_to_all(f_loc, f_sorted, r_list, s_list)
    else:
        p_loc, f_loc = pts, f
    # 4. the sharded build: global nodes summed by the library's NCCL communicator (in place, on the
    #    library stream), or — in-process / gloo communicators — through the callback
    if getattr(comm, "library_nccl", False):
        comm.ensure_library_comm(fmi)
        d = fmi.FmiDist()
        d.rank, d.world, d.shard_depth = rank, world, s
        for a in range(3):
            d.lo[a] = float(lo[a])
        d.width = float(width)
        tree = fmi.build_dist(p_loc, f_loc, degree, tol, max_depth, d)
        st = ShardedTree(tree, comm, lo, width, s, owner, kernels)
        st._keep = (p_loc, f_loc)
        return st
    xbytes = fmi.dist_xbuf_bytes(degree, s)
    xbuf = torch.empty(xbytes, dtype=torch.uint8, device=dev)
    views = {0: torch.float64, 1: torch.int64, 2: torch.float32}

    def _allreduce(ctx, count, dtype):
        try:
            t = xbuf.view(views[dtype])[:count]
            comm.allreduce_sum(t)
            return 0
        except Exception:  # reported to the library as FMI_ENCCL
            return 1

    cb = fmi.ALLREDUCE_FN(_allreduce)
    d = fmi.FmiDist()
    d.rank, d.world, d.shard_depth = rank, world, s
    for a in range(3):
        d.lo[a] = float(lo[a])
    d.width = float(width)
    d.xbuf = ctypes.c_void_p(xbuf.data_ptr())
    d.xbuf_bytes = xbytes
    d.allreduce = cb
    d.ctx = None
    tree = fmi.build_dist(p_loc, f_loc, degree, tol, max_depth, d)
    st = ShardedTree(tree, comm, lo, width, s, owner, kernels)
    st._keep = (xbuf, cb, p_loc, f_loc)
    return st
