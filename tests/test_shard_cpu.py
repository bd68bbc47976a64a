"""Host logic of the sharded (multi-GPU) path, on CPU: shard choice, point exchange, query routing and
the collective-sum plumbing of fmi_build_dist, with torch.distributed gloo at world size 2.

The point-wise kernels (cell histogram, partition, scatter, the build itself) are replaced by a numpy
stub here — test scaffolding only; the product path calls the library (tests/test_gpu_shard.py runs
the real sharded build on a GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch

from paper_1511_01353_b200 import fmi as _fmi
from paper_1511_01353_b200 import shard


# ---------------------------------------------------------------------------------------------
# pure host logic
# ---------------------------------------------------------------------------------------------

def test_assign_cells_contiguous_balanced_deterministic():
    rng = np.random.default_rng(0)
    for world in (2, 3, 4, 8):
        counts = rng.poisson(50, 512)
        owner = shard.assign_cells(counts, world)
        assert np.all(np.diff(owner) >= 0) and owner[0] == 0 and owner[-1] == world - 1  # contiguous ranges
        assert set(np.unique(owner)) == set(range(world))                                # every shard a cell
        load = shard.shard_loads(counts, owner, world)
        assert load.max() <= 1.05 * counts.sum() / world
        assert np.array_equal(owner, shard.assign_cells(counts.copy(), world))


def test_assign_cells_handles_empty_and_skewed():
    counts = np.zeros(64, dtype=np.int64)
    counts[10] = 1000
    owner = shard.assign_cells(counts, 4)
    assert set(np.unique(owner)) == {0, 1, 2, 3}
    assert np.all(np.diff(owner) >= 0)
    assert np.array_equal(shard.assign_cells(np.zeros(8, dtype=np.int64), 8), np.arange(8))


def test_coarsen_counts_follows_morton_nesting():
    c = np.arange(512)
    c1 = shard.coarsen_counts(c, 3, 1)
    assert c1.shape == (8,) and c1[0] == np.arange(64).sum()
    assert shard.coarsen_counts(c, 3, 3) is not None and np.array_equal(shard.coarsen_counts(c, 3, 3), c)


def test_choose_shard_depth():
    rng = np.random.default_rng(1)
    uniform = rng.poisson(1000, 8 ** 4)
    s, owner = shard.choose_shard_depth(uniform, 8, 10)
    assert s == 1 and owner.shape == (8,)
    skew = np.zeros(8 ** 4, dtype=np.int64)
    skew[:64] = 1000                      # all points in one depth-2 cell
    s2, owner2 = shard.choose_shard_depth(skew, 4, 10)
    assert s2 >= 3
    assert shard.choose_shard_depth(uniform, 4, 1)[0] == 1
    assert shard.choose_shard_depth(uniform, 4, 0) == (1, None)
    assert shard.choose_shard_depth(uniform, 1, 10)[0] == 0


def test_root_cube_rule():
    lo, w = shard.root_cube_from_bbox([0.1, 0.0, 0.2], [0.9, 1.0, 0.5])
    assert np.array_equal(lo, np.zeros(3)) and w == 1.0
    lo, w = shard.root_cube_from_bbox([-1.0, 4.0, 0.5], [2.0, 5.0, 2.5])
    assert np.array_equal(lo, [-1.0, 4.0, 0.5]) and w == 3.0


# ---------------------------------------------------------------------------------------------
# world size 2 over gloo: exchange, routing, collective plumbing
# ---------------------------------------------------------------------------------------------

def _labels(p, lo, w, s):
    """Morton label of the depth-s cell (S:324 octant numbering), numpy (test stub)."""
    u = (np.asarray(p) - lo) / w if not (np.all(lo == 0) and w == 1.0) else np.asarray(p)
    q = np.clip(np.floor(u * 2 ** s), 0, 2 ** s - 1).astype(np.int64)
    lab = np.zeros(len(q), dtype=np.int64)
    for b in range(s):
        for a in range(3):
            lab |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return lab


class _FakeTree:
    def __init__(self, pts, rank):
        self.pts = pts
        self.rank = rank

    def eval(self, q, out=None):
        v = q.sum(dim=1) + 1000.0 * self.rank   # records which shard evaluated
        if out is not None:
            out.copy_(v)
            return out
        return v

    def free(self):
        pass


class _Stub:
    """numpy stand-ins for the library's point-wise kernels (CPU test scaffolding)."""
    FmiDist = _fmi.FmiDist
    ALLREDUCE_FN = _fmi.ALLREDUCE_FN

    def __init__(self, rank):
        self.rank = rank
        self.reduced = None

    def bbox(self, pts):
        p = pts.numpy()
        return np.concatenate([p.min(axis=0), p.max(axis=0)])

    def cell_counts(self, pts, lo, width, depth, out):
        lab = _labels(pts.numpy(), lo, width, depth)
        out.copy_(torch.from_numpy(np.bincount(lab, minlength=8 ** depth).astype(np.int64)))

    def partition(self, pts, f, lo, width, depth, owner, world, pts_out, f_out, idx_out, send_counts):
        lab = _labels(pts.numpy(), lo, width, depth)
        dst = owner.numpy()[lab]
        order = np.argsort(dst, kind="stable")
        pts_out.copy_(pts[torch.from_numpy(order)])
        if f_out is not None:
            f_out.copy_(f[torch.from_numpy(order)])
        if idx_out is not None:
            idx_out.copy_(torch.from_numpy(order))
        send_counts.copy_(torch.from_numpy(np.bincount(dst, minlength=world).astype(np.int64)))

    def scatter(self, vals, idx, out):
        out[idx] = vals

    def dist_xbuf_bytes(self, degree, s):
        return 1 << 12

    def build_dist(self, pts, f, degree, tol, max_depth, d):
        # exercise the collective-sum callback the library would call: fp64, int64 and fp32 views
        import ctypes
        buf = (ctypes.c_char * 64).from_address(d.xbuf)
        arr = np.frombuffer(buf, dtype=np.float64, count=4)
        arr[:] = [1.0 + d.rank, 2.0, 3.0, 4.0]
        assert d.allreduce(None, 4, 0) == 0
        self.reduced = arr.copy()
        ints = np.frombuffer(buf, dtype=np.int64, count=2)
        ints[:] = [len(pts), 7]
        assert d.allreduce(None, 2, 1) == 0
        self.total_points = int(ints[0])
        self.shard_depth = d.shard_depth
        return _FakeTree(pts, self.rank)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = shard.TorchComm()
        rng = np.random.default_rng(10 + rank)
        n = 3000 + 500 * rank
        pts = torch.from_numpy(rng.random((n, 3)))
        f = pts[:, 0] * 2.0 + rank
        stub = _Stub(rank)
        st = shard.build_sharded(pts, f, 3, 1e-6, 6, comm, smax=3, kernels=stub)
        mine = st.tree.pts.numpy()
        q = torch.from_numpy(rng.random((777 + 11 * rank, 3)))
        vals = st.eval(q)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), mine=mine, owner=st.owner, s=st.shard_depth,
                 q=q.numpy(), vals=vals.numpy(), reduced=stub.reduced, total=stub.total_points,
                 lo=st.lo, width=st.width)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world2_exchange_routing_and_collectives(tmp_path):
    world = 2
    torch.multiprocessing.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    s = int(res[0]["s"])
    owner = res[0]["owner"]
    assert s >= 1 and np.array_equal(owner, res[1]["owner"])          # same shard map everywhere
    # every point went to the owner of its depth-s cell, none lost or duplicated
    allpts = np.concatenate([np.random.default_rng(10 + r).random((3000 + 500 * r, 3)) for r in range(world)])
    got = np.concatenate([res[r]["mine"] for r in range(world)])
    assert got.shape == allpts.shape
    assert np.array_equal(np.sort(got.view("f8,f8,f8"), axis=0), np.sort(allpts.view("f8,f8,f8"), axis=0))
    for r in range(world):
        lab = _labels(res[r]["mine"], res[r]["lo"], float(res[r]["width"]), s)
        assert np.all(owner[lab] == r)
    # collective sums through the library callback (fp64 and int64 views of the exchange buffer)
    for r in range(world):
        assert np.allclose(res[r]["reduced"], [1.0 + 2.0, 4.0, 6.0, 8.0])
        assert int(res[r]["total"]) == len(allpts)
    # query routing: value evaluated by the owner shard, returned in the caller's order
    for r in range(world):
        q, vals = res[r]["q"], res[r]["vals"]
        lab = _labels(q, res[r]["lo"], float(res[r]["width"]), s)
        assert np.allclose(vals, q.sum(axis=1) + 1000.0 * owner[lab])
