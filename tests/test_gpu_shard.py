"""Sharded build on one GPU with virtual shards (threads + an in-process communicator): the global
nodes and every shard's subtrees must reproduce the single-GPU tree (same topology and point counts,
coefficients and values within the parity tolerance), and routed evaluation must match it.

This exercises the exact library path of a multi-GPU run (fmi_build_dist with its collective
callbacks, fmi_partition exchange, routed fmi_eval); only the communicator differs (NCCL there)."""
import threading

import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run_shards(world, pts, f, q, p, tau, D, smax=3):
    from paper_1511_01353_b200 import fmi, shard
    comms = shard.LocalComm.group(world)
    n, m = len(pts), len(q)
    res = [None] * world
    err = []

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                fmi.set_stream(st)
                sl = slice(r * n // world, (r + 1) * n // world)
                ql = slice(r * m // world, (r + 1) * m // world)
                dp = torch.from_numpy(np.ascontiguousarray(pts[sl])).cuda()
                df = torch.from_numpy(np.ascontiguousarray(f[sl])).cuda()
                dq = torch.from_numpy(np.ascontiguousarray(q[ql])).cuda()
                tr = shard.build_sharded(dp, df, p, tau, D, comms[r], smax=smax)
                vals = tr.eval(dq).cpu().numpy()
                res[r] = (tr.shard_depth, tr.tree.export(), vals, ql)
                tr.free()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            for c in comms:  # unblock the others
                c.shared.barrier.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    from paper_1511_01353_b200 import fmi as _f
    _f.set_stream(None)
    return res


def _merge(res):
    """Global nodes (depth < s) from shard 0, local nodes from every shard: key -> per-node data."""
    s = res[0][0]
    nodes = {}
    for r, (sd, ex, _, _) in enumerate(res):
        for i in range(len(ex["depth"])):
            d = int(ex["depth"][i])
            if d < s and r > 0:
                continue
            key = (d, *map(int, ex["cell"][i]))
            assert key not in nodes, f"node {key} on two shards"
            nodes[key] = {k: ex[k][i] for k in ("n_points", "child_count", "coeffs", "residual_rms")}
    return s, nodes


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_shards_match_single_gpu(world):
    from paper_1511_01353_b200 import fmi
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    q = q[:200_000]
    res = _run_shards(world, pts, f, q, cfg.degree, cfg.tol, cfg.max_depth)
    s, nodes = _merge(res)
    assert s >= 1
    with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol,
                   cfg.max_depth) as one:
        ex = one.export()
        ref_vals = one.eval(torch.from_numpy(q).cuda()).cpu().numpy()
    single = {(int(ex["depth"][i]), *map(int, ex["cell"][i])): i for i in range(len(ex["depth"]))}
    assert set(nodes) == set(single)                                   # identical topology
    scale = float(np.max(np.abs(f)))
    for key, i in single.items():
        nd = nodes[key]
        assert nd["n_points"] == ex["n_points"][i], key
        assert np.array_equal(nd["child_count"], ex["child_count"][i]), key
        assert abs(nd["residual_rms"] - ex["residual_rms"][i]) <= 1e-9 * scale + 1e-6 * ex["residual_rms"][i]
    vals = np.concatenate([r[2] for r in res])
    assert np.max(np.abs(vals - ref_vals)) <= 1e-9 * scale
    # and against the oracle on a sample of the queries
    ora = fo.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth)
    sel = np.arange(0, len(q), 97)
    assert np.max(np.abs(vals[sel] - fo.evaluate(ora, q[sel]))) <= 1e-9 * scale


def test_virtual_shards_all_global_and_empty_shard():
    """max_depth small enough that every node is global (no exchange), and a shard without points."""
    rng = np.random.default_rng(3)
    pts = rng.random((5000, 3)) * 0.4          # all points in one corner: some shards get none
    f = workloads.franke3d(pts)
    q = rng.random((3000, 3)) * 0.4
    for D in (0, 1, 3):
        res = _run_shards(3, pts, f, q, 3, 1e-9, D)
        vals = np.concatenate([r[2] for r in res])
        ora = fo.build(pts, f, 3, 1e-9, D)
        assert np.max(np.abs(vals - fo.evaluate(ora, q))) <= 1e-9 * np.max(np.abs(f))


def test_library_nccl_communicator_world1():
    """The library-owned NCCL communicator (fmi_get_unique_id / fmi_dist_init): an in-place device
    allreduce, and a sharded build at world 1 whose global levels (shard depth 2) are summed by NCCL on
    the library stream (no callback, no exchange buffer) reproduces the single-GPU tree."""
    from paper_1511_01353_b200 import fmi
    fmi.load_library()
    uid = fmi.get_unique_id()
    assert len(uid) == 128
    fmi.dist_init(0, 1, uid)
    try:
        t = torch.arange(10, dtype=torch.float64, device="cuda")
        fmi.dist_allreduce(t)
        assert torch.equal(t.cpu(), torch.arange(10, dtype=torch.float64))
        cfg = workloads.CONFIGS[2]
        pts, f, q = workloads.make_inputs(cfg)
        q = q[:50_000]
        dp, df, dq = (torch.from_numpy(a).cuda() for a in (pts, f, q))
        d = fmi.FmiDist()
        d.rank, d.world, d.shard_depth = 0, 1, 2
        d.width = 1.0
        with fmi.build_dist(dp, df, cfg.degree, cfg.tol, cfg.max_depth, d) as tn, \
                fmi.build(dp, df, cfg.degree, cfg.tol, cfg.max_depth) as one:
            a, b = tn.export(), one.export()
            for k in ("depth", "cell", "n_points", "child_count", "child"):
                assert np.array_equal(a[k], b[k]), k
            va, vb = tn.eval(dq).cpu().numpy(), one.eval(dq).cpu().numpy()
            assert np.max(np.abs(va - vb)) <= 1e-9 * np.max(np.abs(f))
        # a communicator of another world size is refused
        d.world = 2
        with pytest.raises(fmi.FmiError) as ei:
            fmi.build_dist(dp, df, cfg.degree, cfg.tol, cfg.max_depth, d)
        assert ei.value.code == fmi.FMI_ENCCL
    finally:
        fmi.dist_finalize()
