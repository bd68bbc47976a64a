"""Parity at BASELINE.json's full sizes (cfg 3, 4, 5), in the configuration bench.py times.

The full oracle is too slow at these sizes, so every GPU node's integer work is
checked exhaustively and the floating-point results on a sample of nodes one by one:
  * every exported node's point count and octant counts = brute-force cell counts of the inputs;
  * for sampled nodes (depth >= 3), the oracle's least-squares fit of the ORIGINAL f over the node's
    points (the telescoping identity: the path sum down to a node IS that fit) decides the node's
    children (E_o > τ, n_o >= 𝓛, depth guard) — the GPU's child table must agree — and, for sampled
    leaves, gives the interpolant at sampled queries inside the leaf (1e-9·max|f|);
  * E_rms against the analytic function on the sampled queries within 1% of the oracle's.
"""
import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _labels(u, depth):
    q = np.minimum(np.floor(u * 2.0 ** depth), 2 ** depth - 1).astype(np.int64)
    return q[:, 0] | (q[:, 1] << depth) | (q[:, 2] << (2 * depth)), q


def _check(cfg_id, n_sample_nodes=6, n_queries=4000, seed=0):
    import paper_1511_01353_b200 as fmi
    cfg = workloads.CONFIGS[cfg_id]
    pts, f, q = workloads.make_inputs(cfg)
    L = fo.rank(cfg.degree)
    with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol,
                   cfg.max_depth) as tree:
        ex = tree.export()
        lo, width = tree.root_cube()
        u = fo.to_unit(pts, lo, width)
        # -- integer work, every node: counts by brute force per depth ---------------------------
        depth = ex["depth"]
        for d in range(int(depth.max()) + 1):
            sel = np.flatnonzero(depth == d)
            lab, _ = _labels(u, d)
            counts = np.bincount(lab, minlength=8 ** d) if d <= 6 else None
            child_lab, _ = _labels(u, d + 1)
            for i in sel:
                cx, cy, cz = (int(v) for v in ex["cell"][i])
                key = cx | (cy << d) | (cz << (2 * d))
                n_brute = counts[key] if counts is not None else int(np.sum(lab == key))
                assert ex["n_points"][i] == n_brute, (d, (cx, cy, cz))
            if len(sel) and d <= 5:
                cc = np.bincount(child_lab, minlength=8 ** (d + 1))
                for i in sel[:: max(1, len(sel) // 200)]:
                    cx, cy, cz = (int(v) for v in ex["cell"][i])
                    for o in range(8):
                        x, y, z = 2 * cx + (o & 1), 2 * cy + ((o >> 1) & 1), 2 * cz + ((o >> 2) & 1)
                        assert ex["child_count"][i][o] == cc[x | (y << (d + 1)) | (z << (2 * d + 2))]
        # -- sampled nodes: oracle LS fit of the original f over the node's points ---------------
        rng = np.random.default_rng(seed)
        cand = np.flatnonzero(depth >= 3)
        leaves = [i for i in cand if np.all(ex["child"][i] < 0)]
        inner = [i for i in cand if np.any(ex["child"][i] >= 0)]
        pick = list(rng.choice(leaves, size=min(len(leaves), n_sample_nodes // 2 + 1), replace=False))
        if inner:
            pick += list(rng.choice(inner, size=min(len(inner), n_sample_nodes // 2), replace=False))
        scale = float(np.max(np.abs(f)))
        errs_gpu, errs_ora = [], []
        for i in pick:
            d = int(depth[i])
            cell = ex["cell"][i]
            lab, qc = _labels(u, d)
            inside = np.all(qc == cell, axis=1)
            ul = fo.local_coords(u[inside], d, cell)
            fit = fo.fit_node(ul, f[inside], cfg.degree)
            r = f[inside] - fo.vandermonde(ul, cfg.degree) @ fit.coeffs
            oc = fo.octant(ul)
            for o in range(8):
                no = int(np.sum(oc == o))
                e = np.sqrt(np.sum(r[oc == o] ** 2) / no) if no else 0.0
                if no and abs(e / cfg.tol - 1.0) < 1e-6:
                    continue  # a tie at roundoff level: either decision is correct (G17)
                make = no > 0 and e > cfg.tol and no >= L and d + 1 <= cfg.max_depth
                assert (ex["child"][i][o] >= 0) == make, (d, tuple(cell), o, e / cfg.tol, no)
            if np.all(ex["child"][i] < 0):  # leaf: the interpolant inside it is the node's LS fit
                h = 2.0 ** -(d + 1)
                c = (2.0 * cell + 1.0) * h
                qs = lo + width * (c - h + 2 * h * rng.random((200, 3)))
                uq = fo.to_unit(qs, lo, width)
                got = tree.eval(torch.from_numpy(np.ascontiguousarray(qs)).cuda()).cpu().numpy()
                ref = fo.vandermonde(fo.local_coords(uq, d, cell), cfg.degree) @ fit.coeffs
                assert np.max(np.abs(got - ref)) <= 1e-9 * scale, (d, tuple(cell))
                truth = workloads.exact_values(cfg, qs)
                errs_gpu.append(got - truth)
                errs_ora.append(ref - truth)
        if errs_gpu:
            eg, _ = workloads.rms_and_max(np.concatenate(errs_gpu))
            eo, _ = workloads.rms_and_max(np.concatenate(errs_ora))
            assert abs(eg - eo) <= 0.01 * eo + 1e-300
        # -- bookkeeping identity on a sample of the fit points -------------------------
        res = tree.residual()
        sel = rng.choice(len(pts), size=min(len(pts), n_queries), replace=False)
        val = tree.eval(torch.from_numpy(np.ascontiguousarray(pts[sel])).cuda()).cpu().numpy()
        assert np.max(np.abs(val + res[sel] - f[sel])) <= 1e-9 * scale


def test_cfg3_full_size():
    _check(3)


def test_cfg4_full_size():
    _check(4)


@pytest.mark.slow
def test_cfg5_full_size():
    _check(5, n_sample_nodes=4)
