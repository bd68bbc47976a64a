"""Full-size parity against the oracle's golden node lists (tests/golden/oracle_cfg*.npz, written by
tools/make_golden.py, which calls only oracle/ and workloads/).

  cfg3  the whole tree: every node, every decision, 1e5 queries.
  cfg4  every depth-0/1 node and decision, and 8 whole depth-2 subtrees (the oracle ran Alg. 1 from
        the root, expanding only those subtrees); the config's own queries (the same mixture) inside them.
  cfg5  8 whole depth-2 subtrees, each Alg. 1 called on the depth-2 node with the original values
        (telescoping start; the root fit of 2e8 points is beyond the CPU oracle): compared (a) inside
        the full-size GPU tree and (b) as stand-alone problems mapped exactly onto the unit cube.

Bars (BASELINE.json north_star): identical topology and node point counts (decisions within
|E/τ - 1| < the tie band are roundoff-level ties, G17: reported, their subtrees skipped); interpolant
within 1e-9·max|f|; E_rms against the analytic function within 1% of the oracle's; post-fit node RMS
within 1e-6 relative + 1e-12·max|f|.  PAPER.md Alg. 1/2, evaluation P:275-280.
"""
import os

import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo
from parity import compare_with_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
# GPU vs oracle on the same residual: both carry ~1e-13·max|f| of roundoff in E (cfg 3's closest
# decision is 1.9e-3 from τ = 1e-10).  cfg 5 vs a telescoping-start golden: the depth-2 node's
# residual differs from the root-started one by the roundoff of the root and depth-1 fits,
# ~1e-13 absolute against τ = 1e-11.
TIE_BAND = {3: 1e-3, 4: 1e-3, 5: 2e-2}


def _golden(c):
    path = os.path.join(GOLDEN, f"oracle_cfg{c}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (python tools/make_golden.py cfg{c})")
    return dict(np.load(path))


def _queries(gold, c):
    if str(gold["mode"]) == "full":
        return workloads.uniform_points(int(gold["q_n"]), int(gold["q_seed"]))
    if "q_index" in gold:   # the config's own queries (cfg 4: the mixture) inside the sampled subtrees
        cfg = workloads.CONFIGS[c]
        q = workloads.mixture_points(cfg.m, 1, workloads.mixture_centres(0))
        return np.ascontiguousarray(q[gold["q_index"]])
    per = int(gold["q_per_cell"])
    return np.concatenate([workloads.cell_queries(2, tuple(int(v) for v in cell), per, int(gold["q_seed0"]) + t)
                           for t, cell in enumerate(gold["pick"])])


def _in_picked(pick):
    cells = {tuple(int(v) for v in c) for c in pick}

    def within(d, c):
        return d >= 2 and tuple(v >> (d - 2) for v in c) in cells
    return within


def _check_values(cfg, got, gold, q, scale):
    ref = gold["values"]
    err = float(np.max(np.abs(got - ref)))
    assert err <= 1e-9 * scale, f"max|gpu - oracle| = {err:.3e}"
    truth = workloads.exact_values(cfg, q)
    e_gpu, _ = workloads.rms_and_max(got - truth)
    e_ora, _ = workloads.rms_and_max(ref - truth)
    assert abs(e_gpu - e_ora) <= 0.01 * e_ora, (e_gpu, e_ora)
    return err, e_gpu, e_ora


def _full_size(c):
    import paper_1511_01353_b200 as fmi
    cfg = workloads.CONFIGS[c]
    gold = _golden(c)
    pts, f, _ = workloads.make_inputs(cfg.scaled(m=1))
    scale = float(np.max(np.abs(f)))
    q = _queries(gold, c)
    L = fo.rank(cfg.degree)
    with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol,
                   cfg.max_depth) as tree:
        ex = tree.export()
        got = tree.eval(torch.from_numpy(q).cuda()).cpu().numpy()
    within = None
    if str(gold["mode"]) == "top+subtrees":
        inner = _in_picked(gold["pick"])
        within = lambda d, cell: d <= 1 or inner(d, cell)  # noqa: E731
    elif str(gold["mode"]) == "subtrees-telescoped":
        within = _in_picked(gold["pick"])
    rep = compare_with_golden(ex, gold, cfg.tol, L, cfg.max_depth, TIE_BAND[c], scale, within=within)
    err, e_gpu, e_ora = _check_values(cfg, got, gold, q, scale)
    print(f"cfg{c}: {rep['nodes']} golden nodes, {rep['decisions']} decisions, ties {rep['ties']}, "
          f"worst node-rms / bound {rep['worst_rms_over_bound']:.3g}, max|d| {err:.3e}, "
          f"E_rms gpu {e_gpu:.6e} oracle {e_ora:.6e}")
    return rep


def test_cfg3_whole_tree_vs_oracle():
    rep = _full_size(3)
    assert rep["nodes"] == 4467


def test_cfg4_top_levels_and_depth2_subtrees_vs_oracle():
    _full_size(4)


@pytest.mark.slow
def test_cfg5_depth2_subtrees_in_full_tree_vs_oracle():
    _full_size(5)


def test_cfg5_depth2_subtrees_standalone_vs_oracle():
    """Each sampled cfg-5 depth-2 cell as its own problem: x' = (x - cell/4)·4 maps the cell onto the unit
    cube exactly (Sterbenz subtraction, power-of-two scaling), so the GPU's root is the depth-2 node with
    the original values — the same computation as the golden subtree (Alg. 1 on that node), depth
    limit D - 2."""
    import paper_1511_01353_b200 as fmi
    cfg = workloads.CONFIGS[5]
    gold = _golden(5)
    pts = workloads.uniform_points(cfg.n, 0)
    c2 = workloads.cell_of(pts, 2)
    L = fo.rank(cfg.degree)
    per = int(gold["q_per_cell"])
    scale = 0.0
    subs = []
    for t, cell in enumerate(gold["pick"]):
        cell = tuple(int(v) for v in cell)
        x = np.ascontiguousarray(pts[np.all(c2 == np.array(cell), axis=1)])
        subs.append((t, cell, x, workloads.franke3d(x)))
        scale = max(scale, float(np.max(np.abs(subs[-1][3]))))
    del pts, c2
    gd = {(int(gold["depth"][i]), tuple(int(v) for v in gold["cell"][i])): i for i in range(len(gold["depth"]))}
    for t, cell, x, f in subs:
        xm = (x - np.array(cell) / 4.0) * 4.0
        assert xm.min() >= 0.0 and xm.max() <= 1.0
        q = workloads.cell_queries(2, cell, per, int(gold["q_seed0"]) + t)
        qm = np.ascontiguousarray((q - np.array(cell) / 4.0) * 4.0)
        with fmi.build(torch.from_numpy(xm).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol,
                       cfg.max_depth - 2) as tree:
            ex = tree.export()
            got = tree.eval(torch.from_numpy(qm).cuda()).cpu().numpy()
        sel = [i for (d, c), i in gd.items() if tuple(v >> (d - 2) for v in c) == cell]
        sub = {k: v[sel] for k, v in gold.items() if isinstance(v, np.ndarray) and v.shape[:1] == gold["depth"].shape}
        rep = compare_with_golden(ex, sub, cfg.tol, L, cfg.max_depth, 1e-3, scale, depth_offset=2, cell_offset=cell)
        ref = gold["values"][t * per:(t + 1) * per]
        err = float(np.max(np.abs(got - ref)))
        assert err <= 1e-9 * scale, (cell, err)
        print(f"cfg5 cell {cell}: {rep['nodes']} nodes, {rep['decisions']} decisions, ties {rep['ties']}, "
              f"max|d| {err:.3e}")
