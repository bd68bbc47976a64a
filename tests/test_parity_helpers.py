"""Host-side checks of the golden comparison used by the full-size GPU parity tests
(tests/parity.py compare_with_golden): an oracle tree compared with its own golden table passes, a
flipped decision, a wrong count or an extra node fails, and a restricted / stand-alone (mapped) subtree
is compared in the right coordinates."""
import os
import sys

import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo
from parity import compare_with_golden

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import make_golden  # noqa: E402


def _export(t):
    """An oracle tree in the layout of paper_1511_01353_b200.Tree.export()."""
    return {"depth": t.depth, "cell": t.cell, "n_points": t.n_points, "child_count": t.child_count,
            "residual_rms": t.residual_rms, "child": np.where(t.child_index >= 0, t.child_index, -1)}


@pytest.fixture(scope="module")
def small():
    pts = workloads.uniform_points(8000, 21)
    f = workloads.franke3d(pts)
    p, tau, D = 2, 2e-4, 3
    return pts, f, p, tau, D, fo.build(pts, f, p, tau, D)


def test_identical_tree_passes_and_flips_fail(small):
    pts, f, p, tau, D, t = small
    gold = make_golden._node_table([t])
    ex = _export(t)
    rep = compare_with_golden(ex, gold, tau, fo.rank(p), D, 0.0, 1.0)
    assert rep["nodes"] == t.node_count and rep["decisions"] > 10 and not rep["ties"]
    # a decision flipped on the "GPU" side
    i = int(np.flatnonzero((t.child_index >= 0).any(axis=1) & (t.depth > 0))[0])
    o = int(np.flatnonzero(t.child_index[i] >= 0)[0])
    bad = {k: v.copy() for k, v in ex.items()}
    bad["child"][i][o] = -1
    with pytest.raises(AssertionError):
        compare_with_golden(bad, gold, tau, fo.rank(p), D, 0.0, 1.0)
    # ... but accepted as a tie when the oracle margin is inside the band
    m = abs(gold_margin(gold, t, i, o, tau))
    compare_with_golden(bad, gold, tau, fo.rank(p), D, m * 1.01 + 1e-300, 1.0, within=lambda d, c: False)
    # a wrong octant count
    bad = {k: v.copy() for k, v in ex.items()}
    bad["child_count"][0][3] += 1
    with pytest.raises(AssertionError):
        compare_with_golden(bad, gold, tau, fo.rank(p), D, 0.0, 1.0)
    # a node RMS off by more than roundoff
    bad = {k: v.copy() for k, v in ex.items()}
    bad["residual_rms"][2] *= 1.001
    with pytest.raises(AssertionError):
        compare_with_golden(bad, gold, tau, fo.rank(p), D, 0.0, 1.0)


def gold_margin(gold, t, i, o, tau):
    d, c = int(t.depth[i]), tuple(int(v) for v in t.cell[i])
    j = [k for k in range(len(gold["depth"])) if gold["depth"][k] == d and tuple(gold["cell"][k]) == c][0]
    return gold["child_rms"][j][o] / tau - 1.0


def test_extra_gpu_node_fails(small):
    pts, f, p, tau, D, t = small
    # golden without one leaf: the "GPU" tree then has an extra node
    leaf = int(np.flatnonzero((t.child_index < 0).all(axis=1) & (t.depth == t.depth.max()))[0])
    gold = make_golden._node_table([t])
    keep = [k for k in range(len(gold["depth"]))
            if not (gold["depth"][k] == t.depth[leaf] and tuple(gold["cell"][k]) == tuple(t.cell[leaf]))]
    g2 = {k: v[keep] for k, v in gold.items()}
    with pytest.raises(AssertionError):
        compare_with_golden(_export(t), g2, tau, fo.rank(p), D, 0.0, 1.0)


def test_restricted_golden_and_mapped_subtree(small):
    pts, f, p, tau, D, t = small
    cell = (1, 2, 1)
    top = fo.build(pts, f, p, tau, D, descend=lambda d, c: d <= 1)
    inside = np.all(workloads.cell_of(pts, 2) == np.array(cell), axis=1)
    sub = fo.build_subtree(pts[inside], top.residual[inside], p, tau, D, 2, cell)
    gold = make_golden._node_table([top, sub])

    def within(d, c):
        return d <= 1 or tuple(v >> (d - 2) for v in c) == cell
    rep = compare_with_golden(_export(t), gold, tau, fo.rank(p), D, 0.0, 1.0, within=within)
    assert rep["nodes"] == top.node_count + sub.node_count
    # the same subtree solved as its own problem on the unit cube (telescoping start: original f)
    tel = fo.build_subtree(pts[inside], f[inside], p, tau, D, 2, cell)
    xm = (pts[inside] - np.array(cell) / 4.0) * 4.0
    alone = fo.build(xm, f[inside], p, tau, D - 2)
    assert alone.node_count == tel.node_count
    g3 = make_golden._node_table([tel])
    compare_with_golden(_export(alone), g3, tau, fo.rank(p), D, 0.0, 1.0, depth_offset=2, cell_offset=cell)
