"""the unscoped high-order fit (one node, max_depth = 0, degree up to 14) —
PAPER.md §3 / Fig. 1 (L_max = 6, 10, 14) — through the QR path of
csrc/unscoped.cu (R of the monomial Vandermonde as R_V·C through the Legendre basis, then the G9
rejection walk), against the oracle (Householder QR of the monomial Vandermonde, Algorithm 2,
P:330-331).

Bars: the rank (kept columns) equal to the oracle's; the evaluated interpolant within 1e-9·max|f| (the
north_star bar) at every degree — measured differences are ~3e-13·max|f| at p = 14 (N = 5000,
profiles/round1_fig1_f2.jsonl), so the bar holds with a wide margin although both sides evaluate the
monomial form Σ a_α u^α, whose conditioning grows with p.
"""
import os

import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EVAL_TOL = 1e-9
EVAL_TOL_HI = 1e-9


def _fmi():
    import paper_1511_01353_b200 as fmi
    fmi.load_library()
    return fmi


class _UnscopedQR:
    """Route max_depth = 0 builds of any degree through the QR path (FMI_UNSCOPED_QR=1)."""

    def __enter__(self):
        os.environ["FMI_UNSCOPED_QR"] = "1"

    def __exit__(self, *a):
        os.environ.pop("FMI_UNSCOPED_QR", None)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(pts, f, p, q):
    fmi = _fmi()
    with fmi.build(_dev(pts), _dev(f), p, 1e-12, 0) as tree:
        ex = tree.export()
        val = tree.eval(_dev(q)).cpu().numpy()
        res = tree.residual()
    return ex, val, res


def _oracle(pts, f, p, q):
    ora = fo.build(pts, f, p, 1e-12, 0)
    return ora, fo.evaluate(ora, q)


@pytest.mark.parametrize("p", [0, 2, 6, 10])
def test_qr_path_matches_oracle_low_degree(p):
    L = fo.rank(p)
    rng = np.random.default_rng(300 + p)
    N = 20 * L + 13
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    q = rng.random((3000, 3))
    with _UnscopedQR():
        ex, val, res = _run(pts, f, p, q)
    ora, ref = _oracle(pts, f, p, q)
    assert ex["depth"].tolist() == [0]
    assert int(ex["rank"][0]) == int(ora.kept[0].sum())
    assert np.max(np.abs(val - ref)) <= EVAL_TOL * np.max(np.abs(f))
    # residual bookkeeping: interpolant(x_i) + r_i = f_i
    with _UnscopedQR():
        _, at_pts, _ = _run(pts, f, p, pts)
    assert np.max(np.abs(at_pts + res - f)) <= 1e-12 * np.max(np.abs(f)) * max(1, L)
    assert np.array_equal(ex["child_count"][0], ora.child_count[0])
    assert abs(ex["residual_rms"][0] - ora.residual_rms[0]) <= 1e-6 * ora.residual_rms[0]


def test_qr_path_agrees_with_level_path():
    """max_depth = 0 at p = 8: the moment-Gram solve (K5) and the QR path give the same fit."""
    rng = np.random.default_rng(77)
    pts = rng.random((50_000, 3))
    f = workloads.franke3d(pts)
    q = rng.random((5000, 3))
    _, a, _ = _run(pts, f, 8, q)
    with _UnscopedQR():
        _, b, _ = _run(pts, f, 8, q)
    assert np.max(np.abs(a - b)) <= EVAL_TOL * np.max(np.abs(f))


@pytest.mark.parametrize("p", [11, 12, 13, 14])
def test_high_degree_vs_oracle(p):
    L = fo.rank(p)
    rng = np.random.default_rng(400 + p)
    N = 6 * L + 5
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    q = rng.random((2000, 3))
    ex, val, res = _run(pts, f, p, q)
    ora, ref = _oracle(pts, f, p, q)
    assert int(ex["rank"][0]) == int(ora.kept[0].sum())
    err = float(np.max(np.abs(val - ref)))
    assert err <= EVAL_TOL_HI * np.max(np.abs(f)), err
    assert abs(ex["residual_rms"][0] - ora.residual_rms[0]) <= 1e-3 * ora.residual_rms[0]


def test_degree14_reproduces_polynomials():
    """A polynomial of total degree 14 is reproduced (the fit's space contains it): residual ~ 0."""
    rng = np.random.default_rng(5)
    P = 14
    pts = rng.random((8000, 3))
    q = rng.random((3000, 3))

    def poly(x):
        u = 2.0 * x - 1.0
        v = np.zeros(len(x))
        c = np.random.default_rng(6)
        for a in range(P + 1):
            for b in range(P + 1 - a):
                for d in range(P + 1 - a - b):
                    k = c.standard_normal() / (1 + a + b + d) ** 2
                    v += k * (np.polynomial.legendre.legval(u[:, 0], [0] * a + [1])
                              * np.polynomial.legendre.legval(u[:, 1], [0] * b + [1])
                              * np.polynomial.legendre.legval(u[:, 2], [0] * d + [1]))
        return v

    f = poly(pts)
    ex, val, res = _run(pts, f, P, q)
    assert int(ex["rank"][0]) == fo.rank(P)
    scale = np.max(np.abs(f))
    assert np.max(np.abs(res)) <= 1e-8 * scale
    assert np.max(np.abs(val - poly(q))) <= 1e-7 * scale


def test_degree14_needs_enough_points():
    fmi = _fmi()
    pts = np.random.default_rng(0).random((fo.rank(14) - 1, 3))
    with pytest.raises(fmi.FmiError) as ei:
        fmi.build(pts, np.zeros(pts.shape[0]), 14, 1e-6, 0)
    assert ei.value.code == -2


@pytest.mark.parametrize("p", [8, 12])
def test_coplanar_points_rank_truncation(p):
    """Points on the plane z = 0.3: every column with a z power lies in the span of the z-free ones
    (G9 rejects them; rank = (p+1)(p+2)/2), the Legendre Gram is singular (zero pivots, kZeroPivot)."""
    rng = np.random.default_rng(500 + p)
    L = fo.rank(p)
    pts = rng.random((4 * L, 3))
    pts[:, 2] = 0.3
    f = workloads.franke3d(pts)
    q = np.column_stack([rng.random((1500, 2)), np.full(1500, 0.3)])
    with _UnscopedQR():
        ex, val, res = _run(pts, f, p, q)
    ora, ref = _oracle(pts, f, p, q)
    assert int(ora.kept[0].sum()) == (p + 1) * (p + 2) // 2
    assert int(ex["rank"][0]) == int(ora.kept[0].sum())
    assert np.max(np.abs(val - ref)) <= EVAL_TOL * np.max(np.abs(f))


# ---------------------------------------------------------------------------------------------
# the QR path on the octree (max_depth > 0): SURVEY §8 f3 at L_max = 12
# ---------------------------------------------------------------------------------------------

def _tree_parity(pts, f, p, tau, D, q, env=None):
    from parity import compare_trees
    fmi = _fmi()
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        with fmi.build(_dev(pts), _dev(f), p, tau, D) as tree:
            gpu = tree.export()
            val = tree.eval(_dev(q)).cpu().numpy()
            res = tree.residual()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ora = fo.build(pts, f, p, tau, D)
    ref = fo.evaluate(ora, q)
    g, o = compare_trees(gpu, ora, tau)
    scale = float(np.max(np.abs(f)))
    assert np.max(np.abs(val - ref)) <= EVAL_TOL * scale, float(np.max(np.abs(val - ref)))
    for key, gi in g.items():
        a, b = gpu["residual_rms"][gi], ora.residual_rms[o[key]]
        assert abs(a - b) <= 1e-6 * b + 1e-12 * scale, (key, a, b)
        assert gpu["rank"][gi] == int(ora.kept[o[key]].sum()), key
    return gpu, ora, val, res


@pytest.mark.parametrize("p,N,D,tau", [(12, 40_000, 2, 1e-9), (11, 30_000, 3, 1e-8)])
def test_qr_levels_high_degree_octree_vs_oracle(p, N, D, tau):
    """Degrees above the moment-Gram limit on the octree: every node by the QR path, level by level
    (Alg. 1): identical topology, counts and ranks, values within 1e-9·max|f|."""
    rng = np.random.default_rng(600 + p)
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    q = rng.random((4000, 3))
    gpu, ora, _, _ = _tree_parity(pts, f, p, tau, D, q)
    assert ora.node_count > 9 and gpu["depth"].max() == 2


@pytest.mark.parametrize("p", [3, 6])
def test_qr_levels_low_degree_vs_oracle_and_level_path(p):
    """FMI_QR_PATH=1 routes an octree build of any degree through the QR path: same tree as the oracle
    and as the moment-Gram level path."""
    rng = np.random.default_rng(700 + p)
    pts = rng.random((30_000, 3))
    f = workloads.franke3d(pts)
    q = rng.random((3000, 3))
    gpu, ora, val, _ = _tree_parity(pts, f, p, 1e-7, 4, q, env={"FMI_QR_PATH": "1"})
    fmi = _fmi()
    with fmi.build(_dev(pts), _dev(f), p, 1e-7, 4) as t:
        lv = t.eval(_dev(q)).cpu().numpy()
        assert t.node_count == gpu["depth"].shape[0]
    assert np.max(np.abs(val - lv)) <= EVAL_TOL * np.max(np.abs(f))
