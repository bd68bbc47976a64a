"""Pins for the oracle (oracle/fmt_oracle.py) against what the paper and mathematics fix.

None of these checks re-types the oracle's own formula: each compares it with a value the
paper prints, a closed form, a special case that reduces to a library routine using an
independent basis (Legendre products + SVD least squares), or a brute-force rebuild of the
tree.  A plausible mistake (dropped basis term, wrong sign or index, a transposed operand,
wrong residual used for a decision, wrong block bookkeeping) fails at least one of them.
"""
import os

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

import workloads
from oracle import fmt_oracle as fo

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------------------------------------
# independent least-squares machinery (Legendre-product basis in root-cube coordinates, SVD lstsq)
# ---------------------------------------------------------------------------------------------

def _leg_total(x, p):
    """Total-degree-p Legendre-product basis at points x in [-1,1]^3 (an independent basis of the
    same polynomial space as Λ)."""
    V = npleg.legvander3d(x[:, 0], x[:, 1], x[:, 2], [p, p, p])
    keep = [i * (p + 1) ** 2 + j * (p + 1) + k
            for i in range(p + 1) for j in range(p + 1) for k in range(p + 1) if i + j + k <= p]
    return V[:, keep]


def _ls_fit(x, f, p):
    V = _leg_total(2 * x - 1, p)
    c, *_ = np.linalg.lstsq(V, f, rcond=None)
    return c


def _ls_eval(c, x, p):
    return _leg_total(2 * x - 1, p) @ c


def _random_poly(rng, p, ncoef=6):
    """A random degree-<=p polynomial given as a sum of products of p random affine forms —
    no monomial basis involved."""
    A = rng.standard_normal((ncoef, p, 3))
    b = rng.standard_normal((ncoef, p))
    w = rng.standard_normal(ncoef)

    def f(x):
        out = np.zeros(x.shape[0])
        for t in range(ncoef):
            prod = np.ones(x.shape[0])
            for k in range(p):
                prod *= x @ A[t, k] + b[t, k]
            out += w[t] * prod
        return out
    return f


# ---------------------------------------------------------------------------------------------
# basis and rank
# ---------------------------------------------------------------------------------------------

def test_rank_matches_printed_ranks():
    for lmax, L in _read_golden("ranks.txt"):
        assert fo.rank(int(lmax)) == int(L)
        assert len(fo.basis(int(lmax))) == int(L)


def test_basis_order_alg2_loops():
    expect = [tuple(int(v) for v in row) for row in _read_golden("basis_p1.txt")]
    assert fo.basis(1) == expect
    b = fo.basis(5)
    assert len(set(b)) == len(b) and all(sum(t) <= 5 for t in b)


def test_vandermonde_special_values():
    # x = 0: only the constant column survives; x = (2,0,0): Λ_200 = 2^2/2! = 2 (geometric moment)
    V = fo.vandermonde(np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [1.0, 1.0, 1.0]]), 2)
    assert V[0, 0] == 1.0 and np.all(V[0, 1:] == 0.0)
    assert V[1, fo.basis(2).index((2, 0, 0))] == 2.0
    assert V[2, fo.basis(2).index((1, 1, 0))] == 1.0
    assert V[2, fo.basis(2).index((0, 0, 2))] == 0.5


# ---------------------------------------------------------------------------------------------
# node fit (Algorithm 2)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", [0, 1, 3, 4, 6])
def test_fit_reproduces_polynomials(p):
    """Closed form: f a degree-<=p polynomial => the LS fit is exact, residual ~ 0 (BJ north_star pin 1)."""
    rng = np.random.default_rng(10 + p)
    u = rng.uniform(-1, 1, (max(3 * fo.rank(p), 50), 3))
    poly = _random_poly(rng, p) if p > 0 else (lambda x: np.full(x.shape[0], 0.37))
    f = poly(u)
    fit = fo.fit_node(u, f, p)
    r = f - fo.vandermonde(u, p) @ fit.coeffs
    assert np.max(np.abs(r)) <= 1e-11 * np.max(np.abs(f))
    q = rng.uniform(-1, 1, (200, 3))
    assert np.max(np.abs(fo.vandermonde(q, p) @ fit.coeffs - poly(q))) <= 1e-10 * np.max(np.abs(f))


@pytest.mark.parametrize("p", [1, 2, 4])
def test_fit_unisolvent_interpolates(p):
    """Special case: N = 𝓛 points in general position => interpolation (BJ north_star pin 2)."""
    rng = np.random.default_rng(20 + p)
    L = fo.rank(p)
    u = rng.uniform(-1, 1, (L, 3))
    f = rng.standard_normal(L)
    fit = fo.fit_node(u, f, p)
    assert fit.kept.all()
    assert np.max(np.abs(fo.vandermonde(u, p) @ fit.coeffs - f)) <= 1e-9


@pytest.mark.parametrize("p", [12, 14])
def test_fit_high_degree_equals_independent_lstsq(p):
    """The unscoped high-order fits of Fig. 1 (L_max up to 14): the oracle's Householder QR of
    the monomial Vandermonde keeps every column on a random point set and gives the fitted values of an
    SVD least-squares fit in the Legendre product basis."""
    rng = np.random.default_rng(30 + p)
    u = rng.uniform(-1, 1, (4 * fo.rank(p), 3))
    f = workloads.franke3d((u + 1) / 2)
    fit = fo.fit_node(u, f, p)
    assert fit.kept.all()
    ours = fo.vandermonde(u, p) @ fit.coeffs
    ref = _ls_eval(_ls_fit((u + 1) / 2, f, p), (u + 1) / 2, p)
    assert np.max(np.abs(ours - ref)) <= 1e-11


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_fit_equals_independent_lstsq(p):
    """Library routine with an independent basis: same fitted values as SVD lstsq on Legendre products."""
    rng = np.random.default_rng(30 + p)
    u = rng.uniform(-1, 1, (400, 3))
    f = workloads.franke3d((u + 1) / 2)
    fit = fo.fit_node(u, f, p)
    ours = fo.vandermonde(u, p) @ fit.coeffs
    c = _ls_fit((u + 1) / 2, f, p)
    ref = _ls_eval(c, (u + 1) / 2, p)
    assert np.max(np.abs(ours - ref)) <= 1e-12


def test_fit_p0_is_mean():
    """p = 0: Λ is the column of ones, the LS constant is the mean."""
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, (101, 3))
    f = rng.standard_normal(101)
    fit = fo.fit_node(u, f, 0)
    assert abs(fit.coeffs[0] - np.mean(f)) <= 1e-15 * 101


def test_fit_annihilates_fitted_subspace():
    """Λᵀ r = 0 for the LS residual, relative to ‖Λ‖ ‖f‖."""
    rng = np.random.default_rng(4)
    u = rng.uniform(-1, 1, (1000, 3))
    f = workloads.franke3d((u + 1) / 2)
    for p in (2, 4, 6):
        fit = fo.fit_node(u, f, p)
        V = fo.vandermonde(u, p)
        r = f - V @ fit.coeffs
        g = V.T @ r / (np.linalg.norm(V, axis=0) * np.linalg.norm(f))
        assert np.max(np.abs(g)) <= 1e-12


@pytest.mark.parametrize("zval", [0.0, -0.4])
def test_fit_coplanar_truncates_to_2d(zval):
    """Rank deficiency (reading G9): all points on a plane z = const.  The columns with n >= 1 are
    zero (zval = 0) or in the span of earlier columns (zval != 0) and must be dropped, never NaN; the
    fitted values equal the 2-D least-squares fit (Legendre products in x, y)."""
    rng = np.random.default_rng(5)
    p = 3
    u = rng.uniform(-1, 1, (300, 3))
    u[:, 2] = zval
    f = workloads.franke3d((u + 1) / 2)
    fit = fo.fit_node(u, f, p)
    assert np.all(np.isfinite(fit.coeffs))
    assert fit.kept.sum() == (p + 1) * (p + 2) // 2
    # kept columns are exactly those with n == 0 (the first column of each (l, m) run)
    if zval == 0.0:
        assert all(fit.kept[i] == (n == 0) for i, (l, m, n) in enumerate(fo.basis(p)))
    V2 = npleg.legvander2d(u[:, 0], u[:, 1], [p, p])
    keep = [i * (p + 1) + j for i in range(p + 1) for j in range(p + 1) if i + j <= p]
    c2, *_ = np.linalg.lstsq(V2[:, keep], f, rcond=None)
    assert np.max(np.abs(fo.vandermonde(u, p) @ fit.coeffs - V2[:, keep] @ c2)) <= 1e-12


def test_fit_duplicate_points():
    rng = np.random.default_rng(6)
    u = rng.uniform(-1, 1, (60, 3))
    u = np.vstack([u, u])
    f = np.concatenate([np.sin(u[:60, 0]), np.sin(u[:60, 0])])
    fit = fo.fit_node(u, f, 2)
    c = _ls_fit((u + 1) / 2, f, 2)
    assert np.max(np.abs(fo.vandermonde(u, 2) @ fit.coeffs - _ls_eval(c, (u + 1) / 2, 2))) <= 1e-12


# ---------------------------------------------------------------------------------------------
# partition (Alg. 1 FMT_Ordered_by_Octant, FMT_New_Octant)
# ---------------------------------------------------------------------------------------------

def test_octant_numbering_and_ties():
    ul = np.array([[-0.5, -0.5, -0.5], [0.5, -0.5, -0.5], [-0.5, 0.5, -0.5], [0.5, 0.5, 0.5],
                   [0.0, -0.1, -0.1], [0.0, 0.0, 0.0]])
    assert list(fo.octant(ul)) == [0, 1, 2, 7, 1, 7]   # x fastest; 0 -> upper side


def test_local_coords_child_frames():
    # child of the root in octant (+,+,+): centre (3/4,3/4,3/4), half-width 1/4
    u = np.array([[0.75, 0.75, 0.75], [0.5, 0.5, 0.5], [1.0, 1.0, 1.0]])
    ul = fo.local_coords(u, 1, np.array([1, 1, 1]))
    assert np.array_equal(ul, [[0, 0, 0], [-1, -1, -1], [1, 1, 1]])
    assert fo.morton_prefix(1, (1, 0, 0)) == 1 and fo.morton_prefix(1, (0, 0, 1)) == 4
    assert fo.morton_prefix(2, (3, 0, 0)) == 0b001001


# ---------------------------------------------------------------------------------------------
# whole tree (Algorithm 1)
# ---------------------------------------------------------------------------------------------

def _brute_tree(pts, f, p, tau, D):
    """Independent rebuild: every node's fitted values = LS fit of the ORIGINAL f on its points
    (telescoping identity), membership by direct coordinate comparison with the
    dyadic split planes, decisions from that LS residual."""
    L = fo.rank(p)
    nodes = {}
    todo = [(0, (0, 0, 0), np.arange(pts.shape[0]))]
    while todo:
        d, cell, idx = todo.pop()
        c = _ls_fit(pts[idx], f[idx], p)
        res = f[idx] - _ls_eval(c, pts[idx], p)
        h = 0.5 ** (d + 1)
        ctr = (2 * np.array(cell) + 1) * h
        up = pts[idx] >= ctr
        o = up[:, 0] * 1 + up[:, 1] * 2 + up[:, 2] * 4
        child = {}
        for oc in range(8):
            sel = o == oc
            n_o = int(sel.sum())
            e = float(np.sqrt(np.mean(res[sel] ** 2))) if n_o else np.nan
            child[oc] = (n_o, e)
            if n_o and e > tau and n_o >= L and d + 1 <= D:
                cc = (2 * cell[0] + (oc & 1), 2 * cell[1] + ((oc >> 1) & 1), 2 * cell[2] + ((oc >> 2) & 1))
                todo.append((d + 1, cc, idx[sel]))
        nodes[(d, cell)] = dict(n=idx.size, coef=c, rms=float(np.sqrt(np.mean(res ** 2))), child=child)
    return nodes


def _deepest(nodes, x, D):
    d, cell = 0, (0, 0, 0)
    while True:
        h = 0.5 ** (d + 1)
        ctr = (2 * np.array(cell) + 1) * h
        up = x >= ctr
        cc = (2 * cell[0] + int(up[0]), 2 * cell[1] + int(up[1]), 2 * cell[2] + int(up[2]))
        if (d + 1, cc) in nodes:
            d, cell = d + 1, cc
        else:
            return d, cell


@pytest.mark.parametrize("p,N,D,seed", [(1, 300, 2, 0), (2, 300, 2, 1), (2, 2000, 3, 2), (0, 200, 3, 3)])
def test_tree_matches_brute_force(p, N, D, seed):
    rng = np.random.default_rng(seed)
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    # choose tau between two observed child E values so that tau prunes some nodes with a margin
    full = _brute_tree(pts, f, p, 0.0, D)
    es = sorted({round(v[1], 15) for nd in full.values() for v in nd["child"].values() if v[0] >= fo.rank(p)})
    tau = float(np.sqrt(es[len(es) // 3] * es[len(es) // 3 + 1]))
    ref = _brute_tree(pts, f, p, tau, D)
    tree = fo.build(pts, f, p, tau, D)
    got = {(int(tree.depth[i]), tuple(int(v) for v in tree.cell[i])): i for i in range(tree.node_count)}
    assert set(got) == set(ref), "topology differs from the brute-force tree"
    assert 1 < len(ref) < len(full) or len(full) == 1
    for key, i in got.items():
        assert tree.n_points[i] == ref[key]["n"]
        assert abs(tree.residual_rms[i] - ref[key]["rms"]) <= 1e-13
        for oc in range(8):
            n_o, e = ref[key]["child"][oc]
            assert tree.child_count[i][oc] == n_o
            if n_o:
                assert abs(tree.child_rms[i][oc] - e) <= 1e-13
    # evaluation: path sum == LS fit of the deepest node containing the query (telescoping)
    q = rng.random((500, 3))
    val = fo.evaluate(tree, q)
    for t in range(q.shape[0]):
        key = _deepest(ref, q[t], D)
        assert abs(val[t] - _ls_eval(ref[key]["coef"], q[t:t + 1], p)[0]) <= 1e-11
    # bookkeeping: interpolant at the fit points + final residual == original samples
    assert np.max(np.abs(fo.evaluate(tree, pts) + tree.residual - f)) <= 1e-12


def test_tree_polynomial_is_one_node():
    """A global degree-<=p polynomial is fitted exactly at the root: 1 node."""
    rng = np.random.default_rng(7)
    p = 4
    poly = _random_poly(rng, p)
    pts = rng.random((3000, 3))
    f = poly(pts)
    tree = fo.build(pts, f, p, 1e-9 * np.max(np.abs(f)), 5)
    assert tree.node_count == 1
    q = rng.random((300, 3))
    assert np.max(np.abs(fo.evaluate(tree, q) - poly(q))) <= 1e-10 * np.max(np.abs(f))


def test_tree_constant_and_large_tau():
    rng = np.random.default_rng(8)
    pts = rng.random((500, 3))
    assert fo.build(pts, np.full(500, 2.5), 2, 1e-12, 4).node_count == 1
    assert fo.build(pts, workloads.franke3d(pts), 2, 1e30, 4).node_count == 1


def test_tree_residual_never_increases():
    """LS minimality: each node's post-fit RMS <= the RMS of the residual it received."""
    pts = workloads.uniform_points(5000, 0)
    f = workloads.franke3d(pts)
    tree = fo.build(pts, f, 3, 1e-7, 3)
    assert tree.node_count > 9
    assert tree.residual_rms[0] <= np.sqrt(np.mean(f ** 2))
    for i in range(tree.node_count):
        for oc in range(8):
            c = tree.child_index[i][oc]
            if c >= 0:
                assert tree.residual_rms[c] <= tree.child_rms[i][oc] * (1 + 1e-12)


def test_tree_depth_cap_and_count_guard():
    pts = workloads.uniform_points(4000, 1)
    f = workloads.franke3d(pts)
    L = fo.rank(2)
    tree = fo.build(pts, f, 2, 0.0, 2)
    assert tree.depth.max() <= 2
    assert np.all(tree.n_points >= L)
    # every octant block with n_o >= 𝓛 below the cap has a child (tau = 0 and E > 0)
    for i in range(tree.node_count):
        for oc in range(8):
            want = tree.child_count[i][oc] >= L and tree.depth[i] + 1 <= 2
            assert (tree.child_index[i][oc] >= 0) == want


def test_tree_rejects_too_few_points():
    with pytest.raises(ValueError):
        fo.build(np.random.default_rng(0).random((10, 3)), np.zeros(10), 3, 1e-6, 2)


def test_evaluate_outside_root_uses_root_only():
    pts = workloads.uniform_points(3000, 2)
    f = workloads.franke3d(pts)
    tree = fo.build(pts, f, 2, 1e-9, 2)
    q = np.array([[1.5, 0.2, 0.2], [-0.1, 0.5, 0.5]])
    ul = fo.local_coords(q, 0, np.zeros(3, dtype=np.int64))
    assert np.allclose(fo.evaluate(tree, q), fo.vandermonde(ul, 2) @ tree.coeffs[0], rtol=0, atol=1e-15)


def test_general_root_cube():
    """Data outside [0,1]^3: isotropic bounding cube (G6).  An affine image of a unit-cube problem
    gives the same topology and the same interpolant."""
    rng = np.random.default_rng(9)
    pts = np.vstack([rng.random((3000, 3)), [[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]]])
    f = workloads.franke3d(pts)
    t1 = fo.build(pts, f, 2, 1e-4, 2)
    shift = np.array([-3.0, 5.0, 0.25])
    t2 = fo.build(pts * 4.0 + shift, f, 2, 1e-4, 2)
    lo, w = fo.root_cube(pts * 4.0 + shift)
    assert np.array_equal(lo, shift) and w == 4.0
    assert t1.node_count == t2.node_count > 1
    assert np.array_equal(t1.cell[t1.key_order()], t2.cell[t2.key_order()])
    q = rng.random((100, 3))
    assert np.max(np.abs(fo.evaluate(t1, q) - fo.evaluate(t2, q * 4.0 + shift))) <= 1e-10


@pytest.mark.slow
def test_beats_prior_work_franke():
    """PAPER.md:398-402 (§4): the method beats the prior-work errors E_rms = 6e-5, E_inf = 6e-3."""
    (n, lmax, tau, erms_b, einf_b), = _read_golden("prior_work.txt")
    n, lmax, tau = int(n), int(lmax), float(tau)
    pts = workloads.uniform_points(n, 0)
    tree = fo.build(pts, workloads.franke3d(pts), lmax, tau, 8)
    q = workloads.uniform_points(n, 1)
    erms, einf = workloads.rms_and_max(fo.evaluate(tree, q) - workloads.franke3d(q))
    assert erms < float(erms_b) and einf < float(einf_b)


# ---------------------------------------------------------------------------------------------
# row-streamed QR (TSQR branch of _qr_r and of fit_node, nodes above 2^16 rows)
# ---------------------------------------------------------------------------------------------

def test_qr_r_tsqr_branch_equals_lapack():
    """_qr_r above _TSQR_ROWS rows streams blocks (R <- qr([R; block])).  Householder R is unique up
    to the signs of its rows: |R| must equal LAPACK's one-shot dgeqrf R of the same matrix, and RᵀR
    must equal AᵀA."""
    rng = np.random.default_rng(11)
    n = fo._TSQR_ROWS + 4_321
    A = rng.standard_normal((n, 24))
    A[:, 5] *= 1e-3
    R = fo._qr_r(A)
    R0 = np.linalg.qr(A, mode="r")
    assert R.shape == R0.shape == (24, 24)
    s = np.sign(np.diag(R)) * np.sign(np.diag(R0))
    assert np.max(np.abs(R * s[:, None] - R0)) <= 1e-10 * np.max(np.abs(R0))
    G = A.T @ A
    assert np.max(np.abs(R.T @ R - G)) <= 1e-11 * np.max(np.abs(G))


@pytest.mark.parametrize("coplanar", [False, True])
def test_fit_node_streamed_equals_single_block(coplanar, monkeypatch):
    """fit_node on more than _TSQR_ROWS rows (column norms and TSQR streamed over row blocks) gives the
    same fit as the single-block path on the same rows, including the rank-truncation walk."""
    rng = np.random.default_rng(12)
    u = rng.uniform(-1, 1, (3_000, 3))
    if coplanar:
        u[:, 2] = -0.25
    f = workloads.franke3d((u + 1) / 2)
    p = 4
    one = fo.fit_node(u, f, p)
    monkeypatch.setattr(fo, "_TSQR_ROWS", 700)
    many = fo.fit_node(u, f, p)
    assert np.array_equal(one.kept, many.kept)
    V = fo.vandermonde(u, p)
    assert np.max(np.abs(V @ one.coeffs - V @ many.coeffs)) <= 1e-12
    assert np.max(np.abs(fo.apply_fit(u, many.coeffs, p) - V @ many.coeffs)) <= 1e-15


def test_fit_node_above_tsqr_threshold_equals_independent_lstsq():
    """A node with more than 2^16 points (the real streaming threshold): fitted values equal an SVD
    least-squares fit in the Legendre product basis (independent basis and routine)."""
    rng = np.random.default_rng(13)
    u = rng.uniform(-1, 1, (fo._TSQR_ROWS + 3_777, 3))
    f = workloads.franke3d((u + 1) / 2)
    p = 3
    fit = fo.fit_node(u, f, p)
    assert fit.kept.all()
    ours = fo.apply_fit(u, fit.coeffs, p)
    ref = _ls_eval(_ls_fit((u + 1) / 2, f, p), (u + 1) / 2, p)
    assert np.max(np.abs(ours - ref)) <= 1e-12


def test_restricted_and_node_started_runs_reproduce_the_full_tree():
    """Alg. 1 called on a node (build_subtree) with the residual that node receives, and a run whose
    expansion is restricted to a few cells (descend), reproduce the unrestricted run's nodes exactly:
    the recursion only reads the node's own block."""
    pts = workloads.uniform_points(6_000, 3)
    f = workloads.franke3d(pts)
    p, tau, D = 2, 1e-5, 3
    full = fo.build(pts, f, p, tau, D)
    fk = {(int(full.depth[i]), tuple(int(v) for v in full.cell[i])): i for i in range(full.node_count)}
    pick = {(2, (1, 2, 0)), (2, (3, 3, 3))}

    def descend(d, cell):
        return d < 2 or any(d >= dd and tuple(c >> (d - dd) for c in cell) == cc for dd, cc in pick)

    part = fo.build(pts, f, p, tau, D, descend=descend)
    assert 9 < part.node_count < full.node_count
    for i in range(part.node_count):
        key = (int(part.depth[i]), tuple(int(v) for v in part.cell[i]))
        j = fk[key]
        assert np.array_equal(part.coeffs[i], full.coeffs[j])
        assert np.array_equal(part.child_count[i], full.child_count[j])
        assert np.array_equal(part.child_index[i] != -1, full.child_index[j] >= 0)
        if key[0] == 2 and key not in pick:
            raise AssertionError("expanded a node outside the restriction")
    # node-started run: depth-1 node (1,0,1) with the residual the root leaves on its points
    cell = (1, 0, 1)
    inside = np.all(np.minimum(np.floor(pts * 2), 1).astype(int) == cell, axis=1)
    root_only = fo.build(pts, f, p, tau, D, descend=lambda d, c: False)
    sub = fo.build_subtree(pts[inside], root_only.residual[inside], p, tau, D, 1, cell)
    for i in range(sub.node_count):
        j = fk[(int(sub.depth[i]), tuple(int(v) for v in sub.cell[i]))]
        assert np.array_equal(sub.coeffs[i], full.coeffs[j])
        assert sub.residual_rms[i] == full.residual_rms[j]
    assert sub.node_count == sum(1 for k in fk if k[0] >= 1 and tuple(c >> (k[0] - 1) for c in k[1]) == cell)
    # evaluation inside the subtree: same path sum as the full tree minus the root term
    q = (np.array(cell) + workloads.uniform_points(300, 4)) / 2
    ul0 = fo.local_coords(q, 0, np.zeros(3, dtype=np.int64))
    got = fo.evaluate(sub, q) + fo.apply_fit(ul0, full.coeffs[0], p)
    assert np.max(np.abs(got - fo.evaluate(full, q))) <= 1e-14


def _walk_by_lstsq(u, p, delta):
    """Reading G9 computed independently: walk the equilibrated Λ columns in Algorithm-2 order and keep
    column j iff its distance from the span of the kept columns (SVD least squares, not the oracle's
    Householder re-triangularisation) exceeds delta; returns the kept mask and every distance."""
    lam = fo.vandermonde(u, p)
    a = lam / np.linalg.norm(lam, axis=0)
    kept, dist = [], []
    for j in range(a.shape[1]):
        if kept:
            c, *_ = np.linalg.lstsq(a[:, kept], a[:, j], rcond=None)
            d = float(np.linalg.norm(a[:, j] - a[:, kept] @ c))
        else:
            d = float(np.linalg.norm(a[:, j]))
        dist.append(d)
        if d > delta:
            kept.append(j)
    mask = np.zeros(a.shape[1], dtype=bool)
    mask[kept] = True
    return mask, np.array(dist)


@pytest.mark.parametrize("eps", [1e-4, 1e-5, 3e-6, 1e-6, 3e-7, 1e-7, 1e-8])
def test_g9_walk_near_threshold(eps):
    """Column rejection near δ = 1e-6 (reading G9; PAPER.md P:330 is silent on rank deficiency): points
    on the curved sheet z = x² + ε·w, so the column x² is at distance ~ε from the span of the columns
    before it (z is one of them).  The oracle's kept set equals an independent SVD-least-squares walk
    for every decision whose distance is not within 1% of δ, and the sheet's x²-type columns flip from
    kept to dropped as ε crosses δ."""
    rng = np.random.default_rng(11)
    n = 400
    x, y, w = rng.uniform(-1, 1, (3, n))
    u = np.stack([x, y, x * x + eps * w], axis=1)
    p = 2
    fit = fo.fit_node(u, workloads.franke3d((u + 1) / 2), p)
    mask, dist = _walk_by_lstsq(u, p, fo.DELTA)
    clear = np.abs(dist / fo.DELTA - 1.0) > 1e-2
    assert np.array_equal(fit.kept[clear], mask[clear])
    j_x2 = fo.basis(p).index((2, 0, 0))
    assert fit.kept[j_x2] == (dist[j_x2] > fo.DELTA)
    if eps >= 1e-6:
        assert fit.kept[j_x2]
    if eps <= 3e-7:
        assert not fit.kept[j_x2]
