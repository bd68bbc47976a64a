"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): identical topology and node point counts (bit-exact integer work),
evaluated interpolant within 1e-9·max|f| absolute, E_rms against the analytic function within 1%
relative of the oracle's.
"""
import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo
from parity import coeff_and_rms_errors, compare_trees, rms_agreement

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EVAL_TOL = 1e-9


def _fmi():
    import paper_1511_01353_b200 as fmi
    fmi.load_library()
    return fmi


def gpu_build(pts, f, p, tau, D, host=False):
    fmi = _fmi()
    if host:
        return fmi.build(pts, f, p, tau, D)
    return fmi.build(torch.from_numpy(np.ascontiguousarray(pts)).cuda(),
                     torch.from_numpy(np.ascontiguousarray(f)).cuda(), p, tau, D)


def gpu_eval(tree, q, host=False):
    if host:
        return tree.eval(np.ascontiguousarray(q))
    return tree.eval(torch.from_numpy(np.ascontiguousarray(q)).cuda()).cpu().numpy()


def check_parity(pts, f, p, tau, D, q, erms_vs=None):
    ora = fo.build(pts, f, p, tau, D)
    ref = fo.evaluate(ora, q)
    with gpu_build(pts, f, p, tau, D) as tree:
        gpu = tree.export()
        val = gpu_eval(tree, q)
    g, o = compare_trees(gpu, ora, tau)
    scale = float(np.max(np.abs(f))) if f.size else 1.0
    err = float(np.max(np.abs(val - ref))) if q.shape[0] else 0.0
    assert err <= EVAL_TOL * max(scale, 1e-300), f"max|gpu - oracle| = {err:.3e} > {EVAL_TOL * scale:.3e}"
    drms = coeff_and_rms_errors(gpu, ora, g, o)
    rms_agreement(gpu, ora, g, o, scale)  # every common node's post-fit RMS (asserted per node)
    if erms_vs is not None:
        truth = erms_vs(q)
        e_gpu, _ = workloads.rms_and_max(val - truth)
        e_ora, _ = workloads.rms_and_max(ref - truth)
        assert abs(e_gpu - e_ora) <= 0.01 * e_ora, (e_gpu, e_ora)
    return ora, gpu, val, ref, err, drms


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs small enough for the full oracle
# ---------------------------------------------------------------------------------------------

def test_cfg1_full_parity():
    cfg = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(cfg)
    ora, gpu, val, ref, err, drms = check_parity(pts, f, cfg.degree, cfg.tol, cfg.max_depth, q,
                                                 erms_vs=workloads.franke3d)
    assert ora.node_count == 29


def test_cfg2_full_parity():
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    q = q[:100_000]  # the oracle's evaluator is slow; the GPU evaluates all 1e6 in test_cfg2_eval_all
    ora, gpu, val, ref, err, drms = check_parity(pts, f, cfg.degree, cfg.tol, cfg.max_depth, q,
                                                 erms_vs=workloads.franke3d)
    assert ora.node_count == 585


def test_cfg2_eval_all_queries_host_pointers():
    """Full 1e6 queries through host pointers equal the device-pointer path bit for bit."""
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    with gpu_build(pts, f, cfg.degree, cfg.tol, cfg.max_depth, host=True) as th, \
            gpu_build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as td:
        a = gpu_eval(th, q, host=True)
        b = gpu_eval(td, q)
        assert np.array_equal(a, b)
        assert th.node_count == td.node_count == 585


# ---------------------------------------------------------------------------------------------
# sweeps over degree, ragged sizes, depth caps
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", list(range(0, 11)))
def test_degree_sweep(p):
    L = fo.rank(p)
    N = 9 * L + 37  # several chunks per node, ragged tail
    rng = np.random.default_rng(100 + p)
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    q = rng.random((3001, 3))
    check_parity(pts, f, p, 1e-12, 2, q)


@pytest.mark.parametrize("N,D,tau", [(5000, 0, 1e-6), (5000, 3, 0.0), (20011, 4, 1e-4), (777, 6, 1e-9)])
def test_depth_and_tau(N, D, tau):
    rng = np.random.default_rng(N + D)
    pts = rng.random((N, 3))
    f = workloads.franke3d(pts)
    q = rng.random((2000, 3))
    check_parity(pts, f, 3, tau, D, q)


def test_halton_split_plane_points():
    """Halton's first point has x = 0.5 exactly (on the root split plane); dyadic coordinates everywhere."""
    pts = workloads.halton_points(30_000)
    pts[:64] = np.array([[i / 8, j / 8, k / 4] for i in range(4) for j in range(4) for k in range(4)])
    f = workloads.franke3d(pts)
    q = np.vstack([workloads.uniform_points(5000, 1), pts[:64]])
    check_parity(pts, f, 4, 1e-7, 4, q)


def test_clipped_mixture_small():
    """Config-4 shaped data (clustered, clipped to the faces) at a size the oracle finishes quickly."""
    centres = workloads.mixture_centres(0)
    pts = workloads.mixture_points(60_000, 0, centres)
    f = workloads.mixture_values(pts, centres)
    q = workloads.mixture_points(20_000, 1, centres)
    check_parity(pts, f, 6, 1e-9, 12, q)


# ---------------------------------------------------------------------------------------------
# degenerate cases
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", [1, 3, 5])
def test_unisolvent_interpolates(p):
    L = fo.rank(p)
    rng = np.random.default_rng(7 + p)
    pts = rng.random((L, 3))
    f = rng.standard_normal(L)
    with gpu_build(pts, f, p, 0.0, 3) as tree:
        assert tree.node_count == 1
        assert np.max(np.abs(gpu_eval(tree, pts) - f)) <= 1e-8 * np.max(np.abs(f))
    check_parity(pts, f, p, 0.0, 3, rng.random((500, 3)))


def test_too_few_points_is_precondition_error():
    fmi = _fmi()
    pts = np.random.default_rng(0).random((fo.rank(4) - 1, 3))
    with pytest.raises(fmi.FmiError) as ei:
        fmi.build(pts, np.zeros(pts.shape[0]), 4, 1e-6, 2)
    assert ei.value.code == -2


def test_nonfinite_input_rejected():
    fmi = _fmi()
    pts = np.random.default_rng(0).random((100, 3))
    f = np.zeros(100)
    f[5] = np.nan
    with pytest.raises(fmi.FmiError) as ei:
        fmi.build(pts, f, 2, 1e-6, 2)
    assert ei.value.code == -1


@pytest.mark.parametrize("zval", [0.5, 0.3])
def test_coplanar_rank_truncation(zval):
    rng = np.random.default_rng(11)
    pts = rng.random((3000, 3))
    pts[:, 2] = zval
    f = workloads.franke3d(pts)
    ora, gpu, *_ = check_parity(pts, f, 3, 1e-8, 2, np.column_stack([rng.random((500, 2)), np.full(500, zval)]))
    assert np.all(gpu["rank"] == 10) and np.all(ora.kept.sum(axis=1) == 10)


def test_duplicate_points():
    rng = np.random.default_rng(12)
    base = rng.random((2000, 3))
    pts = np.vstack([base, base, base[:500]])
    f = workloads.franke3d(pts)
    check_parity(pts, f, 3, 1e-8, 3, rng.random((1000, 3)))


def test_general_root_cube():
    rng = np.random.default_rng(13)
    pts = rng.random((8000, 3)) * np.array([3.0, 1.0, 2.0]) + np.array([-1.0, 4.0, 0.5])
    f = np.sin(pts[:, 0]) + np.cos(pts[:, 1] * pts[:, 2])
    q = rng.random((3000, 3)) * np.array([3.0, 1.0, 2.0]) + np.array([-1.0, 4.0, 0.5])
    check_parity(pts, f, 4, 1e-9, 3, q)


def test_outside_queries_use_root_polynomial():
    rng = np.random.default_rng(14)
    pts = rng.random((5000, 3))
    f = workloads.franke3d(pts)
    q = np.array([[1.5, 0.5, 0.5], [-0.2, 0.1, 0.9], [0.5, 0.5, 1.0000001], [1.0, 1.0, 1.0], [0.0, 0.0, 0.0]])
    check_parity(pts, f, 3, 1e-9, 3, q)


def test_empty_eval_and_polynomial_one_node():
    rng = np.random.default_rng(15)
    pts = rng.random((4000, 3))
    f = 1.0 + pts[:, 0] * pts[:, 1] - 2.0 * pts[:, 2] ** 3 + pts[:, 0] ** 2 * pts[:, 2]
    with gpu_build(pts, f, 3, 1e-10, 4) as tree:
        assert tree.node_count == 1
        assert gpu_eval(tree, np.zeros((0, 3)), host=True).shape == (0,)
        q = rng.random((1000, 3))
        exact = 1.0 + q[:, 0] * q[:, 1] - 2.0 * q[:, 2] ** 3 + q[:, 0] ** 2 * q[:, 2]
        assert np.max(np.abs(gpu_eval(tree, q) - exact)) <= 1e-12


def test_residual_bookkeeping_and_determinism():
    """interpolant(x_i) + r_i = f_i; two builds are bit-identical."""
    cfg = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(cfg)
    with gpu_build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t1, \
            gpu_build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t2:
        r = t1.residual()
        assert np.max(np.abs(gpu_eval(t1, pts) + r - f)) <= 1e-13
        e1, e2 = t1.export(), t2.export()
        assert np.array_equal(e1["coeffs"], e2["coeffs"])
        assert np.array_equal(gpu_eval(t1, q), gpu_eval(t2, q))
        ora = fo.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth)
        assert np.max(np.abs(r - ora.residual)) <= 1e-9 * np.max(np.abs(f))


def test_deep_cluster_resorts_all_levels():
    """A tight cluster drives the tree far deeper than the sorted key prefix (Dsort ~ log8(N/𝓛) + 1 = 6
    levels here): the build detects it (KeysShort) and re-sorts all levels; the result is the oracle's."""
    rng = np.random.default_rng(21)
    n_bg, n_cl = 2000, 30_000
    pts = np.vstack([rng.random((n_bg, 3)), 0.3 + 1e-4 * rng.random((n_cl, 3))])
    f = workloads.franke3d(pts)
    q = np.vstack([rng.random((1000, 3)), 0.3 + 1e-4 * rng.random((1000, 3))])
    ora, gpu, *_ = check_parity(pts, f, 1, 1e-12, 16, q)
    assert int(np.max(ora.depth)) >= 8


@pytest.mark.parametrize("split_min", ["0", "1000000000000"])
def test_k6_split_and_fused_match_the_oracle(split_min, monkeypatch):
    """The split K6 (Horner-only pass + projections of the created children; used on levels of >= 2^25
    points) and the fused pass (Horner + projections of every potential child) give the oracle's tree at
    a size where every level is small: FMI_K6_SPLIT_MIN forces the choice."""
    monkeypatch.setenv("FMI_K6_SPLIT_MIN", split_min)
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    q = q[:50_000]
    ora, gpu, *_ = check_parity(pts, f, cfg.degree, cfg.tol, cfg.max_depth, q, erms_vs=workloads.franke3d)
    assert ora.node_count == 585


@pytest.mark.parametrize("mode", ["0", "2"])
def test_bucket_sort_modes_match_the_oracle(mode, monkeypatch):
    """Bucketed keys (top sort digit first, records in bucket order; keys.cu bucket_sort_keys): mode 2
    also buckets the build's points (records gathered bucket by bucket, the root projection in stride
    mode, perm composed back to input indices), mode 0 is the plain LSD sort for the queries too.  Both
    give the oracle's tree and values (the default, queries only, is every other test); the residual
    in input order checks the composed permutation."""
    monkeypatch.setenv("FMI_BUCKET_SORT", mode)
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    q = q[:50_000]
    ora, gpu, *_ = check_parity(pts, f, cfg.degree, cfg.tol, cfg.max_depth, q, erms_vs=workloads.franke3d)
    assert ora.node_count == 585
    with gpu_build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as tree:
        res = tree.residual()
    scale = float(np.max(np.abs(f)))
    ref = f - fo.evaluate(ora, pts)
    assert np.max(np.abs(res - ref)) <= EVAL_TOL * scale


# ---------------------------------------------------------------------------------------------
# sort edge cases: query counts around the K2 tile (3072 items), the bucket tile (1536) and warp (32)
# boundaries, and
# point sets of one, two and three points (p = 0: 𝓛 = 1)
# ---------------------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def _tile_tree():
    rng = np.random.default_rng(21)
    pts = rng.random((20_000, 3))
    f = workloads.franke3d(pts)
    ora = fo.build(pts, f, 4, 1e-8, 4)
    tree = gpu_build(pts, f, 4, 1e-8, 4)
    yield ora, tree, float(np.max(np.abs(f)))
    tree.free()


@pytest.mark.parametrize("M", [1, 2, 31, 33, 1535, 1536, 1537, 3071, 3072, 3073, 4609, 6145])
def test_eval_query_counts_around_sort_tiles(_tile_tree, M):
    ora, tree, scale = _tile_tree
    q = np.random.default_rng(1000 + M).random((M, 3))
    val = gpu_eval(tree, q)
    ref = fo.evaluate(ora, q)
    assert np.max(np.abs(val - ref)) <= EVAL_TOL * scale


@pytest.mark.parametrize("N", [1, 2, 3])
def test_degree0_one_to_three_points(N):
    rng = np.random.default_rng(40 + N)
    pts = rng.random((N, 3))
    f = rng.standard_normal(N)
    check_parity(pts, f, 0, 0.0, 3, rng.random((100, 3)))


@pytest.mark.parametrize("eps", [1e-5, 3e-6, 3e-7, 1e-7])
@pytest.mark.parametrize("p", [2, 4])
def test_g9_near_threshold_sheet(p, eps):
    """Column rejection near δ = 1e-6 (reading G9): points on the curved sheet z = x² + ε·w (root frame),
    so the x²-type columns sit at distance ~1.25ε from the span of the columns before them.  The GPU
    (K5 Gram pivots ~ε², hence the K5q Householder re-fit) keeps exactly the oracle's columns, and the
    fitted values at the points agree within 1e-9·max|f|."""
    rng = np.random.default_rng(11)
    n = 2000
    x, y, w = rng.uniform(-1, 1, (3, n))
    u = np.stack([x, y, x * x + eps * w], axis=1)
    pts = (u + 1.0) / 2.0
    f = workloads.franke3d(pts)
    ora = fo.build(pts, f, p, 0.0, 0)
    with gpu_build(pts, f, p, 0.0, 0) as tree:
        ex = tree.export()
        got = gpu_eval(tree, pts)
    ref = fo.evaluate(ora, pts)
    assert int(ex["rank"][0]) == int(ora.kept[0].sum())
    assert np.array_equal(ex["coeffs"][0] != 0, ora.kept[0])
    assert np.max(np.abs(got - ref)) <= EVAL_TOL * np.max(np.abs(f))
