"""Input generators (shared by oracle and CUDA path; they hold none of the method's arithmetic)."""
import numpy as np

import workloads


def test_configs_match_baseline_json():
    import json, os
    bj = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "BASELINE.json")))
    assert len(bj["configs"]) == len(workloads.CONFIGS) == 5
    c = workloads.CONFIGS
    assert (c[1].n, c[1].m, c[1].degree, c[1].max_depth, c[1].tol) == (2000, 10_000, 4, 2, 1e-6)
    assert (c[5].n, c[5].m, c[5].degree, c[5].max_depth, c[5].tol) == (200_000_000, 100_000_000, 10, 10, 1e-11)


def test_franke_gaussian_centres():
    # at (2/9,2/9,2/9) the first term's exponent vanishes; at (4/9,7/9,5/9) the fourth's
    x = np.array([[2 / 9, 2 / 9, 2 / 9], [4 / 9, 7 / 9, 5 / 9]])
    f = workloads.franke3d(x)
    a = 9 * x
    t2 = np.exp(-(a[:, 0] + 1) ** 2 / 49 - (a[:, 1] + 1) ** 2 / 10 - (a[:, 2] + 1) ** 2 / 10)
    t3 = np.exp(-0.25 * ((a[:, 0] - 7) ** 2 + (a[:, 1] - 3) ** 2 + (a[:, 2] - 5) ** 2))
    t1 = np.exp(-0.25 * ((a[:, 0] - 2) ** 2 + (a[:, 1] - 2) ** 2 + (a[:, 2] - 2) ** 2))
    t4 = np.exp(-(a[:, 0] - 4) ** 2 - (a[:, 1] - 7) ** 2 - (a[:, 2] - 5) ** 2)
    assert abs(f[0] - (0.75 + 0.75 * t2[0] + 0.5 * t3[0] - 0.2 * t4[0])) < 1e-15
    assert abs(f[1] - (0.75 * (t1[1] + t2[1]) + 0.5 * t3[1] - 0.2)) < 1e-15


def test_halton_and_uniform_determinism():
    h = workloads.halton_points(8)
    assert h[0, 0] == 0.5 and h[0, 1] == 1 / 3 and h[0, 2] == 0.2
    assert h[3, 0] == 0.125
    assert np.array_equal(workloads.uniform_points(10, 0), np.random.default_rng(0).random((10, 3)))


def test_mixture_clipped_and_seeded():
    c = workloads.mixture_centres(0)
    assert np.all((c >= 0.2) & (c <= 0.8))
    x = workloads.mixture_points(100_000, 0, c)
    assert x.min() == 0.0 or x.min() >= 0.0
    assert np.all((x >= 0) & (x <= 1))
    assert np.array_equal(x, workloads.mixture_points(100_000, 0, c))
    f = workloads.mixture_values(x[:10], c)
    assert np.all(f > 0) and np.all(f <= 8)
