"""Spot checks of the §4 scoping sweep (tools/sweep.py): sweep points
at the paper's orders L_max = 4, 8, 12 recomputed through the same library call and compared
with the oracle — identical tree, interpolant within 1e-9·max|f| on the sweep's own queries (N_q = N_p,
uniform, seed 1), and E_rms / E_inf against the analytic Franke function (the sweep's reported
quantities) within 1% of the oracle's."""
import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo
from parity import compare_trees

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,log8n,tau", [(4, 4, 1e-6), (4, 5, 1e-12), (8, 5, 1e-8), (12, 5, 1e-12),
                                         (12, 4, 1e-6)])
def test_sweep_point_vs_oracle(p, log8n, tau):
    import paper_1511_01353_b200 as fmi
    n = 8 ** log8n
    D = 10                                            # tools/sweep.py default max_depth
    pts = workloads.uniform_points(n, 0)
    f = workloads.franke3d(pts)
    q = workloads.uniform_points(n, 1)[:5000]
    with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), p, tau, D) as tree:
        gpu = tree.export()
        val = tree.eval(torch.from_numpy(q).cuda()).cpu().numpy()
    ora = fo.build(pts, f, p, tau, D)
    ref = fo.evaluate(ora, q)
    compare_trees(gpu, ora, tau)
    assert np.max(np.abs(val - ref)) <= 1e-9 * np.max(np.abs(f))
    truth = workloads.franke3d(q)
    eg, ig = workloads.rms_and_max(val - truth)
    eo, io = workloads.rms_and_max(ref - truth)
    assert abs(eg - eo) <= 0.01 * eo and abs(ig - io) <= 0.01 * io
