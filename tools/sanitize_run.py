"""Workload for memory-safety runs — compute-sanitizer (memcheck / racecheck / synccheck) where the pool
allows it, else the library's own guard bands (FMI_GUARD=1 python tools/sanitize_run.py): every kernel family of the
hot path (keys, sort, gather, K4 moments, M2M TMA copies, K5 solve + refinement, K5q QR, K6 split and
fused passes, decisions, presum, K7 eval, the unscoped f2 path) on BASELINE.json cfg 1 and a reduced
cfg 2, through the C ABI.  Each phase checks its result against the oracle so a run that the
sanitizer slows down still proves it computed the right thing.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py [--quick]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402
from oracle import fmt_oracle as fo  # noqa: E402


def run(pts, f, q, p, tau, D, label):
    scale = float(np.max(np.abs(f)))
    with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), p, tau, D) as tree:
        got = tree.eval(torch.from_numpy(q).cuda()).cpu().numpy()
        nodes = tree.node_count
    ora = fo.build(pts, f, p, tau, D)
    ref = fo.evaluate(ora, q)
    err = float(np.max(np.abs(got - ref)))
    ok = nodes == ora.node_count and err <= 1e-9 * scale
    print(f"{label}: nodes gpu={nodes} oracle={ora.node_count} max|d|={err:.3e} {'ok' if ok else 'MISMATCH'}",
          flush=True)
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="cfg 1 + small cases only (racecheck)")
    a = ap.parse_args()
    fmi.load_library()
    ok = True
    c1 = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(c1)
    ok &= run(pts, f, q[:2000], c1.degree, c1.tol, c1.max_depth, "cfg1")
    # clustered mixture: deep levels, direct moments, K5q/refinement
    cen = workloads.mixture_centres(0)
    x = workloads.mixture_points(20_000 if a.quick else 60_000, 0, cen)
    ok &= run(x, workloads.mixture_values(x, cen), x[:1000].copy(), 4, 1e-9, 6, "mixture p=4")
    # split K6 on every level (FMI_K6_SPLIT_MIN=0) vs fused (default for small levels)
    os.environ["FMI_K6_SPLIT_MIN"] = "0"
    ok &= run(pts, f, q[:2000], c1.degree, c1.tol, c1.max_depth, "cfg1 split-K6")
    os.environ.pop("FMI_K6_SPLIT_MIN")
    if not a.quick:
        c2 = workloads.CONFIGS[2]
        pts2, f2, q2 = workloads.make_inputs(c2)
        ok &= run(pts2, f2, q2[:5000], c2.degree, c2.tol, c2.max_depth, "cfg2")
        rng = np.random.default_rng(5)
        x = rng.random((3000, 3))
        ok &= run(x, workloads.franke3d(x), rng.random((500, 3)), 10, 1e-12, 1, "p=10 D=1")
    # the QR path on the octree (degrees 11-14 at depth > 0: Legendre Gram, CholeskyQR2 pass, walk)
    rng = np.random.default_rng(9)
    x = rng.random((8 ** 4, 3))
    ok &= run(x, workloads.franke3d(x), rng.random((500, 3)), 11, 1e-6, 2, "QR path p=11 D=2")
    # unscoped f2 path (DMMA SYRK + single-CTA Cholesky + rejection walk)
    rng = np.random.default_rng(7)
    x = rng.random((4000, 3))
    ok &= run(x, workloads.franke3d(x), rng.random((500, 3)), 12, 0.0, 0, "unscoped p=12")
    gv = fmi.guard_violations()
    if os.environ.get("FMI_GUARD"):
        print(f"guard bands overwritten: {gv}", flush=True)
        ok &= gv == 0
    print("ALL OK" if ok else "FAILED", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
