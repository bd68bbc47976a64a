"""Diagnostics for a sweep point (tools/sweep.py) against the oracle: per node the rank, minimum pivot,
flags and residual RMS on both sides, and the largest interpolant difference among the queries whose
deepest node it is.  Usage: python tools/diag_sweep.py --p 12 --log8n 4 --tau 1e-6"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402
from oracle import fmt_oracle as fo  # noqa: E402
from parity import node_key_map  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=12)
ap.add_argument("--log8n", type=int, default=4)
ap.add_argument("--tau", type=float, default=1e-6)
ap.add_argument("--depth", type=int, default=10)
a = ap.parse_args()
n = 8 ** a.log8n
pts = workloads.uniform_points(n, 0)
f = workloads.franke3d(pts)
q = workloads.uniform_points(n, 1)[:5000]
with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), a.p, a.tau, a.depth) as tree:
    ex = tree.export()
    val = tree.eval(torch.from_numpy(q).cuda()).cpu().numpy()
ora = fo.build(pts, f, a.p, a.tau, a.depth)
ref = fo.evaluate(ora, q)
g = node_key_map(ex["depth"], ex["cell"])
o = node_key_map(ora.depth, ora.cell)
# deepest oracle node of every query
D = int(ora.depth.max())
owner = []
for x in q:
    best = None
    for d in range(D + 1):
        c = tuple(int(v) for v in np.minimum(np.floor(x * 2 ** d), 2 ** d - 1))
        if (d,) + c in o:
            best = (d,) + c
    owner.append(best)
diff = np.abs(val - ref)
print(f"p={a.p} N={n} tau={a.tau}: nodes gpu {len(g)} oracle {len(o)}; max|d| {diff.max():.3e}")
for key in sorted(o):
    oi, gi = o[key], g.get(key)
    sel = [i for i, w in enumerate(owner) if w == key]
    md = diff[sel].max() if sel else 0.0
    rk_o = int(ora.kept[oi].sum())
    s = (f"{key} n={ora.n_points[oi]} rank o={rk_o}" + (f" g={ex['rank'][gi]} flags={ex['flags'][gi]}"
         f" minpiv o={ora.min_pivot[oi]:.2e} g={ex['min_pivot'][gi]:.2e} rms o={ora.residual_rms[oi]:.3e}"
         f" g={ex['residual_rms'][gi]:.3e}" if gi is not None else " MISSING") + f" q={len(sel)} max|d|={md:.2e}")
    if gi is not None:
        kg = ex["coeffs"][gi] != 0
        s += f" kept-set diff={int(np.sum(kg != ora.kept[oi]))}"
    print(s)
