"""Scoping sweep of PAPER.md §4 (Figs. 2-4): interpolation errors E_rms / E_inf of the 3-D
Franke function against the number of octree nodes, over degree (L_max), residual
threshold τ and grid size N_p = N_q (random p -> q grids in [0,1]^3), on the GPU path.

The paper's figures are placeholders ([FIGURE]), so only the SHAPE can be compared: errors falling with
τ until the degree/size limit, node counts growing like O(N) at low order and O(lg N) at high order
(P:396), and its headline (< 10^3 nodes with E_rms < 1e-11, E_inf < 1e-8) — which this
sweep reports for the (p, τ, N) that reach it.  One JSON line per run.

  python tools/sweep.py [--degrees 4 8 12] [--taus 1e-6 1e-8 1e-10 1e-12] [--log8n 4 5 6 7 8 9]

Degrees above 10 run the QR path on the octree (csrc/unscoped.cu).  Sweep points are checked against the
oracle by tests/test_gpu_sweep.py (this tool does not import it).
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--degrees", type=int, nargs="+", default=[4, 8, 12])  # L_max of P:383
ap.add_argument("--taus", type=float, nargs="+", default=[1e-6, 1e-8, 1e-10, 1e-12])
ap.add_argument("--log8n", type=int, nargs="+", default=[4, 5, 6, 7, 8, 9])  # N_p = 8^4..8^9
ap.add_argument("--max-depth", type=int, default=10)
a = ap.parse_args()

fmi.set_stream(torch.cuda.current_stream())
for k in a.log8n:
    n = 8 ** k
    pts = workloads.uniform_points(n, 0)
    f = workloads.franke3d(pts)
    q = workloads.uniform_points(n, 1)            # N_q = N_p
    truth = workloads.franke3d(q)
    dp, df, dq = (torch.from_numpy(x).cuda() for x in (pts, f, q))
    for p in a.degrees:
        L = (p + 1) * (p + 2) * (p + 3) // 6
        if n < L:
            continue
        for tau in a.taus:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr = fmi.build(dp, df, p, tau, a.max_depth)
            val = tr.eval(dq)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            err = val.cpu().numpy() - truth
            erms, einf = workloads.rms_and_max(err)
            rec = {"path": "qr" if p > 10 else "moments", "N": n, "log8N": k, "degree": p, "rank": L, "tau": tau, "max_depth": a.max_depth,
                   "nodes": tr.node_count, "levels": int(len(tr.level_stats()[0])), "E_rms": erms, "E_inf": einf,
                   "build_eval_s": dt,
                   "paper_headline": bool(tr.node_count < 1000 and erms < 1e-11 and einf < 1e-8)}
            print(json.dumps(rec), flush=True)
            tr.free()
