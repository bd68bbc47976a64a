"""Which nodes take the K5q Householder re-fit (flag bit 0) at a config: count and sizes per depth."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = workloads.CONFIGS[c].scaled(m=1000)
pts, f, _ = workloads.make_inputs(cfg)
with fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol, cfg.max_depth) as t:
    ex = t.export()
for d in range(int(ex["depth"].max()) + 1):
    sel = ex["depth"] == d
    q = sel & ((ex["flags"] & 1) != 0)
    r = sel & ((ex["flags"] & 2) != 0)
    n = ex["n_points"][q]
    print(f"depth {d}: nodes {sel.sum()} qr {q.sum()} (points {n.sum()}, max {n.max() if len(n) else 0}) "
          f"refine {r.sum()} minpiv<1e-9 {(sel & (ex['min_pivot'] < 1e-9)).sum()}")
