"""Run fmi_build + fmi_eval of a config (profiling driver for ncu / compute-sanitizer; not a benchmark)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
if a.n or a.m:
    cfg = cfg.scaled(n=a.n, m=a.m)
pts, f, q = workloads.make_inputs(cfg)
dp, df, dq = (torch.from_numpy(x).cuda() for x in (pts, f, q))
for _ in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    tr = fmi.build(dp, df, cfg.degree, cfg.tol, cfg.max_depth)
    out = tr.eval(dq)
    torch.cuda.synchronize()
    print(f"{cfg.name} N={cfg.n} M={cfg.m}: nodes {tr.node_count} levels {tr.level_stats()} "
          f"step {1e3 * (time.perf_counter() - t):.1f} ms {tr.build_stats()}", flush=True)
    tr.free()
