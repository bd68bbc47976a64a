"""Run fmi_build + fmi_eval of a config (profiling driver for ncu / compute-sanitizer; not a benchmark).

--profile prints the library's per-kernel device time (CUDA events on the library stream) per rep."""
import argparse
import json
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
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
if a.n or a.m:
    cfg = cfg.scaled(n=a.n, m=a.m)
pts, f, q = workloads.make_inputs(cfg)
dp, df, dq = (torch.from_numpy(x).cuda() for x in (pts, f, q))
fmi.set_stream(torch.cuda.current_stream())
for _ in range(a.reps):
    if a.profile:
        fmi.profile_reset()
        fmi.profile_enable(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    tr = fmi.build(dp, df, cfg.degree, cfg.tol, cfg.max_depth)
    tb = time.perf_counter()
    out = tr.eval(dq)
    torch.cuda.synchronize()
    te = time.perf_counter()
    print(f"{cfg.name} N={cfg.n} M={cfg.m}: nodes {tr.node_count} levels {tr.level_stats()[0].tolist()} "
          f"build {1e3 * (tb - t):.1f} ms eval {1e3 * (te - tb):.1f} ms {tr.build_stats()}", flush=True)
    if a.profile:
        fmi.profile_enable(False)
        prof = {k: round(v[0], 3) for k, v in sorted(fmi.profile_get().items()) if v[1]}
        print("  kernels ms:", json.dumps(prof), flush=True)
    tr.free()
