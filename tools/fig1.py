"""PAPER.md §3 / Fig. 1 on the GPU path — SURVEY §8(f) row f2: the unscoped
(single-node, max_depth = 0) interpolation of the 3-D Franke function on random grids
N_p = N_q = 8^6 in [0,1]^3 with L_max = 6, 10, 14 (𝓛 = 84, 286, 680).  Fig. 1 itself is a placeholder
([FIGURE]); the text says only L_max = 14 is qualitatively right, so this reports the errors against
the exact function per degree, the fitted rank, and the device time of build + eval.  With --oracle N
it also compares against the oracle at a reduced N (parity diagnostics: max |gpu - oracle| / max|f|).

  python tools/fig1.py [--log8n 6] [--degrees 6 10 14] [--oracle 5000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log8n", type=int, default=6)
ap.add_argument("--degrees", type=int, nargs="+", default=[6, 10, 14])
ap.add_argument("--oracle", type=int, default=0, help="also compare with the oracle at this N")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

fmi.set_stream(torch.cuda.current_stream())
n = 8 ** a.log8n
pts = workloads.uniform_points(n, 0)
f = workloads.franke3d(pts)
q = workloads.uniform_points(n, 1)
truth = workloads.franke3d(q)
dp, df, dq = (torch.from_numpy(x).cuda() for x in (pts, f, q))
for p in a.degrees:
    times = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tree = fmi.build(dp, df, p, 0.0, 0)
        out = tree.eval(dq)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        ex = tree.export()
        tree.free()
    err = out.cpu().numpy() - truth
    rec = {"N_p": n, "N_q": n, "degree": p, "rank_basis": (p + 1) * (p + 2) * (p + 3) // 6,
           "rank_kept": int(ex["rank"][0]), "E_rms": float(np.sqrt(np.mean(err ** 2))),
           "E_inf": float(np.max(np.abs(err))), "fit_rms": float(ex["residual_rms"][0]),
           "build_eval_ms": float(np.median(times)),
           "path": "unscoped QR (csrc/unscoped.cu)" if p > 10 else "level path (K4/K5), max_depth = 0"}
    if a.oracle:
        from oracle import fmt_oracle as fo
        rng = np.random.default_rng(1000 + p)
        m = max(a.oracle, 2 * rec["rank_basis"])
        ps = rng.random((m, 3))
        fs = workloads.franke3d(ps)
        qs = rng.random((2000, 3))
        t0 = time.perf_counter()
        ora = fo.build(ps, fs, p, 0.0, 0)
        ref = fo.evaluate(ora, qs)
        t_ora = time.perf_counter() - t0
        with fmi.build(torch.from_numpy(ps).cuda(), torch.from_numpy(fs).cuda(), p, 0.0, 0) as t2:
            got = t2.eval(torch.from_numpy(qs).cuda()).cpu().numpy()
            rk = int(t2.export()["rank"][0])
        rec["oracle_check"] = {"N": m, "max_abs_diff_over_max_f": float(np.max(np.abs(got - ref)) / np.max(np.abs(fs))),
                               "rank_gpu": rk, "rank_oracle": int(ora.kept[0].sum()), "oracle_s": t_ora}
    print(json.dumps(rec), flush=True)
