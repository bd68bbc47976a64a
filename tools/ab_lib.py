"""A/B of library variants (tools/build_variant.sh): per-kernel device ms of one config's build + eval.
python tools/ab_lib.py CONFIG LIB [LIB ...]  (each LIB in a fresh process so that load_library binds it)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 3 or (len(sys.argv) == 3 and sys.argv[1] != "--one"):
    cfg = sys.argv[1]
    for lib in sys.argv[2:]:
        out = subprocess.run([sys.executable, __file__, "--one", cfg + ":" + lib], capture_output=True, text=True)
        print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
    sys.exit(0)
cfg_s, lib = sys.argv[2].split(":", 1)
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_01353_b200 as fmi  # noqa: E402
import workloads  # noqa: E402

fmi.load_library(lib)
cfg = workloads.CONFIGS[int(cfg_s)]
pts, f, q = workloads.make_inputs(cfg)
dp, df, dq = (torch.from_numpy(x).cuda() for x in (pts, f, q))
fmi.set_stream(torch.cuda.current_stream())
res = []
for rep in range(3):
    fmi.profile_reset()
    fmi.profile_enable(True)
    with fmi.build(dp, df, cfg.degree, cfg.tol, cfg.max_depth) as tr:
        out = tr.eval(dq)
        torch.cuda.synchronize()
        nodes = tr.node_count
    fmi.profile_enable(False)
    res.append({k: round(v[0], 3) for k, v in fmi.profile_get().items() if v[1]})
best = {k: min(r[k] for r in res[1:]) for k in res[-1]}
print(json.dumps({"nodes": nodes, "total": round(sum(best.values()), 2),
                  **dict(sorted(best.items(), key=lambda kv: -kv[1])[:8])}))
