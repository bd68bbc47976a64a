import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1511_01353_b200 as fmi, workloads
for c in (1, 3, 4):
    cfg = workloads.CONFIGS[c]
    pts, f, q = workloads.make_inputs(cfg)
    h = [torch.from_numpy(x).pin_memory() for x in (pts, f, q)]
    out = torch.empty(q.shape[0], dtype=torch.float64).pin_memory()
    P, F, Q, O = (x.numpy() for x in (*h, out))
    for mode in ("transfer", "build+eval", "transfer", "build+eval"):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3):
            if mode == "transfer":
                fmi.transfer(P, F, Q, cfg.degree, cfg.tol, cfg.max_depth, out=O)
            else:
                t = fmi.build(P, F, cfg.degree, cfg.tol, cfg.max_depth); t.eval(Q, out=O); t.free()
        torch.cuda.synchronize(); print(c, os.environ.get("FMI_NO_OVERLAP", "-"), mode, round((time.perf_counter() - t0) / 3 * 1e3, 2), "ms", flush=True)
