import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np
import paper_1511_01353_b200 as fmi, workloads
cfg = workloads.CONFIGS[5]
pts, f, q = workloads.make_inputs(cfg)
h = [torch.from_numpy(x).pin_memory() for x in (pts, f, q)]
out = torch.empty(q.shape[0], dtype=torch.float64).pin_memory()
P, F, Q, O = (x.numpy() for x in (*h, out))
for mode in ("transfer", "build+eval", "transfer", "build+eval"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if mode == "transfer":
        fmi.transfer(P, F, Q, cfg.degree, cfg.tol, cfg.max_depth, out=O)
    else:
        t = fmi.build(P, F, cfg.degree, cfg.tol, cfg.max_depth); t.eval(Q, out=O); t.free()
    torch.cuda.synchronize(); print(mode, round((time.perf_counter() - t0) * 1e3, 1), "ms", flush=True)
# pure copy bandwidth
d = torch.empty_like(h[0], device="cuda"); torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h[0]); torch.cuda.synchronize()
print("H2D GB/s", h[0].numel() * 8 / (time.perf_counter() - t0) / 1e9)
