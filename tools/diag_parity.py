"""Diagnostics: per-node comparison of GPU vs oracle for a small case (not a test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import workloads
from oracle import fmt_oracle as fo
import paper_1511_01353_b200 as fmi
from parity import node_key_map

def run(name, pts, f, p, tau, D, q):
    ora = fo.build(pts, f, p, tau, D)
    ref = fo.evaluate(ora, q)
    t = fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), p, tau, D)
    g = t.export(); val = t.eval(torch.from_numpy(q).cuda()).cpu().numpy()
    gm = node_key_map(g["depth"], g["cell"]); om = node_key_map(ora.depth, ora.cell)
    print(f"== {name}: nodes gpu {len(gm)} oracle {len(om)} max|dval| {np.max(np.abs(val-ref)):.3e} maxf {np.max(np.abs(f)):.3f}")
    rows = []
    for k, gi in gm.items():
        if k not in om: print('  only gpu', k); continue
        oi = om[k]
        V = fo.vandermonde(np.zeros((1,3)), p)
        # coefficient difference measured at the node's own points (fitted values)
        u = fo.to_unit(pts, ora.lo, ora.width)
        d, c = k[0], np.array(k[1:])
        h = 2.0**-d
        sel = np.all((u >= c*h) & ((u < (c+1)*h) | ((c+1)*h == 1.0)), axis=1)
        ul = fo.local_coords(u[sel], d, c)
        Vn = fo.vandermonde(ul, p)
        dfit = np.max(np.abs(Vn @ (g["coeffs"][gi] - ora.coeffs[oi])))
        rows.append((dfit, k, g["flags"][gi], g["min_pivot"][gi], ora.min_pivot[oi], g["rank"][gi], ora.kept[oi].sum(), g["n_points"][gi], ora.residual_rms[oi]))
    rows.sort(reverse=True)
    for r in rows[:6]:
        print("  dfit %.2e node %s flag %d gpu_minpiv %.2e ora_minpiv %.2e rank %d/%d n %d rms %.2e" % r)
    for k in om:
        if k not in gm: print('  only oracle', k)

if __name__ == "__main__":
    for p in (7, 10):
        L = fo.rank(p); N = 9 * L + 37
        rng = np.random.default_rng(100 + p)
        pts = rng.random((N, 3)); f = workloads.franke3d(pts); q = rng.random((3001, 3))
        run(f"degree {p}", pts, f, p, 1e-12, 2, q)
    L = fo.rank(5); rng = np.random.default_rng(12)
    pts = rng.random((L, 3)); f = rng.standard_normal(L)
    run("unisolvent p5", pts, f, 5, 0.0, 3, rng.random((500, 3)))
    centres = workloads.mixture_centres(0)
    pts = workloads.mixture_points(60_000, 0, centres); f = workloads.mixture_values(pts, centres)
    q = workloads.mixture_points(20_000, 1, centres)
    run("mixture 6e4", pts, f, 6, 1e-9, 12, q)
