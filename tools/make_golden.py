"""Write the oracle's golden node lists for the full-size parity tests (tests/test_gpu_golden.py).

Calls only ``oracle/`` and ``workloads/`` (no product code): every stored value is the oracle's.

  cfg3  the FULL tree of BASELINE.json config 3 (Alg. 1 from the root) and the
        interpolant at the first 1e5 queries of the config.
  cfg4  Alg. 1 from the root with every depth-0/1 node expanded and ``--subtrees`` depth-2
        subtrees expanded completely (the depth-2 nodes receive the residual of the real root
        and depth-1 fits); the interpolant at the config's own queries (the mixture) inside them,
        up to 25,000 per subtree.
  cfg5  the root fit of 2e8 points is beyond this host (Λ alone is 459 GB, ~4 h of QR), so each
        sampled depth-2 subtree is Alg. 1 called on the depth-2 node with the ORIGINAL f: by the
        telescoping identity the depth-2 node's fit of f equals the root + depth-1 +
        depth-2 path sum, so the subtree receives the same residual up to rounding (~1e-13 absolute,
        SURVEY.md §8(c)); decisions closer to τ than that are reported as ties by the test.

Stored per node (canonical (depth, Morton) order): depth, cell, n, child counts, child E_RMS
(P:305), child state (-1 none, 1 expanded, 2 created but outside the sampled subtrees),
post-fit RMS.  Stored per query: the oracle's interpolant.  The queries themselves are regenerated
by ``workloads`` from the recorded seeds.

    python tools/make_golden.py cfg3 [--jobs 6]
"""
import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import fmt_oracle as fo  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
NQ = 100_000


def _log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def _node_table(trees):
    """Concatenate oracle trees into one canonical node table (depth, Morton prefix order)."""
    rows = []
    for t in trees:
        for i in range(t.node_count):
            ci = t.child_index[i]
            state = np.where(ci >= 0, 1, np.where(ci == -2, 2, -1)).astype(np.int8)
            rows.append((int(t.depth[i]), int(t.prefix[i]), tuple(int(v) for v in t.cell[i]), int(t.n_points[i]),
                         t.child_count[i].astype(np.int64), t.child_rms[i].astype(np.float64), state,
                         float(t.residual_rms[i]), float(t.min_pivot[i]), int(t.kept[i].sum())))
    rows.sort(key=lambda r: (r[0], r[1]))
    seen = set()
    out = []
    for r in rows:                       # a subtree root also appears in the top run as a created child
        key = (r[0], r[2])
        if key in seen:
            continue
        seen.add(key)
        out.append(r)
    return dict(
        depth=np.array([r[0] for r in out], dtype=np.int32),
        cell=np.array([r[2] for r in out], dtype=np.int64).reshape(-1, 3),
        n=np.array([r[3] for r in out], dtype=np.int64),
        child_count=np.array([r[4] for r in out]).reshape(-1, 8),
        child_rms=np.array([r[5] for r in out]).reshape(-1, 8),
        child_state=np.array([r[6] for r in out]).reshape(-1, 8),
        residual_rms=np.array([r[7] for r in out]),
        min_pivot=np.array([r[8] for r in out]),
        kept=np.array([r[9] for r in out], dtype=np.int32),
    )


def _subtree_job(args):
    u, r, p, tau, D, depth, cell, qs = args
    t0 = time.time()
    sub = fo.build_subtree(u, r, p, tau, D, depth, cell)
    val = fo.evaluate(sub, qs)
    _log(f"  subtree {depth}:{cell} n={u.shape[0]} nodes={sub.node_count} {time.time() - t0:.0f}s")
    return sub, val


def _summary(name, cfg, table, extra):
    tau = cfg.tol
    L = fo.rank(cfg.degree)
    cr = table["child_rms"]
    cnt = table["child_count"]
    dec = (cnt >= L) & (table["depth"][:, None] + 1 <= cfg.max_depth) & np.isfinite(cr)
    m = np.abs(cr[dec] / tau - 1.0)
    lines = [f"# oracle golden for BASELINE.json {cfg.name} (tools/make_golden.py; PAPER.md Alg. 1/2, P:294-336)",
             f"# {extra}",
             f"nodes {len(table['depth'])}",
             f"max_depth_seen {int(table['depth'].max())}",
             f"decisions_with_guards_met {int(dec.sum())}",
             f"closest_margins |E/tau-1| {' '.join(f'{v:.3e}' for v in np.sort(m)[:8])}",
             f"truncated_nodes {int(np.sum(table['kept'] < L))}"]
    with open(os.path.join(GOLDEN, f"oracle_{name}.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    _log("\n".join(lines))


def make_cfg3(jobs):
    cfg = workloads.CONFIGS[3]
    pts, f, _ = workloads.make_inputs(cfg.scaled(m=1))
    q = workloads.uniform_points(NQ, 1)          # = the config's first 1e5 queries (same stream)
    t0 = time.time()
    tree = fo.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth)
    _log(f"cfg3 build: {tree.node_count} nodes, {time.time() - t0:.0f}s")
    val = fo.evaluate(tree, q)
    table = _node_table([tree])
    np.savez_compressed(os.path.join(GOLDEN, "oracle_cfg3.npz"), mode="full", cfg=3, q_seed=1, q_n=NQ,
                        values=val, **table)
    _summary("cfg3", cfg, table, f"full tree; values at workloads.uniform_points({NQ}, 1); build {time.time() - t0:.0f}s")


def _pick_cells(created, counts, k, seed, n_big):
    """k depth-2 cells: the n_big most populated, then uniform random (seeded) among the rest."""
    order = np.argsort(-counts, kind="stable")
    pick = [created[i] for i in order[:n_big]]
    rest = [c for c in created if c not in pick]
    rng = np.random.default_rng(seed)
    for i in rng.choice(len(rest), size=min(k - n_big, len(rest)), replace=False):
        pick.append(rest[i])
    return pick


def make_cfg4(jobs, k):
    cfg = workloads.CONFIGS[4]
    pts, f, _ = workloads.make_inputs(cfg.scaled(m=1))
    p, tau, D = cfg.degree, cfg.tol, cfg.max_depth
    t0 = time.time()
    top = fo.build(pts, f, p, tau, D, descend=lambda d, c: d <= 1)
    _log(f"cfg4 top (depth 0-1): {top.node_count} nodes, {time.time() - t0:.0f}s")
    created, counts = [], []
    for i in range(top.node_count):
        if top.depth[i] != 1:
            continue
        for o in range(8):
            if top.child_index[i][o] == -2:
                c = tuple(2 * int(top.cell[i][a]) + ((o >> a) & 1) for a in range(3))
                created.append(c)
                counts.append(int(top.child_count[i][o]))
    pick = _pick_cells(created, np.array(counts), k, seed=4, n_big=2)
    _log(f"cfg4 created depth-2 cells: {len(created)}; picked {pick}")
    u = pts                                         # unit cube: root-cube coordinates = points (G6)
    c2 = workloads.cell_of(u, 2)
    # queries: the config's own (the same mixture, seed 1, BASELINE.json) that fall in the picked cells,
    # the first NQ/len(pick) of each cell in query order — uniform queries in a cell would ask for the
    # polynomials far outside their data (clustered points), where no fit is meaningful
    qall = workloads.mixture_points(cfg.m, 1, workloads.mixture_centres(0))
    qc2 = workloads.cell_of(qall, 2)
    jobsl, qidx = [], []
    for t, cell in enumerate(pick):
        inside = np.all(c2 == np.array(cell), axis=1)
        qi = np.flatnonzero(np.all(qc2 == np.array(cell), axis=1))[:2 * NQ // len(pick)]
        qidx.append(qi)
        jobsl.append((u[inside], top.residual[inside], p, tau, D, 2, cell, np.ascontiguousarray(qall[qi])))
    with mp.get_context("fork").Pool(jobs) as pool:
        res = pool.map(_subtree_job, jobsl, chunksize=1)
    vals = []
    for (sub, v), job in zip(res, jobsl):
        qs = job[7]
        # full path sum: root and depth-1 terms + the subtree's
        vals.append(v + _top_terms(top, qs, p))
    table = _node_table([top] + [s for s, _ in res])
    # mark the picked subtrees' roots as expanded in their parents' child_state
    qidx = np.concatenate(qidx)
    np.savez_compressed(os.path.join(GOLDEN, "oracle_cfg4.npz"), mode="top+subtrees", cfg=4,
                        pick=np.array(pick, dtype=np.int64), q_index=qidx.astype(np.int64),
                        values=np.concatenate(vals), **table)
    _summary("cfg4", cfg, table, f"depth 0-1 complete + depth-2 subtrees {pick} (2 most populated + random seed 4); "
                                 f"values at the config's queries (mixture, seed 1) in those cells, up to "
                                 f"{2 * NQ // len(pick)} per cell ({qidx.size} in all); {time.time() - t0:.0f}s")


def _top_terms(top, qs, p):
    """Root + depth-1 polynomial terms of the path sum at queries inside a depth-2 cell."""
    out = fo.apply_fit(fo.local_coords(qs, 0, np.zeros(3, dtype=np.int64)), top.coeffs[0], p)
    c1 = workloads.cell_of(qs, 1)
    for i in range(top.node_count):
        if top.depth[i] == 1:
            sel = np.all(c1 == top.cell[i], axis=1)
            if np.any(sel):
                out[sel] += fo.apply_fit(fo.local_coords(qs[sel], 1, top.cell[i]), top.coeffs[i], p)
    return out


def make_cfg5(jobs, k):
    cfg = workloads.CONFIGS[5]
    p, tau, D = cfg.degree, cfg.tol, cfg.max_depth
    t0 = time.time()
    pts = workloads.uniform_points(cfg.n, 0)
    c2 = workloads.cell_of(pts, 2)
    rng = np.random.default_rng(5)
    allc = [(i, j, l) for l in range(4) for j in range(4) for i in range(4)]
    pick = [allc[i] for i in rng.choice(64, size=k, replace=False)]
    _log(f"cfg5 picked depth-2 cells {pick}")
    jobsl = []
    for t, cell in enumerate(pick):
        inside = np.all(c2 == np.array(cell), axis=1)
        x = np.ascontiguousarray(pts[inside])
        qs = workloads.cell_queries(2, cell, NQ // len(pick), 5000 + t)
        jobsl.append((x, workloads.franke3d(x), p, tau, D, 2, cell, qs))
    del pts, c2
    with mp.get_context("fork").Pool(jobs) as pool:
        res = pool.map(_subtree_job, jobsl, chunksize=1)
    table = _node_table([s for s, _ in res])
    np.savez_compressed(os.path.join(GOLDEN, "oracle_cfg5.npz"), mode="subtrees-telescoped", cfg=5,
                        pick=np.array(pick, dtype=np.int64), q_seed0=5000, q_per_cell=NQ // len(pick),
                        values=np.concatenate([v for _, v in res]), **table)
    _summary("cfg5", cfg, table, f"depth-2 subtrees {pick} (random, seed 5), each Alg. 1 on the depth-2 node with the "
                                 f"original f (telescoping); values at workloads.cell_queries(2, cell, {NQ // len(pick)}, "
                                 f"5000+t); {time.time() - t0:.0f}s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg3", "cfg4", "cfg5"])
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--subtrees", type=int, default=8)
    a = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    if a.which == "cfg3":
        make_cfg3(a.jobs)
    elif a.which == "cfg4":
        make_cfg4(a.jobs, a.subtrees)
    else:
        make_cfg5(a.jobs, a.subtrees)


if __name__ == "__main__":
    main()
