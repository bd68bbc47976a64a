"""ORACLE for the free-mesh-transform hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementation (numpy, float64) of what the
CUDA path computes: the top-down octree residual fit (Algorithm 1,
P:294-314, and Algorithm 2) and the interpolant evaluation
(§2, §4).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  It
shares no code with ``paper_1511_01353_b200`` (the product path): no kernels,
headers, helpers, tables or constants; the only common dependency is the input
generator module ``workloads`` (which holds none of the method's arithmetic).

Citation convention: ``P:<line>`` = /root/reference/PAPER.md line (section /
algorithm given); ``S:<line>`` = SPEC.md line (interface/test ideas only);
``G<k>`` = reading k of the paper-gap ledger in DESIGN.md §2.

Parity status of each function (the pins live in tests/test_oracle.py):
  rank, basis ............ pinned (printed ranks P:292; Alg. 2 loop order P:322-324)
  vandermonde ............ pinned (polynomial reproduction, brute-force lstsq)
  fit_node ............... pinned (polynomial reproduction, unisolvent interpolation,
                           brute-force lstsq with an independent basis, p=0 mean,
                           annihilation, coplanar rank truncation vs 2-D lstsq)
  _qr_r, TSQR branch ..... pinned (R of a > 2^16-row matrix = LAPACK's up to row signs; fit_node
                           streamed vs single-block and vs independent lstsq above 2^16 rows)
  build, build_subtree ... pinned (brute-force tree on tiny inputs, telescoping identity,
                           non-increasing residual, constant/polynomial -> 1 node; a restricted
                           or node-started run reproduces the full run's nodes)
  evaluate ............... pinned (path-sum == per-leaf lstsq; polynomial reproduction)
"""
from __future__ import annotations

import dataclasses
from math import factorial

import numpy as np
from threadpoolctl import threadpool_limits

# Rank-truncation threshold (reading G9): a column of the column-equilibrated
# Vandermonde matrix whose distance to the span of the previously KEPT columns
# is <= DELTA (i.e. |R_jj| <= DELTA for unit-norm columns) is dropped and its
# coefficient set to 0.  Chosen so that the same decision is resolvable in the
# Gram (normal-equation) form used on the GPU: there it reads s_jj <= DELTA**2
# = 1e-12, far above fp64 rounding of a unit-diagonal Gram (G9).
DELTA = 1e-6

# Rows per block of the row-streamed (TSQR) QR for large nodes.
_TSQR_ROWS = 1 << 16


def rank(p: int) -> int:
    """𝓛 = ℓ³_{p+1} = (p+1)(p+2)(p+3)/6 (P:141 rank stride; §3 prints 84/286/680 for
    L_max = 6/10/14; reading G1: the ℓ³_{L_max} of P:158 is off by one)."""
    return (p + 1) * (p + 2) * (p + 3) // 6


def basis(p: int) -> list[tuple[int, int, int]]:
    """Multi-indices (l, m, n), l+m+n <= p, in the loop order of Algorithm 2:
    l = 0..L outer, m = 0..L-l, n = 0..L-l-m inner."""
    out = []
    for l in range(p + 1):
        for m in range(p - l + 1):
            for n in range(p - l - m + 1):
                out.append((l, m, n))
    return out


def vandermonde(u: np.ndarray, p: int) -> np.ndarray:
    """Λ(1:N, lmn) = x1^l x2^m x3^n / (l! m! n!) (§2 geometric moments; Alg. 2)."""
    u = np.asarray(u, dtype=np.float64).reshape(-1, 3)
    # pw[a][k] = u_a ** k, each power formed once (the same `**` as inline, so the same bits)
    pw = [[u[:, a] ** k for k in range(p + 1)] for a in range(3)]
    cols = []
    for (l, m, n) in basis(p):
        cols.append(pw[0][l] * pw[1][m] * pw[2][n] / (factorial(l) * factorial(m) * factorial(n)))
    return np.stack(cols, axis=1) if cols else np.zeros((u.shape[0], 0))


def _qr_r(a: np.ndarray) -> np.ndarray:
    """R factor of a Householder QR (LAPACK dgeqrf, the call named at P:330), row-streamed
    (TSQR: R <- qr([R; block])) for tall matrices.  Run with one BLAS thread: the threaded
    OpenBLAS dgeqrf is ~20x slower on tall-skinny inputs on these hosts."""
    with threadpool_limits(limits=1, user_api="blas"):
        if a.shape[0] <= _TSQR_ROWS:
            return np.linalg.qr(a, mode="r")
        r = np.linalg.qr(a[:_TSQR_ROWS], mode="r")
        for s in range(_TSQR_ROWS, a.shape[0], _TSQR_ROWS):
            r = np.linalg.qr(np.vstack([r, a[s:s + _TSQR_ROWS]]), mode="r")
        return r


@dataclasses.dataclass
class NodeFit:
    coeffs: np.ndarray      # P_F (Λ basis, Alg. 2 column order), dropped columns = 0
    kept: np.ndarray        # bool mask of kept columns
    min_pivot: float        # smallest |R_jj| among kept columns (equilibrated), for diagnostics


def fit_node(u: np.ndarray, r: np.ndarray, p: int, delta: float = DELTA) -> NodeFit:
    """Algorithm 2: Λ, QR, P_F = R⁻¹ Qᵀ f, with the rank-truncation reading G9.

    1. Λ(u); columns equilibrated by their 2-norms d_j (a zero column is dropped).
    2. Householder QR of [Λ D⁻¹ | r]; the last column of R holds Qᵀr.
    3. Column rejection: walk j = 0..𝓛-1; QR of the kept columns so far plus column j; if the new
       diagonal |R_jj| <= delta the column is dropped.  QR of any column subset of [Λ D⁻¹ | r] equals
       the QR of the same subset of R (orthogonal invariance), so the walk runs on R.
    4. P_F = D⁻¹ R_S⁻¹ (Qᵀr)_S on the kept set S, 0 elsewhere.
    """
    u = np.asarray(u, dtype=np.float64).reshape(-1, 3)
    r = np.asarray(r, dtype=np.float64)
    L = rank(p)
    if u.shape[0] <= _TSQR_ROWS:
        lam = vandermonde(u, p)
        d = np.sqrt(np.sum(lam * lam, axis=0))
        nonzero = d > 0
        a = np.zeros_like(lam)
        a[:, nonzero] = lam[:, nonzero] / d[nonzero]
        R = _qr_r(np.hstack([a, r[:, None]]))  # (L+1) x (L+1)
    else:
        # The same two steps, streamed over row blocks so that Λ is never held whole (a node of
        # 2e7 points at p = 6 would need 13 GB): first the column norms, then the row-streamed
        # QR (TSQR) of the equilibrated [Λ D⁻¹ | r] block by block.
        d2 = np.zeros(L)
        for s in range(0, u.shape[0], _TSQR_ROWS):
            lam = vandermonde(u[s:s + _TSQR_ROWS], p)
            d2 += np.sum(lam * lam, axis=0)
        d = np.sqrt(d2)
        nonzero = d > 0
        dd = np.where(nonzero, d, 1.0)
        R = None
        with threadpool_limits(limits=1, user_api="blas"):
            for s in range(0, u.shape[0], _TSQR_ROWS):
                lam = vandermonde(u[s:s + _TSQR_ROWS], p)
                a = np.where(nonzero, lam / dd, 0.0)
                blk = np.hstack([a, r[s:s + _TSQR_ROWS, None]])
                R = np.linalg.qr(blk if R is None else np.vstack([R, blk]), mode="r")
    R = np.vstack([R, np.zeros((L + 1 - R.shape[0], L + 1))]) if R.shape[0] < L + 1 else R
    kept: list[int] = []
    diag_ok = np.abs(np.diag(R)[:L]) > delta
    if np.all(diag_ok & nonzero):
        kept = list(range(L))
        Rs = R[:L, :L]
        qtr = R[:L, L]
        piv = np.abs(np.diag(Rs))
    else:
        piv_list = []
        for j in range(L):
            if not nonzero[j]:
                continue
            cand = kept + [j]
            Rc = _qr_r(R[:, cand])
            if abs(Rc[len(cand) - 1, len(cand) - 1]) > delta:
                kept = cand
                piv_list.append(abs(Rc[len(cand) - 1, len(cand) - 1]))
        Rk = _qr_r(R[:, kept + [L]])
        k = len(kept)
        Rs = Rk[:k, :k]
        qtr = Rk[:k, k]
        piv = np.array(piv_list)
    c = np.zeros(L)
    if kept:
        from scipy.linalg import solve_triangular  # LAPACK dtrtrs: R⁻¹
        c_s = solve_triangular(Rs, qtr, lower=False)
        c[kept] = c_s / d[kept]
    mask = np.zeros(L, dtype=bool)
    mask[kept] = True
    return NodeFit(coeffs=c, kept=mask, min_pivot=float(np.min(piv)) if len(kept) else 0.0)


def apply_fit(u: np.ndarray, coeffs: np.ndarray, p: int) -> np.ndarray:
    """Λ(u)·P_F (the update term of P:332 and the per-node term of f(r) = Λ(r)·F_p),
    formed in row blocks so that Λ is never held whole for large nodes or query sets."""
    u = np.asarray(u, dtype=np.float64).reshape(-1, 3)
    out = np.empty(u.shape[0])
    for s in range(0, u.shape[0], _TSQR_ROWS):
        out[s:s + _TSQR_ROWS] = vandermonde(u[s:s + _TSQR_ROWS], p) @ coeffs
    return out


def morton_prefix(depth: int, cell: tuple[int, int, int]) -> int:
    """Label of a node: interleave the bits of its cell (i, j, k) at ``depth`` with x fastest, so that
    the digit of level t is o = bx + 2 by + 4 bz (S:324 octant numbering; reading G7).  Labels only."""
    i, j, k = cell
    out = 0
    for t in range(depth):
        b = depth - 1 - t
        o = ((i >> b) & 1) | (((j >> b) & 1) << 1) | (((k >> b) & 1) << 2)
        out = (out << 3) | o
    return out


@dataclasses.dataclass
class Tree:
    p: int
    tau: float
    max_depth: int
    lo: np.ndarray               # root cube origin (3,)
    width: float                 # root cube edge W
    depth: np.ndarray            # (nodes,)
    cell: np.ndarray             # (nodes, 3) int64
    prefix: np.ndarray           # (nodes,) uint64 label
    n_points: np.ndarray         # (nodes,)
    coeffs: np.ndarray           # (nodes, 𝓛) P_F in the Λ basis
    kept: np.ndarray             # (nodes, 𝓛) bool
    min_pivot: np.ndarray        # (nodes,)
    residual_rms: np.ndarray     # (nodes,) post-fit RMS over the node's points
    child_rms: np.ndarray        # (nodes, 8) E_RMS of each octant block (nan if n_o == 0)
    child_count: np.ndarray      # (nodes, 8) n_o
    child_index: np.ndarray      # (nodes, 8) index of the child node, -1 none, -2 created but not expanded
    residual: np.ndarray         # (N,) final residual in INPUT order (bookkeeping)

    @property
    def node_count(self) -> int:
        return int(self.depth.shape[0])

    def key_order(self) -> np.ndarray:
        """Canonical node order: (depth, prefix)."""
        return np.lexsort((self.prefix, self.depth))


def root_cube(points: np.ndarray) -> tuple[np.ndarray, float]:
    """Root frame (reading G6): the unit cube when every point lies in [0,1]^3 (all paper
    experiments), else the isotropic bounding cube of the data."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.size == 0 or (np.all(pts >= 0.0) and np.all(pts <= 1.0)):
        return np.zeros(3), 1.0
    lo = pts.min(axis=0)
    w = float(np.max(pts.max(axis=0) - lo))
    return lo, (w if w > 0 else 1.0)


def to_unit(points: np.ndarray, lo: np.ndarray, width: float) -> np.ndarray:
    """Global coordinates -> root-cube coordinates in [0,1]: (x - lo) / W, one subtraction and one
    division per coordinate (identity for the unit cube)."""
    pts = np.asarray(points, dtype=np.float64)
    if width == 1.0 and not np.any(lo):
        return pts.copy()
    return (pts - lo) / width


def local_coords(u: np.ndarray, depth: int, cell: np.ndarray) -> np.ndarray:
    """Alg. 1 line 2: x <- (x - P_C) * P_Scale, with the node of ``depth`` and cell (i,j,k):
    half-width h = 2^-(depth+1), centre c = (2i+1) h (FMT_New_Octant), scale 1/h."""
    h = 2.0 ** (-(depth + 1))
    c = (2.0 * np.asarray(cell, dtype=np.float64) + 1.0) * h
    return (u - c) * (2.0 ** (depth + 1))


def octant(ul: np.ndarray) -> np.ndarray:
    """FMT_Ordered_by_Octant key: o = [x1>=0] + 2[x2>=0] + 4[x3>=0] (tie -> upper)."""
    return (ul[:, 0] >= 0).astype(np.int64) + 2 * (ul[:, 1] >= 0) + 4 * (ul[:, 2] >= 0)


def build(points: np.ndarray, f: np.ndarray, p: int, tau: float, max_depth: int,
          delta: float = DELTA, descend=None) -> Tree:
    """FMT_Mesh_to_Tree (Algorithm 1) called on the root node: the root cube (G6), then
    ``build_subtree`` from depth 0.  The caller's arrays are not modified (the paper overwrites x and
    f in place).  ``descend`` (test harness only) restricts which created children are expanded;
    see ``build_subtree``."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(f, dtype=np.float64).reshape(-1)
    N = pts.shape[0]
    L = rank(p)
    if N < L:
        raise ValueError(f"N={N} < 𝓛={L}: the root fit is underdetermined (S:348)")
    lo, width = root_cube(pts)
    u = to_unit(pts, lo, width)
    tree = build_subtree(u, f, p, tau, max_depth, 0, (0, 0, 0), delta, descend)
    tree.lo, tree.width = lo, width
    return tree


def build_subtree(u: np.ndarray, f: np.ndarray, p: int, tau: float, max_depth: int, depth0: int,
                  cell0: tuple[int, int, int], delta: float = DELTA, descend=None) -> Tree:
    """FMT_Mesh_to_Tree (Algorithm 1) called on the node P of depth ``depth0`` and cell
    ``cell0`` (Alg. 1 is stated for any node P: its recursion calls itself on each created octant,
    P:308-309).  ``u``: root-cube coordinates of P's points (all inside P's box); ``f``: the residual
    P receives (the original values when P is the root).  Run depth-first exactly as printed:

      line 2  map to the node frame                  -> local_coords
      line 3  FMT_Mesh_to_Moments: fit, f <- f - Λ P_F (Alg. 2)  -> fit_node, apply_fit
      line 4  FMT_Ordered_by_Octant: stable partition into 8 blocks
      lines 6-12 for each octant o with n_o points:
              E_RMS = sqrt(sum_block f^2 / n_o) on the post-fit residual (G3)
              recurse iff E_RMS > tau and n_o >= 𝓛 (G4) and depth+1 <= max_depth (G5)
              block bounds: running start j, end j + n_o (G2)

    ``descend(depth, cell) -> bool`` (None = always) is a test-harness restriction, not part of the
    method: a child that Alg. 1 creates but ``descend`` rejects is recorded with child_index -2
    ("created, not expanded in this run") and its subtree is skipped.  Subtrees are independent given
    the residual they receive, so every expanded node is exactly the node of the unrestricted run.
    Returned nodes are in creation (pre-)order; node 0 is P.  ``residual`` is the final residual in
    the order of ``u`` (entries of skipped subtrees hold their received residual)."""
    u = np.asarray(u, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(f, dtype=np.float64).reshape(-1)
    N = u.shape[0]
    L = rank(p)
    perm = np.arange(N)          # current order of the points (Alg. 1 permutes in place)
    res = f.copy()               # the residual, in 'perm' order
    nodes = []                   # dicts, in creation (pre-)order

    # explicit stack of (depth, cell, start, end, parent, octant-in-parent)
    stack = [(depth0, tuple(int(v) for v in cell0), 0, N, -1, -1)]
    while stack:
        depth, cell, j0, j1, parent, oct_in_parent = stack.pop()
        idx = perm[j0:j1]
        ul = local_coords(u[idx], depth, np.array(cell))
        fit = fit_node(ul, res[j0:j1], p, delta)
        res[j0:j1] = res[j0:j1] - apply_fit(ul, fit.coeffs, p)              # Alg. 2 last line
        n = j1 - j0
        me = len(nodes)
        node = dict(depth=depth, cell=cell, n=n, coeffs=fit.coeffs, kept=fit.kept,
                    min_pivot=fit.min_pivot,
                    rms=float(np.sqrt(np.sum(res[j0:j1] ** 2) / n)) if n else 0.0,
                    child_rms=np.full(8, np.nan), child_count=np.zeros(8, dtype=np.int64),
                    child_index=np.full(8, -1, dtype=np.int64))
        nodes.append(node)
        if parent >= 0:
            nodes[parent]["child_index"][oct_in_parent] = me
        # FMT_Ordered_by_Octant: stable partition of this node's block
        o = octant(ul)
        order = np.argsort(o, kind="stable")
        perm[j0:j1] = idx[order]
        res[j0:j1] = res[j0:j1][order]
        counts = np.bincount(o, minlength=8)
        node["child_count"][:] = counts
        j = j0
        children = []
        for oc in range(8):
            n_o = int(counts[oc])
            k = j + n_o
            if n_o > 0:
                e_rms = float(np.sqrt(np.sum(res[j:k] ** 2) / n_o))
                node["child_rms"][oc] = e_rms
                if e_rms > tau and n_o >= L and depth + 1 <= max_depth:        # P:306 (+ G5)
                    ccell = (2 * cell[0] + (oc & 1), 2 * cell[1] + ((oc >> 1) & 1), 2 * cell[2] + ((oc >> 2) & 1))
                    if descend is None or descend(depth + 1, ccell):
                        children.append((depth + 1, ccell, j, k, me, oc))      # FMT_New_Octant
                    else:
                        node["child_index"][oc] = -2
            j = k                                                               # G2
        # push in reverse so that octant 1 is processed first (depth-first, as Alg. 1)
        stack.extend(reversed(children))

    residual = np.empty(N)
    residual[perm] = res
    T = len(nodes)
    return Tree(
        p=p, tau=tau, max_depth=max_depth, lo=np.zeros(3), width=1.0,
        depth=np.array([nd["depth"] for nd in nodes], dtype=np.int64),
        cell=np.array([nd["cell"] for nd in nodes], dtype=np.int64).reshape(T, 3),
        prefix=np.array([morton_prefix(nd["depth"], nd["cell"]) for nd in nodes], dtype=np.uint64),
        n_points=np.array([nd["n"] for nd in nodes], dtype=np.int64),
        coeffs=np.array([nd["coeffs"] for nd in nodes]).reshape(T, L),
        kept=np.array([nd["kept"] for nd in nodes]).reshape(T, L),
        min_pivot=np.array([nd["min_pivot"] for nd in nodes]),
        residual_rms=np.array([nd["rms"] for nd in nodes]),
        child_rms=np.array([nd["child_rms"] for nd in nodes]).reshape(T, 8),
        child_count=np.array([nd["child_count"] for nd in nodes]).reshape(T, 8),
        child_index=np.array([nd["child_index"] for nd in nodes]).reshape(T, 8),
        residual=residual,
    )


def evaluate(tree: Tree, q: np.ndarray) -> np.ndarray:
    """f(r) = Λ(r)·F_p summed over the root-to-deepest-existing-node path (§2; "only
    downward recursion to accumulate local polynomial representation of the residual", P:367-368;
    reading G11).  Queries outside the root cube get the root polynomial only."""
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    M = q.shape[0]
    out = np.zeros(M)
    if M == 0:
        return out
    u = to_unit(q, tree.lo, tree.width)
    inside = np.all((u >= 0.0) & (u <= 1.0), axis=1)
    node_of = np.zeros(M, dtype=np.int64)       # every query starts at the root (node 0)
    active = np.arange(M)
    while active.size:
        nxt = []
        nodes_here = node_of[active]
        for nd in np.unique(nodes_here):
            sel = active[nodes_here == nd]
            ul = local_coords(u[sel], int(tree.depth[nd]), tree.cell[nd])
            out[sel] += apply_fit(ul, tree.coeffs[nd], tree.p)
            sel_in = sel[inside[sel]]
            if sel_in.size == 0:
                continue
            o = octant(local_coords(u[sel_in], int(tree.depth[nd]), tree.cell[nd]))
            ch = tree.child_index[nd][o]
            if np.any(ch == -2):
                raise ValueError("query reaches a node that this restricted run did not expand")
            go = ch >= 0
            node_of[sel_in[go]] = ch[go]
            nxt.append(sel_in[go])
        active = np.concatenate(nxt) if nxt else np.zeros(0, dtype=np.int64)
    return out
