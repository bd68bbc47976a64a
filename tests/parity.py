"""Helpers comparing a GPU tree (paper_1511_01353_b200.Tree.export()) with an oracle tree."""
import numpy as np


def node_key_map(depth, cell):
    return {(int(depth[i]), int(cell[i][0]), int(cell[i][1]), int(cell[i][2])): i for i in range(len(depth))}


def compare_trees(gpu, ora, tau, rel_rms=1e-6):
    """Topology, point counts and octant counts bit-exact; decisions' margins reported."""
    g = node_key_map(gpu["depth"], gpu["cell"])
    o = node_key_map(ora.depth, ora.cell)
    only_g = sorted(set(g) - set(o))
    only_o = sorted(set(o) - set(g))
    msgs = []
    if only_g or only_o:
        # report E/tau margins of the mismatching decisions
        for key in only_g + only_o:
            d, i, j, k = key
            if d == 0:
                continue
            pk = (d - 1, i >> 1, j >> 1, k >> 1)
            oc = (i & 1) | ((j & 1) << 1) | ((k & 1) << 2)
            eo = ora.child_rms[o[pk]][oc] if pk in o else np.nan
            eg = gpu["child_rms"][g[pk]][oc] if pk in g else np.nan
            msgs.append(f"{key}: oracle E/tau={eo / tau if tau else np.inf:.6g} gpu E/tau={eg / tau if tau else np.inf:.6g}")
    assert not only_g and not only_o, "topology differs:\n" + "\n".join(msgs[:20])
    for key, gi in g.items():
        oi = o[key]
        assert gpu["n_points"][gi] == ora.n_points[oi], key
        assert np.array_equal(gpu["child_count"][gi], ora.child_count[oi]), key
    return g, o


def coeff_and_rms_errors(gpu, ora, g, o):
    """max relative differences of node residual RMS and of the P_F coefficients (scaled by node data)."""
    drms = 0.0
    for key, gi in g.items():
        oi = o[key]
        a, b = gpu["residual_rms"][gi], ora.residual_rms[oi]
        drms = max(drms, abs(a - b) / max(abs(b), 1e-300))
    return drms


def rms_agreement(gpu, ora, g, o, scale, rel=1e-6, abs_=1e-12):
    """Every common node's post-fit RMS agrees: |Δ| <= rel·rms_oracle + abs_·max|f| (the
    residuals of the two paths differ by roundoff only, ~1e-13·max|f| at the worst-conditioned nodes)."""
    worst = 0.0
    for key, gi in g.items():
        oi = o[key]
        a, b = gpu["residual_rms"][gi], ora.residual_rms[oi]
        bound = rel * abs(b) + abs_ * scale
        worst = max(worst, abs(a - b) / bound)
        assert abs(a - b) <= bound, (key, a, b)
    return worst


def compare_with_golden(ex, gold, tau, L, max_depth, tie_band, scale, within=None, depth_offset=0,
                        cell_offset=None):
    """GPU tree export ``ex`` against an oracle golden node table (tools/make_golden.py).

    Every golden node must exist on the GPU with the same point count and octant counts (bit-exact
    integer work); every octant decision (child created iff E > τ ∧ n_o >= 𝓛 ∧ depth+1 <= D)
    must agree, except decisions whose oracle margin |E/τ - 1| < tie_band (roundoff-level ties, G17),
    under which the subtree is not compared; every GPU node inside the covered region must be a golden
    node; post-fit node RMS within rms_agreement's bound.  ``within(depth, cell)``: the covered region
    (default everything).  ``depth_offset``/``cell_offset``: map golden coordinates to the GPU tree's
    (a subtree solved as a stand-alone problem).  Returns a report dict."""
    def to_gpu(d, c):
        if cell_offset is None:
            return (d - depth_offset, c)
        s = 1 << (d - depth_offset)
        return (d - depth_offset, tuple(int(c[a] - cell_offset[a] * s) for a in range(3)))

    g = node_key_map(ex["depth"], ex["cell"])
    gd = {(int(gold["depth"][i]), tuple(int(v) for v in gold["cell"][i])): i for i in range(len(gold["depth"]))}
    skipped = set()          # (depth, cell) roots of tie subtrees (golden coordinates)
    ties, decisions, worst_rms = [], 0, 0.0

    def under_tie(d, c):
        for (sd, sc) in skipped:
            if d >= sd and tuple(v >> (d - sd) for v in c) == sc:
                return True
        return False

    for (d, c), i in sorted(gd.items()):
        if under_tie(d, c):
            continue
        key = to_gpu(d, c)
        gk = (key[0],) + tuple(key[1])
        assert gk in g, f"golden node {d}:{c} missing on the GPU"
        gi = g[gk]
        assert ex["n_points"][gi] == gold["n"][i], (d, c)
        assert np.array_equal(ex["child_count"][gi], gold["child_count"][i]), (d, c)
        a, b = ex["residual_rms"][gi], gold["residual_rms"][i]
        bound = 1e-6 * abs(b) + 1e-12 * scale
        assert abs(a - b) <= bound, ("node rms", d, c, a, b)
        worst_rms = max(worst_rms, abs(a - b) / bound)
        for o in range(8):
            n_o = int(gold["child_count"][i][o])
            if n_o < L or d + 1 > max_depth:
                continue
            decisions += 1
            want = gold["child_state"][i][o] != -1
            got = ex["child"][gi][o] >= 0
            margin = abs(gold["child_rms"][i][o] / tau - 1.0) if tau > 0 else np.inf
            cc = tuple(2 * c[a] + ((o >> a) & 1) for a in range(3))
            if margin < tie_band:
                ties.append((d + 1, cc, float(margin), bool(want), bool(got)))
                if want != got:
                    skipped.add((d + 1, cc))
                continue
            assert want == got, f"decision differs at {d}:{c} octant {o}: oracle E/tau={gold['child_rms'][i][o] / tau:.6g}"
    # no extra GPU nodes inside the covered region
    for key, gi in g.items():
        d = key[0] + depth_offset
        c = tuple(int(v) for v in key[1:])
        if cell_offset is not None:
            s = 1 << key[0]
            c = tuple(int(c[a] + cell_offset[a] * s) for a in range(3))
        if within is not None and not within(d, c):
            continue
        if under_tie(d, c):
            continue
        assert (d, c) in gd, f"GPU node {d}:{c} is not in the oracle's tree"
    return {"decisions": decisions, "ties": ties, "worst_rms_over_bound": worst_rms, "nodes": len(gd)}
