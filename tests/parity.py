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
