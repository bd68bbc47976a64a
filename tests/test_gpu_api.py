"""The remaining public calls on a GPU: mesh-to-mesh transfer (fmi_transfer) and tree
files (fmi_save / fmi_load): a loaded tree evaluates bit-identically and exports the same nodes."""
import numpy as np
import pytest

import workloads
from oracle import fmt_oracle as fo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_transfer_matches_build_eval_and_oracle():
    import paper_1511_01353_b200 as fmi
    from paper_1511_01353_b200 import fmi as f_
    cfg = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(cfg)
    got = f_.transfer(pts, f, q, cfg.degree, cfg.tol, cfg.max_depth)
    with fmi.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t:
        ref = t.eval(q)
    assert np.array_equal(got, ref)
    ora = fo.evaluate(fo.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth), q)
    assert np.max(np.abs(got - ora)) <= 1e-9 * np.max(np.abs(f))


def test_save_load_roundtrip(tmp_path):
    import paper_1511_01353_b200 as fmi
    from paper_1511_01353_b200 import fmi as f_
    cfg = workloads.CONFIGS[2]
    pts, f, q = workloads.make_inputs(cfg)
    q = q[:50_000]
    path = tmp_path / "tree.fmi"
    with fmi.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t:
        v1 = t.eval(q)
        e1 = t.export()
        t.save(str(path))
    t2 = f_.load(str(path))
    try:
        v2 = t2.eval(q)
        e2 = t2.export()
        assert np.array_equal(v1, v2)
        for k in ("depth", "cell", "n_points", "child_count", "child", "coeffs", "residual_rms", "rank"):
            assert np.array_equal(e1[k], e2[k]), k
        with pytest.raises(f_.FmiError):
            t2.residual()
    finally:
        t2.free()
    bad = tmp_path / "bad.fmi"
    bad.write_bytes(b"not a tree file at all")
    with pytest.raises(f_.FmiError) as ei:
        f_.load(str(bad))
    assert ei.value.code == f_.FMI_EVERSION


def test_pipelined_host_eval_matches_device_eval():
    """M > 2^24 queries in page-locked host memory take the chunked path (H2D / keys+sort+eval / D2H of
    neighbouring chunks overlapped); every value equals the device-pointer evaluation bit for bit, and
    a pageable output buffer (unpipelined path) gives the same values."""
    import paper_1511_01353_b200 as fmi
    cfg = workloads.CONFIGS[2]
    pts, f, _ = workloads.make_inputs(cfg)
    M = (1 << 24) * 2 + 12345  # three chunks, ragged tail
    q = workloads.uniform_points(M, 7)
    hq = torch.from_numpy(q).pin_memory()
    hout = torch.empty(M, dtype=torch.float64).pin_memory()
    with fmi.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t:
        ref = t.eval(hq.cuda()).cpu().numpy()
        t.eval(hq.numpy(), out=hout.numpy())
        assert np.array_equal(hout.numpy(), ref)
        pageable = t.eval(q)
        assert np.array_equal(pageable, ref)
    # transfer: queries uploaded during the fit, values pipelined back
    out2 = torch.empty(M, dtype=torch.float64).pin_memory()
    fmi.transfer(pts, f, hq.numpy(), cfg.degree, cfg.tol, cfg.max_depth, out=out2.numpy())
    assert np.array_equal(out2.numpy(), ref)


def test_pinned_host_values_uploaded_late():
    """Page-locked host values (N >= 2^20) take the side-stream upload and join the build after the
    moment passes (gathered with the root projection, checked for finiteness there): same tree and
    values as device inputs; a NaN is still rejected with FMI_EINPUT."""
    import paper_1511_01353_b200 as fmi
    from types import SimpleNamespace
    cfg = SimpleNamespace(degree=4, tol=1e-7, max_depth=5)
    pts = workloads.uniform_points((1 << 20) + 12345, 3)
    f = workloads.franke3d(pts)
    q = workloads.uniform_points(20_000, 4)
    hp = torch.from_numpy(pts).pin_memory()
    hf = torch.from_numpy(f).pin_memory()
    with fmi.build(hp.numpy(), hf.numpy(), cfg.degree, cfg.tol, cfg.max_depth) as a, \
            fmi.build(hp.cuda(), hf.cuda(), cfg.degree, cfg.tol, cfg.max_depth) as b:
        assert a.node_count == b.node_count
        assert np.array_equal(a.eval(q), b.eval(q))
    hf[123] = float("nan")
    with pytest.raises(fmi.FmiError) as ei:
        fmi.build(hp.numpy(), hf.numpy(), cfg.degree, cfg.tol, cfg.max_depth)
    assert ei.value.code == -1


@pytest.mark.parametrize("what", ["depth", "child", "parent", "cell", "header_D"])
def test_load_rejects_corrupt_node_records(tmp_path, what):
    """A tree file is untrusted input: a node record whose depth, parent, child index or cell is
    inconsistent is rejected with FMI_EVERSION naming the node (before any kernel follows it)."""
    import struct
    import paper_1511_01353_b200 as fmi
    from paper_1511_01353_b200 import fmi as f_
    cfg = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(cfg)
    path = tmp_path / "tree.fmi"
    with fmi.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t:
        t.save(str(path))
        n = t.node_count
    raw = bytearray(path.read_bytes())
    H = 88                                   # FileHeader: magic, 4 int32, 2 int64, 5 doubles, 2 int32
    cell, parent, child = H, H + 16 * n, H + 20 * n
    if what == "depth":
        struct.pack_into("<i", raw, cell + 5 * 16 + 12, 7)
    elif what == "child":
        struct.pack_into("<i", raw, child + 4 * 3, 1_000_000)
    elif what == "parent":
        struct.pack_into("<i", raw, parent + 4 * (n - 1), n + 5)
    elif what == "cell":
        struct.pack_into("<i", raw, cell + 2 * 16, 9)
    else:
        struct.pack_into("<i", raw, 80, 99)
    bad = tmp_path / "bad.fmi"
    bad.write_bytes(bytes(raw))
    with pytest.raises(f_.FmiError) as ei:
        f_.load(str(bad))
    assert ei.value.code == f_.FMI_EVERSION
    assert ("node" in str(ei.value)) or what == "header_D"
    # the untouched file still loads
    fmi.load(str(path)).free()


def test_profile_select_times_only_the_named_kernels():
    """fmi_profile_select (include/fmi.h): events only around the named kernels; launch and unit counters and
    the results are unaffected (bench.py times its rooflined kernels this way inside the timed region)."""
    import paper_1511_01353_b200 as fmi
    cfg = workloads.CONFIGS[1]
    pts, f, q = workloads.make_inputs(cfg)

    def run(select):
        fmi.profile_reset()
        fmi.profile_select(select)
        fmi.profile_enable(True)
        n0 = fmi.launch_count()
        with fmi.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth) as t:
            v = t.eval(q)
        fmi.profile_enable(False)
        timed = {k for k, (ms, n) in fmi.profile_get().items() if n}
        return v, timed, fmi.launch_count() - n0, fmi.profile_units()

    try:
        v_all, timed_all, n_all, u_all = run(None)
        v_sel, timed_sel, n_sel, u_sel = run(["residual", "solve"])
    finally:
        fmi.profile_select(None)
    assert {"residual", "solve", "keys", "eval"} <= timed_all
    assert timed_sel == {"residual", "solve"}
    assert n_sel == n_all and u_sel == u_all
    assert np.array_equal(v_all, v_sel)
