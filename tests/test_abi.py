"""C-ABI checks that need no GPU: the library loads, exports every symbol include/fmi.h declares, and
rejects bad arguments (or reports the missing device) with the documented codes — never a CPU fallback."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmi.h")
LIB = os.path.join(ROOT, "paper_1511_01353_b200", "libfmi.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmi_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.dirname(LIB), "-j8"], check=True)
    import paper_1511_01353_b200 as fmi
    return fmi.load_library()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("fmi_build", "fmi_eval", "fmi_free", "fmi_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fmi_[a-z_]+)\b", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    import paper_1511_01353_b200 as fmi
    assert set(fmi.EXPORTED) == set(_declared())


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_without_gpu(lib):
    import paper_1511_01353_b200 as fmi
    pts = np.random.default_rng(0).random((100, 3))
    f = np.zeros(100)
    h = lib.fmi_build(None, None, 100, 2, 1e-6, 2)
    assert not h and fmi.last_error()[0] == fmi.fmi.FMI_EINPUT
    for args, code in [((pts, f, 100, 11, 1e-6, 2), fmi.fmi.FMI_EPRECOND),   # p > 10 needs max_depth = 0
                       ((pts, f, 100, 15, 1e-6, 0), fmi.fmi.FMI_EPRECOND),   # p > 14
                       ((pts, f, 100, 12, 1e-6, 0), fmi.fmi.FMI_EPRECOND),   # N < 𝓛 = 455
                       ((pts, f, 100, 2, -1.0, 2), fmi.fmi.FMI_EPRECOND),
                       ((pts, f, 100, 2, float("nan"), 2), fmi.fmi.FMI_EPRECOND),
                       ((pts, f, 100, 2, 1e-6, 21), fmi.fmi.FMI_EPRECOND),
                       ((pts, f, 5, 2, 1e-6, 2), fmi.fmi.FMI_EPRECOND),
                       ((pts, f, -1, 2, 1e-6, 2), fmi.fmi.FMI_EINPUT)]:
        a, b, n, p, tau, d = args
        h = lib.fmi_build(a.ctypes.data, b.ctypes.data, n, p, tau, d)
        assert not h
        assert fmi.last_error()[0] == code, (args[2:], fmi.last_error())
    assert lib.fmi_eval(None, None, 0, None) == fmi.fmi.FMI_EINPUT
    lib.fmi_free(None)  # NULL-safe


def test_profile_select_names(lib):
    """fmi_profile_select: every documented kernel name (and NULL / "" = all) is accepted; an unknown name is
    FMI_EINPUT and leaves the selection alone (include/fmi.h)."""
    import paper_1511_01353_b200 as fmi
    assert lib.fmi_profile_select(None) == 0
    assert lib.fmi_profile_select(b"") == 0
    assert lib.fmi_profile_select(",".join(fmi.fmi.KERNELS).encode()) == 0
    assert lib.fmi_profile_select(b"residual,moments") == 0
    assert lib.fmi_profile_select(b"residual,nope") == fmi.fmi.FMI_EINPUT
    assert "unknown kernel name" in fmi.last_error()[1]
    assert lib.fmi_profile_select(b"resid") == fmi.fmi.FMI_EINPUT  # prefixes are not names
    with pytest.raises(fmi.FmiError):
        fmi.profile_select(["keys", "bogus"])
    fmi.profile_select(None)


def test_no_cpu_fallback_without_device(lib):
    """Valid arguments on a host without a GPU must fail loudly with FMI_ECUDA."""
    import paper_1511_01353_b200 as fmi
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    pts = np.random.default_rng(0).random((200, 3))
    with pytest.raises(fmi.FmiError) as ei:
        fmi.build(pts, np.zeros(200), 2, 1e-6, 2)
    assert ei.value.code == fmi.fmi.FMI_ECUDA


def test_oracle_is_not_imported_by_the_product():
    pkg = os.path.join(ROOT, "paper_1511_01353_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or fn == "fmi.py" and "oracle" not in txt, fn


def test_result_buffer_validation_without_gpu():
    """transfer()/eval() write M doubles through `out`: a wrong dtype, layout or length is rejected before
    the library is called (no silent converted copy, no overrun)."""
    import paper_1511_01353_b200 as fmi
    pts = np.random.default_rng(0).random((100, 3))
    f = pts[:, 0].copy()
    q = pts[:10].copy()
    for bad, exc in [(np.empty(10, dtype=np.float32), TypeError), (np.empty(9), ValueError),
                     (np.empty((10, 2))[:, 0], TypeError), (np.empty(11), ValueError), ([0.0] * 10, TypeError)]:
        with pytest.raises(exc):
            fmi.transfer(pts, f, q, 1, 1e-6, 1, out=bad)
