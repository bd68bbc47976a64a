"""Memory-safety check through the library's guard bands (compute-sanitizer is closed on the GPU pool):
tools/sanitize_run.py --quick under FMI_GUARD=1 runs every kernel family of the hot path (keys, sort,
gather, K4, M2M, K5/K5q/K5r, K6 split and fused, decisions, presum, K7, the QR path at depth > 0 and the
unscoped f2 path; Alg. 1/2) against the oracle, and every library buffer's 4 KiB guard
bands must be intact when it is freed (include/fmi.h fmi_guard_violations)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_intact():
    env = dict(os.environ, FMI_GUARD="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--quick"], env=env,
                         capture_output=True, text=True, timeout=1200)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "guard bands overwritten: 0" in out.stdout
    assert "ALL OK" in out.stdout
