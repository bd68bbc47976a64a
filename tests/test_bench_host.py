"""Host logic of bench.py (no GPU): the algorithmic-work accounting behind the roofline fields and the
reference arm's JSON line.  The work counts are the method's, never the kernels'
instruction counts."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads  # noqa: E402


def test_ranks_are_the_paper_ranks():
    # 𝓛 = (p+1)(p+2)(p+3)/6 (84, 286, 680 for p = 6, 10, 14); K = moments of degree <= 2p
    assert [bench.ranks(p)[1] for p in (6, 10, 14)] == [84, 286, 680]
    assert bench.ranks(10)[0] == 1771


class _Tree:
    def __init__(self, depth, flags, child_count, child):
        self.ex = {"depth": np.array(depth), "flags": np.array(flags),
                   "child_count": np.array(child_count), "child": np.array(child)}

    def export(self):
        return self.ex


def test_projected_points_counts_guarded_and_deferred_blocks():
    L = 10
    # node 0 (depth 0, not deferred): blocks with n_o >= 𝓛 are projected (the kernel's guard)
    # node 1 (depth 1, deferred): only its created children's points were projected (K6_PROJ)
    # node 2 (depth 2 = max_depth): no block may become a child
    t = _Tree(depth=[0, 1, 2], flags=[0, 8, 0],
              child_count=[[12, 9, 10, 0, 0, 0, 0, 30], [20, 20, 5, 0, 0, 0, 0, 0], [50] * 8],
              child=[[1, -1, -1, -1, -1, -1, -1, 2], [3, -1, -1, -1, -1, -1, -1, -1], [-1] * 8])
    assert bench.projected_points(t, L, max_depth=2) == (12 + 10 + 30) + 20


def test_kernel_work_definitions():
    cfg = workloads.CONFIGS[5]
    K, L = bench.ranks(cfg.degree)
    pts = [cfg.n, cfg.n // 2]
    w = bench.kernel_work(cfg, pts, depth_max=1, projected=cfg.n)
    assert w["moments"] == ("flop", 2 * K * cfg.n)
    assert w["residual"] == ("flop", sum(n * (2 * L + 2) for n in pts) + 2 * L * cfg.n)
    assert w["project"] == ("flop", 2 * L * cfg.n)
    assert w["eval"] == ("flop", 2 * L * cfg.m)
    assert w["gather"] == ("byte", 68 * cfg.n)


def test_rooflines_divide_work_per_launch_by_mean_launch_time():
    cfg = workloads.CONFIGS[5]
    prof = {"eval": (20.0, 2)}  # 2 launches over 2 steps, 10 ms each
    r = bench.rooflines(cfg, [cfg.n], 0, prof, steps=2, ms_per_step=100.0, hbm_peak=6000.0)
    e = r["eval"]
    K, L = bench.ranks(cfg.degree)
    assert e["launches_per_step"] == 1.0
    assert e["achieved"] == pytest.approx(2 * L * cfg.m / 10e-3 / 1e12)
    assert e["frac"] == pytest.approx(e["achieved"] / e["peak"])
    assert e["share_of_step"] == pytest.approx(0.1)


def test_reference_arm_line_contract():
    """`bench.py --impl reference` on a small config: the oracle timed on the host, one JSON line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_kernel_work_uses_executed_units():
    """Sort bytes come from the 8-bit passes the library actually ran, solve flops from the nodes it
    factored, key bytes from the library's own per-launch count (fmi_profile_units)."""
    cfg = workloads.CONFIGS[5]
    K, L = bench.ranks(cfg.degree)
    units = {"sort": 20 * (3 * cfg.n + 2 * cfg.m), "solve": 4880, "keys": 76 * cfg.n + 68 * cfg.m}
    w = bench.kernel_work(cfg, [cfg.n], depth_max=0, projected=0, units=units)
    assert w["sort"] == ("byte", 20 * (3 * cfg.n + 2 * cfg.m))
    assert w["solve"] == ("flop", 4880 * (L ** 3 / 3 + 3 * L * L))
    assert w["keys"] == ("byte", 76 * cfg.n + 68 * cfg.m)
    # per-step units: the roofline divides the timed region's units by the step count
    prof = {"sort": (14.6, 12)}   # 2 steps x (3 + 3 passes) x ... launches; 7.3 ms per step
    r = bench.rooflines(cfg, [cfg.n], 0, prof, steps=2, ms_per_step=100.0, hbm_peak=6456.8,
                        units={"sort": 2 * units["sort"]})
    per_launch = units["sort"] / 6
    assert r["sort"]["achieved"] == pytest.approx(per_launch / (14.6e-3 / 12) / 1e9)


def test_self_launch_under_torchrun_reference_arm():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (the driver's launch line);
    rank 0 alone prints the reference line."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--gpus", "1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr


def test_oracle_sample_uses_every_core_on_large_configs():
    """The cpu_baseline sample of a large config: one process per core over random cells of the workload."""
    cfg = workloads.CONFIGS[2].scaled(m=20_000)
    pts, f, q = workloads.make_inputs(cfg)
    v, dt, cores, sample = bench.time_oracle_sample(cfg, pts, f, q, target_points=15_000, cells=2)
    assert v > 0 and cores == min(2, bench.host_cores())
    assert "depth-1 cells" in sample
