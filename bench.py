#!/usr/bin/env python
"""Benchmark of the octree fit + evaluation hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl {fmi,reference}]

One step = fmi_build over the config's N points + fmi_eval at its M queries (+ fmi_free), i.e. every
§8(a) row of SURVEY.md once.  value = (N + M) points / step time (points/s), inputs resident in HBM
before the timed region; e2e = the same through the C ABI with pinned HOST buffers (H2D of points,
values and queries and D2H of the result inside the timed region).  Timing: CUDA events on the stream
the library launches on, barrier + synchronize on both sides, max over ranks.  Inputs (>= 6 GB at
the default config) exceed the 126 MB L2, so no explicit flush is needed between steps.

--impl reference times the oracle (oracle/fmt_oracle.py, CPU) on a bounded sample of the same
workload (there is no reference implementation to install: the paper ships no code).

Multi-GPU (torchrun, N > 1): one sharded build of the SAME global workload (strong scaling): every rank
starts with 1/N of the points and queries, the points are exchanged by Morton cells of the shard depth,
nodes above it are summed with NCCL allreduce (paper_1511_01353_b200/shard.py), queries
are routed to their owner rank and back.  value = (N + M) / step time (max over ranks).
FMI_BENCH_BACKEND=gloo + FMI_BENCH_ONE_DEVICE=1 run the multi-rank path on one GPU (functional check
only; the numbers of such a run are not measurements).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: SMs × FP64 FMA/clk/SM × 2 × max SM clock
PEAK_SOURCE = ("alu: fp64 derived 148 SM x 64 FMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s (measured on this pool: DMMA "
               "37.0, DFMA 34.2 TFLOP/s, profiles/round1_fp64_peak.txt); hbm: MEASURED_PEAKS.json hbm_gbs")


def measured_hbm_peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6456.8  # the pool's measured copy bandwidth at the time of writing


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="fmi", choices=["fmi", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="override N (debugging; not a bench line)")
    ap.add_argument("--m", type=int, default=None, help="override M (debugging; not a bench line)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        if os.environ.get("FMI_BENCH_NO_CLOCKS"):  # diagnostics: no NVML sampling
            self.nv = None
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # one untimed query of each kind: NVML's lazy first-call set-up (which can hold driver locks
            # for a long time) must not land inside the timed region
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands on a bounded sample of the workload
# ------------------------------------------------------------------------------------------------
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_cell_job(args):
    """One sampled subtree: Alg. 1 called on the cell's node with the original values (telescoping
    start) + the interpolant at the config's queries inside the cell."""
    u, f, q, p, tau, D, depth, cell = args
    from oracle import fmt_oracle
    t0 = time.perf_counter()
    tree = fmt_oracle.build_subtree(u, f, p, tau, D, depth, cell)
    fmt_oracle.evaluate(tree, q)
    return time.perf_counter() - t0, tree.node_count


def time_oracle_sample(cfg: workloads.Config, pts, f, q, target_points: int, cells: int | None = None, seed: int = 0):
    """The oracle (as it stands, never tuned) on a bounded sample of the SAME workload, on every host core.

    If the config holds <= target_points points the sample is the whole workload (one process).  Else the
    sample is ``cells`` (default: one per core) random octree cells of the shallowest depth d whose mean
    cell holds <= target_points points (cells with >= 𝓛 points), each fitted as Alg. 1 called on that node
    with the original values and evaluated at the config's queries inside it, one process per cell, all
    cores busy.  value = (sampled points + sampled queries) / wall time."""
    from oracle import fmt_oracle
    cores = host_cores()
    if cfg.n <= target_points:
        t0 = time.perf_counter()
        tree = fmt_oracle.build(pts, f, cfg.degree, cfg.tol, cfg.max_depth)
        fmt_oracle.evaluate(tree, q)
        dt = time.perf_counter() - t0
        sample = (f"the whole {cfg.name} workload (N={cfg.n:,}, M={cfg.m:,}) -> {tree.node_count} nodes; "
                  f"one process (numpy + single-threaded LAPACK QR)")
        return (cfg.n + cfg.m) / dt, dt, 1, sample
    d = 0
    while cfg.n / 8 ** d > target_points:
        d += 1
    L = ranks(cfg.degree)[1]
    cp = workloads.cell_of(pts, d)
    lab = cp[:, 0] | (cp[:, 1] << d) | (cp[:, 2] << (2 * d))
    cnt = np.bincount(lab, minlength=8 ** d)
    cand = np.flatnonzero(cnt >= L)
    k = min(len(cand), cells or cores)
    pick = np.random.default_rng(seed).choice(cand, size=k, replace=False)
    cq = workloads.cell_of(q, d)
    qlab = cq[:, 0] | (cq[:, 1] << d) | (cq[:, 2] << (2 * d))
    jobs, npts, nq = [], 0, 0
    for c in pick:
        cell = (int(c & (2 ** d - 1)), int((c >> d) & (2 ** d - 1)), int(c >> (2 * d)))
        sel = lab == c
        qsel = qlab == c
        jobs.append((np.ascontiguousarray(pts[sel]), np.ascontiguousarray(f[sel]), np.ascontiguousarray(q[qsel]),
                     cfg.degree, cfg.tol, cfg.max_depth, d, cell))
        npts += int(sel.sum())
        nq += int(qsel.sum())
    import multiprocessing as mp
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(min(cores, k)) as pool:
        res = pool.map(_oracle_cell_job, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    nodes = sum(r[1] for r in res)
    sample = (f"{k} random depth-{d} cells of the {cfg.name} workload ({npts:,} points, {nq:,} queries, {nodes} nodes), "
              f"each = Alg. 1 called on the cell's node with the original values (telescoping start) + the "
              f"interpolant at the config's queries in it; {min(cores, k)} processes on {cores} cores "
              f"({cpu_model()}), numpy + single-threaded LAPACK QR per process.  Only levels >= {d} are fitted, "
              f"so this overstates the oracle's whole-workload throughput")
    return (npts + nq) / dt, dt, min(cores, k), sample


# ------------------------------------------------------------------------------------------------
# algorithmic work per kernel: counted from the method's definition, never from the
# instructions the kernels issue (monomial generation, padding and masking are not useful work)
def ranks(p: int):
    K = (2 * p + 1) * (2 * p + 2) * (2 * p + 3) // 6  # raw moments |γ| <= 2p
    L = (p + 1) * (p + 2) * (p + 3) // 6              # basis size 𝓛
    return K, L


def projected_points(t, L: int, max_depth: int) -> int:
    """Points whose child-frame projection K6 computes in one build, from the exported tree: blocks of
    non-deferred nodes that may become children (n_o >= 𝓛, depth+1 <= max_depth; the kernel's guard),
    plus, for nodes whose projections were deferred (flag bit 3), the children actually created
    (the K6_PROJ pass)."""
    ex = t.export()
    cc, child = ex["child_count"], ex["child"]
    pot = (cc >= L) & ((ex["depth"] + 1) <= max_depth)[:, None]
    deferred = (ex["flags"] & 8) != 0
    proj = np.where(deferred[:, None], np.where(child >= 0, cc, 0), np.where(pot, cc, 0))
    return int(proj.sum())


def kernel_work(cfg, levels_points, depth_max: int, projected=None, units=None):
    """Per-step algorithmic work of the main kernels: (unit, amount) — flops or bytes.
    ``units``: per-kernel work units the library counted in the timed region (fmi_profile_units),
    divided by the number of steps — the sort passes and solved nodes actually executed."""
    K, L = ranks(cfg.degree)
    N, M = cfg.n, cfg.m
    pts = [int(x) for x in levels_points]
    units = units or {}
    if projected is None:  # every point of every level projected (upper bound)
        projected = sum(pts)
    w = {
        # K4: one FMA per raw moment per point, once per build (owner pass)
        "moments": ("flop", 2 * K * N),
        # K6 per level: Horner (𝓛 FMA) + Σr² (1 FMA) per point, child projection (𝓛 FMA) per point
        # of a block that may become a child (deferred blocks: only those that did)
        "residual": ("flop", sum(n * (2 * L + 2) for n in pts) + 2 * L * projected),
        # K6 root mode (single GPU: fused with the Morton-order gather): projection of f onto the root
        # frame (𝓛 FMA per point)
        "project": ("flop", 2 * L * N),
        # K7: one Horner of the pre-summed polynomial per query
        "eval": ("flop", 2 * L * M),
        # gather (sharded builds; fused into "project" on one GPU): perm (4 B) + record (32 B) read,
        # 4 SoA doubles (32 B) written
        "gather": ("byte", 68 * N),
    }
    if "sort" in units:   # bytes of the 8-bit passes actually executed, counted by the library: per item the key
        # read by the histogram + key and index read and written by the scatter (32 B with 64-bit keys,
        # 20 B with the 32-bit sort keys)
        w["sort"] = ("byte", units["sort"])
    if "keys" in units:   # bytes counted per launch by the library (coordinates, values, keys, records)
        w["keys"] = ("byte", units["keys"])
    if "solve" in units:  # bordered Cholesky 𝓛³/3 + substitutions and assembly 3𝓛² per factored node
        w["solve"] = ("flop", units["solve"] * (L ** 3 / 3 + 3 * L * L))
    return w


# Kernels whose launches are bracketed by events inside the timed region (the ones kernel_work gives a
# roofline; "gather" only launches on sharded builds).  Events around all ~200 launches of a step slow the
# host launch path of the many small per-level kernels: cfg 5 120.7 -> 122.7 ms/step.
ROOFLINED = ("moments", "residual", "project", "eval", "gather", "sort", "keys", "solve")
EXTRA_PROFILED_STEPS = 2


def rooflines(cfg, levels_points, depth_max, prof, steps, ms_per_step, hbm_peak, projected=None, units=None,
              traffic=None):
    out = {}
    per_step_units = {k: v / steps for k, v in (units or {}).items() if v}
    for name, (unit, work) in kernel_work(cfg, levels_points, depth_max, projected, per_step_units).items():
        ms, n = prof.get(name, (0.0, 0))
        if not n or ms <= 0:
            continue
        launches = n / steps
        per_launch = work / launches
        mean_s = (ms / n) / 1e3
        if unit == "flop":
            achieved, peak, u, bound = per_launch / mean_s / 1e12, FP64_PEAK_TFLOPS, "TFLOP/s", "alu"
        else:
            achieved, peak, u, bound = per_launch / mean_s / 1e9, hbm_peak, "GB/s", "hbm"
        out[name] = {"bound": bound, "achieved": achieved, "peak": peak, "unit": u, "frac": achieved / peak,
                     "traffic": None, "work_per_launch": per_launch, "launches_per_step": launches,
                     "mean_launch_ms": ms / n, "share_of_step": (ms / steps) / ms_per_step}
        t = (traffic or {}).get(name)
        if t:
            out[name]["traffic"] = t["dram_bytes_per_launch"]
            out[name]["traffic_note"] = t["source"]
    return out


def load_traffic(cfg) -> dict:
    """Per-kernel DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the committed
    ncu capture of this config (profiles/traffic_cfg<c>.json, written by tools/ncu_traffic.py with the
    capture file and commit it came from); {} if there is none."""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_cfg{cfg.cfg}.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def run_reference(args, cfg, rank, world):
    """The base contract's reference arm for this tier: the oracle (oracle/fmt_oracle.py, CPU, as it stands)
    timed on this host's cores, each step a bounded sample of the workload (time_oracle_sample)."""
    if rank != 0:
        return
    pts, f, q = workloads.make_inputs(cfg)
    target = 60_000
    times, vals = [], []
    for i in range(args.warmup + args.steps):
        v, dt, cores, sample = time_oracle_sample(cfg, pts, f, q, target, seed=i)
        if i >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = statistics.median(vals)
    t = statistics.median(times)
    line = {
        "impl": "reference", "metric": "fp64 octree fit + eval points/sec", "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: N={cfg.n:,} M={cfg.m:,} p={cfg.degree} max_depth={cfg.max_depth} "
                               f"tol={cfg.tol:g} ({cfg.points}/{cfg.values})"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "host_cores": host_cores(), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-run this command under torch.distributed.run with N ranks
    (the driver's own launch line), so that N processes, one per GPU, are always what is measured."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    cfg = workloads.CONFIGS[args.config]
    if args.n or args.m:
        cfg = cfg.scaled(n=args.n, m=args.m)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1511_01353_b200 as fmi

    if os.environ.get("FMI_BENCH_ONE_DEVICE"):  # functional multi-rank check on one GPU (not a measurement)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("FMI_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    fmi.set_stream(stream)

    t_gen = time.perf_counter()
    pts, f, q = workloads.make_inputs(cfg)
    gen_s = time.perf_counter() - t_gen
    N, M = cfg.n, cfg.m
    pts_all, f_all, q_all = pts, f, q
    if world > 1:  # this rank's slice of the global workload (the sharded build exchanges by cell)
        pts, f = pts[rank * N // world:(rank + 1) * N // world], f[rank * N // world:(rank + 1) * N // world]
        q = q[rank * M // world:(rank + 1) * M // world]
        pts, f, q = (np.ascontiguousarray(a) for a in (pts, f, q))
    d_pts = torch.from_numpy(pts).to(dev)
    d_f = torch.from_numpy(f).to(dev)
    d_q = torch.from_numpy(q).to(dev)
    d_out = torch.empty(q.shape[0], dtype=torch.float64, device=dev)
    comm = None
    if world > 1:
        from paper_1511_01353_b200 import shard
        comm = shard.TorchComm()

    class _Step:
        """one step: build + eval + free (sharded over the ranks when world > 1)"""

        def build(self, p, ff):
            if comm is None:
                return fmi.build(p, ff, cfg.degree, cfg.tol, cfg.max_depth)
            return shard.build_sharded(p, ff, cfg.degree, cfg.tol, cfg.max_depth, comm)

    stepper = _Step()

    def tree_of(t):
        return t if comm is None else t.tree

    def step_device():
        tree = stepper.build(d_pts, d_f)
        tree.eval(d_q, out=d_out)
        return tree

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warm-up (also the tree statistics used for the roofline)
    tree = None
    for _ in range(args.warmup):
        if tree is not None:
            tree.free()
        tree = step_device()
    levels_nodes, levels_points = tree_of(tree).level_stats()
    node_count = tree_of(tree).node_count
    proj_pts = projected_points(tree_of(tree), ranks(cfg.degree)[1], cfg.max_depth)
    shard_depth = getattr(tree, "shard_depth", None)
    tree.free()

    # ---- timed region: device-resident inputs ------------------------------------------------
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    build_ms = []
    fmi.profile_reset()
    fmi.profile_select(ROOFLINED)  # events only around the kernels with a roofline (see ROOFLINED)
    fmi.profile_enable(True)
    launches0 = fmi.launch_count()
    barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            e_s = torch.cuda.Event(enable_timing=True)
            e_s.record(stream)
            tree = stepper.build(d_pts, d_f)
            ev_b.record(stream)
            tree.eval(d_q, out=d_out)
            tree.free()
            torch.cuda.synchronize(dev)
            build_ms.append(e_s.elapsed_time(ev_b))
        ev1.record(stream)
        barrier()
    launches = fmi.launch_count() - launches0
    fmi.profile_enable(False)
    prof = fmi.profile_get()
    units = fmi.profile_units()
    total_ms = ev0.elapsed_time(ev1)
    # untimed extra pass with events around EVERY launch: the device time of the remaining (small) kernels
    # for kernels_ms_per_step / kernel_time_fraction; nothing of it enters value, ms_per_step or the rooflines
    fmi.profile_reset()
    fmi.profile_select(None)
    fmi.profile_enable(True)
    for _ in range(EXTRA_PROFILED_STEPS):
        tree = stepper.build(d_pts, d_f)
        tree.eval(d_q, out=d_out)
        tree.free()
    barrier()
    fmi.profile_enable(False)
    prof_all = fmi.profile_get()
    kernels_ms = {k: v[0] / EXTRA_PROFILED_STEPS for k, v in prof_all.items() if v[1]}
    kernels_ms.update({k: v[0] / args.steps for k, v in prof.items() if v[1]})  # the timed region's own
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = (N + M) / (ms_per_step / 1e3)  # the global workload (all ranks together)
    build_pts_s = N / (statistics.median(build_ms) / 1e3)
    eval_pts_s = M / ((ms_per_step - statistics.median(build_ms)) / 1e3)

    # rooflines: algorithmic work per launch / mean launch time (library events on the launching
    # stream, inside the timed region); the dominant kernel is the bench line's "roofline"
    pt_levels = int(np.sum(levels_points))
    hbm_peak = measured_hbm_peak()
    roofs = rooflines(cfg, levels_points, len(levels_points) - 1, prof, args.steps, ms_per_step, hbm_peak,
                      proj_pts, units, load_traffic(cfg) if world == 1 else None)
    dominant = max(roofs, key=lambda k: roofs[k]["share_of_step"]) if roofs else None
    # correctness of the timed step's output: interpolation error against the analytic function on a
    # sample of this rank's queries, next to the oracle-parity tests (tests/test_gpu_*.py)
    out_host = d_out.cpu().numpy()
    chk = np.random.default_rng(0).choice(q.shape[0], size=min(q.shape[0], 1_000_000), replace=False)
    e_rms, e_inf = workloads.rms_and_max(out_host[chk] - workloads.exact_values(cfg, q[chk]))
    step_kernel_ms = sum(kernels_ms.values())

    # ---- e2e through the C ABI with pinned host buffers -----------------------------------------
    h_pts = torch.from_numpy(pts).pin_memory()
    h_f = torch.from_numpy(f).pin_memory()
    h_q = torch.from_numpy(q).pin_memory()
    h_out = torch.empty(q.shape[0], dtype=torch.float64).pin_memory()
    np_pts, np_f, np_q, np_out = h_pts.numpy(), h_f.numpy(), h_q.numpy(), h_out.numpy()

    def e2e_step():
        if comm is None:  # host pointers through the C ABI (fmi_transfer = build + eval): the
            # library uploads the points, the fit runs while the queries upload on a side stream, then
            # the values come back — every byte crosses PCIe inside the timed call
            fmi.transfer(np_pts, np_f, np_q, cfg.degree, cfg.tol, cfg.max_depth, out=np_out)
        else:             # sharded: this rank's host slice -> device, sharded build, routed eval -> host
            tp, tf, tq = (h.to(dev, non_blocking=True) for h in (h_pts, h_f, h_q))
            tr = stepper.build(tp, tf)
            h_out.copy_(tr.eval(tq))
            tr.free()

    for _ in range(args.warmup):  # untimed: first-call costs of the host-buffer paths (streams, modules)
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    e2e_step_ms = []  # per-step host wall clock (visibility of host-side jitter on the short configs)
    for _ in range(args.steps):
        ts = time.perf_counter()
        e2e_step()
        e2e_step_ms.append(round((time.perf_counter() - ts) * 1e3, 3))
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = (N + M) / e2e_s
    gpu_out_max = float(np.max(np.abs(np_out)))

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, dt, cores, sample = time_oracle_sample(cfg, pts_all, f_all, q_all, 400_000)
            cpu = {"value": v, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample,
                   "seconds": dt, "host_cores": host_cores(), "cpu_model": cpu_model()}
        line = {
            "metric": "fp64 octree fit + eval points/sec",
            "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"{cfg.name}: N={N:,} M={M:,} p={cfg.degree} max_depth={cfg.max_depth} tol={cfg.tol:g} "
                            f"({cfg.points} points, {cfg.values} values)",
                "parallelism": (f"sharded x{world}: Morton cells of depth {shard_depth} per rank, global nodes "
                                f"of depth < {shard_depth} summed by NCCL allreduce") if world > 1 else "single-gpu",
                "l2": (f"inputs {(N * 32 + M * 24) / 1e9:.2f} GB vs 126 MB L2: "
                       + ("no flush needed" if N * 32 + M * 24 > 2e9 else "the step's own 40 B/point/level "
                          "passes evict the inputs (no explicit flush)")),
                "nodes": node_count, "levels": len(levels_nodes), "point_levels": pt_levels,
                "projected_points": proj_pts,
                "build_points_per_s": build_pts_s, "eval_points_per_s": eval_pts_s,
                "build_ms_per_step": [round(x, 3) for x in build_ms],
                "input_gen_s": gen_s,
            },
            "roofline": dict(kernel=dominant, **roofs[dominant], peak_source=PEAK_SOURCE) if dominant else None,
            "rooflines": roofs,
            "kernels_ms_per_step": dict(sorted(kernels_ms.items())),
            "kernels_ms_note": (f"{', '.join(ROOFLINED)}: library events inside the timed region; the other kernels: "
                                f"{EXTRA_PROFILED_STEPS} extra untimed steps with events around every launch"),
            "kernel_time_fraction": step_kernel_ms / ms_per_step,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "points/s",
                    "h2d_bytes_per_step": N * 24 + N * 8 + M * 24, "d2h_bytes_per_step": M * 8,
                    "note": ("host wall clock around K steps of fmi_transfer with pinned host buffers (H2D of "
                             "points, values, queries and D2H of the values inside the call; the query upload "
                             "overlaps the fit), max over ranks") if world == 1 else
                            "host wall clock around K steps (H2D of points, values, queries and D2H of the values "
                            "inside), max over ranks",
                    "step_ms": e2e_step_ms},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "check": {"queries": int(chk.size), "e_rms_vs_exact": e_rms, "e_inf_vs_exact": e_inf,
                      "max_abs_out_e2e": gpu_out_max},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
