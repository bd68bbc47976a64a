"""Per-kernel DRAM traffic of one config's build + eval (the bench step), for bench.py's roofline `traffic`.

python tools/ncu_traffic.py CONFIG   (on the GPU box; runs ncu over tools/run_build.py --config CONFIG)

Every launch of the library's main kernels is profiled with dram__bytes_read.sum + dram__bytes_write.sum
(clock control off); launches are grouped by the library's kernel ids (the names of fmi_profile_get /
the bench line's `kernels_ms_per_step`) and written as bytes per launch to profiles/traffic_cfg<C>.json
with the command and the commit they came from.  The numbers of a run under ncu are not timings."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# CUDA kernel name prefix -> library kernel id (csrc/fmi_internal.cuh KID_*)
KIDS = [("k_residual_reduce", None), ("k_residual", "residual"), ("k_moments_reduce", None), ("k_moments", "moments"),
        ("k_solve_qr", None), ("k_solve", "solve"), ("k_gather_root", "project"), ("k_eval", "eval"),
        ("k_rs_", "sort"), ("k_bk_", "keys"), ("k_keys", "keys")]


def kid_of(name: str):
    base = name.split("(")[0].split("<")[0].split("::")[-1].strip()
    for pre, kid in KIDS:
        if base.startswith(pre):
            return kid
    return None


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "--csv",
           "-k", "regex:^(k_residual|k_moments|k_solve|k_gather_root|k_eval|k_rs_|k_bk_|k_keys)",
           sys.executable, os.path.join(ROOT, "tools", "run_build.py"), "--config", str(cfg)]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    lines = out[out.index('"ID"'):] if '"ID"' in out else ""
    rows = list(csv.DictReader(io.StringIO(lines)))
    per = collections.defaultdict(dict)  # launch id -> metric -> bytes
    names = {}
    for r in rows:
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        per[r["ID"]][r["Metric Name"]] = v * scale
        names[r["ID"]] = r["Kernel Name"]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for lid, m in per.items():
        kid = kid_of(names[lid])
        if kid:
            agg[kid][0] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            agg[kid][1] += 1
    commit = os.environ.get("FMI_COMMIT") or subprocess.run(
        ["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True, cwd=ROOT).stdout.strip() or "?"
    src = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over tools/run_build.py --config {cfg} "
           f"(tools/ncu_traffic.py, tree of commit {commit})")
    res = {k: {"dram_bytes_per_launch": b / n, "launches": n, "source": src} for k, (b, n) in sorted(agg.items())}
    path = os.path.join(ROOT, "profiles", f"traffic_cfg{cfg}.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
