# p = 12 sweep-point diagnostics + per-launch K5 times at cfg 3/4/5 (FMI_PROF_LOG)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/diag_sweep.py --p 12 --log8n 4 --tau 1e-6 > gpurun_out/r2_diag_p12.log 2>&1; echo "diag rc=$?"
for c in 3 4 5; do
  FMI_PROF_LOG=1 timeout 300 python tools/run_build.py --config $c --m 1000 --reps 2 --profile > gpurun_out/r2_launch_cfg$c.log 2>&1
  echo "cfg$c rc=$?"
done
