# compute-sanitizer memcheck over every kernel family (tools/sanitize_run.py) + eval kernel A/B at cfg 5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 1 0; do
  echo "FMI_EVAL_PIPE=$v" >> gpurun_out/r2_eval_ab.log
  FMI_EVAL_PIPE=$v timeout 300 python tools/run_build.py --config 5 --reps 3 --profile 2>&1 | grep -o '"eval": [0-9.]*\|eval [0-9.]* ms' | tail -2 | tr '\n' ' ' >> gpurun_out/r2_eval_ab.log
  echo >> gpurun_out/r2_eval_ab.log
done
cat gpurun_out/r2_eval_ab.log
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
tail -12 gpurun_out/r2_memcheck.log
