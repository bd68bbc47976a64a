# K5 shared-memory-resident variant: parity suites + solve times at cfg 3/4 (resident vs global kernel)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_k5res_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_k5res_tests.log; tail -3 gpurun_out/r2_k5res_tests.log
: > gpurun_out/r2_k5res_times.log
for c in 2 3 4; do
 for v in 1 0; do
  echo "cfg$c FMI_K5_RES=$v" >> gpurun_out/r2_k5res_times.log
  FMI_K5_RES=$v timeout 300 python tools/run_build.py --config $c --m 1000 --reps 3 --profile 2>&1 | grep -o '"solve": [0-9.]*\|"refine_solve": [0-9.]*\|build [0-9.]* ms' | tail -3 | tr '\n' ' ' >> gpurun_out/r2_k5res_times.log
  echo >> gpurun_out/r2_k5res_times.log
 done
done
cat gpurun_out/r2_k5res_times.log
