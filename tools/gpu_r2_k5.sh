# golden full-size tests for cfg4/cfg5 + K5 experiments (persistent CTAs per SM) + ncu of the level-4 k_solve (cfg5)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_golden.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r2_golden.log 2>&1
echo "golden rc=$?" >> gpurun_out/r2_golden.log; tail -12 gpurun_out/r2_golden.log
for c in 3 4 5; do
 for k in 0 1 2 3; do
  if [ $k = 0 ]; then unset FMI_K5_CTAS_PER_SM; else export FMI_K5_CTAS_PER_SM=$k; fi
  echo "cfg$c ctas/sm=$k" >> gpurun_out/r2_k5grid.log
  timeout 300 python tools/run_build.py --config $c --m 1000 --reps 3 --profile 2>&1 | grep -o '"solve": [0-9.]*\|"refine_solve": [0-9.]*\|build [0-9.]* ms' | tail -3 >> gpurun_out/r2_k5grid.log
 done
done
unset FMI_K5_CTAS_PER_SM
cat gpurun_out/r2_k5grid.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve --launch-skip 4 --launch-count 1 -o gpurun_out/r2_k5_cfg5_l4 python tools/run_build.py --config 5 --m 1000 > gpurun_out/r2_k5_ncu.log 2>&1
echo "ncu rc=$?"
