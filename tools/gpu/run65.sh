mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size > gpurun_out/pytest_r65.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r65.log
for c in 3 4 5; do for v in 0 def; do
  if [ $v = def ]; then unset FMI_K5_SMALL; else export FMI_K5_SMALL=$v; fi
  timeout 600 python tools/run_build.py --config $c --reps 3 --profile > gpurun_out/run_cfg${c}_k5s${v}.log 2>&1
  echo "== cfg$c small=$v $(grep -o 'build [0-9.]* ms eval [0-9.]* ms' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1) $(grep -o '"solve": [0-9.]*' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1) $(grep -o '"refine_solve": [0-9.]*' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1)" >> gpurun_out/k5s_summary.log
done; done
unset FMI_K5_SMALL
