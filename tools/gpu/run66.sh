mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 3 4; do for v in 1000 5000 100000000; do
  export FMI_K5_SMALL=$v
  timeout 600 python tools/run_build.py --config $c --reps 3 --profile > gpurun_out/run_cfg${c}_k5s${v}.log 2>&1
  echo "== cfg$c small=$v $(grep -o 'build [0-9.]* ms eval [0-9.]* ms' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1) $(grep -o '"solve": [0-9.]*' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1) $(grep -o '"refine_solve": [0-9.]*' gpurun_out/run_cfg${c}_k5s${v}.log | tail -1)" >> gpurun_out/k5s2_summary.log
done; done
