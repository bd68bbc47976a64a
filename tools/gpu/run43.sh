mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 3 4; do
  timeout 600 python tools/run_build.py --config $c --reps 3 --profile > gpurun_out/run_cfg${c}_v57.log 2>&1
  FMI_TRACE=1 timeout 600 python tools/run_build.py --config $c --reps 2 > gpurun_out/trace_cfg${c}_v57.log 2>&1
done
