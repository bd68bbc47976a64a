mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_TRACE=1 timeout 900 python tools/run_build.py --config 4 --reps 10 > gpurun_out/trace_cfg4_reps.log 2>&1
