mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
FMI_TRACE=1 timeout 600 python tools/run_build.py --config 5 --reps 4 > gpurun_out/trace1_cfg5.log 2>&1
FMI_TRACE=2 timeout 600 python tools/run_build.py --config 5 --reps 2 > gpurun_out/trace2_cfg5.log 2>&1
FMI_TRACE=2 timeout 600 python tools/run_build.py --config 3 --reps 3 > gpurun_out/trace2_cfg3.log 2>&1
