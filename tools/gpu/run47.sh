mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_K6_SPLIT=1 timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:"k_residual$" --csv --log-file gpurun_out/k6split_launches.csv python tools/run_build.py --config 5 --reps 1 > gpurun_out/k6split_ncu.log 2>&1
