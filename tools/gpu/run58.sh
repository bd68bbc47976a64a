mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_TRACE=1 timeout 900 python bench.py --config 4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_trace.log 2> gpurun_out/bench_cfg4_trace.err
