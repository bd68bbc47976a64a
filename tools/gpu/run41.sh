mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5_r1f.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r1f.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_r1f.log 2>&1
