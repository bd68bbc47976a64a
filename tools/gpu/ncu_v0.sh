mkdir -p gpurun_out
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moments -c 2 -o gpurun_out/k4_v0 -f python tools/run_build.py --config 5 --n 20000000 --m 100000 > gpurun_out/ncu_k4_v0.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v0.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_v0.log 2>&1
echo done
