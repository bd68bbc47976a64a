mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5_r1e.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r1e.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1e.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r1e.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_r1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_residual$" -s 4 -c 1 -o gpurun_out/k6_r1e -f python tools/run_build.py --config 5 > gpurun_out/ncu_k6_r1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_moments$" -c 1 -o gpurun_out/k4_r1e -f python tools/run_build.py --config 5 > gpurun_out/ncu_k4_r1e.log 2>&1
