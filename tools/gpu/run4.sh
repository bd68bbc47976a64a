mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v5.log
for c in 3 4; do timeout 300 python tools/run_build.py --config $c --reps 3 > gpurun_out/run_cfg${c}_v5.log 2>&1; done
timeout 600 python tools/run_build.py --config 5 --reps 2 > gpurun_out/run_cfg5_v5.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_v5.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_v5.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_residual<" -s 3 -c 1 -o gpurun_out/k6_v5 -f python tools/run_build.py --config 5 --n 20000000 --m 1000000 > gpurun_out/ncu_k6_v5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_solve<" -s 4 -c 1 -o gpurun_out/k5_v5 -f python tools/run_build.py --config 5 --n 20000000 --m 1000000 > gpurun_out/ncu_k5_v5.log 2>&1
