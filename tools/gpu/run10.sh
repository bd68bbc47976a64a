mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_v15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v15.log
for c in 3 4; do timeout 300 python tools/run_build.py --config $c --reps 3 --profile > gpurun_out/run_cfg${c}_v15.log 2>&1; done
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v15.log 2>&1; timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_v15.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_v15.log
