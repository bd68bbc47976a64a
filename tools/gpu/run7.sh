mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v7.log
timeout 300 python tools/run_build.py --config 3 --reps 3 --profile > gpurun_out/run_cfg3_v7.log 2>&1
timeout 300 python tools/run_build.py --config 4 --reps 3 --profile > gpurun_out/run_cfg4_v7.log 2>&1
timeout 600 python tools/run_build.py --config 5 --reps 3 --profile > gpurun_out/run_cfg5_v7.log 2>&1
