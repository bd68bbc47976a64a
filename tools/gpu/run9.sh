mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_v12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v12.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_rs_scatter$" -c 1 -o gpurun_out/sort_v12 -f python tools/run_build.py --config 5 > gpurun_out/ncu_k4_v12.log 2>&1
