mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v29.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v29.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v29.log 2>&1
