mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_unscoped.py -q -x > gpurun_out/pytest_unscoped_v5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_unscoped_v5.log
