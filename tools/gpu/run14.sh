mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_v17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v17.log
