mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_api.py -q -x > gpurun_out/pytest_api_v2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_api_v2.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_v2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_e2e_v2.log
