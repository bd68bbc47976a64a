mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r71.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r71.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r71.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r71.log
timeout 900 python bench.py > gpurun_out/bench_cfg5_r71.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r71.log
