mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_full_v3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_v3.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v3.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_v3.log
