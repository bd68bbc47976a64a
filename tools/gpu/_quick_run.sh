mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size > gpurun_out/pytest_v94.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v94.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v94.log 2>&1
