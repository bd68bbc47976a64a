mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size > gpurun_out/pytest_gpu_v26.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v26.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v26.log 2>&1
timeout 300 python tools/run_build.py --config 4 --reps 2 --profile > gpurun_out/run_cfg4_v26.log 2>&1
FMI_TRACE=2 timeout 300 python tools/run_build.py --config 4 --reps 2 > gpurun_out/trace_cfg4_v26.log 2>&1
timeout 300 python tools/run_build.py --config 3 --reps 2 --profile > gpurun_out/run_cfg3_v26.log 2>&1
