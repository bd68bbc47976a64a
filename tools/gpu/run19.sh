mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_K4=batch timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_k4b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k4b.log
FMI_K4=batch timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_k4b.log 2>&1
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_k4a.log 2>&1
