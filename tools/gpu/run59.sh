mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_K4_STAGED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg2 or degree_sweep or mixture" > gpurun_out/pytest_k4b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k4b.log
FMI_K4_STAGED=1 timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/k4b_cfg5.log 2>&1
