mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v39.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v39.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_v39.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_moments$" -c 1 python tools/run_build.py --config 5 > gpurun_out/ncu_k4_v39.log 2>&1
