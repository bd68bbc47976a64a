mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 -o gpurun_out/k6_v4 -f python tools/run_build.py --config 5 --n 20000000 --m 1000000 > gpurun_out/ncu_k6_v4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 4 -c 1 -o gpurun_out/k5_v4 -f python tools/run_build.py --config 5 --n 20000000 --m 1000000 > gpurun_out/ncu_k5_v4.log 2>&1
