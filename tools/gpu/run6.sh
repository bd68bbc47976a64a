mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
timeout 300 python tools/run_build.py --config 3 --reps 6 --profile > gpurun_out/run_cfg3_v6.log 2>&1
timeout 600 python tools/run_build.py --config 5 --reps 3 --profile > gpurun_out/run_cfg5_v6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_moments$" -c 1 -o gpurun_out/k4_v6 -f python tools/run_build.py --config 5 > gpurun_out/ncu_k4_v6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_residual$" -s 4 -c 1 -o gpurun_out/k6_v6 -f python tools/run_build.py --config 5 > gpurun_out/ncu_k6_v6.log 2>&1
