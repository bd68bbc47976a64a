mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_solve$" -s 4 -c 1 -o gpurun_out/k5_v9 -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k5_v9.log 2>&1
