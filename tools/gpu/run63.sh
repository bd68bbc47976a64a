mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_gather_root$" -c 1 -o gpurun_out/gr_r1k -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_gr_r1k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_solve$" -c 3 -o gpurun_out/k5_cfg4_r1k -f python tools/run_build.py --config 4 --reps 1 > gpurun_out/ncu_k5_cfg4_r1k.log 2>&1
