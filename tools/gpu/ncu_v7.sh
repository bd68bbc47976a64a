mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_solve$" -s 8 -c 1 -o gpurun_out/k5_v7 -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k5_v7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_eval$" -c 1 -o gpurun_out/k7_v7 -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k7_v7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_syrk$" -c 1 -o gpurun_out/syrk_v7 -f python tools/fig1.py --log8n 6 --degrees 14 --reps 1 > gpurun_out/ncu_syrk_v7.log 2>&1
