mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_residual$" --csv --log-file gpurun_out/k6_traffic_r1g.csv python tools/run_build.py --config 5 --reps 1 > gpurun_out/k6_traffic_r1g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_residual$" -s 7 -c 2 -o gpurun_out/k6_r1g -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k6_r1g.log 2>&1
