mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in 0 32 64 0 32; do
  FMI_L2_FETCH=$v timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_l2f${v}.log 2>&1
  echo "== $v" >> gpurun_out/l2f_summary.log
  grep -o "build [0-9.]* ms eval [0-9.]* ms" gpurun_out/run_cfg5_l2f${v}.log | tail -1 >> gpurun_out/l2f_summary.log
  grep -o '"[a-z_]*": [0-9.]*' gpurun_out/run_cfg5_l2f${v}.log | tail -18 | tr '\n' ' ' >> gpurun_out/l2f_summary.log; echo >> gpurun_out/l2f_summary.log
done
FMI_L2_FETCH=32 timeout 900 ncu --set full --clock-control none -k regex:"^k_gather_root$" -c 1 -o gpurun_out/gr_l2f32 -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_gr_l2f32.log 2>&1
