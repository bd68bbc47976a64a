mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for nc in 1 0; do
  if [ $nc = 1 ]; then export FMI_BENCH_NO_CLOCKS=1; else unset FMI_BENCH_NO_CLOCKS; fi
  timeout 900 python bench.py --config 4 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_nc$nc.log 2>&1
done
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; free -g >> gpurun_out/nvsmi.txt; nproc >> gpurun_out/nvsmi.txt; uptime >> gpurun_out/nvsmi.txt
