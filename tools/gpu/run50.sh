mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for sp in 1 0; do
  FMI_K6_SPLIT=$sp timeout 900 python bench.py --config 4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_split$sp.log 2>&1
done
