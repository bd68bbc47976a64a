mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r1.log
done
