mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r1j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r1j.log
done
