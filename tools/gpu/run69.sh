mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_cfg5_r69.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r69.log
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r69.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r69.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r69.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r69.log
