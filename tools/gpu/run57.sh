mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r1k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r1k.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_r1k.log 2>&1
for c in 5 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r1k.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r1k.log
done
