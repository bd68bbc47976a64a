mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r67.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r67.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r67.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r67.log
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r67.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r67.log
done
