mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size > gpurun_out/pytest_v67.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v67.log
for c in 4 3; do
  timeout 900 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg${c}_v67.log 2>&1
done
