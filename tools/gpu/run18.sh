mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for fill in 8 3 1.5 0; do
  echo "== fill $fill" >> gpurun_out/refine_sweep.log
  FMI_REFINE_FILL=$fill timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size 2>&1 | tail -n 8 >> gpurun_out/refine_sweep.log
  FMI_REFINE_FILL=$fill timeout 300 python tools/run_build.py --config 4 --reps 2 --profile 2>&1 | tail -n 2 >> gpurun_out/refine_sweep.log
  FMI_REFINE_FILL=$fill timeout 300 python tools/run_build.py --config 3 --reps 2 --profile 2>&1 | tail -n 2 >> gpurun_out/refine_sweep.log
done
