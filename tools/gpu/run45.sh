mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for th in 1 1e300; do
  FMI_DEFER_THETA=$th timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/split_th${th}.log 2>&1
done
