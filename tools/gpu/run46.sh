mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for sp in 1; do
  for c in 5; do
    FMI_K6_SPLIT=$sp timeout 600 python tools/run_build.py --config $c --reps 2 --profile > gpurun_out/k6split_${sp}_cfg${c}.log 2>&1
  done
done
