mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for mf in 2 4 8 16; do
  for c in 5 4 3; do
    FMI_MT_FILL=$mf timeout 600 python tools/run_build.py --config $c --reps 2 > gpurun_out/mtfill_${mf}_cfg${c}.log 2>&1
  done
done
