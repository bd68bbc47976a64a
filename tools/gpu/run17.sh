mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
for k in k_m2m k_gather k_eval; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}\$" -c 1 -o gpurun_out/${k}_v20 -f python tools/run_build.py --config 5 > gpurun_out/ncu_${k}_v20.log 2>&1
done
