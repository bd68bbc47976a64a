mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5_r1j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r1j.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1j.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r1j.log
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r1j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r1j.log
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1j.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_r1j.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_residual$" -s 1 -c 2 -o gpurun_out/k6_r1j -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k6_r1j.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_moments$" -c 1 -o gpurun_out/k4_r1j -f python tools/run_build.py --config 5 --reps 1 > gpurun_out/ncu_k4_r1j.log 2>&1
