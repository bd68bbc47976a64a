mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5_r1h.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r1h.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1h.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r1h.log
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_r1h.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg${c}_r1h.log
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_r1h.log 2>&1
