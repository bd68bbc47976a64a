# round-2 final measurements: full GPU suite, smoke, bench lines (cfg5 default + cfg1-4), the reference arm,
# per-kernel DRAM traffic (tools/ncu_traffic.py) and the ncu launch list of the bench command.
# usage (here): gpurun -- "FMI_COMMIT=$(git rev-parse --short HEAD) bash tools/gpu_r2_final.sh TAG"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
tag=${1:-final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python tools/ncu_traffic.py 5 > gpurun_out/${tag}_traffic.log 2>&1; echo "traffic rc=$?"
cp profiles/traffic_cfg5.json gpurun_out/traffic_cfg5.json 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_cfg5.jsonl 2> gpurun_out/${tag}_bench_cfg5.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${tag}_bench_cfg5.jsonl
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${tag}_bench_cfg$c.jsonl 2>> gpurun_out/${tag}_bench_cfg5.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_bench_reference.jsonl 2>> gpurun_out/${tag}_bench_cfg5.err
echo "reference rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_launches_cfg5.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "launch list rc=$?"
