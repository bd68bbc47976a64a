# round-2 GPU check: full GPU test suite (incl. the golden full-size comparisons) + cfg5 bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
tail -3 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_cfg5.jsonl 2> gpurun_out/r2_bench_cfg5.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_cfg5.jsonl
