# K5 global kernel (p = 10): parity suite + cfg 5 solve time
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_k5g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_k5g_tests.log; tail -2 gpurun_out/r2_k5g_tests.log
timeout 300 python tools/run_build.py --config 5 --m 1000 --reps 3 --profile 2>&1 | grep -o '"solve": [0-9.]*\|build [0-9.]* ms' | tail -2 | tee gpurun_out/r2_k5g_times.log
