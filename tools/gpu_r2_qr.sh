# QR path on the octree (p = 11, 12 and FMI_QR_PATH), unscoped regression, sweep spot checks, golden cfg4/cfg5,
# then the f3 sweep at the paper's orders (L_max = 4, 8, 12; N up to 8^9)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_unscoped.py tests/test_gpu_sweep.py tests/test_gpu_golden.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_qr_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_qr_tests.log; tail -15 gpurun_out/r2_qr_tests.log
timeout 2400 python tools/sweep.py > gpurun_out/r2_sweep_f3.jsonl 2> gpurun_out/r2_sweep_f3.err
echo "sweep rc=$?"; wc -l gpurun_out/r2_sweep_f3.jsonl; tail -3 gpurun_out/r2_sweep_f3.err
