# CholeskyQR2 pass on the QR path: the p = 12 sweep point diagnostics + sweep/unscoped suites
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/diag_sweep.py --p 12 --log8n 4 --tau 1e-6 > gpurun_out/r2_diag_p12_qr2.log 2>&1; echo "diag rc=$?"
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_unscoped.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_qr2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_qr2_tests.log; tail -5 gpurun_out/r2_qr2_tests.log
