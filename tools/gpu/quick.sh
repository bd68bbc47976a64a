# usage (from anywhere): bash /root/repo/tools/gpu/quick.sh TAG  -> GPU tests (minus cfg5 fullsize) + cfg5 profile run
cd "$(dirname "$0")/../.." || exit 1
TAG=$1
cat > tools/gpu/_quick_run.sh <<EOS
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_cfg5_full_size > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=\$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python tools/run_build.py --config 5 --reps 2 --profile > gpurun_out/run_cfg5_$TAG.log 2>&1
EOS
timeout 3000 /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu/_quick_run.sh' > /tmp/gpurun_$TAG.out 2>&1
tail -n 1 /tmp/gpurun_$TAG.out
tail -n 2 gpurun_out/pytest_$TAG.log
grep -o "build [0-9.]* ms eval [0-9.]* ms" gpurun_out/run_cfg5_$TAG.log | tail -1
grep -o '"[a-z_]*": [0-9.]*' gpurun_out/run_cfg5_$TAG.log | tail -18 | tr '\n' ' '; echo
