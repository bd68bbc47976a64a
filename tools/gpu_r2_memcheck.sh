set -x
nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
tail -5 gpurun_out/r2_memcheck.log
