mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/microbench/fp64_peak.cu && timeout 120 /tmp/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 3 4; do timeout 300 python tools/run_build.py --config $c --reps 3 > gpurun_out/run_cfg$c.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5.log
