mkdir -p gpurun_out
set -x
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_mix tools/microbench/fp64_mix.cu && timeout 120 /tmp/fp64_mix > gpurun_out/fp64_mix.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v2.log
for c in 3 4; do timeout 300 python tools/run_build.py --config $c --reps 3 > gpurun_out/run_cfg${c}_v2.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_v2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_v2.log
