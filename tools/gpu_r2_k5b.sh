# new GPU tests (NCCL world-1 communicator, loader validation, shards) + K5 launch-shape experiments
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_api.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r2_shard_api.log 2>&1
echo "shard/api rc=$?" >> gpurun_out/r2_shard_api.log; tail -4 gpurun_out/r2_shard_api.log
: > gpurun_out/r2_k5b.log
for c in 3 4 5; do
 for v in "FMI_K5_TINY=0" "FMI_K5_TINY=148" "FMI_K5_TINY=148 FMI_K5_CTAS_PER_SM=1" "FMI_K5_TINY=600"; do
  echo "cfg$c $v" >> gpurun_out/r2_k5b.log
  env $v timeout 300 python tools/run_build.py --config $c --m 1000 --reps 3 --profile 2>&1 | grep -o '"solve": [0-9.]*\|"refine_solve": [0-9.]*\|build [0-9.]* ms' | tail -3 | tr '\n' ' ' >> gpurun_out/r2_k5b.log
  echo >> gpurun_out/r2_k5b.log
 done
done
cat gpurun_out/r2_k5b.log
