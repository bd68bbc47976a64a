mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_BENCH_BACKEND=gloo FMI_BENCH_ONE_DEVICE=1 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 3 --config 5 > gpurun_out/bench_mr2_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_mr2_cfg5.log
