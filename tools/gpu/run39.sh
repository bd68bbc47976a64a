mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
FMI_BENCH_BACKEND=gloo FMI_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --config 3 > gpurun_out/bench_mr2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_mr2.log
