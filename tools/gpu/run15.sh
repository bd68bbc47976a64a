mkdir -p gpurun_out
set -x
export PYTHONUNBUFFERED=1
FMI_BENCH_BACKEND=gloo FMI_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 3 --steps 2 --warmup 1 > gpurun_out/bench_n2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_gloo.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --config 3 --steps 1 --warmup 1 > gpurun_out/bench_n2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_ref.log
