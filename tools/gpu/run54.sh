mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_unscoped.py -q -x > gpurun_out/pytest_unscoped_v8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_unscoped_v8.log
timeout 900 python tools/fig1.py --log8n 6 --degrees 6 10 14 --oracle 5000 > gpurun_out/fig1_v8.jsonl 2> gpurun_out/fig1_v8.err
FMI_UNSCOPED_QR=1 timeout 900 python tools/fig1.py --log8n 6 --degrees 6 10 --oracle 5000 > gpurun_out/fig1_qr_v8.jsonl 2>> gpurun_out/fig1_v8.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fig1_launches_v8.csv python tools/fig1.py --log8n 6 --degrees 14 --reps 1 > /dev/null 2>&1
