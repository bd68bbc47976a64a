mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/fig1.py --log8n 6 --degrees 6 10 14 --oracle 5000 > gpurun_out/fig1_v1.jsonl 2> gpurun_out/fig1_v1.err
FMI_UNSCOPED_QR=1 timeout 900 python tools/fig1.py --log8n 6 --degrees 6 10 --oracle 5000 > gpurun_out/fig1_qr_v1.jsonl 2>> gpurun_out/fig1_v1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fig1_launches_v1.csv python tools/fig1.py --log8n 6 --degrees 14 --reps 1 > /dev/null 2>&1
