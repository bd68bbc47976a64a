# round-2 `ncu --set full` captures of the hot kernels at cfg 5 (one build + eval of tools/run_build.py; run only
# after the same command has exited 0 without ncu).  Reports land in gpurun_out/; summarise them here with
# tools/ncu_summary.py / tools/ncu_lines.py into profiles/.
# usage (here): gpurun --timeout 2400 -- "bash tools/gpu_r2_ncu.sh TAG"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
tag=${1:-round2_ncu}
mkdir -p gpurun_out
timeout 600 python tools/run_build.py --config 5 --profile > gpurun_out/${tag}_plain.log 2>&1
rc=$?; echo "plain rc=$rc"; tail -2 gpurun_out/${tag}_plain.log
[ $rc -ne 0 ] && exit $rc
# build side: gather + root projection, K4, then K5 and the two K6 passes of the first levels
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:^(k_gather_root|k_moments|k_solve|k_residual)$' -c 11 -f -o gpurun_out/${tag}_build \
  python tools/run_build.py --config 5 > gpurun_out/${tag}_build.log 2>&1
echo "ncu build rc=$?"
# query side: K7 (first launches)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:^k_eval$' -c 2 -f -o gpurun_out/${tag}_eval \
  python tools/run_build.py --config 5 > gpurun_out/${tag}_eval.log 2>&1
echo "ncu eval rc=$?"
# summaries on the box (the reports can exceed gpurun_out's 64 MiB return limit): raw metric pages + tools/ncu_summary.py
for r in build eval; do
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/${tag}_$r.ncu-rep > gpurun_out/${tag}_${r}_summary.txt 2>&1
done
ls -la gpurun_out/${tag}_*.ncu-rep
find gpurun_out -name '*.ncu-rep' -size +30M -delete
# cfg 4 bench line again (the v6 run's line had two host-stalled steps)
for k in a b; do
  timeout 600 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_cfg4_$k.jsonl 2> gpurun_out/${tag}_bench_cfg4_$k.err
done
