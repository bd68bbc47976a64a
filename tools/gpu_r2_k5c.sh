# K5 phase timing (clock64 per phase, -DFMI_K5_TIMING) at cfg3 and cfg5 + ncu of the level-4 cfg5 k_solve
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/k5_timing.sh > gpurun_out/r2_k5_phases.log 2>&1; echo "timing rc=$?"
grep "k5 phases" gpurun_out/r2_k5_phases.log | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_solve<" --launch-skip 4 --launch-count 1 -o gpurun_out/r2_k5_cfg5_l4b python tools/run_build.py --config 5 --m 1000 > gpurun_out/r2_k5_ncu2.log 2>&1
echo "ncu rc=$?"
