cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in 3 4; do
timeout 300 python tools/run_build.py --config $c --reps 4 2>&1 | tail -2 | cut -c1-200
FMI_TRACE=1 timeout 300 python tools/run_build.py --config $c --reps 2 2>&1 | grep -v "^cfg" | tail -2 | cut -c1-3000
FMI_TRACE=2 timeout 300 python tools/run_build.py --config $c --reps 2 2>&1 | grep -v "^cfg" | tail -1 | cut -c1-3000
done
