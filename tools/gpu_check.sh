# quick GPU check after a kernel change: parity + golden suites, then per-kernel ms of cfg 3/4/5 builds
# usage: bash tools/gpu_check.sh TAG [configs...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-chk}; shift
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${tag}_tests.log; tail -2 gpurun_out/${tag}_tests.log
for c in ${@:-3 4 5}; do
  timeout 300 python tools/run_build.py --config $c --m 1000 --reps 3 --profile > gpurun_out/${tag}_cfg$c.log 2>&1
  echo "cfg$c: $(grep -o 'build [0-9.]* ms' gpurun_out/${tag}_cfg$c.log | tail -1)"
  tail -1 gpurun_out/${tag}_cfg$c.log | python -c "
import json,sys
s=sys.stdin.read(); d=json.loads(s[s.index('{'):])
print('  ', ', '.join(f'{k} {v:.2f}' for k,v in sorted(d.items(), key=lambda kv:-kv[1])[:10]))"
done
