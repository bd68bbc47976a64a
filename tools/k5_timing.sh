# Phase timing of K5 (k_solve / k_solve_res): builds libfmi_t.so with -DFMI_K5_TIMING and runs one build of
# each config given (default 5): tools/k5_timing.sh 3 4
cd "$(dirname "$0")/../paper_1511_01353_b200" || exit 1
mkdir -p build_t
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I../include"
[ -n "$K5T_SKIP_BUILD" ] || $NV -DFMI_K5_TIMING -c csrc/solve.cu -o build_t/solve.o || exit 1
$NV -gencode arch=compute_100a,code=sm_100a -shared -o libfmi_t.so $(ls build/*.o | grep -v solve.o) build_t/solve.o -lcudart -ldl || exit 1
cd ..
for c in ${@:-5}; do
CFG=$c python - <<'EOP'
import os, paper_1511_01353_b200 as fmi, workloads, torch, numpy as np
fmi.load_library("paper_1511_01353_b200/libfmi_t.so")
cfg = workloads.CONFIGS[int(os.environ['CFG'])]
pts, f, _ = workloads.make_inputs(cfg.scaled(m=1000))
t = fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol, cfg.max_depth)
torch.cuda.synchronize()
print("cfg", cfg.name, "nodes", t.node_count)
EOP
done
