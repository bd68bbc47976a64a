# Phase timing of K5 (k_solve): builds libfmi_t.so with -DFMI_K5_TIMING and runs one cfg-5 build.
cd "$(dirname "$0")/../paper_1511_01353_b200" || exit 1
mkdir -p build_t
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I../include"
$NV -DFMI_K5_TIMING -c csrc/solve.cu -o build_t/solve.o || exit 1
$NV -gencode arch=compute_100a,code=sm_100a -shared -o libfmi_t.so $(ls build/*.o | grep -v solve.o) build_t/solve.o -lcudart || exit 1
cd ..
python - <<'EOP'
import paper_1511_01353_b200 as fmi, workloads, torch, numpy as np
fmi.load_library("paper_1511_01353_b200/libfmi_t.so")
cfg = workloads.CONFIGS[5]
pts = workloads.uniform_points(cfg.n, 0)
f = workloads.franke3d(pts)
t = fmi.build(torch.from_numpy(pts).cuda(), torch.from_numpy(f).cuda(), cfg.degree, cfg.tol, cfg.max_depth)
torch.cuda.synchronize()
print("nodes", t.node_count)
EOP
