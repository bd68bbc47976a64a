# Build libfmi_<name>.so with extra nvcc flags for the listed sources (others from build/): experiments.
#   tools/build_variant.sh k4a "-DFMI_K4_LIM=48 -DFMI_K4_MINB=2" moments.cu
cd "$(dirname "$0")/../paper_1511_01353_b200" || exit 1
name=$1; flags=$2; shift 2
mkdir -p build_$name
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I../include -Xptxas -v"
objs=""
for f in build/*.o; do
  b=$(basename $f .o)
  if echo " $* " | grep -q " $b.cu "; then
    $NV $flags -c csrc/$b.cu -o build_$name/$b.o 2> build_$name/$b.ptxas.log || { cat build_$name/$b.ptxas.log; exit 1; }
    objs="$objs build_$name/$b.o"
  else
    objs="$objs $f"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libfmi_$name.so $objs -lcudart -ldl
