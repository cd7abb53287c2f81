# build a variant of the native library with extra nvcc flags into _variants/<name>.so
# usage: scripts/build_variant.sh <name> "<flags>"
set -e
name=$1; flags=$2
mkdir -p _variants/$name
objs=""
for s in capi elementwise attention attn_tc attn_fa attn_tm gemm peer; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags \
    -c paper_2408_12588_b200/csrc/$s.cu -o _variants/$name/$s.o &
  objs="$objs _variants/$name/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$name.so $objs -lcudart
