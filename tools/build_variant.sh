#!/bin/bash
# Build an A/B variant of libsaturn with extra -D flags into build_variants/<name>/:
#   tools/build_variant.sh nocp -DSAT_GA_CPASYNC=0
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
out=$ROOT/build_variants/$name
mkdir -p "$out"
NI=$(cd "$ROOT" && python -c "import paper_2309_01226_b200.build as b; print(b._nccl_include())")
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -O3 -I$NI"
for s in kernels api peers; do
  /usr/local/cuda/bin/nvcc $F "$@" -c "$ROOT/paper_2309_01226_b200/csrc/$s.cu" -o "$out/$s.o"
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o "$out/libsaturn.so" \
  "$out/kernels.o" "$out/api.o" "$out/peers.o" -ldl -lrt
rm -f "$out"/*.o
echo "$out/libsaturn.so"
